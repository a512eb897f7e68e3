"""What does tcgen05 kind::tf32 do with the 13 low mantissa bits of an fp32
operand in shared memory: truncate, or round? One MMA, M = 128, N = 8, K = 8,
A = fp32 values with low bits set, B = e_0 (so D[m][0] = A[m][0] as the
tensor core saw it)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09063_b200 as P  # noqa: E402

M, N, K = 128, 8, 8
rng = np.random.default_rng(0)
A = (rng.standard_normal((M, K)) * 3).astype(np.float32)
B = np.zeros((N, K), np.float32)
B[0, 0] = 1.0
D = np.zeros((128, N), np.float32)
P._lib.check(P.lib.pgb_debug_umma_probe(0, M, N, K, 0, 0, P._lib.ptr(A), P._lib.ptr(B),
                                        P._lib.ptr(D)))
a = A[:, 0]
bits = a.view(np.uint32)
trunc = (bits & np.uint32(0xFFFFE000)).view(np.float32)
# round to nearest, ties away (cvt.rna) and ties to even
rna = ((bits + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)
got = D[:M, 0]
print("tensor core == truncation:", np.array_equal(got, trunc),
      " == rna:", np.array_equal(got, rna), " == raw fp32:", np.array_equal(got, a))
print("examples", list(zip(a[:4].tolist(), got[:4].tolist(), trunc[:4].tolist(), rna[:4].tolist())))
