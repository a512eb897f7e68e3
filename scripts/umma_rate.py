"""tcgen05 kind::tf32 issue rate for the shapes / layouts the MNIST kernel uses.
mode bits: 1 two accumulators, 2 streaming operand addresses, 4 other threads
poll the mbarrier, 8 launch 1024 threads (else 128), 16 four issuing warps,
32 descriptors advanced by 64-bit adds instead of rebuilt."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09063_b200 as P  # noqa: E402


def rate(M, N, strides, mode=0, reps=256):
    st = np.array(strides, np.uint32)
    cyc = np.zeros(1, np.int64)
    P._lib.check(P.lib.pgb_debug_umma_rate(0, M, N, reps, P._lib.ptr(st), mode, P._lib.ptr(cyc)))
    return cyc[0] / reps


for M, N in [(128, 16), (128, 32), (64, 64), (128, 64), (128, 128), (128, 256)]:
    pm = [M // 8 * 128, 128, N // 8 * 128, 128]
    print(f"M={M:3d} N={N:3d}  rebuild {rate(M, N, pm, 2):6.1f}  descadd {rate(M, N, pm, 2 | 32):6.1f}"
          f"  4warps {rate(M, N, pm, 2 | 16):6.1f}  4warps+descadd {rate(M, N, pm, 2 | 16 | 32):6.1f}"
          f"  same-desc {rate(M, N, pm, 32):6.1f}", flush=True)
