"""tcgen05 kind::tf32 issue rate for the shapes / layouts the MNIST kernel uses."""
import ctypes as C
import sys
import os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09063_b200 as P

def rate(M, N, strides, mode=0, reps=256):
    st = np.array(strides, np.uint32)
    cyc = np.zeros(1, np.int64)
    P._lib.check(P.lib.pgb_debug_umma_rate(0, M, N, reps, P._lib.ptr(st), mode, P._lib.ptr(cyc)))
    return cyc[0] / reps

for M, N in [(128, 16), (128, 32), (64, 32), (128, 64), (128, 128), (128, 256), (64, 16), (64, 256)]:
    packed_m = [M // 8 * 128, 128, N // 8 * 128, 128]      # cores packed along M (LBO = K stride)
    packed_k = [128, 256, 128, 256]                         # cores packed along K (SBO = 256 B)
    ylike = [128, 512, 256, 128]
    print(f"M={M:3d} N={N:3d}  packedM {rate(M, N, packed_m):6.1f}  packedK {rate(M, N, packed_k):6.1f}"
          f"  Ylike {rate(M, N, ylike):6.1f}  2acc {rate(M, N, packed_m, 1):6.1f} cyc/MMA", flush=True)
