"""Does a TMA box start need 16-byte alignment in the innermost dimension?
Loads 32 x 4 boxes at x0 in {-1, 0, 1, 2, 3, 5} from a 64 x 8 array and compares."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_09063_b200 as P
W, H = 64, 8
src = np.arange(W * H, dtype=np.float32).reshape(H, W)
for x0 in [int(a) for a in sys.argv[1:]] or (0,):
    out = np.zeros(128, np.float32)
    P._lib.check(P.lib.pgb_debug_tma_box(0, P._lib.ptr(src), W, H, x0, 1, P._lib.ptr(out)))
    want = np.zeros((4, 32), np.float32)
    for r in range(4):
        for c in range(32):
            x, y = x0 + c, 1 + r
            want[r, c] = src[y, x] if 0 <= x < W else 0.0
    print(x0, "ok" if np.array_equal(out.reshape(4, 32), want) else f"MISMATCH first row {out[:8]}")
