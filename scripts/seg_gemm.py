import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_09063_b200 as P
for (M, N, K) in [(384, 128, 1152), (2048, 64, 576), (4096, 16, 2304)]:
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    out = []
    for sg in ("0", "1", "2", "4", "8", "16", "64"):
        os.environ["PGB_DEBUG_SEG"] = sg
        Cm = np.zeros((M, N), np.float32)
        P._lib.check(P.lib.pgb_debug_tma_gemm(0, M, N, K, P._lib.ptr(A), P._lib.ptr(B), P._lib.ptr(Cm)))
        out.append(f"seg{sg}:{np.linalg.norm(Cm - want) / np.linalg.norm(want):.1e}")
    print(M, N, K, " ".join(out))
