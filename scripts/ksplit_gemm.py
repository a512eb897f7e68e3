import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_09063_b200 as P
for (M, N, K) in [(2048, 64, 576), (1024, 64, 576), (2048, 32, 576), (4096, 128, 1152), (2048, 64, 288)]:
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    out = []
    for S in ("1", "2", "3", "6"):
        os.environ["PGB_DEBUG_KSPLIT"] = S
        Cm = np.zeros((M, N), np.float32)
        P._lib.check(P.lib.pgb_debug_tma_gemm(0, M, N, K, P._lib.ptr(A), P._lib.ptr(B), P._lib.ptr(Cm)))
        err = np.linalg.norm(Cm - want) / np.linalg.norm(want)
        bad = np.argwhere(np.abs(Cm - want) > 1e-3 * np.abs(want).max())
        out.append(f"S={S}:{err:.1e}" + (f" bad{len(bad)} first{bad[:2].tolist()}" if len(bad) else ""))
    print(M, N, K, " ".join(out))
