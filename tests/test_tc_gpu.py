"""tcgen05 building block: 3xTF32 GEMM (UTCHMMA, TMEM accumulators) vs an
fp64 reference. The bar is the per-example-GEMM accuracy the DPSGD path
needs (normwise 1e-6; a single TF32 pass would be ~3e-4)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (256, 64, 64), (200, 100, 77), (16, 10, 512),
                                   (1000, 200, 300)])
def test_tc_gemm_3xtf32(P, M, N, K):
    rng = np.random.default_rng(M * 7 + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    Cm = np.zeros((M, N), np.float32)
    P._lib.check(P.lib.pgb_debug_tc_gemm(0, M, N, K, P._lib.ptr(A), P._lib.ptr(B),
                                         P._lib.ptr(Cm)))
    want = A.astype(np.float64) @ B.astype(np.float64).T
    err = np.linalg.norm(Cm - want) / np.linalg.norm(want)
    assert err < 1e-6, err
