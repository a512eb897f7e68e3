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


@pytest.mark.parametrize("M", [64, 128])
@pytest.mark.parametrize("N", [16, 32])
def test_umma_layouts(P, M, N):
    """K-major (no swizzle) operands and the accumulator lane map (M = 128:
    lane m; M = 64: lane m % 16 + 32 (m / 16)) the tensor-core MNIST kernel
    relies on; small integers, so the product is exact. (tf32 MN-major
    operands need the 128B_BASE32B swizzle: with SWIZZLE_NONE the MMA leaves
    the accumulator untouched, so the kernel uses K-major operands only.)"""
    a_mn = b_mn = 0
    K = 24
    rng = np.random.default_rng(M + N + 2 * a_mn + b_mn)
    A = rng.integers(-4, 5, (M, K)).astype(np.float32)
    B = rng.integers(-4, 5, (N, K)).astype(np.float32)
    D = np.zeros((128, N), np.float32)
    P._lib.check(P.lib.pgb_debug_umma_probe(0, M, N, K, a_mn, b_mn, P._lib.ptr(A),
                                            P._lib.ptr(B), P._lib.ptr(D)))
    want = A @ B.T
    lanes = np.arange(M) if M == 128 else (np.arange(M) % 16 + 32 * (np.arange(M) // 16))
    np.testing.assert_array_equal(D[lanes], want)


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 64, 96), (200, 100, 76), (1000, 16, 288),
                                   (384, 128, 1152), (64, 32, 4)])
def test_tma_gemm_3xtf32(P, M, N, K):
    """The TMA-fed GEMM (tensor maps with the 128-B swizzle, K-major UMMA
    descriptors, hi = the TMA tile itself since tcgen05 truncates tf32, lo
    split on the CUDA cores): normwise 1e-6 against fp64, ragged M/N/K (the
    TMA out-of-bounds fill)."""
    rng = np.random.default_rng(M + 3 * N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    Cm = np.zeros((M, N), np.float32)
    P._lib.check(P.lib.pgb_debug_tma_gemm(0, M, N, K, P._lib.ptr(A), P._lib.ptr(B),
                                          P._lib.ptr(Cm)))
    want = A.astype(np.float64) @ B.astype(np.float64).T
    err = np.linalg.norm(Cm - want) / np.linalg.norm(want)
    assert err < 1e-6, err


@pytest.mark.parametrize("C,H,W,D", [(3, 32, 32, 10), (32, 32, 32, 16), (32, 16, 16, 64),
                                     (64, 8, 8, 10), (128, 8, 8, 32), (128, 4, 4, 256),
                                     (256, 4, 4, 10), (16, 8, 32, 40), (48, 16, 8, 96)])
@pytest.mark.parametrize("env", ["PGB_TMA_ALL=1", "PGB_TMA_ALL=1 PGB_DWH_MIN_C=1",
                                 "PGB_DWH_MIN_C=1 PGB_DWH_ROT=2", "PGB_TMA_ALL=1 PGB_NO_DW_HALO=1",
                                 "PGB_NO_DIRECT_CONV=1", "PGB_TMA_SPLIT=1 PGB_DWH_SPLIT=1"],
                         ids=["tma_all", "tma_all_dwh_all", "dwh_all_rot2", "tma_all_no_dwh",
                              "no_direct", "split_operands"])
def test_tma_conv_gemms_match_oracle(P, O, monkeypatch, C, H, W, D, env):
    """Every 3x3 conv GEMM on the TMA engine (PGB_TMA_ALL=1: forward,
    per-example dW and input gradient, whatever the per-kind default picks;
    the per-example dW on the halo kernel for C >= 16 or, PGB_DWH_MIN_C=1, for
    every channel count, else the tap-slot TMA GEMM): a conv -> relu -> conv ->
    relu -> global-avgpool model over the geometries of the CIFAR CNN and a few
    ragged ones (W != H, channel counts off the 32 grid), per-example gradients
    and norms against the oracle."""
    for kv in env.split():
        k, v = kv.split("=")
        monkeypatch.setenv(k, v)
    layers = [P.LayerSpec(P.LayerKind.conv, C, D, 3, 1, 1), P.LayerSpec(P.LayerKind.relu),
              P.LayerSpec(P.LayerKind.conv, D, 10, 3, 1, 1), P.LayerSpec(P.LayerKind.relu),
              P.LayerSpec(P.LayerKind.global_avgpool)]
    desc = P.custom_desc(P.ModelKind.cifar_cnn, layers, (C, H, W), 10)
    od = O.custom_desc(O.CIFAR_CNN, [(1, C, D, 3, 1, 1), (6, 0, 0, 0, 1, 0), (1, D, 10, 3, 1, 1),
                                     (6, 0, 0, 0, 1, 0), (4, 0, 0, 0, 1, 0)], (C, H, W), 10)
    B = 3
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    st, nr = eng.per_example_flat(data.inputs, data.labels)
    ws, wnsq, _ = O.per_example_grads(od, data.inputs.astype(np.float64),
                                      data.labels.astype(np.float64), O.init_params(od, 0))
    off = 0
    for n in od.blocks:
        g, w = st[off:off + B * n], ws[off:off + B * n]
        assert np.linalg.norm(g - w) <= 1e-5 * np.linalg.norm(w), (off, n)
        off += B * n
    wn = np.sqrt(wnsq)
    assert np.max(np.abs(nr - wn) / wn) < 1e-5
