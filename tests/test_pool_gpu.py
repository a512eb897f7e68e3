"""The 2x2 / stride-2 pooling kernels (pool2_fwd_kernel, pool2_bwd_kernel: one
thread per window, the CIFAR CNN's three average pools and the layer-wise MNIST
max pool) against the generic window kernels (PGB_POOL_GENERIC=1), bitwise:
same fp32 operations in the same window order, first-max routing
(kernels.hpp:377-396). Integer-valued images force max-pool ties and exact-zero
relu inputs, the edge cases the reference's KATs pin."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(P, desc, B, strat, x, y, generic, monkeypatch, steps=2):
    if generic:
        monkeypatch.setenv("PGB_POOL_GENERIC", "1")
    m = P.build_from_desc(desc, 0)
    e = P.GradEngine(m, P.Strategy(strat), B)
    if generic:
        monkeypatch.delenv("PGB_POOL_GENERIC")
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=4)
    norms = []
    for s in range(steps):
        r = P.dpsgd_step(m, e, x, y, cfg, s)
        norms.append(r.pre_clip_norms.copy())
    return m.flat_params(), np.concatenate(norms)


@pytest.mark.parametrize("name,integral", [("cifar", False), ("mnist_layerwise", False),
                                           ("mnist_layerwise", True)])
def test_pool2_bitwise_generic(P, name, integral, monkeypatch):
    if name == "cifar":
        desc = P.build_desc(P.ModelKind.cifar_cnn)
        B, strat = 4, 4
    else:
        monkeypatch.setenv("PGB_NO_FUSED", "1")
        desc = P.build_desc(P.ModelKind.mnist_cnn)
        B, strat = 8, 4
    data = P.synth_for_model(desc, B, 1)
    x = data.inputs
    if integral:  # ties inside pooling windows and exact zeros before the relus
        x = np.floor(np.abs(x) * 2.0).astype(np.float32)
    pa, na = _run(P, desc, B, strat, x, data.labels, False, monkeypatch)
    pb, nb = _run(P, desc, B, strat, x, data.labels, True, monkeypatch)
    np.testing.assert_array_equal(na, nb)
    np.testing.assert_array_equal(pa, pb)
