"""The norms-only two-pass step and the weighted gradient sums on the GPU.

Reference: dpsgd_step's norms branch (proj/core/src/dpsgd.cpp:194-230) takes
per-example norms from the norms-only engine, then the clipped sum as one
weighted backward, GradEngine::weighted_grad_sum (strategies.cpp:432-450);
batch_grad_sum (:453-458) is the all-ones case. On the device the dense blocks
stay factored (a_i, delta_i), so the "second pass" is the aggregation kernel's
weighted outer-product sum with w_i in place of the clip factors.

Checked against the compiled reference itself (oracle/_ref, fp64): its
weighted_grad_sum and its norms-strategy dpsgd_step. Tolerances as in
test_parity_gpu.py (per-block normwise 1e-5; parameters a few fp32 ulps plus
1e-5 of the update).
"""
import numpy as np
import pytest

from test_parity_gpu import CONFIGS, TOL, blockwise_rel, make

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R(O):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    return O


@pytest.mark.parametrize("cfg", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_weighted_grad_sum_matches_reference(P, O, R, cfg):
    name, kind, opts, B, strat = cfg
    desc, od = make(P, O, name, kind, opts, B)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy(strat), B)
    w = np.random.default_rng(1).uniform(0.05, 1.0, B).astype(np.float32)
    got = eng.weighted_grad_sum(data.inputs, data.labels, w)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 0)
    ref = O.RefModel(od, strat, B, p64)
    want = ref.weighted_grad_sum(x64, y64, w.astype(np.float64))
    assert blockwise_rel(got, want, od.blocks) < TOL
    ones = eng.batch_grad_sum(data.inputs, data.labels)
    want1 = ref.weighted_grad_sum(x64, y64, np.ones(B))
    assert blockwise_rel(ones, want1, od.blocks) < TOL


def test_weighted_sum_with_clip_factors_is_the_clipped_sum(P, O):
    """Second pass with w = the clip factors reproduces the one-pass clipped
    sum (same aggregation order: bitwise)."""
    B = 32
    desc = P.build_desc(P.ModelKind.mnist_cnn)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    C = 1.0
    one_pass, norms, _ = eng.clipped_sum(data.inputs, data.labels, C)
    s = np.where(norms > C, np.float32(C) / norms, np.float32(1)).astype(np.float32)
    two_pass = eng.weighted_grad_sum(data.inputs, data.labels, s)
    np.testing.assert_array_equal(two_pass, one_pass)


@pytest.mark.parametrize("name", ["logreg", "fcnn", "fcnn_104_50_2"])
def test_norms_strategy_step_matches_reference_two_pass(P, O, R, name):
    """Strategy.norms engines (dense models) against the reference's own
    norms-only two-pass dpsgd_step, three steps with noise."""
    cfg = next(c for c in CONFIGS if c[0] == name)
    _, kind, opts, B, _ = cfg
    desc, od = make(P, O, name, kind, opts, B)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy.norms, B)
    dp = P.DpConfig(clip_norm=0.5, noise_multiplier=1.1, learning_rate=0.1, seed=3)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 0)
    ref = O.RefModel(od, O.NORMS, B, p64)
    for step in range(3):
        p_old = ref.params()
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, dp, step)
        rn, rclip = ref.step(x64, y64, 0.5, 1.1, 0.1, 1, 3, step)
        assert np.max(np.abs(rep.pre_clip_norms - rn) / rn) < TOL
        assert rep.clipped_count == rclip
        p_new = ref.params()
        got = model.flat_params().astype(np.float64)
        delta = np.abs(p_new - p_old).max()
        assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)
        model.params = P.unflatten(desc, p_new.astype(np.float32))


def test_norms_strategy_rejects_microbatch(P):
    """dpsgd.cpp:195-198: the norms-only strategy supports microbatch = 1 only."""
    B = 8
    desc = P.build_desc(P.ModelKind.fcnn)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy.norms, B)
    dp = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, microbatch=2, seed=0)
    from paper_2010_09063_b200 import _lib
    from paper_2010_09063_b200.errors import ConfigError
    with pytest.raises(ConfigError, match="microbatch = 1 only"):
        P.dpsgd_step(model, eng, data.inputs, data.labels, dp, 0)
    # the C ABI itself refuses it too (the check is not only in the Python mirror)
    import ctypes as C
    norms = np.empty(B // 2, np.float32)
    rep = _lib.StepReportC()
    rc = _lib.lib.pgb_dpsgd_step(eng.handle, _lib.ptr(data.inputs), _lib.ptr(data.labels),
                                 C.byref(dp.to_c()), 0, _lib.ptr(norms), C.byref(rep))
    assert rc == 4 and b"microbatch = 1 only" in _lib.lib.pgb_last_error()
