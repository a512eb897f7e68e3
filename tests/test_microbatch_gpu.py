"""Microbatch m > 1 on the GPU (dpsgd.cpp:102-132: the mean over m consecutive
examples is the clipped unit; B/m units, noise, mean over the units), against
the oracle, in graph and eager mode, and with m changing between calls on one
engine (each m has its own CUDA graph: m and U = B/m are baked into the
microbatch, norm and aggregation launches).

Tolerances as test_parity_gpu.py: unit norms element-wise rel 1e-5, clip
counts exact, parameters a few ulps + 1e-5 of the update.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5

CASES = [
    # (name, kind, options, batch, strategy, microbatches)
    ("logreg", 0, {}, 64, 2, (2, 4)),
    ("fcnn", 1, {}, 32, 1, (2, 4, 32)),
    ("mnist_cnn", 2, {}, 32, 4, (2, 4)),
    ("cifar_cnn", 3, {}, 4, 4, (2,)),
    ("embed_small", 4, dict(seq_len=16, vocab=50, hidden=8), 8, 5, (2, 4)),
]


def _check(rep, model, p_new, wn, wclip, p_old):
    assert np.max(np.abs(rep.pre_clip_norms - wn) / wn) < TOL
    assert rep.clipped_count == wclip
    got = model.flat_params().astype(np.float64)
    delta = np.abs(p_new - p_old).max()
    assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)


@pytest.mark.parametrize("mode", ["graph", "eager"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_microbatch_steps_match_oracle(P, O, case, mode):
    name, kind, opts, B, strat, ms = case
    desc = P.build_desc(P.ModelKind(kind), P.ModelOptions(**opts))
    od = O.build_desc(kind, **opts)
    data = P.synth_for_model(desc, B, 0)
    x64, y64 = O.synth(od, B, 0)
    C = 0.05 if name == "embed_small" else 0.5
    for m in ms:
        model = P.build_from_desc(desc, 0)
        eng = P.GradEngine(model, P.Strategy(strat), B, P.ExecMode[mode])
        cfg = P.DpConfig(clip_norm=C, noise_multiplier=1.1, learning_rate=0.1, microbatch=m,
                         seed=2)
        p64 = O.init_params(od, 0)
        for step in range(2):
            rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, step)
            assert rep.pre_clip_norms.shape == (B // m,)
            p_new, wn, wclip, _ = O.dpsgd_step(od, x64, y64, p64, C, 1.1, 0.1, m, 2, step)
            _check(rep, model, p_new, wn, wclip, p64)
            p64 = p_new


def test_microbatch_switch_on_one_engine(P, O):
    """m = 64, 128, 64, 1, 128 on one B = 256 engine (the round-1 graph cache
    folded every m >= 63 onto one key): each step against the oracle."""
    B = 256
    desc = P.build_desc(P.ModelKind.fcnn)
    od = O.build_desc(O.FCNN)
    data = P.synth_for_model(desc, B, 1)
    x64, y64 = O.synth(od, B, 1)
    model = P.build_from_desc(desc, 0)
    eng = P.GradEngine(model, P.Strategy.vmap, B)
    p64 = O.init_params(od, 0)
    for step, m in enumerate([64, 128, 64, 1, 128]):
        cfg = P.DpConfig(clip_norm=0.3, noise_multiplier=1.1, learning_rate=0.1, microbatch=m,
                         seed=4)
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, step)
        assert rep.pre_clip_norms.shape == (B // m,)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64, y64, p64, 0.3, 1.1, 0.1, m, 4, step)
        _check(rep, model, p_new, wn, wclip, p64)
        p64 = p_new


def test_microbatch_switch_mnist(P, O):
    """The fused MNIST engine switching between m = 1 (tensor-core kernel +
    pair rows) and m = 2, 4 (materialised stacks + microbatch means)."""
    B = 16
    desc = P.build_desc(P.ModelKind.mnist_cnn)
    od = O.build_desc(O.MNIST_CNN)
    data = P.synth_for_model(desc, B, 3)
    x64, y64 = O.synth(od, B, 3)
    model = P.build_from_desc(desc, 0)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    p64 = O.init_params(od, 0)
    for step, m in enumerate([2, 1, 4, 2, 1]):
        cfg = P.DpConfig(clip_norm=0.5, noise_multiplier=1.1, learning_rate=0.1, microbatch=m,
                         seed=1)
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, step)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64, y64, p64, 0.5, 1.1, 0.1, m, 1, step)
        _check(rep, model, p_new, wn, wclip, p64)
        p64 = p_new
