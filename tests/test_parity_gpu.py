"""GPU parity of the sm_100a engine against the oracle (C restatement of the
reference, itself pinned to the compiled reference in tests/test_oracle.py).

Tolerances (north_star: "within fp32 tolerance (rel 1e-5)"): per-example
norms element-wise rel <= 1e-5; clipped sums / stacks / updates per-block
normwise rel <= 1e-5 against the fp64 oracle (an element-wise rel bar fails
even for the reference's own fp32 build); noise <= 1 ulp.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5

CONFIGS = [
    # (name, model kind, options, batch, strategy)
    ("logreg", 0, {}, 64, 2),
    ("fcnn", 1, {}, 32, 1),
    ("fcnn_104_50_2", None, {}, 32, 1),
    ("mnist_cnn", 2, {}, 32, 4),
    ("cifar_cnn", 3, {}, 4, 4),
    ("embed_small", 4, dict(seq_len=16, vocab=50, hidden=8), 8, 5),
]


def make(P, O, name, kind, opts, B):
    if name == "fcnn_104_50_2":
        layers = [P.LayerSpec(P.LayerKind.dense, 104, 50), P.LayerSpec(P.LayerKind.relu),
                  P.LayerSpec(P.LayerKind.dense, 50, 2)]
        desc = P.custom_desc(P.ModelKind.fcnn, layers, (104,), 2)
        od = O.custom_desc(O.FCNN, [(0, 104, 50, 0, 1, 0), (6, 0, 0, 0, 1, 0),
                                    (0, 50, 2, 0, 1, 0)], (104,), 2)
    else:
        desc = P.build_desc(P.ModelKind(kind), P.ModelOptions(**opts))
        od = O.build_desc(kind, **opts)
    return desc, od


def blockwise_rel(got, want, blocks, B=None):
    worst, off = 0.0, 0
    for n in blocks:
        m = n * (B or 1)
        g, w = got[off:off + m], want[off:off + m]
        den = np.linalg.norm(w)
        if den > 0:
            worst = max(worst, np.linalg.norm(g - w) / den)
        else:
            worst = max(worst, np.abs(g).max() if m else 0.0)
        off += m
    return worst


@pytest.mark.parametrize("cfg", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_per_example_grads_and_norms(P, O, cfg):
    name, kind, opts, B, strat = cfg
    desc, od = make(P, O, name, kind, opts, B)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy(strat), B)
    stacks, norms = eng.per_example_flat(data.inputs, data.labels)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 0)
    ws, wnsq, _ = O.per_example_grads(od, x64, y64, p64)
    assert blockwise_rel(stacks, ws, od.blocks, B) < TOL
    wn = np.sqrt(wnsq)
    assert np.max(np.abs(norms - wn) / wn) < TOL


@pytest.mark.parametrize("cfg", CONFIGS, ids=[c[0] for c in CONFIGS])
@pytest.mark.parametrize("sigma", [0.0, 1.1])
def test_dpsgd_step_matches_oracle(P, O, cfg, sigma):
    name, kind, opts, B, strat = cfg
    desc, od = make(P, O, name, kind, opts, B)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy(strat), B)
    C = 1.0 if name != "embed_small" else 0.05
    cfg_ = P.DpConfig(clip_norm=C, noise_multiplier=sigma, learning_rate=0.1, seed=0)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 0)
    for step in range(2):
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg_, step)
        p_new, wn, wclip, cs = O.dpsgd_step(od, x64, y64, p64, C, sigma, 0.1, 1, 0, step)
        assert np.max(np.abs(rep.pre_clip_norms - wn) / wn) < TOL
        assert rep.clipped_count == wclip
        got = model.flat_params().astype(np.float64)
        # fp32 parameters: a few ulps of |p| plus 1e-5 of the update size
        delta = np.abs(p_new - p64).max()
        assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)
        expected_streams = [O.noise_stream(step, p) for p in range(od.n_blocks)] if sigma else []
        assert rep.noise_streams == expected_streams
        p64 = p_new
        model.params = P.unflatten(desc, p64.astype(np.float32))


@pytest.mark.parametrize("cfg", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_clipped_sum_matches_oracle(P, O, cfg):
    """North-star parity: noise-free clipped-sum gradient within fp32
    tolerance (per-block normwise rel <= 1e-5 and element-wise
    |d| <= 1e-5 (|ref| + max|ref|)), norms and clip count."""
    name, kind, opts, B, strat = cfg
    desc, od = make(P, O, name, kind, opts, B)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy(strat), B)
    C = 0.05 if name == "embed_small" else 1.0
    got, norms, nclip = eng.clipped_sum(data.inputs, data.labels, C)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 0)
    _, wn, wclip, want = O.dpsgd_step(od, x64, y64, p64, C, 0.0, 0.1, 1, 0, 0)
    assert np.max(np.abs(norms - wn) / wn) < TOL
    assert nclip == wclip
    assert blockwise_rel(got, want, od.blocks) < TOL
    off = 0
    for n in od.blocks:
        w = want[off:off + n]
        assert np.all(np.abs(got[off:off + n] - w) <= TOL * (np.abs(w) + np.abs(w).max()))
        off += n


def test_noise_bitwise(P, O):
    for seed, stream, n in [(0, 1 << 32, 26010), (7, (1 << 32) + 4096 * 3 + 5, 1001), (1, 4, 7)]:
        got = P.gaussian(seed, stream, n)
        want = O.gaussian(seed, stream, n, np.float32)
        ulps = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
        assert ulps.max() <= 1
        assert (ulps == 0).mean() > 1 - 1e-4


def test_aggregate_matches_reference_fp32_order(P, O):
    """The norm/clip/sum/noise/update kernel over given fp32 stacks follows
    the reference's fp32 views-path arithmetic (dpsgd.cpp:232-322): norms
    within 1 ulp, clip counts exact, parameters within fp32 re-association of
    the clipped sum (the device sums 8 ordered chunks of examples)."""
    desc = P.build_desc(P.ModelKind.mnist_cnn)
    od = O.build_desc(O.MNIST_CNN)
    B = 64
    model = P.build(P.ModelKind.mnist_cnn, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    stacks, _ = eng.per_example_flat(data.inputs, data.labels)
    p0 = model.flat_params()
    for sigma, C in [(1.1, 1.0), (0.0, 5.0), (0.5, 1e9)]:
        cfg = P.DpConfig(clip_norm=C, noise_multiplier=sigma, learning_rate=0.1, seed=3)
        model.params = P.unflatten(desc, p0)
        rep = P.aggregate(eng, model, stacks, cfg, 9)
        got = model.flat_params()
        want, wn, wclip = O.aggregate_f32(od.blocks, stacks, p0, C, sigma, 0.1, 3, 9, B)
        nu = np.abs(rep.pre_clip_norms.view(np.int32).astype(np.int64) -
                    wn.view(np.int32).astype(np.int64))
        assert nu.max() <= 1
        assert rep.clipped_count == wclip
        pu = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
        assert (pu == 0).mean() > 0.9, f"bitwise fraction {(pu == 0).mean()}"
        assert np.max(np.abs(got - want)) <= 2e-6 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("kind,B,strat", [(0, 7, 2), (1, 13, 3), (1, 1, 2), (2, 5, 4)])
def test_ragged_batches_match_oracle(P, O, kind, B, strat):
    """Batches that fill neither a CTA of the fused dense kernel (8 examples)
    nor a pair of the MNIST kernel: three noised steps against the oracle."""
    desc = P.build_desc(P.ModelKind(kind))
    od = O.build_desc(kind)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 4)
    eng = P.GradEngine(model, P.Strategy(strat), B)
    cfg = P.DpConfig(clip_norm=0.7, noise_multiplier=1.1, learning_rate=0.1, seed=6)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 4)
    for step in range(3):
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, step)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64, y64, p64, 0.7, 1.1, 0.1, 1, 6, step)
        assert np.max(np.abs(rep.pre_clip_norms - wn) / wn) < TOL
        assert rep.clipped_count == wclip
        got = model.flat_params().astype(np.float64)
        delta = np.abs(p_new - p64).max()
        assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)
        p64 = p_new
