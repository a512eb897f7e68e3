"""The reference's edge-case known-answer tests, forced on the GPU paths.

* clip / clip_scales KATs (proj/tests/test_dpsgd.cpp:37-47,77-82): (6,8) at
  C=5 -> (3,4); norm == C is not clipped and passes unchanged; a zero
  gradient has scale 1 -- through the aggregation kernel (pgb_aggregate) and,
  for the norm == C boundary, through each fused per-example kernel's own
  clip decision (the step's reported norm used as C);
* first-max routing of max-pool ties (kernels.hpp:377-396) and the relu
  gradient at an exactly-zero pre-activation (gt mask, autodiff.cpp:121-124):
  integer images, conv1 weights on a 1/16 grid (every conv1 output exact, so
  the GPU and the fp64 oracle see the same ties), one all-zero image (every
  relu input exactly 0) -- fused tensor-core kernel and layer-wise schedule;
* checked_id (kernels.hpp:475-489): non-integral and out-of-range ids and
  labels raise IndexError with the reference's text, the first bad value in
  the reference's order wins, parameters stay untouched.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _fcnn_zero(P, B):
    desc = P.build_desc(P.ModelKind.fcnn)
    model = P.build_from_desc(desc, 0)
    model.params = [np.zeros_like(p) for p in model.params]
    eng = P.GradEngine(model, P.Strategy.vmap, B)
    return desc, model, eng


def test_clip_kat_rescales_onto_sphere(P):
    """(6, 8) at C = 5 becomes (3, 4) exactly; the update p - lr * sum / B with
    p = 0, lr = 1, B = 1 exposes the clipped row bit for bit."""
    desc, model, eng = _fcnn_zero(P, 1)
    stacks = np.zeros(eng.P, np.float32)
    stacks[:2] = [6.0, 8.0]
    cfg = P.DpConfig(clip_norm=5.0, noise_multiplier=0.0, learning_rate=1.0, seed=0)
    rep = P.aggregate(eng, model, stacks, cfg, 0)
    got = model.flat_params()
    assert rep.pre_clip_norms[0] == 10.0
    assert rep.clipped_count == 1
    np.testing.assert_array_equal(got[:2], [-3.0, -4.0])
    assert not got[2:].any()


def test_clip_kat_boundary_unchanged(P):
    """norm == C: not clipped (count 0) and the row passes bit-unchanged."""
    desc, model, eng = _fcnn_zero(P, 1)
    stacks = np.zeros(eng.P, np.float32)
    stacks[7:9] = [3.0, 4.0]
    cfg = P.DpConfig(clip_norm=5.0, noise_multiplier=0.0, learning_rate=1.0, seed=0)
    rep = P.aggregate(eng, model, stacks, cfg, 0)
    assert rep.pre_clip_norms[0] == 5.0
    assert rep.clipped_count == 0
    np.testing.assert_array_equal(model.flat_params()[7:9], [-3.0, -4.0])


def test_clip_scales_kat_zero_gradient(P, O):
    """clip_scales({10, 0, 4}, 5) = {0.5, 1, 1}: norms reported exactly, one
    clipped, the zero row contributes nothing (no 0 * inf), the update equals
    the reference's fp32 aggregation."""
    desc, model, eng = _fcnn_zero(P, 3)
    P_ = eng.P
    stacks = np.zeros(3 * P_, np.float32)
    # block-major: block b of example i at off_b * 3 + i * size_b
    od = O.build_desc(O.FCNN)
    sz0 = od.blocks[0]
    stacks[0 * sz0 + 0: 0 * sz0 + 2] = [6.0, 8.0]   # example 0, norm 10
    stacks[2 * sz0 + 1] = 4.0                       # example 2, norm 4 (example 1: zeros)
    cfg = P.DpConfig(clip_norm=5.0, noise_multiplier=0.0, learning_rate=1.0, seed=0)
    p0 = model.flat_params()
    rep = P.aggregate(eng, model, stacks, cfg, 0)
    np.testing.assert_array_equal(rep.pre_clip_norms, [10.0, 0.0, 4.0])
    assert rep.clipped_count == 1
    got = model.flat_params()
    want, wn, wclip = O.aggregate_f32(od.blocks, stacks, p0, 5.0, 0.0, 1.0, 0, 0, 3)
    np.testing.assert_array_equal(wn, [10.0, 0.0, 4.0])
    assert wclip == 1
    np.testing.assert_array_equal(got, want)
    assert np.isfinite(got).all()


CLIP_CASES = [
    # (name, kind, options, batch, strategy, extra env)
    ("mnist_tc", 2, {}, 1, 4, {}),
    ("mnist_tc_b4", 2, {}, 4, 4, {}),
    ("mnist_layerwise", 2, {}, 4, 4, {"PGB_NO_FUSED": "1"}),
    ("fcnn_mlp", 1, {}, 4, 1, {}),
    ("cifar", 3, {}, 2, 4, {}),
    ("embed_small", 4, dict(seq_len=16, vocab=50, hidden=8), 4, 5, {}),
]


@pytest.mark.parametrize("case", CLIP_CASES, ids=[c[0] for c in CLIP_CASES])
def test_clip_boundary_in_each_step_kernel(P, case, monkeypatch):
    """Each step kernel's own clip decision at norm == C (the norms it
    reports, as fp32, used as C): the largest norm is not clipped, so the
    update is bitwise the unclipped one; one ulp below it clips."""
    name, kind, opts, B, strat, env = case
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    desc = P.build_desc(P.ModelKind(kind), P.ModelOptions(**opts))
    data = P.synth_for_model(desc, B, 1)

    def step(C):
        model = P.build_from_desc(desc, 0)
        eng = P.GradEngine(model, P.Strategy(strat), B)
        cfg = P.DpConfig(clip_norm=float(C), noise_multiplier=0.0, learning_rate=0.1, seed=0)
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, 0)
        return model.flat_params(), rep

    loose, rl = step(1e30)
    assert rl.clipped_count == 0
    n = rl.pre_clip_norms
    top = np.float32(n.max())
    at, ra = step(top)
    np.testing.assert_array_equal(ra.pre_clip_norms, n)
    assert ra.clipped_count == 0
    np.testing.assert_array_equal(at, loose)
    # one ulp below clips (the factor fl(C / n) may round the update back)
    _, rb = step(np.nextafter(top, np.float32(0)))
    assert rb.clipped_count == int((n >= top).sum())
    below, _ = step(top * np.float32(0.5))
    assert not np.array_equal(below, loose)
    if B > 1:  # the count at an interior boundary: exactly the norms above it
        mid = np.float32(np.sort(n)[B // 2])
        _, rm = step(mid)
        assert rm.clipped_count == int((n > mid).sum())


def _tie_model(P, O, B, seed=3):
    """MNIST CNN whose conv1 outputs are exact (integer images in {0..3},
    conv1 weights on a 1/16 grid, bias 0): 2x2 max-pool windows hold exact
    ties; example 0 is all zeros (every relu input exactly 0); the left half
    of examples 1..B/2 is zero."""
    desc = P.build_desc(P.ModelKind.mnist_cnn)
    od = O.build_desc(O.MNIST_CNN)
    p = O.init_params(od, 0).astype(np.float32)
    n0 = od.blocks[0]
    p[:n0] = np.round(p[:n0] * 16.0) / 16.0
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 4, size=(B, 1, 28, 28)).astype(np.float32)
    x[0] = 0.0
    x[1:B // 2, :, :, :14] = 0.0
    y = rng.integers(0, 10, size=B).astype(np.float32)
    return desc, od, p, x, y


def _count_ties(x, w1):
    """Number of 2x2 pool windows of relu(conv1) with a tied positive max."""
    import numpy.lib.stride_tricks as st
    B = x.shape[0]
    xp = np.pad(x[:, 0].astype(np.float64), ((0, 0), (3, 3), (3, 3)))
    win = st.sliding_window_view(xp, (8, 8), axis=(1, 2))[:, ::2, ::2]  # (B,14,14,8,8)
    z = np.einsum("bijuv,duv->bdij", win, w1.reshape(16, 8, 8).astype(np.float64))
    r = np.maximum(z, 0.0).reshape(B, 16, 7, 2, 7, 2).transpose(0, 1, 2, 4, 3, 5)
    r = r.reshape(B, 16, 7, 7, 4)
    m = r.max(-1)
    return int(((r == m[..., None]).sum(-1) > 1)[m > 0].sum())


@pytest.mark.parametrize("env", [{}, {"PGB_NO_FUSED": "1"}, {"PGB_MNIST_SIMT": "1"}],
                         ids=["tc_kernel", "layerwise", "simt_kernel"])
def test_maxpool_ties_and_zero_relu_match_oracle(P, O, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    B = 16
    desc, od, p, x, y = _tie_model(P, O, B)
    assert _count_ties(x, p[:od.blocks[0]]) > 100  # the case is really exercised
    model = P.build_from_desc(desc, 0)
    model.params = P.unflatten(desc, p)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    stacks, norms = eng.per_example_flat(x, y)
    ws, wnsq, _ = O.per_example_grads(od, x.astype(np.float64), y.astype(np.float64),
                                      p.astype(np.float64))
    wn = np.sqrt(wnsq)
    assert np.max(np.abs(norms - wn) / wn) < TOL
    off = 0
    for n in od.blocks:
        g, w = stacks[off:off + B * n].reshape(B, n), ws[off:off + B * n].reshape(B, n)
        assert np.linalg.norm(g - w) <= TOL * np.linalg.norm(w)
        for i in range(B):
            # per example and block (a misrouted tie moves a whole pooled
            # gradient: an O(1) error; 1e-4 leaves room for fp32 cancellation
            # in one example's bias sums)
            den = np.linalg.norm(w[i])
            err = np.linalg.norm(g[i] - w[i])
            assert err <= 1e-4 * den or err == 0.0, (off, i, err, den)
        off += B * n
    # the all-zero image: only the last bias has a gradient (every relu closed)
    g0 = [stacks[o:o + B * n].reshape(B, n)[0] for o, n in
          zip(np.cumsum([0] + [B * b for b in od.blocks[:-1]]), od.blocks)]
    assert all(not g.any() for g in g0[:-1]) and g0[-1].any()
    # and a full step against the oracle
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    rep = P.dpsgd_step(model, eng, x, y, cfg, 0)
    p_new, wn2, wclip, _ = O.dpsgd_step(od, x.astype(np.float64), y.astype(np.float64),
                                        p.astype(np.float64), 1.0, 1.1, 0.1, 1, 0, 0)
    assert rep.clipped_count == wclip
    got = model.flat_params().astype(np.float64)
    delta = np.abs(p_new - p).max()
    assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)


# ---- checked_id (kernels.hpp:475-489) --------------------------------------

def _embed(P, B=4, L=16, V=50):
    desc = P.build_desc(P.ModelKind.embed, P.ModelOptions(seq_len=L, vocab=V, hidden=8))
    data = P.synth_for_model(desc, B, 0)
    return desc, data


def _expect_index_error(P, desc, strat, x, y, msg):
    from paper_2010_09063_b200.errors import IndexError_ as PgbIndexError
    B = x.shape[0]
    model = P.build_from_desc(desc, 0)
    eng = P.GradEngine(model, P.Strategy(strat), B)
    p0 = model.flat_params()
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    with pytest.raises(PgbIndexError) as ei:
        P.dpsgd_step(model, eng, x, y, cfg, 0)
    assert str(ei.value).endswith(msg), str(ei.value)
    np.testing.assert_array_equal(model.flat_params(), p0)
    # the engine recovers: a clean step afterwards works
    return eng, model


def test_embedding_id_non_integral(P):
    desc, data = _embed(P)
    x = data.inputs.copy()
    x[2, 5] = 3.5
    _expect_index_error(P, desc, 5, x, data.labels,
                        f"gather_rows: non-integral id at position {2 * 16 + 5}")


def test_embedding_id_out_of_range(P):
    desc, data = _embed(P)
    x = data.inputs.copy()
    x[1, 3] = 50.0
    _expect_index_error(P, desc, 5, x, data.labels,
                        f"gather_rows: id 50 out of range [0,50) at position {16 + 3}")
    x[1, 3] = -2.0
    _expect_index_error(P, desc, 5, x, data.labels,
                        f"gather_rows: id -2 out of range [0,50) at position {16 + 3}")


def test_first_bad_value_in_reference_order_wins(P):
    """Several bad values: the reference throws at the first one it meets --
    the embedding gather (forward) before the labels (loss), ascending
    position within each."""
    desc, data = _embed(P)
    x = data.inputs.copy()
    y = data.labels.copy()
    x[3, 0] = 99.0
    x[1, 7] = 2.25
    x[2, 1] = -1.0
    y[0] = 7.0
    _expect_index_error(P, desc, 5, x, y, f"gather_rows: non-integral id at position {16 + 7}")


@pytest.mark.parametrize("kind,strat,B,bad,msg", [
    (2, 4, 8, 12.0, "softmax_xent label: id 12 out of range [0,10) at position 3"),
    (2, 4, 8, 2.5, "softmax_xent label: non-integral id at position 3"),
    (1, 1, 8, -1.0, "softmax_xent label: id -1 out of range [0,10) at position 3"),
    (0, 2, 8, 2.0, "softmax_xent label: id 2 out of range [0,2) at position 3"),
    (3, 4, 2, 10.0, "softmax_xent label: id 10 out of range [0,10) at position 1"),
])
def test_label_errors(P, kind, strat, B, bad, msg):
    desc = P.build_desc(P.ModelKind(kind))
    data = P.synth_for_model(desc, B, 0)
    y = data.labels.copy()
    y[min(3, B - 1)] = bad
    eng, model = _expect_index_error(P, desc, strat, data.inputs, y, msg)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, 0)


def test_index_messages_match_compiled_reference(P, O):
    """The same bad inputs through the unmodified reference (oracle/_ref):
    identical IndexError text."""
    if not O.ref_available():
        pytest.skip("compiled reference not built")
    desc, data = _embed(P)
    od = O.build_desc(O.EMBED, seq_len=16, vocab=50, hidden=8)
    p = O.ref_init_params(od, 0, np.float32)
    for pos, val in [((2, 5), 3.5), ((1, 3), 50.0)]:
        x = data.inputs.copy()
        x[pos] = val
        R = O.RefModel(od, O.JACMM, 4, p, np.float32)
        with pytest.raises(O.OracleError) as ref_err:
            R.step(x, data.labels, 1.0, 1.1, 0.1, 1, 0, 0)
        model = P.build_from_desc(desc, 0)
        eng = P.GradEngine(model, P.Strategy.jacmm, 4)
        with pytest.raises(Exception) as ours:
            P.dpsgd_step(model, eng, x, data.labels,
                         P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1), 0)
        ref_msg = str(ref_err.value).split("] ", 1)[1]  # OracleError: "[code] what()"
        assert str(ours.value) == ref_msg, (str(ours.value), ref_msg)
