"""The embedding block's aggregation kernels (BASELINE config 5, the sparse
per-example gradient path): embed_agg4_kernel (four elements per lane, the
example list built in parallel) against embed_agg_kernel (scalar,
PGB_EMB_AGG_SCALAR=1), bitwise -- they perform the same fp32 operations per
element in the same ascending example order (dpsgd.cpp:287-317) and draw the
same noise pairs (kernels.hpp:597-614) -- in the one-process step (mode 0) and
the data-parallel schedule (mode 1, a one-rank NCCL communicator), plus the
small config against the oracle with the vector kernel on.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _engine(P, desc, B, monkeypatch, scalar, dist=False):
    model = P.build_from_desc(desc, 0)
    if scalar:
        monkeypatch.setenv("PGB_EMB_AGG_SCALAR", "1")
    if dist:
        from paper_2010_09063_b200.dist import nccl_unique_id
        monkeypatch.setenv("PGB_FORCE_DIST", "1")
        eng = P.GradEngine(model, P.Strategy.jacmm, B, rank=0, world=1,
                           unique_id=nccl_unique_id())
        monkeypatch.delenv("PGB_FORCE_DIST")
    else:
        eng = P.GradEngine(model, P.Strategy.jacmm, B)
    if scalar:
        monkeypatch.delenv("PGB_EMB_AGG_SCALAR")
    return model, eng


@pytest.mark.parametrize("dist", [False, True], ids=["step", "dist"])
@pytest.mark.parametrize("shape", [(512, 256, 10004, 100), (64, 32, 300, 132), (40, 17, 97, 8)],
                         ids=["config5", "E132", "small"])
def test_embed_agg_vector_kernel_bitwise_scalar(P, shape, dist, monkeypatch):
    B, L, V, E = shape
    desc = P.build_desc(P.ModelKind.embed, P.ModelOptions(seq_len=L, vocab=V, hidden=E))
    data = P.synth_for_model(desc, 3 * B, 5)
    cfg = P.DpConfig(clip_norm=0.05, noise_multiplier=1.1, learning_rate=0.5, seed=3)
    m_v, e_v = _engine(P, desc, B, monkeypatch, scalar=False, dist=dist)
    m_s, e_s = _engine(P, desc, B, monkeypatch, scalar=True, dist=dist)
    for s in range(3):
        sl = slice(s * B, (s + 1) * B)
        rv = P.dpsgd_step(m_v, e_v, data.inputs[sl], data.labels[sl], cfg, 7 + s)
        rs = P.dpsgd_step(m_s, e_s, data.inputs[sl], data.labels[sl], cfg, 7 + s)
        np.testing.assert_array_equal(rv.pre_clip_norms, rs.pre_clip_norms)
        assert rv.clipped_count == rs.clipped_count
        np.testing.assert_array_equal(m_v.flat_params(), m_s.flat_params())


def test_embed_agg_vector_kernel_matches_oracle(P, O):
    B, L, V, E = 16, 24, 60, 12
    desc = P.build_desc(P.ModelKind.embed, P.ModelOptions(seq_len=L, vocab=V, hidden=E))
    od = O.build_desc(4, seq_len=L, vocab=V, hidden=E)
    model = P.build_from_desc(desc, 0)
    eng = P.GradEngine(model, P.Strategy.jacmm, B)
    data = P.synth_for_model(desc, B, 0)
    x64, y64 = O.synth(od, B, 0)
    p64 = O.init_params(od, 0)
    np.testing.assert_array_equal(data.inputs, x64.astype(np.float32))
    cfg = P.DpConfig(clip_norm=0.05, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    for step in range(3):
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, step)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64, y64, p64, 0.05, 1.1, 0.1, 1, 0, step)
        assert np.max(np.abs(rep.pre_clip_norms - wn) / wn) < TOL
        assert rep.clipped_count == wclip
        got = model.flat_params().astype(np.float64)
        delta = np.abs(p_new - p64).max()
        assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)
        p64 = p_new
