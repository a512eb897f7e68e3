"""The data-parallel schedule executed on one GPU.

PGB_FORCE_DIST=1 makes pgb_engine_create_dist build a one-rank NCCL
communicator and run the real multi-GPU step: aggregate_kernel in mode 1 (the
rank's clipped sum), ncclAllReduce of that sum and of the clip count, then
noise_update_kernel (shared-seed noise, mean over the global units, update).
Reference basis: proj/core/src/dpsgd.cpp:244-330 (examples are independent;
one noised sum per step).

Checks:
* against the oracle (norms rel 1e-5, exact clip counts, parameters within a
  few ulps + 1e-5 of the update), for the fused MNIST kernel, the fused dense
  kernel and the layer-wise (CIFAR) schedule;
* bitwise against the one-process step (the all-reduce of one rank is the
  identity, and noise_update_kernel performs the aggregation epilogue's exact
  fp32 operations);
* the multi-step CUDA graphs with the all-reduce captured inside
  (pgb_run_steps_device, pgb_run_epoch) bitwise against step calls.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5

CASES = [
    # (name, kind, options, batch, strategy)
    ("mnist_cnn", 2, {}, 32, 4),
    ("fcnn", 1, {}, 32, 1),
    ("cifar_cnn", 3, {}, 4, 4),
]


def _dist_engine(P, model, strat, B, monkeypatch):
    from paper_2010_09063_b200.dist import nccl_unique_id
    monkeypatch.setenv("PGB_FORCE_DIST", "1")
    eng = P.GradEngine(model, P.Strategy(strat), B, rank=0, world=1,
                       unique_id=nccl_unique_id())
    monkeypatch.delenv("PGB_FORCE_DIST")
    return eng


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_dist_schedule_matches_oracle_and_single_process(P, O, case, monkeypatch):
    name, kind, opts, B, strat = case
    desc = P.build_desc(P.ModelKind(kind), P.ModelOptions(**opts))
    od = O.build_desc(kind, **opts)
    data = P.synth_for_model(desc, B, 0)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    md = P.build_from_desc(desc, 0)
    ed = _dist_engine(P, md, strat, B, monkeypatch)
    assert ed.info().world == 1
    m1 = P.build_from_desc(desc, 0)
    e1 = P.GradEngine(m1, P.Strategy(strat), B)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 0)
    for step in range(3):
        rd = P.dpsgd_step(md, ed, data.inputs, data.labels, cfg, step)
        r1 = P.dpsgd_step(m1, e1, data.inputs, data.labels, cfg, step)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64, y64, p64, 1.0, 1.1, 0.1, 1, 0, step)
        assert np.max(np.abs(rd.pre_clip_norms - wn) / wn) < TOL
        assert rd.clipped_count == wclip == r1.clipped_count
        got = md.flat_params()
        delta = np.abs(p_new - p64).max()
        assert np.all(np.abs(got.astype(np.float64) - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)
        np.testing.assert_array_equal(got, m1.flat_params())
        np.testing.assert_array_equal(rd.pre_clip_norms, r1.pre_clip_norms)
        assert rd.noise_streams == r1.noise_streams
        p64 = p_new


@pytest.mark.parametrize("sigma", [0.0, 1.1])
def test_dist_clipped_sum_probe(P, O, sigma, monkeypatch):
    """The noise-free clipped sum of the rank (the all-reduce input) and a
    sigma = 0 step through the dist schedule, against the oracle."""
    B = 16
    desc = P.build_desc(P.ModelKind.mnist_cnn)
    od = O.build_desc(O.MNIST_CNN)
    data = P.synth_for_model(desc, B, 2)
    model = P.build_from_desc(desc, 0)
    eng = _dist_engine(P, model, 4, B, monkeypatch)
    got, norms, nclip = eng.clipped_sum(data.inputs, data.labels, 0.8)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 2)
    p_new, wn, wclip, want = O.dpsgd_step(od, x64, y64, p64, 0.8, sigma, 0.1, 1, 4, 5)
    assert np.max(np.abs(norms - wn) / wn) < TOL
    assert nclip == wclip
    off = 0
    for n in od.blocks:
        w = want[off:off + n]
        assert np.linalg.norm(got[off:off + n] - w) <= TOL * np.linalg.norm(w)
        off += n
    cfg = P.DpConfig(clip_norm=0.8, noise_multiplier=sigma, learning_rate=0.1, seed=4)
    rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, 5)
    assert rep.clipped_count == wclip
    delta = np.abs(p_new - p64).max()
    got = model.flat_params().astype(np.float64)
    assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)


@pytest.mark.parametrize("kind,B,strat,row", [(2, 64, 4, 784), (1, 64, 1, 104)])
def test_dist_multistep_graphs_match_step_calls(P, O, kind, B, strat, row, monkeypatch):
    """pgb_run_steps_device with the NCCL all-reduce captured inside the
    static multi-step graphs (full chunks + a remainder graph) equals the same
    steps one call at a time, bitwise; pgb_prepare_steps builds the graphs
    beforehand without changing the result."""
    torch = pytest.importorskip("torch")
    from paper_2010_09063_b200 import _lib
    NB, STEPS = 5, 21
    desc = P.build_desc(P.ModelKind(kind))
    data = P.synth_for_model(desc, B * NB, 0)
    dx = torch.from_numpy(data.inputs).cuda()
    dy = torch.from_numpy(data.labels).cuda()
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0).to_c()
    out = []
    for mode in ("steps", "calls", "single"):
        model = P.build_from_desc(desc, 0)
        if mode == "single":
            eng = P.GradEngine(model, P.Strategy(strat), B)
        else:
            eng = _dist_engine(P, model, strat, B, monkeypatch)
        if mode in ("steps", "single"):
            _lib.check(_lib.lib.pgb_prepare_steps(eng.handle, C.c_void_p(dx.data_ptr()),
                                                  C.c_void_p(dy.data_ptr()), NB, STEPS,
                                                  C.byref(cfg)))
            n = C.c_int64()
            _lib.check(_lib.lib.pgb_run_steps_device(eng.handle, C.c_void_p(dx.data_ptr()),
                                                     C.c_void_p(dy.data_ptr()), NB, STEPS,
                                                     C.byref(cfg), 3, C.byref(n)))
            assert n.value >= STEPS
        else:
            for i in range(STEPS):
                b = (3 + i) % NB
                _lib.check(_lib.lib.pgb_dpsgd_step_device(
                    eng.handle, C.c_void_p(dx.data_ptr() + b * B * row * 4),
                    C.c_void_p(dy.data_ptr() + b * B * 4), C.byref(cfg), 3 + i))
        _lib.check(_lib.lib.pgb_synchronize(eng.handle, None, None))
        out.append(eng.get_flat_params())
    np.testing.assert_array_equal(out[0], out[1])
    np.testing.assert_array_equal(out[0], out[2])


def test_dist_epoch_driver_matches_single_process(P, O, monkeypatch):
    """pgb_run_epoch through the dist schedule (chunk graphs with the
    all-reduce inside, the clip count reduced into its result slot) equals
    the one-process epoch: parameters, norms and clip total."""
    B = 64
    desc = P.build_desc(P.ModelKind.mnist_cnn)
    data = P.synth_for_model(desc, 21 * B, 1)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=3)
    res = []
    for dist in (True, False):
        model = P.build_from_desc(desc, 0)
        eng = (_dist_engine(P, model, 4, B, monkeypatch) if dist
               else P.GradEngine(model, P.Strategy.groupconv, B))
        norms = np.empty(21 * B, np.float32)
        _, clipped = P.run_epoch(eng, model, data, cfg, 7, norms)
        res.append((model.flat_params(), norms, clipped))
    np.testing.assert_array_equal(res[0][0], res[1][0])
    np.testing.assert_array_equal(res[0][1], res[1][1])
    assert res[0][2] == res[1][2]
