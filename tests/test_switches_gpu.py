"""The round-2 CIFAR / embedding step-path variants against the oracle and
against each other:

* ghost conv norms + clip-scaled summed dW (default) and per-example stacks
  (PGB_NO_GHOST=1), per-example dW on the halo kernel for C >= 16 (default),
  for every layer (PGB_DWH_MIN_C=1; with PGB_NO_GHOST=1 also the 8x8 layers),
  with two accumulators per kernel row (PGB_DWH_ROT=2) or on the register-gather
  GEMM (PGB_NO_DW_HALO=1), the 3-channel first layer's forward and dW on the
  CUDA cores (default) or the gather GEMM (PGB_NO_DIRECT_CONV=1 / _DW=1), halo
  TMA stages (default) and one box per tap, the weight-gradient work on a
  forked graph branch beside the input gradient (default) or in line
  (PGB_NO_DW_FORK=1)
  (PGB_NO_HALO=1), batch-invariant K splits (default) and none
  (PGB_NO_KSPLIT=1): each a full DPSGD step of the CIFAR CNN against the oracle
  (norms rel 1e-5, exact clip counts, parameters within a few ulps + 1e-5 of
  the update);
* the embedding step with the dense head's aggregation on a forked graph
  branch (default) and in line (PGB_NO_EMB_FORK=1): bitwise, through per-call
  steps and the multi-step epoch driver (captured graphs with the fork).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _engine(P, desc, B, strat, monkeypatch, env):
    # env entries: "NAME" (set to 1) or "NAME=VALUE"
    kv = [(e.split("=", 1) + ["1"])[:2] for e in env]
    for k, v in kv:
        monkeypatch.setenv(k, v)
    m = P.build_from_desc(desc, 0)
    e = P.GradEngine(m, P.Strategy(strat), B)
    for k, _ in kv:
        monkeypatch.delenv(k)
    return m, e


@pytest.mark.parametrize("env", [(), ("PGB_NO_GHOST",), ("PGB_NO_HALO",), ("PGB_NO_KSPLIT",),
                                 ("PGB_NO_GHOST", "PGB_NO_HALO"), ("PGB_NO_DW_HALO",),
                                 ("PGB_DWH_MIN_C=1",), ("PGB_DWH_ROT=2",),
                                 ("PGB_NO_GHOST", "PGB_DWH_MIN_C=1"), ("PGB_NO_DIRECT_CONV",),
                                 ("PGB_NO_DIRECT_DW",), ("PGB_NO_DW_FORK",)],
                         ids=["default", "no_ghost", "no_halo", "no_ksplit", "no_ghost_no_halo",
                              "no_dw_halo", "dw_halo_all", "dw_halo_rot2", "no_ghost_dw_halo_all",
                              "no_direct_conv", "no_direct_dw", "no_dw_fork"])
def test_cifar_step_variants_match_oracle(P, O, env, monkeypatch):
    B = 4
    desc = P.build_desc(P.ModelKind.cifar_cnn)
    od = O.build_desc(O.CIFAR_CNN)
    model, eng = _engine(P, desc, B, 4, monkeypatch, env)
    data = P.synth_for_model(desc, B, 0)
    x64, y64 = O.synth(od, B, 0)
    p64 = O.init_params(od, 0)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    for step in range(2):
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, step)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64, y64, p64, 1.0, 1.1, 0.1, 1, 0, step)
        assert np.max(np.abs(rep.pre_clip_norms - wn) / wn) < TOL
        assert rep.clipped_count == wclip
        got = model.flat_params().astype(np.float64)
        delta = np.abs(p_new - p64).max()
        assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)
        p64 = p_new


def test_embed_fork_bitwise_in_line(P, monkeypatch):
    B, L, V, E = 64, 32, 300, 20
    desc = P.build_desc(P.ModelKind.embed, P.ModelOptions(seq_len=L, vocab=V, hidden=E))
    data = P.synth_for_model(desc, 10 * B, 2, pinned=True)
    cfg = P.DpConfig(clip_norm=0.05, noise_multiplier=1.1, learning_rate=0.5, seed=1)
    ma, ea = _engine(P, desc, B, 5, monkeypatch, ())
    mb, eb = _engine(P, desc, B, 5, monkeypatch, ("PGB_NO_EMB_FORK",))
    for s in range(2):
        sl = slice(s * B, (s + 1) * B)
        ra = P.dpsgd_step(ma, ea, data.inputs[sl], data.labels[sl], cfg, s)
        rb = P.dpsgd_step(mb, eb, data.inputs[sl], data.labels[sl], cfg, s)
        np.testing.assert_array_equal(ra.pre_clip_norms, rb.pre_clip_norms)
        assert ra.clipped_count == rb.clipped_count
        np.testing.assert_array_equal(ma.flat_params(), mb.flat_params())
    na = np.empty(10 * B, np.float32)
    nb = np.empty(10 * B, np.float32)
    _, ca = P.run_epoch(ea, ma, data, cfg, 2, na)
    _, cb = P.run_epoch(eb, mb, data, cfg, 2, nb)
    assert ca == cb
    np.testing.assert_array_equal(na, nb)
    np.testing.assert_array_equal(ea.get_flat_params(), eb.get_flat_params())


@pytest.mark.parametrize("C,H,D", [(64, 8, 32), (32, 4, 16)])
def test_first_layer_small_map_conv_step_matches_oracle(P, O, C, H, D):
    """A 3x3 conv on an 8x8 / 4x4 map as the FIRST layer (its input is the
    step input, so it keeps per-example stacks) followed by one that takes the
    ghost path: full DPSGD steps against the oracle."""
    layers = [P.LayerSpec(P.LayerKind.conv, C, D, 3, 1, 1), P.LayerSpec(P.LayerKind.relu),
              P.LayerSpec(P.LayerKind.conv, D, 10, 3, 1, 1), P.LayerSpec(P.LayerKind.relu),
              P.LayerSpec(P.LayerKind.global_avgpool)]
    desc = P.custom_desc(P.ModelKind.cifar_cnn, layers, (C, H, H), 10)
    od = O.custom_desc(O.CIFAR_CNN, [(1, C, D, 3, 1, 1), (6, 0, 0, 0, 1, 0), (1, D, 10, 3, 1, 1),
                                     (6, 0, 0, 0, 1, 0), (4, 0, 0, 0, 1, 0)], (C, H, H), 10)
    B = 6
    model = P.build_from_desc(desc, 0)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    data = P.synth_for_model(desc, B, 0)
    x64, y64 = O.synth(od, B, 0)
    p64 = O.init_params(od, 0)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    for step in range(2):
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, step)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64, y64, p64, 1.0, 1.1, 0.1, 1, 0, step)
        assert np.max(np.abs(rep.pre_clip_norms - wn) / wn) < TOL
        assert rep.clipped_count == wclip
        got = model.flat_params().astype(np.float64)
        delta = np.abs(p_new - p64).max()
        assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)
        p64 = p_new
