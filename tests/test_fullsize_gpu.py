"""Parity at the benchmarked sizes (BASELINE: MNIST CNN at batch 256), through
every entry point bench.py times:

* pgb_dpsgd_step (host buffers, the reference-shaped step call);
* pgb_dpsgd_step_device on device-resident batches at changing addresses (the
  CUDA-graph replay whose per-step arguments are kernel-node updates);
* pgb_run_epoch (the pipelined epoch driver with its device result ring);

each against the oracle (C restatement of the reference, pinned to the
compiled reference in test_oracle.py) on the same seeds. CIFAR at batch 256 is
too slow for the CPU oracle, so there the check is a size-independent property:
the batch-256 clipped sum and norms equal those of batch-8 engines over the
same examples (which are themselves checked against the oracle at B = 8 in
test_parity_gpu.py).

Tolerances as in test_parity_gpu.py: norms element-wise rel 1e-5; parameters a
few fp32 ulps plus 1e-5 of the update; clipped sums per-block normwise 1e-5.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _mnist(P, O, B):
    desc = P.build_desc(P.ModelKind.mnist_cnn)
    od = O.build_desc(O.MNIST_CNN)
    return desc, od


def _check_params(got, p_new, p_old):
    delta = np.abs(p_new - p_old).max()
    assert np.all(np.abs(got.astype(np.float64) - p_new) <= 3e-7 * np.abs(p_new) + TOL * delta)


def test_mnist_b256_steps_match_oracle(P, O):
    B = 256
    desc, od = _mnist(P, O, B)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, 2 * B, 0)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, 2 * B, 0)
    for step in range(3):
        sl = slice((step % 2) * B, (step % 2 + 1) * B)
        rep = P.dpsgd_step(model, eng, data.inputs[sl], data.labels[sl], cfg, step)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64[sl], y64[sl], p64, 1.0, 1.1, 0.1, 1, 0, step)
        assert np.max(np.abs(rep.pre_clip_norms - wn) / wn) < TOL
        assert rep.clipped_count == wclip
        _check_params(model.flat_params(), p_new, p64)
        p64 = p_new


def test_mnist_b256_clipped_sum_matches_oracle(P, O):
    B = 256
    desc, od = _mnist(P, O, B)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    got, norms, nclip = eng.clipped_sum(data.inputs, data.labels, 1.0)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 0)
    _, wn, wclip, want = O.dpsgd_step(od, x64, y64, p64, 1.0, 0.0, 0.1, 1, 0, 0)
    assert np.max(np.abs(norms - wn) / wn) < TOL
    assert nclip == wclip
    off = 0
    for n in od.blocks:
        w = want[off:off + n]
        assert np.linalg.norm(got[off:off + n] - w) <= TOL * np.linalg.norm(w)
        off += n


def test_mnist_b256_device_steps_match_oracle(P, O):
    """The bench.py path: batches already on the device, read in place by the
    graph (the fused kernel's input pointers are node-parameter updates)."""
    torch = pytest.importorskip("torch")
    from paper_2010_09063_b200 import _lib
    B, nb = 256, 3
    desc, od = _mnist(P, O, B)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, nb * B, 0)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=5)
    dx = torch.from_numpy(data.inputs).cuda()
    dy = torch.from_numpy(data.labels).cuda()
    row = 28 * 28
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, nb * B, 0)
    order = [0, 2, 1, 2]
    for step, b in enumerate(order):
        _lib.check(_lib.lib.pgb_dpsgd_step_device(
            eng.handle, C.c_void_p(dx.data_ptr() + b * B * row * 4),
            C.c_void_p(dy.data_ptr() + b * B * 4), C.byref(cfg.to_c()), 100 + step))
        sl = slice(b * B, (b + 1) * B)
        p64, wn, wclip, _ = O.dpsgd_step(od, x64[sl], y64[sl], p64, 1.0, 1.1, 0.1, 1, 5,
                                         100 + step)
    norms = np.empty(B, np.float32)
    rep = _lib.StepReportC()
    _lib.check(_lib.lib.pgb_synchronize(eng.handle, _lib.ptr(norms), C.byref(rep)))
    assert np.max(np.abs(norms - wn) / wn) < TOL
    assert rep.clipped_count == wclip
    got = eng.get_flat_params().astype(np.float64)
    p0 = O.init_params(od, 0)
    assert np.linalg.norm(got - p64) <= TOL * np.linalg.norm(p64 - p0)


def test_mnist_b256_epoch_driver_matches_oracle(P, O):
    B, steps = 256, 4
    desc, od = _mnist(P, O, B)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, steps * B, 0, pinned=True)
    eng = P.GradEngine(model, P.Strategy.groupconv, B)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    norms = np.empty(steps * B, np.float32)
    _, clipped = P.run_epoch(eng, model, data, cfg, 40, norms)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, steps * B, 0)
    total = 0
    for s in range(steps):
        sl = slice(s * B, (s + 1) * B)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64[sl], y64[sl], p64, 1.0, 1.1, 0.1, 1, 0, 40 + s)
        assert np.max(np.abs(norms[sl] - wn) / wn) < TOL, f"step {s}"
        total += wclip
        p_prev, p64 = p64, p_new
    assert clipped == total
    _check_params(eng.get_flat_params(), p64, p_prev)


def test_cifar_b256_matches_batch8_engines(P, O):
    """Size-independent property at the CIFAR config's batch: per-example
    norms and the clipped sum of a batch-256 engine equal the same quantities
    assembled from batch-8 engines (different grids and tilings)."""
    B, b = 256, 8
    desc = P.build_desc(P.ModelKind.cifar_cnn)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    big = P.GradEngine(model, P.Strategy.groupconv, B)
    got, norms, nclip = big.clipped_sum(data.inputs, data.labels, 1.0)
    small = P.GradEngine(model, P.Strategy.groupconv, b)
    want = np.zeros_like(got, dtype=np.float64)
    wnorms = np.empty(B, np.float32)
    wclip = 0
    for i in range(0, B, b):
        s, n, c = small.clipped_sum(data.inputs[i:i + b], data.labels[i:i + b], 1.0)
        want += s
        wnorms[i:i + b] = n
        wclip += c
    assert np.max(np.abs(norms - wnorms) / wnorms) < TOL
    assert nclip == wclip
    od = O.build_desc(O.CIFAR_CNN)
    off = 0
    for n in od.blocks:
        w = want[off:off + n]
        assert np.linalg.norm(got[off:off + n] - w) <= TOL * np.linalg.norm(w)
        off += n


def test_mnist_run_steps_device_matches_step_calls(P, O):
    """pgb_run_steps_device (static multi-step graphs, step index and batch
    picked on the device) gives bitwise the parameters of the same steps
    issued one pgb_dpsgd_step_device call at a time, including a remainder
    that does not fill a graph."""
    torch = pytest.importorskip("torch")
    from paper_2010_09063_b200 import _lib
    B, NB, STEPS = 256, 5, 19
    desc, od = _mnist(P, O, B)
    data = P.synth_for_model(desc, B * NB, 0)
    dx = torch.from_numpy(data.inputs).cuda()
    dy = torch.from_numpy(data.labels).cuda()
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0).to_c()
    out = []
    for mode in ("steps", "calls"):
        model = P.build_from_desc(desc, 0)
        eng = P.GradEngine(model, P.Strategy.groupconv, B)
        if mode == "steps":
            n = C.c_int64()
            _lib.check(_lib.lib.pgb_run_steps_device(eng.handle, C.c_void_p(dx.data_ptr()),
                                                     C.c_void_p(dy.data_ptr()), NB, STEPS,
                                                     C.byref(cfg), 3, C.byref(n)))
            assert n.value >= STEPS
        else:
            for i in range(STEPS):
                b = (3 + i) % NB
                _lib.check(_lib.lib.pgb_dpsgd_step_device(
                    eng.handle, C.c_void_p(dx.data_ptr() + b * B * 784 * 4),
                    C.c_void_p(dy.data_ptr() + b * B * 4), C.byref(cfg), 3 + i))
        _lib.check(_lib.lib.pgb_synchronize(eng.handle, None, None))
        out.append(eng.get_flat_params())
    np.testing.assert_array_equal(out[0], out[1])


def test_mnist_long_graph_run_matches_step_calls(P, O):
    """Cross-step overlap (each step's per-example kernel a programmatic
    dependent of the previous step's aggregation, whose CTAs may start while
    the one before is still updating) leaves no trace: 256 steps through the
    static multi-step graphs equal the same steps one call at a time, bitwise."""
    torch = pytest.importorskip("torch")
    from paper_2010_09063_b200 import _lib
    B, NB, STEPS = 256, 3, 256
    desc, od = _mnist(P, O, B)
    data = P.synth_for_model(desc, B * NB, 1)
    dx = torch.from_numpy(data.inputs).cuda()
    dy = torch.from_numpy(data.labels).cuda()
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.05, seed=9).to_c()
    out = []
    for mode in ("steps", "calls"):
        model = P.build_from_desc(desc, 0)
        eng = P.GradEngine(model, P.Strategy.groupconv, B)
        if mode == "steps":
            n = C.c_int64()
            _lib.check(_lib.lib.pgb_run_steps_device(eng.handle, C.c_void_p(dx.data_ptr()),
                                                     C.c_void_p(dy.data_ptr()), NB, STEPS,
                                                     C.byref(cfg), 0, C.byref(n)))
        else:
            for i in range(STEPS):
                b = i % NB
                _lib.check(_lib.lib.pgb_dpsgd_step_device(
                    eng.handle, C.c_void_p(dx.data_ptr() + b * B * 784 * 4),
                    C.c_void_p(dy.data_ptr() + b * B * 4), C.byref(cfg), i))
        _lib.check(_lib.lib.pgb_synchronize(eng.handle, None, None))
        out.append(eng.get_flat_params())
    np.testing.assert_array_equal(out[0], out[1])


def test_mnist_in_kernel_aggregation_matches(P, O, monkeypatch):
    """PGB_GRID_SYNC=1 (aggregation inside the tensor-core kernel after a grid
    barrier) runs the same tiles in the same order as the aggregation kernel:
    bitwise the same parameters and clip count."""
    B = 256
    desc, od = _mnist(P, O, B)
    data = P.synth_for_model(desc, 2 * B, 0)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    out = []
    monkeypatch.setenv("PGB_C2_PAIRS", "0")  # per-example conv2 rows, as in-kernel
    for flag in (None, "1"):
        if flag:
            monkeypatch.setenv("PGB_GRID_SYNC", flag)
        model = P.build_from_desc(desc, 0)
        eng = P.GradEngine(model, P.Strategy.groupconv, B)
        reps = [P.dpsgd_step(model, eng, data.inputs[s * B:(s + 1) * B],
                             data.labels[s * B:(s + 1) * B], cfg, s).clipped_count
                for s in range(2)]
        out.append((model.flat_params(), reps))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


def test_mnist_conv2_pair_rows_match_per_example_rows(P, O, monkeypatch):
    """The step's default: tc_kernel hands conv2 W to the aggregation as
    clipped pair rows fl(g_2c s_2c) + fl(g_2c+1 s_2c+1). Same norms and clip
    count as the per-example rows (PGB_C2_PAIRS=0); the update differs only by
    the association of the fp32 sum (SURVEY 8(d) tolerance), the other blocks
    bitwise."""
    B = 255  # odd: the last CTA holds one example
    desc, od = _mnist(P, O, B)
    data = P.synth_for_model(desc, B, 3)
    cfg = P.DpConfig(clip_norm=0.5, noise_multiplier=1.1, learning_rate=0.1, seed=5)
    p0 = P.build_from_desc(desc, 0).flat_params()
    out = []
    for flag in ("0", "1"):
        monkeypatch.setenv("PGB_C2_PAIRS", flag)
        model = P.build_from_desc(desc, 0)
        eng = P.GradEngine(model, P.Strategy.groupconv, B)
        rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, 2)
        out.append((model.flat_params(), rep))
    (pa, ra), (pb, rb) = out
    np.testing.assert_array_equal(ra.pre_clip_norms, rb.pre_clip_norms)
    assert ra.clipped_count == rb.clipped_count
    lo = sum(od.blocks[:2])
    hi = lo + od.blocks[2]  # conv2 W
    np.testing.assert_array_equal(np.delete(pa, np.s_[lo:hi]), np.delete(pb, np.s_[lo:hi]))
    delta = np.abs(pa[lo:hi] - p0[lo:hi]).max()
    assert delta > 0
    np.testing.assert_allclose(pb[lo:hi], pa[lo:hi], rtol=0, atol=1e-4 * delta)


def test_embed_full_size_sparse_step_matches_dense_clipped_sum(P, O):
    """BASELINE config 5 shape (V = 10,004, L = 256, E = 100, B = 512): the
    step's sparse embedding path (distinct tokens + counts, per-row example
    bitmaps) gives the same update as the dense per-example stack the
    clipped-sum probe materialises (sigma = 0, p_new = p - lr * sum / B; lr
    large enough that p - p_new carries the sum without fp32 cancellation)."""
    B = 512
    desc = P.build_desc(P.ModelKind.embed, P.ModelOptions(hidden=100))
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    eng = P.GradEngine(model, P.Strategy.jacmm, B)
    p0 = model.flat_params().astype(np.float64)
    got_sum, norms, nclip = eng.clipped_sum(data.inputs, data.labels, 1.0)
    lr = 1000.0
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=0.0, learning_rate=lr, seed=0)
    rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, 0)
    np.testing.assert_allclose(rep.pre_clip_norms, norms, rtol=1e-6)
    assert rep.clipped_count == nclip
    step_sum = (p0 - model.flat_params().astype(np.float64)) * B / lr
    n_emb = 10004 * 100
    want = got_sum[:n_emb].astype(np.float64)
    assert np.linalg.norm(step_sum[:n_emb] - want) <= 1e-5 * np.linalg.norm(want)


@pytest.mark.parametrize("name,kind", [("fcnn", 1), ("logreg", 0)])
def test_dense_run_steps_device_matches_step_calls(P, O, name, kind):
    """Dense models through the fused MLP kernel in static multi-step graphs
    (batch and noise step read on the device): bitwise the parameters of the
    same steps issued one call at a time, with a remainder that does not fill
    a graph."""
    torch = pytest.importorskip("torch")
    from paper_2010_09063_b200 import _lib
    B, NB, STEPS = 64, 3, 21
    desc = P.build_desc(P.ModelKind(kind))
    data = P.synth_for_model(desc, B * NB, 2)
    row = int(np.prod(desc.input_shape))
    dx = torch.from_numpy(data.inputs).cuda()
    dy = torch.from_numpy(data.labels).cuda()
    cfg = P.DpConfig(clip_norm=0.5, noise_multiplier=1.1, learning_rate=0.1, seed=4).to_c()
    out = []
    for mode in ("steps", "calls"):
        model = P.build_from_desc(desc, 0)
        eng = P.GradEngine(model, P.Strategy.outer, B)
        if mode == "steps":
            n = C.c_int64()
            _lib.check(_lib.lib.pgb_run_steps_device(eng.handle, C.c_void_p(dx.data_ptr()),
                                                     C.c_void_p(dy.data_ptr()), NB, STEPS,
                                                     C.byref(cfg), 5, C.byref(n)))
        else:
            for i in range(STEPS):
                b = (5 + i) % NB
                _lib.check(_lib.lib.pgb_dpsgd_step_device(
                    eng.handle, C.c_void_p(dx.data_ptr() + b * B * row * 4),
                    C.c_void_p(dy.data_ptr() + b * B * 4), C.byref(cfg), 5 + i))
        _lib.check(_lib.lib.pgb_synchronize(eng.handle, None, None))
        out.append(eng.get_flat_params())
    np.testing.assert_array_equal(out[0], out[1])


def test_fcnn_epoch_driver_matches_oracle(P, O):
    """pgb_run_epoch on the FCNN (fused MLP kernel, chunk graphs with the
    noise step read on the device) against the oracle, step by step."""
    B, steps = 64, 20
    desc = P.build_desc(P.ModelKind.fcnn)
    od = O.build_desc(O.FCNN)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, steps * B, 0, pinned=True)
    eng = P.GradEngine(model, P.Strategy.norms, B)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    norms = np.empty(steps * B, np.float32)
    _, clipped = P.run_epoch(eng, model, data, cfg, 7, norms)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, steps * B, 0)
    total = 0
    for s in range(steps):
        sl = slice(s * B, (s + 1) * B)
        p_new, wn, wclip, _ = O.dpsgd_step(od, x64[sl], y64[sl], p64, 1.0, 1.1, 0.1, 1, 0, 7 + s)
        assert np.max(np.abs(norms[sl] - wn) / wn) < TOL, f"step {s}"
        total += wclip
        p_prev, p64 = p64, p_new
    assert clipped == total
    _check_params(eng.get_flat_params(), p64, p_prev)


@pytest.mark.parametrize("name", ["embed", "cifar"])
def test_layerwise_epoch_driver_matches_step_calls(P, O, name):
    """pgb_run_epoch on the layer-wise schedule (chunk graphs with each step's
    input pointer baked in, noise step read on the device; head and remainder
    steps launched directly) gives bitwise the parameters, norms and clip
    counts of the same steps issued one dpsgd_step call at a time."""
    if name == "embed":
        desc = P.build_desc(P.ModelKind.embed, P.ModelOptions(seq_len=16, vocab=50, hidden=8))
        B, steps, strat, C_ = 8, 21, P.Strategy.jacmm, 0.05
    else:
        desc = P.build_desc(P.ModelKind.cifar_cnn)
        B, steps, strat, C_ = 4, 19, P.Strategy.groupconv, 1.0
    data = P.synth_for_model(desc, steps * B, 3, pinned=True)
    cfg = P.DpConfig(clip_norm=C_, noise_multiplier=1.1, learning_rate=0.1, seed=2)
    m1 = P.build_from_desc(desc, 0)
    e1 = P.GradEngine(m1, strat, B)
    norms = np.empty(steps * B, np.float32)
    _, clipped = P.run_epoch(e1, m1, data, cfg, 30, norms)
    m2 = P.build_from_desc(desc, 0)
    e2 = P.GradEngine(m2, strat, B)
    total = 0
    for s in range(steps):
        sl = slice(s * B, (s + 1) * B)
        rep = P.dpsgd_step(m2, e2, data.inputs[sl], data.labels[sl], cfg, 30 + s)
        np.testing.assert_array_equal(norms[sl], rep.pre_clip_norms)
        total += rep.clipped_count
    assert clipped == total
    np.testing.assert_array_equal(e1.get_flat_params(), e2.get_flat_params())
