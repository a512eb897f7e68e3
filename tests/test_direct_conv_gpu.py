"""The few-channel first layer on the CUDA cores (conv3x3_smallc_fwd_kernel,
conv3x3_smallc_dw_kernel: staged input rows walked as a three-row register
window, per-warp cotangent slices, shared-memory column sums) over channel
counts 1-4, ragged heights and output-channel counts that leave a warp's
second channel empty (D % 2 != 0 is not a model the reference builds, but
D % 32 != 0 and D % 16 != 0 are): per-example gradients and norms of a
conv -> relu -> conv -> relu -> global-avgpool model against the oracle
(the per-example dW of proj/core/src/strategies.cpp:156-170)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _step_kernels(P, eng, data):
    """Kernel labels of one profiled step (pgb_profile_steps) of the engine."""
    import ctypes as C
    import torch
    from paper_2010_09063_b200 import _lib
    dx = torch.from_numpy(data.inputs).cuda()
    dy = torch.from_numpy(data.labels).cuda()
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0).to_c()
    nk = C.c_int32()
    ms = (C.c_float * 64)()
    names = C.create_string_buffer(64 * 32)
    _lib.check(_lib.lib.pgb_profile_steps(eng.handle, C.c_void_p(dx.data_ptr()),
                                          C.c_void_p(dy.data_ptr()), C.byref(cfg), 0, 1, 64,
                                          C.cast(ms, C.c_void_p), C.cast(names, C.c_void_p),
                                          C.byref(nk)))
    return {names.raw[32 * k:32 * k + 32].split(b"\0")[0].decode() for k in range(nk.value)}


@pytest.mark.parametrize("C,H,D", [(1, 32, 16), (2, 20, 20), (3, 32, 32), (4, 9, 48), (3, 32, 24)])
def test_first_layer_direct_dw_matches_oracle(P, O, C, H, D):
    W = 32  # the direct per-example dW kernel's map width
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
    # the schedule really ran the CUDA-core first-layer kernels
    names = _step_kernels(P, eng, data)
    assert "conv_dw_pex_direct" in names, names
    if D % 16 == 0:
        assert "conv_fwd_direct" in names, names
    # a full step through the same kernels (norm partials, clip, update)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=0)
    x64, y64 = O.synth(od, B, 0)
    p64 = O.init_params(od, 0)
    rep = P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, 0)
    p_new, wn2, wclip, _ = O.dpsgd_step(od, x64, y64, p64, 1.0, 1.1, 0.1, 1, 0, 0)
    assert np.max(np.abs(rep.pre_clip_norms - wn2) / wn2) < 1e-5
    assert rep.clipped_count == wclip
    got = model.flat_params().astype(np.float64)
    delta = np.abs(p_new - p64).max()
    assert np.all(np.abs(got - p_new) <= 3e-7 * np.abs(p_new) + 1e-5 * delta)
