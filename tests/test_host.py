"""Host side of the product, no GPU needed: the C-ABI library loads and
exports every symbol include/pegrad_b200.h declares; model descriptions,
parameter init and synthetic data are bit-identical to the reference; config
validation and the strategy support matrix raise the reference's errors."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "pegrad_b200.h")).read()
    return sorted(set(re.findall(r"\b(pgb_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(P):
    lib = C.CDLL(os.path.join(ROOT, "paper_2010_09063_b200", "libpegrad_b200.so"))
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares each of them
    from paper_2010_09063_b200 import _lib
    assert not [s for s in syms if s not in _lib.EXPORTS]
    assert b"sm_100a" in P.lib.pgb_version()


def test_library_is_sm100a_native():
    so = os.path.join(ROOT, "paper_2010_09063_b200", "libpegrad_b200.so")
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("kind,count", [(0, 105), (1, 5760), (2, 26010), (3, 605226),
                                        (4, 160098), (5, 1081002)])
def test_param_counts(P, kind, count):
    """proj/tests/test_models.cpp:26-35."""
    d = P.build_desc(P.ModelKind(kind))
    assert d.param_count() == count
    assert P.lib.pgb_param_count(C.byref(d.to_c())) == count


def test_param_names_and_shapes(P):
    d = P.build_desc(P.ModelKind.mnist_cnn)
    assert d.param_names == ["l0.W", "l0.b", "l3.W", "l3.b", "l6.W", "l6.b", "l8.W", "l8.b"]
    assert d.param_shapes[0] == (16, 1, 8, 8) and d.param_shapes[4] == (512, 32)
    e = P.build_desc(P.ModelKind.embed, P.ModelOptions(hidden=100))
    assert e.param_names[0] == "l0.table" and e.param_shapes[0] == (10004, 100)


@pytest.mark.parametrize("kind,opts", [(0, {}), (1, {}), (2, {}), (3, {}),
                                       (4, dict(seq_len=16, vocab=50, hidden=8))])
def test_init_and_synth_bit_identical_to_oracle(P, O, kind, opts):
    d = P.build_desc(P.ModelKind(kind), P.ModelOptions(**opts))
    od = O.build_desc(kind, **opts)
    np.testing.assert_array_equal(P.build_from_desc(d, 5).flat_params(),
                                  O.init_params(od, 5, np.float32))
    ds = P.synth_for_model(d, 37, 2)
    x, y = O.synth(od, 37, 2, np.float32)
    np.testing.assert_array_equal(ds.inputs, x)
    np.testing.assert_array_equal(ds.labels, y)


def test_synth_matches_reference_fixture(P):
    import hashlib
    g = np.load(os.path.join(ROOT, "tests", "golden", "mnist_cnn.npz"))
    ds = P.synth_for_model(P.build_desc(P.ModelKind.mnist_cnn), int(g["B"]), 0)
    assert hashlib.sha256(ds.inputs.tobytes()).hexdigest() == str(g["x_sha"])
    assert hashlib.sha256(ds.labels.tobytes()).hexdigest() == str(g["y_sha"])


def test_validate_config_errors(P):
    """proj/tests/test_dpsgd.cpp:285-296, dpsgd.cpp:36-51."""
    from paper_2010_09063_b200.errors import ConfigError
    with pytest.raises(ConfigError, match="clip norm must be positive"):
        P.validate(P.DpConfig(clip_norm=0.0), 8)
    with pytest.raises(ConfigError, match="must divide the batch size 8"):
        P.validate(P.DpConfig(microbatch=3), 8)
    P.validate(P.DpConfig(microbatch=4), 8)
    with pytest.raises(ConfigError, match="non-negative"):
        P.validate(P.DpConfig(noise_multiplier=-1.0), 8)
    with pytest.raises(ConfigError, match="learning rate"):
        P.validate(P.DpConfig(learning_rate=0.0), 8)


def test_strategy_support_matrix_is_enforced_before_device_work(P):
    """strategies.cpp:76-113: 'unsupported layer' raised at engine creation;
    the check runs before any CUDA call, so it holds on a CPU-only host."""
    from paper_2010_09063_b200.errors import UnsupportedError
    for kind, strat in [(P.ModelKind.mnist_cnn, P.Strategy.outer),
                        (P.ModelKind.mnist_cnn, P.Strategy.norms),
                        (P.ModelKind.embed, P.Strategy.groupconv),
                        (P.ModelKind.lstm, P.Strategy.jacmm)]:
        d = P.build_desc(kind)
        h = C.c_void_p()
        st = P.lib.pgb_engine_create(C.byref(d.to_c()), int(strat), 4, 0, C.byref(h))
        assert st == 6
        assert P.lib.pgb_last_error().startswith(b"unsupported layer: ")
        with pytest.raises(UnsupportedError):
            P._lib.check(st)


def test_unknown_model_kind(P):
    from paper_2010_09063_b200.errors import ConfigError
    d = P._lib.ModelDescC()
    st = P.lib.pgb_build_desc(17, None, C.byref(d))
    with pytest.raises(ConfigError, match="unknown model kind"):
        P._lib.check(st)


def test_bad_geometry_is_a_shape_error(P):
    """conv_out_extent rejects non-integral extents (kernels.hpp:400-410): the
    BASELINE 'conv32 4x4/2' after the stride-2 pool is not representable."""
    from paper_2010_09063_b200.errors import ShapeError
    L = P.LayerSpec
    K = P.LayerKind
    with pytest.raises(ShapeError, match="integral extent"):
        layers = [L(K.conv, 1, 16, 8, 2, 3), L(K.relu), L(K.maxpool, 0, 0, 2, 2),
                  L(K.conv, 16, 32, 4, 2, 0), L(K.relu), L(K.flatten), L(K.dense, 128, 10)]
        d = P.custom_desc(P.ModelKind.mnist_cnn, layers, (1, 28, 28), 10)
        h = C.c_void_p()
        P._lib.check(P.lib.pgb_engine_create(C.byref(d.to_c()), 4, 4, 0, C.byref(h)))


def test_noise_stream_ids(P):
    assert P.noise_stream(0, 0) == 1 << 32
    assert P.noise_stream(3, 5) == (1 << 32) + 3 * 4096 + 5


def test_shard_bounds():
    from paper_2010_09063_b200.dist import shard_bounds
    assert [shard_bounds(r, 4, 256) for r in range(4)] == [(0, 64), (64, 128), (128, 192),
                                                           (192, 256)]
    with pytest.raises(ValueError):
        shard_bounds(0, 3, 256)


def test_cpp_shim_header_compiles_and_links():
    """include/pegrad_b200.hpp + the C ABI link against the product .so."""
    import subprocess
    import tempfile
    libdir = os.path.join(ROOT, "paper_2010_09063_b200")
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-L", libdir,
                        "-lpegrad_b200", "-o", os.path.join(d, "t")], check=True)
