"""IDX ingest (io::load_idx / load_mnist, proj/core/src/dataset.cpp:35-112) and
the BenchRecord JSON / CSV emitters (proj/core/src/harness.cpp:219-317),
checked against the compiled reference (oracle/_ref) on the same files."""
import os
import struct

import numpy as np
import pytest


def _write_idx(path, arr, magic=None):
    arr = np.asarray(arr, np.uint8)
    m = magic if magic is not None else (0x0800 | arr.ndim)
    with open(path, "wb") as f:
        f.write(struct.pack(">I", m))
        for d in arr.shape:
            f.write(struct.pack(">I", d))
        f.write(arr.tobytes())


@pytest.fixture
def mnist_dir(tmp_path):
    rng = np.random.default_rng(7)
    _write_idx(tmp_path / "train-images-idx3-ubyte", rng.integers(0, 256, (37, 28, 28)))
    _write_idx(tmp_path / "train-labels-idx1-ubyte", rng.integers(0, 10, 37))
    return tmp_path


def test_load_idx_matches_reference(P, O, mnist_dir):
    if not O.ref_available():
        pytest.skip("compiled reference not built")
    for name, div in (("train-images-idx3-ubyte", 255.0), ("train-labels-idx1-ubyte", 0.0)):
        path = str(mnist_dir / name)
        got = P.load_idx(path, div)
        want, dims = O.ref_load_idx(path)
        assert got.shape == dims
        if div:
            want = want / np.float32(255)
        np.testing.assert_array_equal(got.reshape(-1), want)


def test_load_mnist_dataset(P, mnist_dir):
    d = P.load_mnist(str(mnist_dir))
    assert d.inputs.shape == (37, 1, 28, 28) and d.labels.shape == (37,)
    assert d.name == "mnist-train" and d.classes == 10 and d.count == 37
    assert float(d.inputs.max()) <= 1.0 and float(d.inputs.min()) >= 0.0


@pytest.mark.parametrize("case", ["magic", "rank", "truncated_dims", "size", "short"])
def test_load_idx_format_errors_match_reference(P, O, tmp_path, case):
    path = str(tmp_path / "bad")
    if case == "magic":
        _write_idx(path, np.zeros((2, 2)), magic=0x00000D02)
    elif case == "rank":
        _write_idx(path, np.zeros(3), magic=0x00000805)
    elif case == "truncated_dims":
        with open(path, "wb") as f:
            f.write(struct.pack(">II", 0x00000803, 5))
    elif case == "size":
        _write_idx(path, np.zeros((3, 4)))
        with open(path, "ab") as f:
            f.write(b"\0")
    else:
        with open(path, "wb") as f:
            f.write(b"\0\0")
    with pytest.raises(P.errors.FormatError) as ours:
        P.load_idx(path)
    if O.ref_available():
        with pytest.raises(O.OracleError) as theirs:
            O.ref_load_idx(path)
        assert theirs.value.code == 8  # FormatError
        # the same message, byte offset included
        assert str(ours.value).split("load_idx:")[1] == str(theirs.value).split("load_idx:")[1]


def test_load_idx_missing_file(P, tmp_path):
    with pytest.raises(P.errors.IoError):
        P.load_idx(str(tmp_path / "nope"))


def _records(P):
    return [P.BenchRecord(model="mnist_cnn", strategy="groupconv", mode="graph", vectorized=True,
                          batch_size=256, epochs=3, median_epoch_seconds=0.0276,
                          epoch_seconds=[0.0281, 0.0276, 0.027501],
                          peak_planned_bytes=62914560,
                          optimizer_report=P.OptimizerReport(1, 2, 3, 4, 0.125), seed=0,
                          element_width=32, status="ok", reason=""),
            P.BenchRecord(model="lstm", strategy="groupconv", batch_size=16, status="skip",
                          reason="unsupported layer", vectorized=False)]


def test_records_json_round_trips_through_reference(P, O):
    recs = _records(P)
    text = P.records_to_json(recs)
    assert P.records_from_json(text) == recs
    if not O.ref_available():
        pytest.skip("compiled reference not built")
    # the reference parses our file and re-emits the identical text
    assert O.ref_records_json_roundtrip(text) == text


def test_emit_json_csv_files(P, tmp_path):
    recs = _records(P)
    P.emit_json(recs, str(tmp_path / "r.json"))
    assert P.parse_json_file(str(tmp_path / "r.json")) == recs
    P.emit_csv(recs, str(tmp_path / "r.csv"))
    lines = open(tmp_path / "r.csv").read().splitlines()
    assert lines[0].startswith("model,strategy,mode,vectorized,batch_size")
    assert lines[1].split(",")[7] == "0.0281;0.0276;0.027501"
    assert len(lines) == 3
    with pytest.raises(P.errors.ContractError):
        P.emit_json([], str(tmp_path / "e.json"))


@pytest.mark.gpu
def test_load_idx_device_decode_matches_host(P, mnist_dir):
    """The device path ships the IDX payload as bytes and decodes on the GPU:
    bitwise the host loader's floats."""
    for name, div in (("train-images-idx3-ubyte", 255.0), ("train-labels-idx1-ubyte", 0.0)):
        path = str(mnist_dir / name)
        host = P.load_idx(path, div)
        dev = P.load_idx(path, div, device=0)
        np.testing.assert_array_equal(dev.cpu().numpy(), host)
    d = P.load_mnist(str(mnist_dir), device=0)
    assert tuple(d.inputs.shape) == (37, 1, 28, 28) and d.inputs.is_cuda
