"""Epoch drivers — bench::run_bench and bench::train (proj/core/src/harness.cpp:
85-167, 319-382) over the device engine. Timing covers the DPSGD steps only
(engine construction / graph capture are excluded, harness.hpp:31-33)."""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import asdict, dataclass, field
from typing import List

import numpy as np

from . import _lib
from ._lib import check, lib
from .dataset import Dataset, slice_batch
from .dpsgd import DpConfig, dpsgd_step, sgd_step
from .errors import ConfigError, ContractError, IoError, UnsupportedError
from .models import Model, ModelKind, build, model_name
from .strategies import ExecMode, GradEngine, Strategy, strategy_name


@dataclass
class OptimizerReport:
    removed_nodes: int = 0
    fusion_groups: int = 0
    peak_bytes: int = 0
    no_reuse_bytes: int = 0
    trace_seconds: float = 0.0


@dataclass
class BenchRecord:
    model: str = ""
    strategy: str = ""
    mode: str = "graph"
    vectorized: bool = True
    batch_size: int = 0
    epochs: int = 0
    median_epoch_seconds: float = 0.0
    epoch_seconds: List[float] = field(default_factory=list)
    peak_planned_bytes: int = 0
    optimizer_report: OptimizerReport = field(default_factory=OptimizerReport)
    seed: int = 0
    element_width: int = 32
    status: str = "ok"
    reason: str = ""


@dataclass
class RunOptions:
    batch_sizes: List[int] = field(default_factory=lambda: [16, 32, 64, 128, 256])
    epochs: int = 20
    mode: ExecMode = ExecMode.graph
    vectorize: int = -1
    mem_cap_bytes: int = 0
    clip_norm: float = 1.0
    noise_multiplier: float = 1.0
    learning_rate: float = 0.1
    microbatch: int = 1
    seed: int = 0


def _record_to_obj(r: BenchRecord) -> dict:
    d = asdict(r)
    d["vectorized"] = bool(d["vectorized"])
    return d


def records_to_json(records: List[BenchRecord]) -> str:
    """bench::records_to_json (proj/core/src/harness.cpp:219-267): an array of
    records with snake_case keys, the reference's nlohmann layout (sorted keys,
    2-space indent) so either side parses the other's files."""
    if not records:
        raise ContractError("emit: no records")
    return json.dumps([_record_to_obj(r) for r in records], indent=2, sort_keys=True)


def records_from_json(text: str) -> List[BenchRecord]:
    """bench::records_from_json (proj/core/src/harness.cpp:236-274)."""
    out = []
    for j in json.loads(text):
        o = j["optimizer_report"]
        out.append(BenchRecord(
            model=j["model"], strategy=j["strategy"], mode=j["mode"],
            vectorized=bool(j["vectorized"]), batch_size=int(j["batch_size"]),
            epochs=int(j["epochs"]), median_epoch_seconds=float(j["median_epoch_seconds"]),
            epoch_seconds=[float(v) for v in j["epoch_seconds"]],
            peak_planned_bytes=int(j["peak_planned_bytes"]),
            optimizer_report=OptimizerReport(int(o["removed_nodes"]), int(o["fusion_groups"]),
                                             int(o["peak_bytes"]), int(o["no_reuse_bytes"]),
                                             float(o["trace_seconds"])),
            seed=int(j["seed"]), element_width=int(j["element_width"]), status=j["status"],
            reason=j["reason"]))
    return out


def emit_json(records: List[BenchRecord], path: str) -> None:
    """bench::emit_json (proj/core/src/harness.cpp:276-282)."""
    text = records_to_json(records)
    try:
        with open(path, "w") as f:
            f.write(text + "\n")
    except OSError as e:
        raise IoError(f"emit_json: cannot write '{path}'") from e


def parse_json_file(path: str) -> List[BenchRecord]:
    """bench::parse_json_file (proj/core/src/harness.cpp:284-290)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise IoError(f"parse_json_file: cannot read '{path}'") from e
    return records_from_json(text)


def emit_csv(records: List[BenchRecord], path: str) -> None:
    """bench::emit_csv (proj/core/src/harness.cpp:292-317): header plus one line
    per record, the epoch list joined by ';'."""
    if not records:
        raise ContractError("emit: no records")
    head = ("model,strategy,mode,vectorized,batch_size,epochs,median_epoch_seconds,"
            "epoch_seconds,peak_planned_bytes,removed_nodes,fusion_groups,opt_peak_bytes,"
            "no_reuse_bytes,trace_seconds,seed,element_width,status,reason\n")
    g = lambda v: f"{v:g}"  # noqa: E731  (ostream default precision, 6 significant digits)
    try:
        with open(path, "w") as f:
            f.write(head)
            for r in records:
                o = r.optimizer_report
                f.write(",".join([
                    r.model, r.strategy, r.mode, "true" if r.vectorized else "false",
                    str(r.batch_size), str(r.epochs), g(r.median_epoch_seconds),
                    ";".join(g(v) for v in r.epoch_seconds), str(r.peak_planned_bytes),
                    str(o.removed_nodes), str(o.fusion_groups), str(o.peak_bytes),
                    str(o.no_reuse_bytes), g(o.trace_seconds), str(r.seed),
                    str(r.element_width), r.status, r.reason]) + "\n")
    except OSError as e:
        raise IoError(f"emit_csv: cannot write '{path}'") from e


def median(values: List[float]) -> float:
    v = sorted(values)
    n = len(v)
    if n == 0:
        return 0.0
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def run_epoch(engine: GradEngine, model: Model, data: Dataset, cfg: DpConfig, step0: int,
              norms_out: np.ndarray = None):
    """One epoch of N/B sequential slices through pgb_run_epoch (pipelined
    H2D, CUDA-graph steps). Returns (seconds, clipped_total)."""
    engine.bind(model)
    secs = C.c_double()
    clipped = C.c_int64()
    x = np.ascontiguousarray(data.inputs, np.float32)
    y = np.ascontiguousarray(data.labels, np.float32)
    check(lib.pgb_run_epoch(engine.handle, _lib.ptr(x), _lib.ptr(y), data.count,
                            C.byref(cfg.to_c()), step0, _lib.ptr(norms_out), C.byref(clipped),
                            C.byref(secs)))
    model._engine = engine
    return secs.value, clipped.value


def run_bench(kind: ModelKind, data: Dataset, strategy: Strategy,
              opts: RunOptions) -> List[BenchRecord]:
    cfg = DpConfig(opts.clip_norm, opts.noise_multiplier, opts.learning_rate, opts.microbatch,
                   opts.seed)
    records = []
    for B in opts.batch_sizes:
        rec = BenchRecord(model=model_name(kind), strategy=strategy_name(strategy),
                          mode=opts.mode.name, vectorized=strategy != Strategy.naive,
                          batch_size=B, epochs=opts.epochs, seed=opts.seed)
        model = build(kind, opts.seed)
        if B > data.count:
            rec.status, rec.reason = "skip", "batch larger than the dataset"
            records.append(rec)
            continue
        try:
            engine = GradEngine(model, strategy, B, opts.mode)
        except UnsupportedError as e:
            rec.status, rec.reason = "skip", str(e)
            records.append(rec)
            continue
        rec.peak_planned_bytes = engine.footprint_bytes()
        if opts.mem_cap_bytes and rec.peak_planned_bytes > opts.mem_cap_bytes:
            rec.status = "oom"
            rec.reason = (f"footprint {rec.peak_planned_bytes} bytes exceeds cap "
                          f"{opts.mem_cap_bytes}")
            records.append(rec)
            continue
        rec.optimizer_report.trace_seconds = engine.trace_seconds()
        steps = data.count // B
        for epoch in range(opts.epochs):
            secs, _ = run_epoch(engine, model, data, cfg, epoch * steps)
            rec.epoch_seconds.append(secs)
        rec.median_epoch_seconds = median(rec.epoch_seconds)
        records.append(rec)
    return records


@dataclass
class TrainResult:
    epoch_mean_loss: List[float] = field(default_factory=list)
    final_train_accuracy: float = 0.0
    steps: int = 0


def _shuffle(order: np.ndarray, seed: int, epoch: int) -> np.ndarray:
    """One Fisher-Yates pass with RngState(seed, 2^40 + epoch), in place
    (harness.cpp:330-343: the order starts at 0..n-1 once and every epoch
    reshuffles the previous one), by the library (pgb_shuffle_order)."""
    assert order.dtype == np.int64 and order.flags.c_contiguous
    check(lib.pgb_shuffle_order(seed, epoch, order.size, _lib.ptr(order)))
    return order


def _shuffle_py(order: np.ndarray, seed: int, epoch: int) -> np.ndarray:
    """The same pass restated in Python (checks pgb_shuffle_order)."""
    n = order.size
    key = _stream_key(seed, (1 << 40) + epoch)
    ctr = 0
    for i in range(n - 1, 0, -1):
        u = (_value_at(key, ctr) >> 11) * 2.0 ** -53
        ctr += 1
        j = int(0 + (i + 1 - 0) * u)
        order[i], order[j] = order[j], order[i]
    return order


_M64 = (1 << 64) - 1


def _mix64(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _stream_key(seed, stream):
    return _mix64((seed + 0x9E3779B97F4A7C15 * (stream + 1)) & _M64)


def _value_at(key, i):
    return _mix64((key + 0x9E3779B97F4A7C15 * (i + 1)) & _M64)


def train(model: Model, data: Dataset, strategy: Strategy, mode: ExecMode, cfg: DpConfig,
          batch: int, epochs: int, private_training: bool) -> TrainResult:
    """Deterministic training loop: seeded per-epoch shuffle, DPSGD (or SGD)
    steps, evaluation loss over the first min(N, 1024) examples."""
    if batch <= 0 or batch > data.count:
        raise ConfigError("train: bad batch size")
    engine = GradEngine(model, strategy, batch, mode)
    res = TrainResult()
    steps = data.count // batch
    eval_n = min(data.count, 1024)
    order = np.arange(data.count, dtype=np.int64)
    for epoch in range(epochs):
        _shuffle(order, cfg.seed, epoch)
        for s in range(steps):
            idx = order[s * batch:(s + 1) * batch]
            x, y = data.inputs[idx], data.labels[idx]
            if private_training:
                dpsgd_step(model, engine, x, y, cfg, epoch * steps + s)
            else:
                sgd_step(model, engine, x, y, cfg.learning_rate)
            res.steps += 1
        losses, _ = evaluate(engine, model, data, eval_n)
        res.epoch_mean_loss.append(float(losses.astype(np.float64).sum() / eval_n))
    _, logits = evaluate(engine, model, data, data.count)
    if logits.shape[1] == 1:
        pred = (logits[:, 0] > 0).astype(np.int64)
    else:
        pred = logits.argmax(axis=1)  # first maximum, as models::predict
    res.final_train_accuracy = float((pred == data.labels.astype(np.int64)).mean())
    return res


def evaluate(engine: GradEngine, model: Model, data: Dataset, n: int):
    """Per-example losses and logits of the first n examples, forward-only
    on the device in engine-batch chunks (the tail chunk is padded)."""
    engine.bind(model)
    B = engine.batch()
    K = model.desc.classes
    losses = np.empty(n, np.float32)
    logits = np.empty((n, K), np.float32)
    for start in range(0, n, B):
        cnt = min(B, n - start)
        b = slice_batch(data, start, cnt)
        x, y = b.x, b.y
        if cnt < B:
            x = np.concatenate([x, np.repeat(x[-1:], B - cnt, axis=0)])
            y = np.concatenate([y, np.repeat(y[-1:], B - cnt)])
        lo = np.empty(B, np.float32)
        lg = np.empty((B, K), np.float32)
        check(lib.pgb_forward(engine.handle, _lib.ptr(np.ascontiguousarray(x, np.float32)),
                              _lib.ptr(np.ascontiguousarray(y, np.float32)), _lib.ptr(lo),
                              _lib.ptr(lg)))
        losses[start:start + cnt] = lo[:cnt]
        logits[start:start + cnt] = lg[:cnt]
    return losses, logits
