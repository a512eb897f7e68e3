"""DPSGD step API — the reference's dpsgd.hpp (proj/core/include/pegrad/dpsgd.hpp:24-78)
over the sm_100a engine. ``dpsgd_step`` keeps the reference signature and
semantics: per-example gradients -> (microbatch) -> clip at C -> clipped sum
-> N(0, (sigma C)^2) noise from stream 2^32 + step*4096 + p -> mean -> SGD
update; there is no privacy accountant (sigma is raw configuration).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _lib
from ._lib import check, lib
from .errors import ConfigError, ContractError
from .models import Model
from .strategies import GradEngine


@dataclass
class DpConfig:
    clip_norm: float = 1.0          # C > 0
    noise_multiplier: float = 0.0   # sigma >= 0
    learning_rate: float = 0.1
    microbatch: int = 1
    seed: int = 0

    def to_c(self) -> _lib.DpConfigC:
        return _lib.DpConfigC(self.clip_norm, self.noise_multiplier, self.learning_rate,
                              int(self.microbatch), int(self.seed))


@dataclass
class StepReport:
    pre_clip_norms: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    clipped_count: int = 0
    noise_streams: List[int] = field(default_factory=list)


def validate(cfg: DpConfig, batch: int) -> None:
    """dpsgd.cpp:36-51 (the engine re-validates in C++ with the same messages)."""
    if not (np.float32(cfg.clip_norm) > 0):
        raise ConfigError("DpConfig: clip norm must be positive")
    if np.float32(cfg.noise_multiplier) < 0:
        raise ConfigError("DpConfig: noise multiplier must be non-negative")
    if not (np.float32(cfg.learning_rate) > 0):
        raise ConfigError("DpConfig: learning rate must be positive")
    if cfg.microbatch < 1 or batch % cfg.microbatch != 0:
        raise ConfigError(f"DpConfig: microbatch size {cfg.microbatch} must divide the batch "
                          f"size {batch}")


def noise_stream(step_index: int, param_ordinal: int) -> int:
    """dpsgd.cpp:27-32."""
    return (1 << 32) + step_index * 4096 + param_ordinal


def dpsgd_step(model: Model, engine: GradEngine, x, y, cfg: DpConfig,
               step_index: int) -> StepReport:
    """One DPSGD update of ``model`` (dpsgd.cpp:188-331). The parameters stay
    resident on the device; ``model.params`` fetches them on access."""
    validate(cfg, engine.batch())
    if engine.strategy().name == "norms" and cfg.microbatch != 1:
        raise ConfigError("dpsgd_step: the norms-only strategy supports microbatch = 1 only")
    engine.bind(model)
    x, y = engine._inputs(x, y)
    units = engine.batch() // cfg.microbatch
    norms = np.empty(units, np.float32)
    rep = _lib.StepReportC()
    check(lib.pgb_dpsgd_step(engine.handle, _lib.ptr(x), _lib.ptr(y), C.byref(cfg.to_c()),
                             int(step_index), _lib.ptr(norms), C.byref(rep)))
    model._engine = engine
    return StepReport(norms, int(rep.clipped_count),
                      [int(rep.noise_streams[i]) for i in range(rep.n_streams)])


def sgd_step(model: Model, engine: GradEngine, x, y, learning_rate: float) -> None:
    """Non-private baseline: params -= lr * mean batch gradient (dpsgd.cpp:334-346)."""
    engine.bind(model)
    x, y = engine._inputs(x, y)
    check(lib.pgb_sgd_step(engine.handle, _lib.ptr(x), _lib.ptr(y), float(learning_rate)))
    model._engine = engine


def aggregate(engine: GradEngine, model: Model, stacks_flat: np.ndarray, cfg: DpConfig,
              step_index: int) -> StepReport:
    """The views-path tail (norms, clip, clipped sum, noise, mean, update) on the
    device over caller-supplied per-example stacks (block-major, B*P)."""
    engine.bind(model)
    stacks_flat = np.ascontiguousarray(stacks_flat, np.float32)
    if stacks_flat.size != engine.batch() * engine.P:
        raise ContractError("aggregate: stacks must hold batch * param_count floats")
    norms = np.empty(engine.batch(), np.float32)
    rep = _lib.StepReportC()
    check(lib.pgb_aggregate(engine.handle, _lib.ptr(stacks_flat), C.byref(cfg.to_c()),
                            int(step_index), _lib.ptr(norms), C.byref(rep)))
    model._engine = engine
    return StepReport(norms, int(rep.clipped_count),
                      [int(rep.noise_streams[i]) for i in range(rep.n_streams)])


def gaussian(seed: int, stream: int, n: int, device: int = 0) -> np.ndarray:
    """gaussian<float>(n, RngState(seed, stream)) generated on the device."""
    out = np.empty(n, np.float32)
    check(lib.pgb_gaussian(device, seed, stream, n, _lib.ptr(out)))
    return out
