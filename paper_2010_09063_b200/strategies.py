"""GradEngine — the reference's compiled per-example-gradient pipeline
(proj/core/include/pegrad/strategies.hpp:58-100), here a handle on the
sm_100a engine in libpegrad_b200.so.

Whatever Strategy is requested, the device runs one fixed kernel schedule
(batched implicit-GEMM layers, per-example weight gradients into resident
stacks, fused norm/clip/sum/noise/update); the strategy is kept for API
parity and for the reference's support matrix (strategies.cpp:76-113), which
is enforced identically (UnsupportedError "unsupported layer: ...").
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import check, lib
from .models import Model, ModelDesc, flatten


class Strategy(enum.IntEnum):
    naive = 0
    vmap = 1
    outer = 2
    norms = 3
    groupconv = 4
    jacmm = 5


class ExecMode(enum.IntEnum):
    eager = 0
    graph = 1


def strategy_name(s: Strategy) -> str:
    return Strategy(s).name


def strategy_from_name(name: str) -> Strategy:
    from .errors import ConfigError
    try:
        return Strategy[name]
    except KeyError:
        raise ConfigError(f"unknown strategy '{name}' (expected naive, vmap, outer, norms, "
                          "groupconv, jacmm)") from None


def all_strategies() -> List[Strategy]:
    return list(Strategy)


@dataclass
class PerExampleGrads:
    """PerExampleGrads<T> (strategies.hpp:42-48)."""
    norms_only: bool = False
    stacks: List[np.ndarray] = field(default_factory=list)
    norms: Optional[np.ndarray] = None
    batch: int = 0


class GradEngine:
    def __init__(self, model: Model, strategy: Strategy, batch: int,
                 mode: ExecMode = ExecMode.graph, device: int = 0, *, rank: int = 0,
                 world: int = 1, unique_id: Optional[bytes] = None):
        t0 = time.perf_counter()
        self.desc: ModelDesc = model.desc
        self._desc_c = model.desc.to_c()
        self._strategy = Strategy(strategy)
        self._mode = ExecMode(mode)
        self._batch = int(batch)
        h = C.c_void_p()
        if world > 1 or unique_id is not None:
            # the data-parallel engine (a one-rank communicator when world == 1
            # and PGB_FORCE_DIST=1: the multi-GPU schedule on one GPU)
            uid = _lib.UniqueIdC()
            C.memmove(C.byref(uid), unique_id, 128)
            check(lib.pgb_engine_create_dist(C.byref(self._desc_c), int(strategy), int(batch),
                                             device, rank, world, C.byref(uid), C.byref(h)))
        else:
            check(lib.pgb_engine_create(C.byref(self._desc_c), int(strategy), int(batch),
                                        device, C.byref(h)))
        self.handle = h
        # eager mode re-launches kernel by kernel; graph mode replays a CUDA graph
        check(lib.pgb_engine_set_graph(h, 1 if self._mode == ExecMode.graph else 0))
        self.P = self.desc.param_count()
        self._bound: Optional[Model] = None
        self.set_flat_params(model.flat_params())
        self._bound = model
        self._trace_seconds = time.perf_counter() - t0

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            lib.pgb_engine_destroy(h)
            self.handle = None

    # -- metadata --------------------------------------------------------
    def strategy(self) -> Strategy:
        return self._strategy

    def mode(self) -> ExecMode:
        return self._mode

    def batch(self) -> int:
        return self._batch

    def trace_seconds(self) -> float:
        return self._trace_seconds

    def info(self) -> _lib.EngineInfoC:
        out = _lib.EngineInfoC()
        check(lib.pgb_engine_info_get(self.handle, C.byref(out)))
        return out

    def footprint_bytes(self) -> int:
        return int(self.info().workspace_bytes)

    def supports_views(self) -> bool:  # strategies.cpp:400-403
        return self._mode == ExecMode.graph and self._strategy not in (Strategy.naive,
                                                                       Strategy.norms)

    # -- parameters --------------------------------------------------------
    def set_flat_params(self, flat: np.ndarray):
        flat = np.ascontiguousarray(flat, np.float32)
        assert flat.size == self.P
        # the bound model may hold its newest parameters only on the device
        # (dpsgd_step leaves them there): fetch them before they are replaced,
        # and forget the binding so the next bind() uploads again
        b = self._bound
        if b is not None and b._engine is self:
            b.params  # noqa: B018  (downloads into the model)
        self._bound = None
        check(lib.pgb_set_params(self.handle, _lib.ptr(flat)))

    def get_flat_params(self) -> np.ndarray:
        out = np.empty(self.P, np.float32)
        check(lib.pgb_get_params(self.handle, _lib.ptr(out)))
        return out

    def bind(self, model: Model):
        """Make the device hold `model`'s parameters (uploads only when stale)."""
        if model._engine is self and self._bound is model:
            return
        flat = model.flat_params()
        self.set_flat_params(flat)
        self._bound = model

    def _inputs(self, x, y):
        from .errors import ContractError
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        if x.shape[0] != self._batch or y.shape[0] != self._batch:
            raise ContractError(f"GradEngine: batch extent mismatch (engine built for "
                                f"{self._batch})")
        return x, y

    # -- per-example gradients -------------------------------------------
    def compute(self, x, y, params=None) -> PerExampleGrads:
        x, y = self._inputs(x, y)
        if params is not None:
            self.set_flat_params(flatten(params))
        B = self._batch
        stacks = np.empty(B * self.P, np.float32)
        norms = np.empty(B, np.float32)
        check(lib.pgb_per_example_grads(self.handle, _lib.ptr(x), _lib.ptr(y),
                                        _lib.ptr(stacks), _lib.ptr(norms)))
        out, off = [], 0
        for s in self.desc.param_shapes:
            n = int(np.prod(s))
            out.append(stacks[off: off + B * n].reshape((B,) + tuple(s)))
            off += B * n
        return PerExampleGrads(False, out, norms, B)

    compute_views = compute

    def per_example_flat(self, x, y):
        """Block-major flat stacks (B*P) and norms (B), as pgb_per_example_grads."""
        x, y = self._inputs(x, y)
        stacks = np.empty(self._batch * self.P, np.float32)
        norms = np.empty(self._batch, np.float32)
        check(lib.pgb_per_example_grads(self.handle, _lib.ptr(x), _lib.ptr(y),
                                        _lib.ptr(stacks), _lib.ptr(norms)))
        return stacks, norms


    def clipped_sum(self, x, y, clip_norm: float):
        """Noise-free clipped sum (P), pre-clip norms (B), clipped count."""
        x, y = self._inputs(x, y)
        out = np.empty(self.P, np.float32)
        norms = np.empty(self._batch, np.float32)
        n = C.c_int64()
        check(lib.pgb_clipped_sum(self.handle, _lib.ptr(x), _lib.ptr(y), float(clip_norm),
                                  _lib.ptr(out), _lib.ptr(norms), C.byref(n)))
        return out, norms, n.value

    def weighted_grad_sum(self, x, y, w):
        """sum_i w_i g_i over the batch (P floats, flat parameter order), as
        GradEngine::weighted_grad_sum (strategies.cpp:432-450)."""
        x, y = self._inputs(x, y)
        w = np.ascontiguousarray(w, np.float32)
        if w.shape != (self._batch,):
            raise ValueError(f"weights must have shape ({self._batch},)")
        out = np.empty(self.P, np.float32)
        check(lib.pgb_weighted_grad_sum(self.handle, _lib.ptr(x), _lib.ptr(y), _lib.ptr(w),
                                        _lib.ptr(out)))
        return out

    def batch_grad_sum(self, x, y):
        """sum_i g_i over the batch, as GradEngine::batch_grad_sum (strategies.cpp:453-458)."""
        x, y = self._inputs(x, y)
        out = np.empty(self.P, np.float32)
        check(lib.pgb_batch_grad_sum(self.handle, _lib.ptr(x), _lib.ptr(y), _lib.ptr(out)))
        return out
