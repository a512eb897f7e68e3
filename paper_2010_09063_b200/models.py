"""Model descriptions and parameters — the reference's models API
(proj/core/include/pegrad/models.hpp:24-88), backed by libpegrad_b200.so.

Parameters are fp32 numpy arrays in registry order ("l<i>.W", "l<i>.b",
"l<i>.table"), initialised bit-identically to models::build<float>
(models.cpp:359-375).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib


class ModelKind(enum.IntEnum):
    logreg = 0
    fcnn = 1
    mnist_cnn = 2
    cifar_cnn = 3
    embed = 4
    lstm = 5


class LayerKind(enum.IntEnum):
    dense = 0
    conv = 1
    maxpool = 2
    avgpool = 3
    global_avgpool = 4
    flatten = 5
    relu = 6
    embedding = 7
    seq_avgpool = 8
    lstm = 9


def model_name(kind: ModelKind) -> str:
    return ModelKind(kind).name


def model_kind_from_name(name: str) -> ModelKind:
    from .errors import ConfigError
    try:
        return ModelKind[name]
    except KeyError:
        raise ConfigError(f"unknown model '{name}' (expected one of logreg, fcnn, mnist_cnn, "
                          "cifar_cnn, embed, lstm)") from None


@dataclass
class LayerSpec:
    kind: LayerKind
    in_: int = 0
    out: int = 0
    k: int = 0
    stride: int = 1
    pad: int = 0


@dataclass
class ModelOptions:
    seq_len: int = -1
    vocab: int = -1
    hidden: int = -1


@dataclass
class ModelDesc:
    kind: ModelKind
    layers: List[LayerSpec]
    input_shape: tuple
    classes: int = 2
    token_input: bool = False
    param_names: List[str] = field(default_factory=list)
    param_shapes: List[tuple] = field(default_factory=list)
    param_fan_in: List[int] = field(default_factory=list)

    def param_count(self) -> int:
        return int(sum(int(np.prod(s)) for s in self.param_shapes))

    # -- C ABI conversion ------------------------------------------------
    def to_c(self) -> _lib.ModelDescC:
        d = _lib.ModelDescC()
        d.model_kind = int(self.kind)
        d.n_layers = len(self.layers)
        for i, l in enumerate(self.layers):
            d.layers[i] = _lib.LayerSpecC(int(l.kind), l.in_, l.out, l.k, l.stride, l.pad)
        d.input_rank = len(self.input_shape)
        for i, v in enumerate(self.input_shape):
            d.input_shape[i] = v
        d.classes = self.classes
        d.token_input = int(self.token_input)
        check(lib.pgb_finish_desc(C.byref(d)))
        return d

    @staticmethod
    def from_c(d: _lib.ModelDescC) -> "ModelDesc":
        layers = [LayerSpec(LayerKind(d.layers[i].kind), d.layers[i].in_, d.layers[i].out,
                            d.layers[i].k, d.layers[i].stride, d.layers[i].pad)
                  for i in range(d.n_layers)]
        desc = ModelDesc(ModelKind(d.model_kind), layers,
                         tuple(int(d.input_shape[i]) for i in range(d.input_rank)),
                         int(d.classes), bool(d.token_input))
        desc._fill_registry()
        return desc

    def _fill_registry(self):
        """register_params naming/shape rules (models.cpp:50-83)."""
        self.param_names, self.param_shapes, self.param_fan_in = [], [], []
        for i, l in enumerate(self.layers):
            pre = f"l{i}."
            if l.kind == LayerKind.dense:
                self._add(pre + "W", (l.in_, l.out), l.in_)
                self._add(pre + "b", (l.out,), 0)
            elif l.kind == LayerKind.conv:
                self._add(pre + "W", (l.out, l.in_, l.k, l.k), l.in_ * l.k * l.k)
                self._add(pre + "b", (l.out,), 0)
            elif l.kind == LayerKind.embedding:
                self._add(pre + "table", (l.in_, l.out), l.out)
            elif l.kind == LayerKind.lstm:
                self._add(pre + "Wx", (4 * l.out, l.in_), l.in_)
                self._add(pre + "Wh", (4 * l.out, l.out), l.out)
                self._add(pre + "b", (4 * l.out,), 0)

    def _add(self, name, shape, fan):
        self.param_names.append(name)
        self.param_shapes.append(tuple(shape))
        self.param_fan_in.append(fan)


def build_desc(kind: ModelKind, opts: Optional[ModelOptions] = None) -> ModelDesc:
    o = opts or ModelOptions()
    d = _lib.ModelDescC()
    check(lib.pgb_build_desc(int(kind), C.byref(_lib.ModelOptionsC(o.seq_len, o.vocab, o.hidden)),
                             C.byref(d)))
    return ModelDesc.from_c(d)


def custom_desc(kind: ModelKind, layers: Sequence[LayerSpec], input_shape, classes: int,
                token_input: bool = False) -> ModelDesc:
    desc = ModelDesc(ModelKind(kind), list(layers), tuple(input_shape), classes, token_input)
    desc._fill_registry()
    desc.to_c()  # validates through the library
    return desc


class Model:
    """models::Model<float>: a description plus parameter tensors.

    When bound to a GradEngine the authoritative parameters live on the
    device; ``params`` downloads them lazily (the reference replaces the
    tensors after every step, dpsgd.cpp:173-183).
    """

    def __init__(self, desc: ModelDesc, params: List[np.ndarray]):
        self.desc = desc
        self._params = params
        self._engine = None  # engine holding newer device-side params

    @property
    def params(self) -> List[np.ndarray]:
        if self._engine is not None:
            flat = self._engine.get_flat_params()
            self._params = unflatten(self.desc, flat)
            self._engine = None
        return self._params

    @params.setter
    def params(self, value: List[np.ndarray]):
        self._params = [np.ascontiguousarray(v, np.float32) for v in value]
        self._engine = None

    def flat_params(self) -> np.ndarray:
        return flatten(self.params)


def flatten(params: Sequence[np.ndarray]) -> np.ndarray:
    return np.concatenate([np.asarray(p, np.float32).ravel() for p in params]) \
        if len(params) else np.zeros(0, np.float32)


def unflatten(desc: ModelDesc, flat: np.ndarray) -> List[np.ndarray]:
    out, off = [], 0
    for s in desc.param_shapes:
        n = int(np.prod(s))
        out.append(flat[off: off + n].reshape(s).copy())
        off += n
    return out


def build_from_desc(desc: ModelDesc, seed: int) -> Model:
    flat = np.empty(desc.param_count(), np.float32)
    check(lib.pgb_init_params(C.byref(desc.to_c()), seed, _lib.ptr(flat)))
    return Model(desc, unflatten(desc, flat))


def build(kind: ModelKind, seed: int, opts: Optional[ModelOptions] = None) -> Model:
    return build_from_desc(build_desc(kind, opts), seed)
