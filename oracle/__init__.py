"""TEST INFRASTRUCTURE — the parity oracle, never the product.

Two checkers live here:

* ``port``  — ``oracle/pgb_oracle.c``, our plain-C restatement of the
  reference DPSGD step (built into ``oracle/_build/libpgb_oracle.so``);
* ``ref``   — the UNMODIFIED reference library compiled from
  ``/root/reference/proj/core/src`` (``oracle/_ref/libpegrad_ref.so``,
  built here by ``oracle/Makefile``; it travels to the GPU box as a built
  artefact, the sources do not).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libpgb_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpegrad_ref.so")

MAX_LAYERS = 32
MAX_BLOCKS = 64

# pegrad::models::ModelKind / LayerKind / Strategy ordinals
LOGREG, FCNN, MNIST_CNN, CIFAR_CNN, EMBED, LSTM_MODEL = range(6)
(DENSE, CONV, MAXPOOL, AVGPOOL, GLOBAL_AVGPOOL, FLATTEN, RELU, EMBEDDING,
 SEQ_AVGPOOL, LSTM) = range(10)
NAIVE, VMAP, OUTER, NORMS, GROUPCONV, JACMM = range(6)


class Layer(C.Structure):
    _fields_ = [("kind", C.c_int32), ("in_", C.c_int64), ("out", C.c_int64),
                ("k", C.c_int64), ("stride", C.c_int64), ("pad", C.c_int64)]


class Desc(C.Structure):
    _fields_ = [("model_kind", C.c_int32), ("n_layers", C.c_int32),
                ("layers", Layer * MAX_LAYERS), ("in_rank", C.c_int32),
                ("in_shape", C.c_int64 * 3), ("classes", C.c_int64),
                ("token_input", C.c_int32), ("n_blocks", C.c_int32),
                ("block_size", C.c_int64 * MAX_BLOCKS),
                ("fan_in", C.c_int64 * MAX_BLOCKS)]

    @property
    def blocks(self):
        return [int(self.block_size[i]) for i in range(self.n_blocks)]

    @property
    def param_count(self):
        return sum(self.blocks)

    @property
    def input_shape(self):
        return tuple(int(self.in_shape[i]) for i in range(self.in_rank))

    def layer_rows(self):
        return [(l.kind, l.in_, l.out, l.k, l.stride, l.pad)
                for l in self.layers[: self.n_layers]]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_port = None
_ref = None

_P = C.POINTER
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


def build():
    """Compile the restatement (and the reference when its sources exist)."""
    targets = ["port"]
    if os.path.isdir("/root/reference/proj"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
        L = C.CDLL(PORT_SO)
        L.orc_last_error.restype = C.c_char_p
        L.orc_build_desc.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_int64, _P(Desc)]
        L.orc_finish_desc.argtypes = [_P(Desc)]
        L.orc_param_count.argtypes = [_P(Desc)]
        L.orc_param_count.restype = C.c_int64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_mix64.restype = C.c_uint64
        L.orc_rng_value_at.argtypes = [C.c_uint64] * 3
        L.orc_rng_value_at.restype = C.c_uint64
        L.orc_gaussian_f64.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, f64p]
        L.orc_gaussian_f32.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, f32p]
        L.orc_init_params_f64.argtypes = [_P(Desc), C.c_uint64, f64p]
        L.orc_init_params_f32.argtypes = [_P(Desc), C.c_uint64, f32p]
        L.orc_synth_f64.argtypes = [_P(Desc), C.c_int64, C.c_uint64, f64p, f64p]
        L.orc_synth_f32.argtypes = [_P(Desc), C.c_int64, C.c_uint64, f32p, f32p]
        L.orc_per_example_grads.argtypes = [_P(Desc), C.c_int64, f64p, f64p, f64p,
                                            C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_dpsgd_step.argtypes = [_P(Desc), C.c_int64, f64p, f64p, f64p, C.c_double,
                                     C.c_double, C.c_double, C.c_int64, C.c_uint64,
                                     C.c_int64, C.c_void_p, _P(C.c_int64), C.c_void_p]
        L.orc_sgd_step.argtypes = [_P(Desc), C.c_int64, f64p, f64p, f64p, C.c_double]
        L.orc_aggregate_f32.argtypes = [C.c_int64, C.c_int32, _P(C.c_int64), f32p, f32p,
                                        C.c_float, C.c_float, C.c_float, C.c_uint64,
                                        C.c_int64, C.c_void_p, _P(C.c_int64)]
        _port = L
    return _port


def _chk(rc, lib, errfn):
    if rc != 0:
        raise OracleError(rc, getattr(lib, errfn)().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---- restatement helpers -------------------------------------------------

def build_desc(kind, seq_len=-1, vocab=-1, hidden=-1) -> Desc:
    d = Desc()
    _chk(port().orc_build_desc(kind, seq_len, vocab, hidden, C.byref(d)), port(), "orc_last_error")
    return d


def custom_desc(model_kind, layers, input_shape, classes, token_input=False) -> Desc:
    d = Desc()
    d.model_kind = model_kind
    d.n_layers = len(layers)
    for i, (k, a, b, kk, s, p) in enumerate(layers):
        d.layers[i] = Layer(k, a, b, kk, s, p)
    d.in_rank = len(input_shape)
    for i, v in enumerate(input_shape):
        d.in_shape[i] = v
    d.classes = classes
    d.token_input = int(token_input)
    _chk(port().orc_finish_desc(C.byref(d)), port(), "orc_last_error")
    return d


def init_params(d: Desc, seed: int, dtype=np.float64):
    out = np.empty(d.param_count, dtype=dtype)
    fn = port().orc_init_params_f64 if dtype == np.float64 else port().orc_init_params_f32
    fn(C.byref(d), seed, out)
    return out


def synth(d: Desc, n: int, seed: int, dtype=np.float64):
    x = np.empty((n,) + d.input_shape, dtype=dtype)
    y = np.empty(n, dtype=dtype)
    fn = port().orc_synth_f64 if dtype == np.float64 else port().orc_synth_f32
    _chk(fn(C.byref(d), n, seed, x, y), port(), "orc_last_error")
    return x, y


def gaussian(seed, stream, n, dtype=np.float64):
    out = np.empty(n, dtype=dtype)
    (port().orc_gaussian_f64 if dtype == np.float64 else port().orc_gaussian_f32)(seed, stream, n, out)
    return out


def per_example_grads(d: Desc, x, y, params):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    params = np.ascontiguousarray(params, np.float64)
    B = x.shape[0]
    stacks = np.empty(B * d.param_count)
    normsq = np.empty(B)
    losses = np.empty(B)
    _chk(port().orc_per_example_grads(C.byref(d), B, x, y, params, _ptr(stacks), _ptr(normsq),
                                      _ptr(losses)), port(), "orc_last_error")
    return stacks, normsq, losses


def split_stacks(d: Desc, stacks, B):
    """Block-major flat stacks -> list of (B, block_size) arrays."""
    out, off = [], 0
    for n in d.blocks:
        out.append(stacks[off: off + B * n].reshape(B, n))
        off += B * n
    return out


def dpsgd_step(d: Desc, x, y, params, clip, sigma, lr, microbatch=1, seed=0, step=0):
    """Returns (new_params, norms, clipped_count, noise_free_clipped_sum)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    p = np.array(params, dtype=np.float64, copy=True)
    B = x.shape[0]
    norms = np.empty(B // microbatch)
    cs = np.empty(d.param_count)
    nclip = C.c_int64()
    _chk(port().orc_dpsgd_step(C.byref(d), B, x, y, p, clip, sigma, lr, microbatch, seed, step,
                               _ptr(norms), C.byref(nclip), _ptr(cs)), port(), "orc_last_error")
    return p, norms, nclip.value, cs


def sgd_step(d: Desc, x, y, params, lr):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    p = np.array(params, dtype=np.float64, copy=True)
    _chk(port().orc_sgd_step(C.byref(d), x.shape[0], x, y, p, lr), port(), "orc_last_error")
    return p


def aggregate_f32(blocks, stacks, params, clip, sigma, lr, seed, step, B):
    bs = (C.c_int64 * len(blocks))(*blocks)
    p = np.array(params, dtype=np.float32, copy=True)
    norms = np.empty(B, np.float32)
    nclip = C.c_int64()
    port().orc_aggregate_f32(B, len(blocks), bs, np.ascontiguousarray(stacks, np.float32), p,
                             clip, sigma, lr, seed, step, _ptr(norms), C.byref(nclip))
    return p, norms, nclip.value


def noise_stream(step, p):
    return (1 << 32) + step * 4096 + p


# ---- compiled reference (oracle/_ref) --------------------------------------

def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO + " (run make -C oracle ref where /root/reference exists)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_desc_builtin.restype = C.c_void_p
        L.ref_desc_builtin.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64]
        L.ref_desc_custom.restype = C.c_void_p
        L.ref_desc_custom.argtypes = [C.c_int, C.c_int, _P(C.c_int64), C.c_int, _P(C.c_int64),
                                      C.c_int64, C.c_int]
        L.ref_desc_free.argtypes = [C.c_void_p]
        L.ref_desc_param_count.argtypes = [C.c_void_p]
        L.ref_desc_param_count.restype = C.c_int64
        for sfx, ptr, T in (("f32", f32p, C.c_float), ("f64", f64p, C.c_double)):
            getattr(L, f"ref_init_params_{sfx}").argtypes = [C.c_void_p, C.c_uint64, ptr]
            getattr(L, f"ref_synth_{sfx}").argtypes = [C.c_void_p, C.c_int64, C.c_uint64, ptr, ptr]
            getattr(L, f"ref_gaussian_{sfx}").argtypes = [C.c_uint64, C.c_uint64, C.c_int64, ptr]
            f = getattr(L, f"ref_engine_new_{sfx}")
            f.restype = C.c_void_p
            f.argtypes = [C.c_void_p, C.c_int, C.c_int64, ptr]
            getattr(L, f"ref_engine_free_{sfx}").argtypes = [C.c_void_p]
            getattr(L, f"ref_engine_get_params_{sfx}").argtypes = [C.c_void_p, ptr]
            getattr(L, f"ref_engine_set_params_{sfx}").argtypes = [C.c_void_p, ptr]
            getattr(L, f"ref_engine_per_example_{sfx}").argtypes = [C.c_void_p, ptr, ptr,
                                                                    C.c_void_p, C.c_void_p]
            getattr(L, f"ref_engine_step_{sfx}").argtypes = [C.c_void_p, ptr, ptr, T, T, T,
                                                             C.c_int64, C.c_uint64, C.c_int64,
                                                             C.c_void_p, _P(C.c_int64)]
            getattr(L, f"ref_engine_sgd_step_{sfx}").argtypes = [C.c_void_p, ptr, ptr, T]
            getattr(L, f"ref_engine_weighted_sum_{sfx}").argtypes = [C.c_void_p, ptr, ptr, ptr,
                                                                     C.c_void_p]
        L.ref_run_bench_f32.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_double, C.c_double, C.c_double, C.c_uint64,
                                        _P(C.c_double)]
        L.ref_train_f32.argtypes = [C.c_void_p, f32p, f32p, f32p, C.c_int64, C.c_int,
                                    C.c_double, C.c_double, C.c_double, C.c_int64, C.c_uint64,
                                    C.c_int64, C.c_int64, C.c_int, f64p, _P(C.c_double),
                                    _P(C.c_int64)]
        L.ref_load_idx_f32.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, _P(C.c_int64),
                                       _P(C.c_int), _P(C.c_int64)]
        L.ref_records_json_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_int64,
                                                 _P(C.c_int64)]
        _ref = L
    return _ref


def ref_train(desc: Desc, params, x, y, strategy, clip, sigma, lr, microbatch, seed, batch,
              epochs, private=True):
    """bench::train<float> of the compiled reference (harness.cpp:319-382):
    (final params, per-epoch mean evaluation losses, final accuracy, steps)."""
    L = ref()
    rows = desc.layer_rows()
    l6 = (C.c_int64 * (6 * len(rows)))(*[v for r in rows for v in r])
    ins = (C.c_int64 * desc.in_rank)(*desc.input_shape)
    h = L.ref_desc_custom(desc.model_kind, len(rows), l6, desc.in_rank, ins, desc.classes,
                          desc.token_input)
    p = np.array(params, np.float32, copy=True)
    x = np.ascontiguousarray(x, np.float32)
    y = np.ascontiguousarray(y, np.float32)
    losses = np.zeros(max(1, epochs))
    acc, steps = C.c_double(), C.c_int64()
    try:
        _chk(L.ref_train_f32(h, p, x, y, x.shape[0], strategy, clip, sigma, lr, microbatch,
                             seed, batch, epochs, int(private), losses, C.byref(acc),
                             C.byref(steps)), L, "ref_last_error")
    finally:
        L.ref_desc_free(h)
    return p, losses[:epochs], acc.value, steps.value


def ref_load_idx(path):
    """io::load_idx<float> of the compiled reference: (values, dims) or
    raises RefError (code 8 FormatError, 9 IoError)."""
    L = ref()
    n, rank, dims = C.c_int64(), C.c_int(), (C.c_int64 * 8)()
    _chk(L.ref_load_idx_f32(path.encode(), None, 0, C.byref(n), C.byref(rank), dims), L,
         "ref_last_error")
    out = np.empty(n.value, np.float32)
    _chk(L.ref_load_idx_f32(path.encode(), _ptr(out), n.value, C.byref(n), C.byref(rank), dims),
         L, "ref_last_error")
    return out, tuple(dims[i] for i in range(rank.value))


def ref_records_json_roundtrip(text: str) -> str:
    """bench::records_to_json(bench::records_from_json(text)) of the reference."""
    L = ref()
    n = C.c_int64()
    _chk(L.ref_records_json_roundtrip(text.encode(), None, 0, C.byref(n)), L, "ref_last_error")
    buf = C.create_string_buffer(n.value + 1)
    _chk(L.ref_records_json_roundtrip(text.encode(), buf, n.value + 1, C.byref(n)), L,
         "ref_last_error")
    return buf.value.decode()


class RefModel:
    """The reference's Model<T> + GradEngine<T> (graph mode) behind a handle."""

    def __init__(self, desc: Desc, strategy: int, batch: int, params, dtype=np.float64):
        L = ref()
        self.dtype = dtype
        self.sfx = "f64" if dtype == np.float64 else "f32"
        self.desc = desc
        rows = desc.layer_rows()
        l6 = (C.c_int64 * (6 * len(rows)))(*[v for r in rows for v in r])
        ins = (C.c_int64 * desc.in_rank)(*desc.input_shape)
        self.hdesc = L.ref_desc_custom(desc.model_kind, len(rows), l6, desc.in_rank, ins,
                                       desc.classes, desc.token_input)
        p = np.ascontiguousarray(params, dtype)
        self.h = getattr(L, f"ref_engine_new_{self.sfx}")(self.hdesc, strategy, batch, p)
        if not self.h:
            raise OracleError(-1, L.ref_last_error().decode())
        self.batch = batch

    def _call(self, name, *args):
        L = ref()
        rc = getattr(L, f"ref_{name}_{self.sfx}")(self.h, *args)
        if rc != 0:
            raise OracleError(rc, L.ref_last_error().decode())

    def params(self):
        out = np.empty(self.desc.param_count, self.dtype)
        self._call("engine_get_params", out)
        return out

    def set_params(self, p):
        self._call("engine_set_params", np.ascontiguousarray(p, self.dtype))

    def per_example(self, x, y, want_stacks=True):
        """Stacks (None for want_stacks=False, e.g. the norms-only strategy) and norms."""
        B = self.batch
        stacks = np.empty(B * self.desc.param_count, self.dtype) if want_stacks else None
        norms = np.empty(B, self.dtype)
        self._call("engine_per_example", np.ascontiguousarray(x, self.dtype),
                   np.ascontiguousarray(y, self.dtype),
                   _ptr(stacks) if want_stacks else None, _ptr(norms))
        return stacks, norms

    def step(self, x, y, clip, sigma, lr, microbatch=1, seed=0, step=0):
        norms = np.empty(self.batch // microbatch, self.dtype)
        n = C.c_int64()
        self._call("engine_step", np.ascontiguousarray(x, self.dtype),
                   np.ascontiguousarray(y, self.dtype), clip, sigma, lr, microbatch, seed, step,
                   _ptr(norms), C.byref(n))
        return norms, n.value

    def weighted_grad_sum(self, x, y, w):
        """GradEngine::weighted_grad_sum (strategies.cpp:432-450), flat."""
        out = np.empty(self.desc.param_count, self.dtype)
        self._call("engine_weighted_sum", np.ascontiguousarray(x, self.dtype),
                   np.ascontiguousarray(y, self.dtype), np.ascontiguousarray(w, self.dtype),
                   _ptr(out))
        return out

    def sgd_step(self, x, y, lr):
        self._call("engine_sgd_step", np.ascontiguousarray(x, self.dtype),
                   np.ascontiguousarray(y, self.dtype), lr)

    def __del__(self):
        try:
            L = ref()
            if getattr(self, "h", None):
                getattr(L, f"ref_engine_free_{self.sfx}")(self.h)
            if getattr(self, "hdesc", None):
                L.ref_desc_free(self.hdesc)
        except Exception:
            pass


def ref_gaussian(seed, stream, n, dtype=np.float64):
    out = np.empty(n, dtype)
    sfx = "f64" if dtype == np.float64 else "f32"
    rc = getattr(ref(), f"ref_gaussian_{sfx}")(seed, stream, n, out)
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return out


def ref_synth(desc: Desc, n, seed, dtype=np.float64):
    L = ref()
    rows = desc.layer_rows()
    l6 = (C.c_int64 * (6 * len(rows)))(*[v for r in rows for v in r])
    ins = (C.c_int64 * desc.in_rank)(*desc.input_shape)
    h = L.ref_desc_custom(desc.model_kind, len(rows), l6, desc.in_rank, ins, desc.classes,
                          desc.token_input)
    x = np.empty((n,) + desc.input_shape, dtype)
    y = np.empty(n, dtype)
    sfx = "f64" if dtype == np.float64 else "f32"
    rc = getattr(L, f"ref_synth_{sfx}")(h, n, seed, x, y)
    L.ref_desc_free(h)
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return x, y


def ref_init_params(desc: Desc, seed, dtype=np.float64):
    L = ref()
    rows = desc.layer_rows()
    l6 = (C.c_int64 * (6 * len(rows)))(*[v for r in rows for v in r])
    ins = (C.c_int64 * desc.in_rank)(*desc.input_shape)
    h = L.ref_desc_custom(desc.model_kind, len(rows), l6, desc.in_rank, ins, desc.classes,
                          desc.token_input)
    out = np.empty(desc.param_count, dtype)
    sfx = "f64" if dtype == np.float64 else "f32"
    getattr(L, f"ref_init_params_{sfx}")(h, seed, out)
    L.ref_desc_free(h)
    return out
