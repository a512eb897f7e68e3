"""ctypes binding of include/pegrad_b200.h (libpegrad_b200.so).

The CUDA library is the only implementation: there is no CPU fallback. If
the shared object is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

PKG = os.path.dirname(os.path.abspath(__file__))
# PGB_LIBRARY: an alternative build of the same library (e.g. the PGB_TRACE
# timestamp build used by scripts/trace_phases.py)
SO = os.environ.get("PGB_LIBRARY") or os.path.join(PKG, "libpegrad_b200.so")

MAX_LAYERS = 32
MAX_PARAMS = 64


class LayerSpecC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("in_", C.c_int64), ("out", C.c_int64),
                ("k", C.c_int64), ("stride", C.c_int64), ("pad", C.c_int64)]


class ModelOptionsC(C.Structure):
    _fields_ = [("seq_len", C.c_int64), ("vocab", C.c_int64), ("hidden", C.c_int64)]


class ModelDescC(C.Structure):
    _fields_ = [("model_kind", C.c_int32), ("n_layers", C.c_int32),
                ("layers", LayerSpecC * MAX_LAYERS), ("input_rank", C.c_int32),
                ("input_shape", C.c_int64 * 3), ("classes", C.c_int64),
                ("token_input", C.c_int32), ("n_params", C.c_int32),
                ("param_size", C.c_int64 * MAX_PARAMS),
                ("param_fan_in", C.c_int64 * MAX_PARAMS)]


class DpConfigC(C.Structure):
    _fields_ = [("clip_norm", C.c_float), ("noise_multiplier", C.c_float),
                ("learning_rate", C.c_float), ("microbatch", C.c_int64), ("seed", C.c_uint64)]


class StepReportC(C.Structure):
    _fields_ = [("clipped_count", C.c_int64), ("n_streams", C.c_int32),
                ("noise_streams", C.c_uint64 * MAX_PARAMS)]


class UniqueIdC(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


class EngineInfoC(C.Structure):
    _fields_ = [("batch", C.c_int64), ("global_batch", C.c_int64), ("param_count", C.c_int64),
                ("n_params", C.c_int32), ("world", C.c_int32), ("rank", C.c_int32),
                ("device", C.c_int32), ("workspace_bytes", C.c_int64),
                ("kernels_per_step", C.c_int32), ("graph_enabled", C.c_int32)]


EXPORTS = {
    # name: (restype, argtypes)
    "pgb_last_error": (C.c_char_p, []),
    "pgb_version": (C.c_char_p, []),
    "pgb_build_desc": (C.c_int, [C.c_int32, C.POINTER(ModelOptionsC), C.POINTER(ModelDescC)]),
    "pgb_finish_desc": (C.c_int, [C.POINTER(ModelDescC)]),
    "pgb_param_count": (C.c_int64, [C.POINTER(ModelDescC)]),
    "pgb_init_params": (C.c_int, [C.POINTER(ModelDescC), C.c_uint64, C.c_void_p]),
    "pgb_synth": (C.c_int, [C.POINTER(ModelDescC), C.c_int64, C.c_uint64, C.c_void_p,
                            C.c_void_p]),
    "pgb_engine_create": (C.c_int, [C.POINTER(ModelDescC), C.c_int32, C.c_int64, C.c_int32,
                                    C.POINTER(C.c_void_p)]),
    "pgb_nccl_unique_id": (C.c_int, [C.POINTER(UniqueIdC)]),
    "pgb_engine_create_dist": (C.c_int, [C.POINTER(ModelDescC), C.c_int32, C.c_int64,
                                         C.c_int32, C.c_int32, C.c_int32,
                                         C.POINTER(UniqueIdC), C.POINTER(C.c_void_p)]),
    "pgb_engine_destroy": (None, [C.c_void_p]),
    "pgb_engine_info_get": (C.c_int, [C.c_void_p, C.POINTER(EngineInfoC)]),
    "pgb_engine_set_graph": (C.c_int, [C.c_void_p, C.c_int32]),
    "pgb_set_params": (C.c_int, [C.c_void_p, C.c_void_p]),
    "pgb_get_params": (C.c_int, [C.c_void_p, C.c_void_p]),
    "pgb_dpsgd_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(DpConfigC),
                                 C.c_int64, C.c_void_p, C.POINTER(StepReportC)]),
    "pgb_dpsgd_step_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.POINTER(DpConfigC), C.c_int64]),
    "pgb_synchronize": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(StepReportC)]),
    "pgb_sgd_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float]),
    "pgb_per_example_grads": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]),
    "pgb_clipped_sum": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_void_p,
                                  C.c_void_p, C.POINTER(C.c_int64)]),
    "pgb_weighted_grad_sum": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]),
    "pgb_batch_grad_sum": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "pgb_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "pgb_aggregate": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(DpConfigC), C.c_int64,
                                C.c_void_p, C.POINTER(StepReportC)]),
    "pgb_gaussian": (C.c_int, [C.c_int32, C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]),
    "pgb_run_epoch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                C.POINTER(DpConfigC), C.c_int64, C.c_void_p,
                                C.POINTER(C.c_int64), C.POINTER(C.c_double)]),
    "pgb_profile_steps": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(DpConfigC),
                                    C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                    C.POINTER(C.c_int32)]),
    "pgb_debug_tc_gemm": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                    C.c_void_p, C.c_void_p]),
    "pgb_debug_tma_box": (C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_int32, C.c_void_p]),
    "pgb_debug_tma_gemm": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                     C.c_void_p, C.c_void_p]),
    "pgb_debug_umma_probe": (C.c_int, [C.c_int32] * 6 + [C.c_void_p] * 3),
    "pgb_debug_umma_rate": (C.c_int, [C.c_int32] * 4 + [C.c_void_p, C.c_int32, C.c_void_p]),
    "pgb_run_steps_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                       C.POINTER(DpConfigC), C.c_int64, C.POINTER(C.c_int64)]),
    "pgb_shuffle_order": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.c_void_p]),
    "pgb_prepare_steps": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                    C.POINTER(DpConfigC)]),
    "pgb_idx_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), C.c_void_p,
                               C.POINTER(C.c_int64)]),
    "pgb_load_idx": (C.c_int, [C.c_char_p, C.c_float, C.c_void_p, C.c_int64]),
    "pgb_load_idx_device": (C.c_int, [C.c_char_p, C.c_int32, C.c_float, C.c_void_p, C.c_int64]),
    "pgb_device_params": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "pgb_device_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "pgb_kernels_per_step": (C.c_int32, [C.c_void_p]),
}


def _load():
    if not os.path.exists(SO):
        raise ImportError(
            f"{SO} is missing: build it with `python paper_2010_09063_b200/build.py` "
            "(the engine has no CPU fallback)")
    lib = C.CDLL(SO)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status != 0:
        msg = lib.pgb_last_error().decode(errors="replace")
        raise errors.from_status(status, msg)


def ptr(a):
    """Address of a numpy array / torch tensor / None for the C ABI."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)
