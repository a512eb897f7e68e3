"""pegrad_b200 — a B200-native (sm_100a) DPSGD step engine.

Drop-in for the reference ("pegrad") DPSGD path: the same model descriptions,
DpConfig / StepReport / dpsgd_step contract, GradEngine and run_bench / train
epoch drivers, executed by hand-written CUDA kernels behind the C ABI in
include/pegrad_b200.h. There is no CPU fallback: importing this package
loads libpegrad_b200.so or fails.
"""
from . import errors
from ._lib import lib
from .dataset import Batch, Dataset, load_idx, load_mnist, slice_batch, synth_for_model
from .dpsgd import DpConfig, StepReport, aggregate, dpsgd_step, gaussian, noise_stream, sgd_step, validate
from .harness import (BenchRecord, OptimizerReport, RunOptions, TrainResult, emit_csv, emit_json,
                      evaluate, median, parse_json_file, records_from_json, records_to_json,
                      run_bench, run_epoch, train)
from .models import (LayerKind, LayerSpec, Model, ModelDesc, ModelKind, ModelOptions, build,
                     build_desc, build_from_desc, custom_desc, flatten, unflatten)
from .strategies import ExecMode, GradEngine, PerExampleGrads, Strategy, all_strategies

__all__ = [
    "errors", "lib", "Batch", "Dataset", "load_idx", "load_mnist", "slice_batch",
    "synth_for_model", "DpConfig", "OptimizerReport", "emit_csv", "emit_json",
    "parse_json_file", "records_from_json", "records_to_json",
    "StepReport", "aggregate", "dpsgd_step", "gaussian", "noise_stream", "sgd_step", "validate",
    "BenchRecord", "RunOptions", "TrainResult", "evaluate", "median", "run_bench", "run_epoch",
    "train", "LayerKind", "LayerSpec", "Model", "ModelDesc", "ModelKind", "ModelOptions", "build",
    "build_desc", "build_from_desc", "custom_desc", "flatten", "unflatten", "ExecMode",
    "GradEngine", "PerExampleGrads", "Strategy", "all_strategies",
]
