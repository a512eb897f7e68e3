"""Build libpegrad_b200.so in-tree with nvcc for sm_100a.

    python paper_2010_09063_b200/build.py        # or __graft_entry__.build()

The library bundles the CUDA runtime statically and resolves NCCL with
dlopen at first distributed use, so single-GPU callers need nothing but the
driver.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libpegrad_b200.so")

SOURCES = ["host.cpp", "engine.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "pegrad_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def _nvcc_cmd(out: str, verbose: bool):
    return [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
            "-Xcompiler", "-fPIC,-O3", "-shared", "-I", os.path.join(ROOT, "include"),
            "-I", CSRC, "-Xptxas", "-v" if verbose else "-O3",
            *[os.path.join(CSRC, s) for s in SOURCES], "-o", out, "-ldl"]


def build(force: bool = False, verbose: bool = False) -> str:
    if os.environ.get("PGB_TRACE"):
        return build_trace(verbose)
    if not force and not _stale():
        return OUT
    cmd = _nvcc_cmd(OUT + ".tmp", verbose)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libpegrad_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


TRACE_OUT = os.path.join(PKG, "libpegrad_b200_trace.so")


def build_trace(verbose: bool = False) -> str:
    """The same library with device phase timestamps (-DPGB_TRACE), written
    beside the product build; load it with PGB_LIBRARY=<path>."""
    cmd = _nvcc_cmd(TRACE_OUT + ".tmp", verbose) + ["-DPGB_TRACE"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building the trace library")
    os.replace(TRACE_OUT + ".tmp", TRACE_OUT)
    return TRACE_OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
