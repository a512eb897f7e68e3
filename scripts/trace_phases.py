#!/usr/bin/env python
"""Per-phase timeline of the MNIST step kernels from device timestamps.

Needs the trace build:  PGB_TRACE=1 python paper_2010_09063_b200/build.py
(writes libpegrad_b200_trace.so beside the product library; this script
loads it through PGB_LIBRARY). Then, on a GPU: python scripts/trace_phases.py
Prints, for the fused per-example kernel, the mean duration of every phase
(barrier to barrier) on SMs holding one CTA vs two, and for the aggregation
kernel the start / scales / loop / epilogue split per tile kind.
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("PGB_LIBRARY", os.path.join(HERE, "paper_2010_09063_b200",
                                                  "libpegrad_b200_trace.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09063_b200 as P  # noqa: E402
from paper_2010_09063_b200 import _lib  # noqa: E402

AGG, FUSED, NF = 0, 40000, 32
SLOTS = FUSED + NF * 4096
L = _lib.lib
if not hasattr(L, "pgb_debug_trace"):
    sys.exit("not a trace build (PGB_TRACE=1 python paper_2010_09063_b200/build.py)")
L.pgb_debug_trace.argtypes = [C.c_void_p, C.c_int]
B = 256
desc = P.build_desc(P.ModelKind.mnist_cnn)
model = P.build(P.ModelKind.mnist_cnn, 0)
data = P.synth_for_model(desc, B, 0)
eng = P.GradEngine(model, P.Strategy.groupconv, B)
cfg = P.DpConfig(1.0, 1.1, 0.1, 1, 0)
for s in range(5):
    P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, s)
GRAPH = "--graph" in sys.argv
if GRAPH:
    # the last step of a static 8-step graph (the bench path: tc_kernel a
    # programmatic dependent of the previous step's aggregation)
    import torch
    dx = torch.from_numpy(data.inputs).cuda()
    dy = torch.from_numpy(data.labels).cuda()
    n = C.c_int64()
    ccfg = cfg.to_c()
    _lib.check(L.pgb_run_steps_device(eng.handle, C.c_void_p(dx.data_ptr()),
                                      C.c_void_p(dy.data_ptr()), 1, 16, C.byref(ccfg), 0,
                                      C.byref(n)))
    _lib.check(L.pgb_synchronize(eng.handle, None, None))
    _lib.check(L.pgb_debug_trace(None, 0))
    _lib.check(L.pgb_run_steps_device(eng.handle, C.c_void_p(dx.data_ptr()),
                                      C.c_void_p(dy.data_ptr()), 1, 8, C.byref(ccfg), 16,
                                      C.byref(n)))
    _lib.check(L.pgb_synchronize(eng.handle, None, None))
else:
    _lib.check(L.pgb_debug_trace(None, 0))
    P.dpsgd_step(model, eng, data.inputs, data.labels, cfg, 7)
buf = np.zeros(SLOTS, np.int64)
_lib.check(L.pgb_debug_trace(C.c_void_p(buf.ctypes.data), SLOTS))

F = buf[FUSED:FUSED + NF * B].reshape(B, NF)
F = F[F[:, 0] > 0]  # one row per CTA (the tensor-core kernel runs B/2 CTAs)
t0 = F[:, 0].min()
marks = sorted([k for k in list(range(16)) + [23] if F[:, k].all()], key=lambda k: F[0, k])
end = F[:, marks[-1]]
if GRAPH and F[:, 25].all():
    rel = F[:, 25].min()
    pc = lambda v: np.percentile(v, [0, 50, 100]).astype(int)  # noqa: E731
    print(f"  graph step: CTA start {pc(F[:, 0] - rel)} ns, alloc+barrier {pc(F[:, 21] - rel)}, "
          f"images {pc(F[:, 22] - rel)}, wait returns {pc(F[:, 25] - rel)}, phase 1 "
          f"{pc(F[:, 1] - rel)} ns relative to the first wait return")
    print(f"  graph step: conv1 done {pc(F[:, 2] - rel)}, conv2 done {pc(F[:, 5] - rel)}, "
          f"last mark {pc(end - rel)} ns relative to the first wait return")
if F[:, 26].all() and F[:, 27].all():
    pc = lambda v: np.percentile(v, [0, 50, 100]).astype(int)  # noqa: E731
    print(f"  CTA start: last thread starts {pc(F[:, 26] - F[:, 0])} ns after thread 0, arrives at "
          f"the first barrier {pc(F[:, 27] - F[:, 0])}; thread 0 arrives {pc(F[:, 28] - F[:, 0])}, "
          f"barrier done {pc(F[:, 21] - F[:, 0])}")
    if F[:, 29].all() and F[:, 30].all():
        print(f"  thread 0: TMEM alloc done {pc(F[:, 29] - F[:, 0])}, image address "
              f"{pc(F[:, 30] - F[:, 0])}, image copy issued {pc(F[:, 31] - F[:, 0])}, images "
              f"arrive {pc(F[:, 22] - F[:, 0])} ns after start")
if F[:, 24].all():
    print(f"  conv2 pair rows: last CTA done {(F[:, 24].max() - end.max()) / 1e3:.2f} us after its "
          f"clip factor")
    end = F[:, 24]
order = np.argsort(end)
n = len(F)
one, two = (order[:30], order[-100:]) if n == B else (order[:n // 2], order[n // 2:])
print(f"fused kernel: first CTA start -> last end {(end.max() - t0) / 1e3:.2f} us, "
      f"first end {(end.min() - t0) / 1e3:.2f} us")
print("phase  alone(us)  shared(us)" if n == B else "phase  early-half(us)  late-half(us)")
for a, b in zip(marks[:-1], marks[1:]):
    d = F[:, b] - F[:, a]
    print(f"{a:2d}->{b:2d}  {d[one].mean() / 1e3:8.2f}  {d[two].mean() / 1e3:8.2f}")
if F[:, 21].all() and F[:, 22].all() and not F[:, 19].any():
    print(f"  setup: TMEM alloc + barrier {(F[:, 21] - F[:, 0]).mean() / 1e3:.2f} us, image/W1 TMA wait "
          f"{(F[:, 22] - F[:, 21]).mean() / 1e3:.2f} us, Y build {(F[:, 1] - F[:, 22]).mean() / 1e3:.2f} us")
for k in range(16, 19):
    if F[:, k].all():
        print(f"  mark {k}: {(F[:, k] - F[:, 7]).mean() / 1e3:.2f} us after mark 7")
if F[:, 19].all() and F[:, 21].all():
    e23 = F[:, 23].max()
    print(f"  in-kernel aggregation: barrier arrive {(F[:, 19] - e23).min() / 1e3:.2f}.."
          f"{(F[:, 19] - e23).max() / 1e3:.2f} us after the last example ends, released "
          f"{(F[:, 20] - e23).min() / 1e3:.2f}..{(F[:, 20] - e23).max() / 1e3:.2f}, tiles done "
          f"{(F[:, 21] - e23).min() / 1e3:.2f}..{(F[:, 21] - e23).max() / 1e3:.2f}")
A = buf[AGG:AGG + 8 * 4096].reshape(4096, 8)
A = A[A[:, 0] > 0]
if len(A):
    if GRAPH and F[:, 25].all():
        print(f"  graph step: aggregation ends {(A[:, 4].max() - F[:, 25].min()) / 1e3:.2f} us after "
              f"the first wait return of the tensor-core kernel")
    print(f"aggregate: {len(A)} CTAs; first start {(A[:, 0].min() - end.max()) / 1e3:.2f} us after "
          f"the fused kernel's last CTA, last end {(A[:, 4].max() - end.max()) / 1e3:.2f} us after")
    if (A[:, 5] > 0).all():
        rel = (A[:, 5] - end.max()) / 1e3
        print(f"  PDL release (griddepcontrol.wait returns): {rel.min():.2f}..{rel.max():.2f} us after "
              f"the fused kernel's last CTA")
        for k, col in ((0, 1), (1, 2)):
            m = A[:, col] > 0
            if m.any():
                a = A[m]
                pc = lambda v: np.percentile(v, [0, 50, 100]).astype(int)  # noqa: E731
                print(f"  kind {k}: release->loads+scales+sync {pc(a[:, col] - a[:, 5])} ns")
                if k == 0 and (a[:, 6] > 0).all():
                    print(f"    first rows arrive {pc(a[:, 6] - a[:, 5])} ns, scales done "
                          f"{pc(a[:, 7] - a[:, 5])} ns after release")
    for k, col in ((0, 1), (1, 2)):
        m = A[:, col] > 0
        if m.any():
            a = A[m]
            pc = lambda v: np.percentile(v, [0, 50, 100]).astype(int)  # noqa: E731
            print(f"  kind {k}: n={m.sum()} scales+sync {pc(a[:, col] - a[:, 0])} ns, "
                  f"loop {pc(a[:, 3] - a[:, col])}, epilogue {pc(a[:, 4] - a[:, 3])}")
