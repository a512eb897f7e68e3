#!/usr/bin/env python
"""Benchmark: DPSGD examples/sec, MNIST CNN (reference topology, P=26,010),
batch 256 per GPU, C=1.0, sigma=1.1, lr=0.1, synthetic MNIST-shaped data.

    python bench.py [--gpus N --steps K --warmup W]           # our engine
    python bench.py --impl reference ...                       # reference CPU path

Under torchrun each rank drives one GPU with 256 examples per step (weak
scaling: global DP batch 256*N, one NCCL all-reduce of the clipped sum per
step). Prints ONE JSON line on rank 0.

value  : device-resident inputs (a 60,000-example synthetic dataset, 188 MB >
         the 126 MB L2, cycled batch by batch), K steps timed with CUDA events
         on the engine stream, max over ranks.
e2e    : the public epoch driver pgb_run_epoch on PINNED HOST batches: every
         step copies its batch H2D and reads its result (per-example norms +
         clipped count) back D2H; wall time, max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DPSGD examples/sec at batch 256 (MNIST CNN); median epoch time vs CPU ref"
UNIT = "examples/s"
BATCH = 256
CLIP, SIGMA, LR, SEED = 1.0, 1.1, 0.1, 0
DATA_N = 60000  # the paper's MNIST epoch; 188 MB of fp32 pixels > L2


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML every 5 ms."""

    def __init__(self, index=0):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None

    def _run(self):
        N = self.N
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.N:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified reference library compiled here)
# ---------------------------------------------------------------------------

def _ref_worker(steps, warmup, time_cap, q):
    import numpy as np
    import oracle as O
    d = O.build_desc(O.MNIST_CNN)
    p = O.ref_init_params(d, SEED, np.float32)
    nb = 16
    x, y = O.ref_synth(d, BATCH * nb, SEED, np.float32)
    R = O.RefModel(d, O.GROUPCONV, BATCH, p, np.float32)
    for s in range(warmup):
        b = s % nb
        R.step(x[b * BATCH:(b + 1) * BATCH], y[b * BATCH:(b + 1) * BATCH], CLIP, SIGMA, LR, 1,
               SEED, s)
    t0 = time.perf_counter()
    done = 0
    while done < steps and (time.perf_counter() - t0) < time_cap:
        b = done % nb
        R.step(x[b * BATCH:(b + 1) * BATCH], y[b * BATCH:(b + 1) * BATCH], CLIP, SIGMA, LR, 1,
               SEED, warmup + done)
        done += 1
    q.put((done, time.perf_counter() - t0))


def cpu_reference(steps, procs, warmup=1, time_cap=20.0):
    """The reference's own dpsgd_step (groupconv strategy, graph mode, fp32,
    its 2-thread intra-op split) on `procs` independent processes, each over
    its own batches; returns (aggregate ex/s, steps per process, seconds)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ref_worker, args=(steps, warmup, time_cap, q))
          for _ in range(procs)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    value = sum(n * BATCH / t for n, t in res)
    return value, [n for n, _ in res], max(t for _, t in res)


def run_reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    ncpu = os.cpu_count() or 1
    procs = max(1, ncpu // 2)
    value, nsteps, t = cpu_reference(args.steps, procs, warmup=args.warmup,
                                     time_cap=args.ref_seconds)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": int(min(nsteps)), "warmup": args.warmup,
        "ms_per_step": 1e3 * t / max(1, min(nsteps)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (io::synth_for_model, seed 0)", "impl": "reference",
        "config": workload_config(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 2 * procs, "kind": "reference",
                         "sample": f"{procs} processes x up to {args.steps} reference "
                                   f"dpsgd_step(B=256, groupconv, graph, fp32) capped at "
                                   f"{args.ref_seconds:.0f} s each (ran {nsteps}); host "
                                   f"nproc={ncpu}; 2 threads per process, the reference's "
                                   f"maximum (parallel.cpp:30-75)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(world):
    return {"workload": "mnist_cnn DPSGD step (reference topology conv16 8x8/2 p3, maxpool2, "
                        "conv32 4x4, fc512-32, fc32-10; P=26,010)",
            "model": "mnist_cnn", "global_batch": BATCH * world, "per_gpu_batch": BATCH,
            "seq_len": None, "parallelism": f"dp{world}",
            "clip_norm": CLIP, "noise_multiplier": SIGMA, "learning_rate": LR,
            "l2": f"inputs larger than L2: {DATA_N}-example resident dataset (188 MB) cycled "
                  "one batch per step"}


# ---------------------------------------------------------------------------
# our engine
# ---------------------------------------------------------------------------

def algorithmic(name, B, P, nb):
    """Algorithmic bytes per launch for the HBM-bound kernels:
    per-example stacks are B*P fp32 values."""
    if name == "aggregate":
        return B * P * 4 + 2 * P * 4 + B * nb * 8 + B * 4
    if name == "sumsq":
        return B * P * 4 + B * nb * 8
    return None


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2010_09063_b200 as Pk
    from paper_2010_09063_b200 import _lib

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    dev = local
    desc = Pk.build_desc(Pk.ModelKind.mnist_cnn)
    model = Pk.build(Pk.ModelKind.mnist_cnn, SEED)
    if world > 1:
        uid = bytearray(128)
        if rank == 0:
            u = _lib.UniqueIdC()
            _lib.check(_lib.lib.pgb_nccl_unique_id(C.byref(u)))
            uid = bytearray(bytes(u)[:128])
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        engine = Pk.GradEngine(model, Pk.Strategy.groupconv, BATCH, device=dev, rank=rank,
                               world=world, unique_id=obj[0])
    else:
        engine = Pk.GradEngine(model, Pk.Strategy.groupconv, BATCH, device=dev)
    cfg = Pk.DpConfig(CLIP, SIGMA, LR, 1, SEED)
    ccfg = cfg.to_c()

    # synthetic dataset (this rank's shard of the stream: seed + rank)
    data = Pk.synth_for_model(desc, DATA_N, SEED + rank, pinned=True)
    dx = torch.from_numpy(data.inputs).to(f"cuda:{dev}")
    dy = torch.from_numpy(data.labels).to(f"cuda:{dev}")
    nbatches = DATA_N // BATCH
    row = int(np.prod(desc.input_shape))

    sp = C.c_void_p()
    _lib.check(_lib.lib.pgb_device_stream(engine.handle, C.byref(sp)))
    stream = torch.cuda.ExternalStream(sp.value, device=f"cuda:{dev}")

    def step(i):
        b = i % nbatches
        _lib.check(_lib.lib.pgb_dpsgd_step_device(
            engine.handle, C.c_void_p(dx.data_ptr() + b * BATCH * row * 4),
            C.c_void_p(dy.data_ptr() + b * BATCH * 4), C.byref(ccfg), i))

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(args.warmup):
        step(i)
    _lib.check(_lib.lib.pgb_synchronize(engine.handle, None, None))
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        ev0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i)
        ev1.record(stream)
        ev1.synchronize()
        _lib.check(_lib.lib.pgb_synchronize(engine.handle, None, None))
    barrier()
    t = max_over_ranks(ev0.elapsed_time(ev1) * 1e-3)
    value = args.steps * BATCH * world / t
    kps = engine.info().kernels_per_step

    # ---- e2e: public epoch driver from pinned host memory -------------------
    e_steps = max(1, min(args.steps, nbatches))
    sub = Pk.Dataset(data.inputs[: e_steps * BATCH], data.labels[: e_steps * BATCH],
                     data.name, e_steps * BATCH, data.classes)
    norms = np.empty(e_steps * BATCH, np.float32)
    Pk.run_epoch(engine, model, Pk.Dataset(data.inputs[:BATCH * 2], data.labels[:BATCH * 2],
                                            data.name, BATCH * 2, 10), cfg, 0)  # warm
    barrier()
    w0 = time.perf_counter()
    secs, _ = Pk.run_epoch(engine, model, sub, cfg, 10 ** 6, norms)
    w1 = time.perf_counter()
    barrier()
    e2e_t = max_over_ranks(w1 - w0)
    e2e = e_steps * BATCH * world / e2e_t

    # ---- dominant kernel: per-kernel event timing of the same schedule -------
    hbm, bf16, peak_kind = peaks()
    nk = C.c_int32()
    ms = np.zeros(64, np.float32)
    names = C.create_string_buffer(64 * 32)
    _lib.check(_lib.lib.pgb_profile_steps(
        engine.handle, C.c_void_p(dx.data_ptr()), C.c_void_p(dy.data_ptr()), C.byref(ccfg),
        5 * 10 ** 6, 16, 64, _lib.ptr(ms), names, C.byref(nk)))
    kernels = [(names.raw[32 * k:32 * k + 32].split(b"\0")[0].decode(), float(ms[k]))
               for k in range(nk.value)]
    step_ms = sum(m for _, m in kernels)
    P = engine.P
    nb = len(desc.param_shapes)
    roof = None
    hbm_kernels = [(n, m) for n, m in kernels if algorithmic(n, BATCH, P, nb)]
    dom_name, dom_ms = max(kernels, key=lambda km: km[1])
    if hbm_kernels:
        hn, hm = max(hbm_kernels, key=lambda km: km[1])
        ach = algorithmic(hn, BATCH, P, nb) / (hm * 1e-3) / 1e9
        roof = {"kernel": hn, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": None, "peak_kind": peak_kind,
                "share_of_step": hm / step_ms if step_ms else None,
                "avg_launch_us": hm * 1e3}
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                import oracle
                if oracle.ref_available():
                    v, nst, tt = cpu_reference(args.ref_steps, 1, 2, args.ref_seconds)
                    cpu = {"value": v, "unit": UNIT, "cores": 2, "kind": "reference",
                           "sample": f"{nst[0]} reference dpsgd_step calls (B=256, groupconv, "
                                     f"graph mode, fp32; {nst[0] * BATCH} examples) in 1 "
                                     f"process, {tt:.1f} s; host nproc={os.cpu_count()}"}
            except Exception as e:  # pragma: no cover
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                       "sample": f"unavailable: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (bit-identical to io::synth_for_model, seed 0+rank); random-init "
                    "params (models::build seed 0)",
            "config": workload_config(world),
            "e2e": {"value": e2e, "unit": UNIT,
                    "h2d_bytes_per_step": BATCH * row * 4 + BATCH * 4,
                    "d2h_bytes_per_step": BATCH * 4 + 8,
                    "api": "pgb_run_epoch (pinned host batches, per-step H2D + D2H)"},
            "roofline": roof,
            "dominant_kernel": {"name": dom_name, "avg_us": dom_ms * 1e3,
                                "share_of_step": dom_ms / step_ms if step_ms else None},
            "kernels_us": {n: round(m * 1e3, 3) for n, m in kernels},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "gpu_launches": kps * args.steps,
            "kernels_per_step": kps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-steps", type=int, default=200)
    ap.add_argument("--ref-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
