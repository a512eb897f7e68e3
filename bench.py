#!/usr/bin/env python
"""Benchmark: DPSGD examples/sec at batch 256 (MNIST CNN, reference topology,
P=26,010), C=1.0, sigma=1.1, lr=0.1, synthetic MNIST-shaped data.

    python bench.py [--gpus N --steps K --warmup W] [--model cifar_cnn ...]
    python bench.py --impl reference ...          # the reference's CPU path

Under torchrun the global DP batch (256) is sharded across the N ranks
(rank r takes examples [r*B/N, (r+1)*B/N) of every global batch;
strong scaling), one NCCL all-reduce of the clipped sum per step captured in
the engine's multi-step CUDA graphs, the same noise on every rank from the
shared seed. --weak keeps the per-GPU batch at 256 instead. Prints ONE JSON
line on rank 0.

value  : device-resident inputs (a synthetic dataset larger than the 126 MB
         L2 -- 60,000 MNIST images, 188 MB -- cycled batch by batch), W warm-up
         steps, every CUDA graph of the timed call built untimed
         (pgb_prepare_steps), then K steps timed with CUDA events on the engine
         stream, max over ranks.
e2e    : the public epoch driver pgb_run_epoch on PINNED HOST batches over
         full epochs of the dataset (MNIST: 60,000 examples = 234 steps): every
         step copies its batch H2D and reads its result (per-example norms +
         clipped count) back D2H; the median epoch time over --epochs timed
         epochs after one untimed one (harness.cpp:85-167 reports the median
         epoch), max over ranks.
roofline: per-kernel device times from CUDA events around each launch of the
         same schedule (pgb_profile_steps), algorithmic work per SURVEY 8(d).
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

UNIT = "examples/s"
CLIP, SIGMA, LR, SEED = 1.0, 1.1, 0.1, 0

# model -> (ModelKind, options, strategy, per-GPU batch, dataset size, metric, MFLOP/ex)
MODELS = {
    "mnist_cnn": (2, {}, 4, 256, 60000,
                  "DPSGD examples/sec at batch 256 (MNIST CNN); median epoch time vs CPU ref",
                  1.689, "reference topology conv16 8x8/2 p3, maxpool2, conv32 4x4, "
                         "fc512-32, fc32-10; P=26,010"),
    "cifar_cnn": (3, {}, 4, 256, 12800, "DPSGD examples/sec at batch 256 (CIFAR-10 CNN)",
                  260.6, "8 conv3x3 + 3 avgpool + GAP; P=605,226"),
    "fcnn": (1, {}, 2, 256, 200000, "DPSGD examples/sec at batch 256 (FCNN 104-50-10)",
             0.0238, "dense 104-50-10; P=5,760"),
    "logreg": (0, {}, 2, 256, 300000, "DPSGD examples/sec at batch 256 (logistic regression)",
               0.0006, "dense 104-1, sigmoid head; P=105"),
    "embed": (4, {"hidden": 100}, 5, 512, 16384,
              "DPSGD examples/sec at batch 512 (IMDb-shaped embedding)", 0.05,
              "embedding 10,004x100, mean-pool, dense 100-2; P=1,000,602"),
}


def tc_peaks():
    """Measured TF32 dense and FP32 SGEMM peaks of this pool's B200s
    (scripts/measure_peaks.py -> profiles/*_peaks.json; SURVEY 8(d) asks for
    them beside the bf16 number): the 3xTF32 ceiling of an fp32-accurate
    tensor-core kernel is tf32 / 3."""
    import glob
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_peaks.json")), reverse=True):
        try:
            with open(f) as fh:
                d = json.load(fh)
            return float(d["tf32_tflops"]), float(d["fp32_sgemm_tflops"]), os.path.relpath(f, ROOT)
        except Exception:
            pass
    return None, None, None


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


def ncu_traffic(model, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed ncu --set full capture (profiles/*_<model>_ncu_traffic.json),
    or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_{model.split('_')[0]}_ncu_traffic.json")))
    for f in reversed(files):
        try:
            with open(f) as fh:
                k = json.load(fh)["kernels"].get(kernel)
            if k:
                return k["traffic_bytes"], os.path.relpath(f, ROOT)
        except Exception:
            pass
    return None, None


def ncu_counters(model, kernel):
    """The other per-kernel counters of the same committed capture (or {})."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_{model.split('_')[0]}_ncu_traffic.json")))
    for f in reversed(files):
        try:
            with open(f) as fh:
                k = json.load(fh)["kernels"].get(kernel)
            if k:
                return k
        except Exception:
            pass
    return {}


def workload_config(model, world, per_gpu=0, global_batch=0):
    kind, opts, strat, batch, data_n, _, _, arch = MODELS[model]
    per_gpu = per_gpu or batch
    global_batch = global_batch or per_gpu * world
    return {"workload": f"{model} DPSGD step ({arch})", "model": model,
            "global_batch": global_batch, "per_gpu_batch": per_gpu, "seq_len": None,
            "parallelism": f"dp{world}", "clip_norm": CLIP, "noise_multiplier": SIGMA,
            "learning_rate": LR,
            "l2": f"inputs larger than L2 where the dataset allows: {data_n}-example resident "
                  "synthetic dataset cycled one batch per step"}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified reference library compiled here)
# ---------------------------------------------------------------------------

def _ref_worker(model, steps, warmup, time_cap, q, batch_override=0):
    import numpy as np
    import oracle as O
    kind, opts, strat, batch, _, _, _, _ = MODELS[model]
    batch = batch_override or batch
    strat = {4: O.GROUPCONV, 2: O.OUTER, 5: O.JACMM}.get(strat, strat)
    if model == "fcnn":
        strat = O.NORMS  # the reference's fastest FCNN strategy
    d = O.build_desc(kind, **opts)
    p = O.ref_init_params(d, SEED, np.float32)
    nb = 4
    x, y = O.ref_synth(d, batch * nb, SEED, np.float32)
    R = O.RefModel(d, strat, batch, p, np.float32)
    for s in range(warmup):
        b = s % nb
        R.step(x[b * batch:(b + 1) * batch], y[b * batch:(b + 1) * batch], CLIP, SIGMA, LR, 1,
               SEED, s)
    t0 = time.perf_counter()
    done = 0
    while done < steps and (time.perf_counter() - t0) < time_cap:
        b = done % nb
        R.step(x[b * batch:(b + 1) * batch], y[b * batch:(b + 1) * batch], CLIP, SIGMA, LR, 1,
               SEED, warmup + done)
        done += 1
    q.put((done, time.perf_counter() - t0))


def cpu_reference(model, steps, procs, warmup=1, time_cap=20.0, batch=0):
    """The reference's own dpsgd_step (its fastest strategy, graph mode, fp32,
    its 2-thread intra-op split) on `procs` independent processes, each over
    its own batches; returns (aggregate ex/s, steps per process, seconds)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ref_worker, args=(model, steps, warmup, time_cap, q, batch))
          for _ in range(procs)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    batch = batch or MODELS[model][3]
    value = sum(n * batch / t for n, t in res if n)
    return value, [n for n, _ in res], max(t for _, t in res)


def run_reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    ncpu = os.cpu_count() or 1
    procs = max(1, ncpu // 2)
    value, nsteps, t = cpu_reference(args.model, args.steps, procs, warmup=args.warmup,
                                     time_cap=args.ref_seconds, batch=args.batch)
    batch = args.batch or MODELS[args.model][3]
    line = {
        "metric": MODELS[args.model][5], "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": int(min(nsteps)), "warmup": args.warmup,
        "ms_per_step": 1e3 * t / max(1, min(nsteps)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (io::synth_for_model, seed 0)", "impl": "reference",
        "config": workload_config(args.model, 1, args.batch or MODELS[args.model][3]),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 2 * procs, "kind": "reference",
                         "sample": f"{procs} processes x up to {args.steps} reference "
                                   f"dpsgd_step(B={batch}, graph, fp32) capped at "
                                   f"{args.ref_seconds:.0f} s each (ran {nsteps}); host "
                                   f"nproc={ncpu}; 2 threads per process, the reference's "
                                   f"maximum (parallel.cpp:30-75)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our engine
# ---------------------------------------------------------------------------

def conv_gemm_flops(desc, B):
    """Algorithmic FLOPs of the convolution GEMMs of one step: forward,
    per-example dW and input gradient (2*M*N*K each, single pass; the 3xTF32
    split is not counted as work)."""
    from paper_2010_09063_b200 import LayerKind
    shape = tuple(desc.input_shape)
    first = True
    total = 0
    for l in desc.layers:
        if l.kind == LayerKind.conv:
            C_, H, W = shape
            Ho = (H + 2 * l.pad - l.k) // l.stride + 1
            Wo = (W + 2 * l.pad - l.k) // l.stride + 1
            mnk = B * Ho * Wo * l.out * C_ * l.k * l.k
            total += 2 * mnk * (2 if first else 3)
            shape = (l.out, Ho, Wo)
            first = False
        elif l.kind in (LayerKind.maxpool, LayerKind.avgpool):
            shape = (shape[0], (shape[1] - l.k) // l.stride + 1, (shape[2] - l.k) // l.stride + 1)
        elif l.kind == LayerKind.global_avgpool:
            shape = (shape[0],)
    return total


def aggregate_bytes(desc, B, fused, c2_pairs=False, sparse_embed=False, ghost=False):
    """Bytes the aggregation kernel must read/write: per-example gradient
    sources (materialised rows: B*|p|*4; factored dense blocks: B*(in+out)*4;
    with c2_pairs the MNIST kernel's second conv weight block arrives as
    ceil(B/2) clipped pair rows), the parameters (read + write), norms partials.
    With ghost, the weight blocks of 3x3 / stride-1 convs on 4x4 and 8x8 maps
    are summed by the clip-scaled GEMM (DESIGN 3.2a), not the aggregation."""
    from paper_2010_09063_b200 import LayerKind
    total = 0
    pi = 0
    nconv = 0
    skip_p = 0
    H = W = None
    if len(desc.input_shape) == 3:
        H, W = int(desc.input_shape[1]), int(desc.input_shape[2])
    for l in desc.layers:
        if l.kind == LayerKind.dense:
            total += B * (l.in_ + l.out) * 4 + B * l.out * 4
            pi += 2
        elif l.kind == LayerKind.conv:
            Ho = (H + 2 * l.pad - l.k) // l.stride + 1 if H else None
            Wo = (W + 2 * l.pad - l.k) // l.stride + 1 if W else None
            is_ghost = (ghost and l.k == 3 and l.stride == 1 and l.pad == 1 and Ho
                        and Ho * Wo in (16, 64))
            rows = (B + 1) // 2 if (c2_pairs and nconv == 1) else B
            if is_ghost:
                total += B * l.out * 4
                skip_p += l.out * l.in_ * l.k * l.k
            else:
                total += (rows * l.out * l.in_ * l.k * l.k + B * l.out) * 4
            H, W = Ho, Wo
            nconv += 1
            pi += 2
        elif l.kind in (LayerKind.maxpool, LayerKind.avgpool) and H:
            H, W = (H - l.k) // l.stride + 1, (W - l.k) // l.stride + 1
        elif l.kind == LayerKind.embedding:
            # the sparse step path: embed_agg_kernel (its own roofline line),
            # not the aggregation kernel, sums this block
            if not sparse_embed:
                total += B * l.in_ * l.out * 4
            else:
                skip_p += l.in_ * l.out
            pi += 1
    P = desc.param_count() - skip_p
    return total + 2 * P * 4 + B * 8 * (1 if fused else pi) + B * 4


_PINNED = []


def _pinned(a):
    """A copy of `a` in page-locked host memory (the e2e leg's H2D source)."""
    import numpy as np
    import torch
    t = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
    out = t.numpy()
    np.copyto(out, a)
    _PINNED.append(t)  # the buffer lives as long as the process
    return out


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2010_09063_b200 as Pk
    from paper_2010_09063_b200 import _lib
    from paper_2010_09063_b200.dist import exchange_unique_id

    kind, opts, strat, GBATCH, DATA_N, METRIC, MFLOP, _ = MODELS[args.model]
    if args.batch:  # batch sweeps (BASELINE config 2: FFNN at batch 16-512)
        METRIC = METRIC.replace(f"batch {GBATCH}", f"batch {args.batch}")
        GBATCH = args.batch
    rank, local, world = dist_env()
    if args.weak:
        BATCH = GBATCH            # per-GPU batch fixed, global batch grows with N
        GBATCH = BATCH * world
    else:
        if GBATCH % world:
            raise SystemExit(f"global batch {GBATCH} is not divisible by {world} ranks")
        BATCH = GBATCH // world   # the global batch sharded across the ranks
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    dev = local
    desc = Pk.build_desc(Pk.ModelKind(kind), Pk.ModelOptions(**opts))
    model = Pk.build_from_desc(desc, SEED)
    if world > 1:
        uid = exchange_unique_id(rank)
        engine = Pk.GradEngine(model, Pk.Strategy(strat), BATCH, device=dev, rank=rank,
                               world=world, unique_id=uid)
    elif args.dist_schedule:
        # one GPU running the data-parallel step (aggregate mode 1 -> one-rank
        # ncclAllReduce -> noise_update_kernel): the per-rank cost at N = 256 / B
        from paper_2010_09063_b200.dist import nccl_unique_id
        os.environ["PGB_FORCE_DIST"] = "1"
        engine = Pk.GradEngine(model, Pk.Strategy(strat), BATCH, device=dev, rank=0, world=1,
                               unique_id=nccl_unique_id())
        del os.environ["PGB_FORCE_DIST"]
    else:
        engine = Pk.GradEngine(model, Pk.Strategy(strat), BATCH, device=dev)
    cfg = Pk.DpConfig(CLIP, SIGMA, LR, 1, SEED)
    ccfg = cfg.to_c()

    # synthetic dataset (io::synth_for_model, seed 0), the same on every rank;
    # this rank keeps its shard of every global batch, pinned on the host
    nbatches = DATA_N // GBATCH
    full = Pk.synth_for_model(desc, nbatches * GBATCH, SEED)
    row = int(np.prod(desc.input_shape))
    G = GBATCH // BATCH
    from paper_2010_09063_b200.dist import shard_batches
    xs, ys = shard_batches(full.inputs, full.labels, nbatches, GBATCH, G, rank % G)
    data = Pk.Dataset(_pinned(xs), _pinned(ys), full.name, nbatches * BATCH, full.classes)
    del full
    dx = torch.from_numpy(data.inputs).to(f"cuda:{dev}")
    dy = torch.from_numpy(data.labels).to(f"cuda:{dev}")

    sp = C.c_void_p()
    _lib.check(_lib.lib.pgb_device_stream(engine.handle, C.byref(sp)))
    stream = torch.cuda.ExternalStream(sp.value, device=f"cuda:{dev}")

    def run_steps(i0, n):
        """n steps from step index i0; step i reads resident batch i mod nbatches
        (pgb_run_steps_device: static multi-step CUDA graphs for the fused MNIST
        schedule, one pgb_dpsgd_step_device-equivalent step each)."""
        launches = C.c_int64()
        _lib.check(_lib.lib.pgb_run_steps_device(
            engine.handle, C.c_void_p(dx.data_ptr()), C.c_void_p(dy.data_ptr()), nbatches, n,
            C.byref(ccfg), i0, C.byref(launches)))
        return launches.value

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

    run_steps(0, args.warmup)
    _lib.check(_lib.lib.pgb_synchronize(engine.handle, None, None))
    # one-time setup of the timed call (its multi-step graphs), untimed
    _lib.check(_lib.lib.pgb_prepare_steps(
        engine.handle, C.c_void_p(dx.data_ptr()), C.c_void_p(dy.data_ptr()), nbatches,
        args.steps, C.byref(ccfg)))
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        # hold the stream ~0.2 ms (before the timed region) so the host has
        # queued the timed launches when the first one starts: the events then
        # bracket K back-to-back device steps, not host launch latency
        with torch.cuda.stream(stream):
            torch.cuda._sleep(400_000)
        ev0.record(stream)
        h0 = time.perf_counter()
        timed_launches = run_steps(args.warmup, args.steps)
        host_issue = (time.perf_counter() - h0) / args.steps
        ev1.record(stream)
        ev1.synchronize()
        _lib.check(_lib.lib.pgb_synchronize(engine.handle, None, None))
    barrier()
    t = max_over_ranks(ev0.elapsed_time(ev1) * 1e-3)
    value = args.steps * GBATCH / t
    kps = engine.info().kernels_per_step

    # ---- e2e: public epoch driver from pinned host memory, full epochs ------
    e_steps = nbatches
    norms = np.empty(e_steps * BATCH, np.float32)
    # one untimed epoch: builds the driver's multi-step graphs for every
    # input-chunk slot and touches the pinned pages (one-time setup)
    Pk.run_epoch(engine, model, data, cfg, 0)
    barrier()
    epoch_s = []
    for ep in range(args.epochs):
        barrier()
        w0 = time.perf_counter()
        Pk.run_epoch(engine, model, data, cfg, (ep + 1) * e_steps, norms)
        w1 = time.perf_counter()
        epoch_s.append(max_over_ranks(w1 - w0))
    barrier()
    e2e_t = statistics.median(epoch_s)
    e2e = e_steps * GBATCH / e2e_t

    # ---- per-kernel device time of the same schedule ------------------------
    hbm, bf16, peak_kind = peaks()
    tf32, fp32_sgemm, tf32_src = tc_peaks()
    nk = C.c_int32()
    ms = np.zeros(64, np.float32)
    names = C.create_string_buffer(64 * 32)
    _lib.check(_lib.lib.pgb_profile_steps(
        engine.handle, C.c_void_p(dx.data_ptr()), C.c_void_p(dy.data_ptr()), C.byref(ccfg),
        5 * 10 ** 6, 8, 64, _lib.ptr(ms), names, C.byref(nk)))
    kernels = [(names.raw[32 * k:32 * k + 32].split(b"\0")[0].decode(), float(ms[k]))
               for k in range(nk.value)]
    step_ms = sum(m for _, m in kernels)
    by_name = {}
    for n, m in kernels:
        by_name[n] = by_name.get(n, 0.0) + m
    dom_name, dom_ms = max(by_name.items(), key=lambda kv: kv[1])
    fused = dom_name in ("mnist_fused", "mnist_tc") or "mnist_fused" in by_name or "mnist_tc" in by_name
    roof = None
    if dom_name == "mnist_fused":
        # fp32 CUDA-core kernel: algorithmic FLOPs / time
        flops = MFLOP * 1e6 * BATCH
        ach = flops / (dom_ms * 1e-3) / 1e12
        fp32_peak = 148 * 128 * 2 * (clocks.max_mhz or 1965) * 1e6 / 1e12
        traffic, tsrc = ncu_traffic(args.model, "fused_kernel")
        roof = {"kernel": dom_name, "bound": "tensor", "achieved": ach, "peak": bf16,
                "unit": "TFLOP/s", "frac": ach / bf16, "traffic": traffic,
                "traffic_source": tsrc, "peak_kind": peak_kind,
                "engine": "fp32 FFMA/FFMA2 on CUDA cores; per-example GEMMs are 16-256 wide and "
                          "run shared-memory-bandwidth bound (DESIGN.md 3.1)",
                "fp32_simt_peak_tflops": fp32_peak, "frac_of_fp32_simt_peak": ach / fp32_peak,
                "fp32_sgemm_tflops_measured": fp32_sgemm,
                "share_of_step": dom_ms / step_ms, "avg_launch_us": dom_ms * 1e3}
    elif dom_name == "mnist_tc":
        # the whole per-example pass with its conv GEMMs on tcgen05: algorithmic
        # FLOPs (fwd + input grads + per-example dW, counted once)
        flops = MFLOP * 1e6 * BATCH
        ach = flops / (dom_ms * 1e-3) / 1e12
        traffic, tsrc = ncu_traffic(args.model, "tc_kernel")
        tk = ncu_counters(args.model, "tc_kernel")
        roof = {"kernel": dom_name, "bound": "tensor", "achieved": ach, "peak": bf16,
                "unit": "TFLOP/s", "frac": ach / bf16, "traffic": traffic,
                "traffic_source": tsrc, "peak_kind": peak_kind,
                "engine": "tcgen05.mma kind::tf32 with the 3xTF32 split folded into M/N "
                          "(fp32 parity); conv fwd / per-example dW / input grad on tensor "
                          "cores, pooling, dense layers and the loss on CUDA cores",
                "tf32x3_effective_peak_tflops": (tf32 or bf16 / 2) / 3,
                "frac_of_tf32x3_effective_peak": ach / ((tf32 or bf16 / 2) / 3),
                "tf32_peak_tflops_measured": tf32, "tf32_peak_source": tf32_src,
                "tensor_pipe_active_pct_ncu": tk.get("tensor_pipe_active_pct"),
                "issue_active_pct_ncu": tk.get("issue_active_pct"),
                "share_of_step": dom_ms / step_ms, "avg_launch_us": dom_ms * 1e3}
    elif dom_name.endswith("_tc") or dom_name.endswith("_tma"):
        # every kernel doing the conv GEMM work the algorithmic FLOPs count:
        # forward, input gradient, per-example dW -- or, for the ghost layers,
        # their Gram norms and the clip-scaled summed dW GEMM
        conv = [n for n in by_name if n.endswith("_tc") or n.endswith("_tma")
                or n in ("conv_dw_gram", "conv_dw_sum", "conv_fwd_direct", "conv_dw_pex_direct")]
        tc_ms = sum(by_name[n] for n in conv)
        flops = conv_gemm_flops(desc, BATCH)
        ach = flops / (tc_ms * 1e-3) / 1e12
        roof = {"kernel": "conv GEMMs on tcgen05 (" + ", ".join(conv) + ")",
                "bound": "tensor", "achieved": ach, "peak": bf16, "unit": "TFLOP/s",
                "frac": ach / bf16, "traffic": None, "peak_kind": peak_kind,
                "engine": "tcgen05.mma kind::tf32, 3xTF32 split (work counted once); "
                          "3x3 convs fed by tensor-map TMA (128-B swizzle), the others by "
                          "register gathers; the 3-channel first layer's forward and per-example dW "
                          "(conv_*_direct) on the CUDA cores in fp32, their time counted here",
                "tf32x3_effective_peak_tflops": (tf32 or bf16 / 2) / 3,
                "frac_of_tf32x3_effective_peak": ach / ((tf32 or bf16 / 2) / 3),
                "tf32_peak_tflops_measured": tf32, "tf32_peak_source": tf32_src,
                "share_of_step": tc_ms / step_ms, "avg_launch_us": tc_ms * 1e3}
    if "aggregate" in by_name:
        agg_b = aggregate_bytes(desc, BATCH, fused,
                                c2_pairs=("mnist_tc" in by_name and
                                          os.environ.get("PGB_C2_PAIRS", "1") != "0"),
                                sparse_embed="embed_agg" in by_name,
                                ghost="conv_dw_gram" in by_name)
        am = by_name["aggregate"]
        atraffic, _ = ncu_traffic(args.model, "aggregate_kernel")
        agg = {"kernel": "aggregate", "bound": "hbm", "achieved": agg_b / (am * 1e-3) / 1e9,
               "peak": hbm, "unit": "GB/s", "frac": agg_b / (am * 1e-3) / 1e9 / hbm,
               "traffic": atraffic, "algorithmic_bytes": agg_b, "share_of_step": am / step_ms,
               "avg_launch_us": am * 1e3}
        if roof is None:
            roof = agg
    else:
        agg = None
    if "embed_agg" in by_name:
        # sparse embedding aggregation: per table row the clipped sum over the
        # examples holding it, noise, mean, update. Algorithmic bytes: the
        # table read + write, the pooled cotangents, the per-example distinct
        # tokens and counts, the row bitmaps
        from paper_2010_09063_b200 import LayerKind
        el = next(l for l in desc.layers if l.kind == LayerKind.embedding)
        V, E = el.in_, el.out
        Lq = int(desc.input_shape[0])
        eb = 2 * V * E * 4 + BATCH * E * 4 + 2 * BATCH * Lq * 4 + V * ((BATCH + 31) // 32) * 4
        em = by_name["embed_agg"]
        roof = {"kernel": "embed_agg", "bound": "hbm", "achieved": eb / (em * 1e-3) / 1e9,
                "peak": hbm, "unit": "GB/s", "frac": eb / (em * 1e-3) / 1e9 / hbm,
                "traffic": None, "algorithmic_bytes": eb, "share_of_step": em / step_ms,
                "avg_launch_us": em * 1e3,
                "note": "latency-bound (per-row example lists, fp64 Box-Muller noise for V*E "
                        "elements)"}
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                import oracle
                if oracle.ref_available():
                    v, nst, tt = cpu_reference(args.model, args.ref_steps, 1, 1,
                                               args.ref_seconds, batch=args.batch)
                    cpu = {"value": v, "unit": UNIT, "cores": 2, "kind": "reference",
                           "sample": f"{nst[0]} reference dpsgd_step calls (B={BATCH}, graph "
                                     f"mode, fp32; {nst[0] * BATCH} examples) in 1 process, "
                                     f"{tt:.1f} s; the reference uses 2 threads; host "
                                     f"nproc={os.cpu_count()}"}
            except Exception as e:  # pragma: no cover
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                       "sample": f"unavailable: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (bit-identical to io::synth_for_model, seed 0; rank r takes its "
                    "shard of every global batch); random-init params (models::build seed 0)",
            "config": dict(workload_config(args.model, world, BATCH, GBATCH),
                           **({"schedule": "data-parallel kernels on a one-rank NCCL "
                               "communicator (--dist-schedule)"} if args.dist_schedule else {})),
            "e2e": {"value": e2e, "unit": UNIT,
                    "h2d_bytes_per_step": BATCH * row * 4 + BATCH * 4,
                    "d2h_bytes_per_step": BATCH * 4 + 8,
                    "median_epoch_s": e2e_t, "epoch_examples": e_steps * GBATCH,
                    "epochs_timed": args.epochs,
                    "epoch_s": [round(v, 6) for v in epoch_s],
                    "api": "pgb_run_epoch over full epochs (pinned host batches; every step's inputs copied H2D and its norms + clip count read back D2H inside the timed region, 8 steps per copy / graph launch); value = examples per epoch / median epoch seconds"},
            "roofline": roof,
            "aggregate_roofline": agg,
            "kernels_us": {n: round(m * 1e3, 3) for n, m in by_name.items()},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "gpu_launches": timed_launches,
            "kernels_per_step": kps,
            "host_issue_us_per_step": round(host_issue * 1e6, 2),
            "e2e_us_per_step": round(e2e_t / e_steps * 1e6, 2),
            "median_epoch_s": e2e_t,
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
    ap.add_argument("--model", default="mnist_cnn", choices=sorted(MODELS))
    ap.add_argument("--ref-steps", type=int, default=200)
    ap.add_argument("--ref-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=0,
                    help="global batch override (default: the config's batch)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: --batch (or the config's batch) per GPU")
    ap.add_argument("--dist-schedule", action="store_true",
                    help="one GPU: run the multi-GPU step schedule on a one-rank NCCL "
                         "communicator (per-rank cost proxy for N > 1)")
    ap.add_argument("--epochs", type=int, default=5,
                    help="timed full epochs of the e2e leg (median reported)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
