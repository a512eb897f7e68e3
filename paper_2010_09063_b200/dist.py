"""Data-parallel DPSGD over one process per GPU.

Each rank owns a contiguous shard of every minibatch, computes its local
clipped sum  S_r = sum_{i in shard} min(1, C/||g_i||) g_i  on its GPU, and
ONE NCCL all-reduce (inside the engine's CUDA graph, over NVLink/NVSwitch)
produces S = sum_r S_r on every rank. Each rank then adds the SAME Gaussian
noise -- drawn from the shared seed and the step's counter-based stream --
divides by the global number of clipped units and updates its replica, so
the replicas stay bitwise identical and the privacy accounting is that of a
single noise draw per step.

torch.distributed is used only to exchange the NCCL unique id; the
collective itself is issued by libpegrad_b200.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Tuple

from . import _lib


def shard_bounds(rank: int, world: int, batch: int) -> Tuple[int, int]:
    """Examples [lo, hi) of the global batch owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if batch % world:
        raise ValueError(f"global batch {batch} is not divisible by world size {world}")
    per = batch // world
    return rank * per, (rank + 1) * per


def shard_batches(x, y, n_batches: int, global_batch: int, world: int, rank: int):
    """This rank's examples of every global batch of a dataset laid out as
    n_batches consecutive global batches: batch b's rows
    [b*G + lo, b*G + hi) with (lo, hi) = shard_bounds(rank, world, G),
    concatenated -- the per-rank ring pgb_run_steps_device / pgb_run_epoch
    walk (bench.py --gpus N)."""
    import numpy as np
    lo, hi = shard_bounds(rank, world, global_batch)
    per = hi - lo
    row = int(np.prod(x.shape[1:]))
    xs = np.ascontiguousarray(
        x[: n_batches * global_batch].reshape(n_batches, global_batch, row)[:, lo:hi]).reshape(
            (n_batches * per,) + tuple(x.shape[1:]))
    ys = np.ascontiguousarray(
        y[: n_batches * global_batch].reshape(n_batches, global_batch)[:, lo:hi]).reshape(-1)
    return xs, ys


def nccl_unique_id() -> bytes:
    u = _lib.UniqueIdC()
    _lib.check(_lib.lib.pgb_nccl_unique_id(C.byref(u)))
    return bytes(u)[:128]


def exchange_unique_id(rank: int) -> bytes:
    """Rank 0 creates the NCCL id; torch.distributed broadcasts it."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]
