"""The N>1 data-parallel decomposition, checked on CPU with world_size 2
over gloo: per-rank shard clipped sums (oracle) all-reduced equal the
full-batch clipped sum; shared-seed noise keeps replicas identical; the
DPSGD update computed from the reduced sum equals the single-process step."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2010_09063_b200.dist import shard_bounds

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    d = O.build_desc(O.MNIST_CNN)
    B, C, sigma, lr, seed, step = 16, 1.0, 1.1, 0.1, 0, 4
    p = O.init_params(d, 0)
    x, y = O.synth(d, B, 0)
    lo, hi = shard_bounds(rank, world, B)
    # local clipped sum of this rank's shard
    _, norms, nclip, local = O.dpsgd_step(d, x[lo:hi], y[lo:hi], p, C, 0.0, lr, 1, seed, step)
    t = torch.from_numpy(local.copy())
    dist.all_reduce(t)
    c = torch.tensor([nclip], dtype=torch.int64)
    dist.all_reduce(c)
    # shared-seed noise, global mean, update -- what noise_update_kernel does
    noise = np.concatenate([O.gaussian(seed, O.noise_stream(step, q), n)
                            for q, n in enumerate(d.blocks)])
    newp = p - lr * ((t.numpy() + sigma * C * noise) / B)
    out[rank] = (t.numpy(), int(c.item()), newp)
    dist.destroy_process_group()


def test_two_rank_shards_reduce_to_the_full_batch_step():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    import oracle as O
    d = O.build_desc(O.MNIST_CNN)
    p = O.init_params(d, 0)
    x, y = O.synth(d, 16, 0)
    want_p, _, want_clip, want_sum = O.dpsgd_step(d, x, y, p, 1.0, 1.1, 0.1, 1, 0, 4)
    s0, c0, p0 = out[0]
    s1, c1, p1 = out[1]
    np.testing.assert_array_equal(s0, s1)          # all-reduce gives identical bytes
    np.testing.assert_array_equal(p0, p1)          # replicas stay in sync
    assert c0 == c1 == want_clip
    assert np.linalg.norm(s0 - want_sum) <= 1e-12 * np.linalg.norm(want_sum)
    np.testing.assert_allclose(p0, want_p, rtol=1e-12, atol=1e-15)


def _host_worker(rank, world, port, out):
    """The library's host side of the data-parallel path over gloo: the NCCL
    unique id created by rank 0 (pgb_nccl_unique_id) reaches every rank
    byte-identical (dist.exchange_unique_id), and bench.py's shard of every
    global batch (dist.shard_batches) partitions the dataset."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_2010_09063_b200 as P
    from paper_2010_09063_b200.dist import exchange_unique_id, shard_batches

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    uid = exchange_unique_id(rank)
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    desc = P.build_desc(P.ModelKind.mnist_cnn)
    data = P.synth_for_model(desc, 3 * 8, 0)
    xs, ys = shard_batches(data.inputs, data.labels, 3, 8, world, rank)
    parts_x = [None] * world
    parts_y = [None] * world
    dist.all_gather_object(parts_x, xs)
    dist.all_gather_object(parts_y, ys)
    out[rank] = (len(uid), all(i == ids[0] for i in ids), parts_x, parts_y, data.inputs,
                 data.labels)
    dist.destroy_process_group()


def test_host_side_of_data_parallel_path_gloo_world2():
    import numpy as np
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_host_worker, args=(world, port, out), nprocs=world, join=True)
    n, same, px, py, x, y = out[0]
    assert n == 128 and same and out[1][1]
    per = 8 // world
    for b in range(3):
        for r in range(world):
            np.testing.assert_array_equal(px[r][b * per:(b + 1) * per],
                                          x[b * 8 + r * per:b * 8 + (r + 1) * per])
            np.testing.assert_array_equal(py[r][b * per:(b + 1) * per],
                                          y[b * 8 + r * per:b * 8 + (r + 1) * per])
