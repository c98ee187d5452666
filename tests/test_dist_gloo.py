"""Multi-process (world_size 2, gloo, CPU) tests of the view-sharded data-parallel
host logic (paper_2509_03775_b200/dist.py).  The device kernels are not
involved: what is exercised is the sharding, the gradient pre-scaling, the
flat-buffer sum allreduce and the max-over-ranks timing reduction."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_03775_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        views = list(range(8))
        mine = D.shard_views(views, rank, world)
        # per-view "gradients": a flat buffer [pos | logit | sh | sr] per view
        rng = np.random.default_rng(0)
        per_view = rng.normal(size=(len(views), 37)).astype(np.float32)
        scale = D.grad_scale(len(mine), world)
        flat = torch.zeros(37, dtype=torch.float32)
        for v in mine:
            flat += torch.from_numpy(per_view[v])
        flat *= scale
        D.make_allreduce()(flat)
        slow = D.max_over_ranks(1.0 + rank)
        out.put((rank, mine, flat.numpy().copy(), slow))
    finally:
        dist.destroy_process_group()


def test_shard_views_partition():
    views = list(range(10))
    for world in (1, 2, 3, 4, 8):
        shards = [D.shard_views(views, r, world) for r in range(world)]
        assert sum(shards, []) == views
        assert max(map(len, shards)) - min(map(len, shards)) <= 1
    with pytest.raises(ValueError):
        D.shard_views(views, 2, 2)


def test_two_rank_allreduce_is_mean_over_views():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, m0, f0, s0), (r1, m1, f1, s1) = res
    assert m0 + m1 == list(range(8))
    # identical replicas after the allreduce, equal to the mean over all views
    assert np.array_equal(f0, f1)
    per_view = np.random.default_rng(0).normal(size=(8, 37)).astype(np.float32)
    assert np.allclose(f0, per_view.mean(0), rtol=1e-6, atol=1e-7)
    assert s0 == s1 == 2.0
