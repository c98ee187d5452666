"""Data parallelism by camera view.

One process per GPU.  The scene state (positions, logits, indices, both
codebooks and the host refcount / lineage / free-list mirrors) is replicated;
each rank renders its own shard of the step's views; the only exchange is one
sum-allreduce of the flat gradient buffer ``[d_pos | d_logit | d_SH | d_SR]``
(``GradientSet.flat``), over NCCL on NVLink/NVSwitch, issued in two parts
(engine.Trainer._enqueue_backward): ``[d_pos | d_logit]`` on a side stream as
soon as the per-Gaussian gradients are written, overlapping the codebook
reduce kernels, then ``[d_SH | d_SR]``.  The gradients are
pre-scaled by 1 / (views per rank * world) so the sum is the mean over all
views of the step.  Every rank then applies the identical SGLD update (same
device Philox seed and offset) and the identical MCMC decisions (same host
Generator seed), so replicas stay bit-identical with no broadcast.

Nothing in the reference is distributed (it is single-process numpy); the
batch semantics (mean of per-view gradients) reduce to the reference's
single-view update for one view on one rank.
"""

from __future__ import annotations

import os


def world_info():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_views(views: list, rank: int, world: int) -> list:
    """Contiguous, balanced shard of the step's views for one rank."""
    n = len(views)
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return views[start:start + base + (1 if rank < extra else 0)]


def grad_scale(views_per_rank: int, world: int) -> float:
    """Scale each rank's summed per-view gradients so the allreduced sum is the mean."""
    return 1.0 / (views_per_rank * world)


def make_allreduce(group=None):
    """In-place sum allreduce of a flat gradient tensor (NCCL for CUDA tensors)."""
    import torch.distributed as dist

    def allreduce(flat):
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        return flat

    return allreduce


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (bench timing: the slowest rank defines the step)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
