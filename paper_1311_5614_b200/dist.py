"""Multi-GPU plumbing for the replica-parallel configurations.

C2/C3 run one problem per rank and C5 shards its batch of independent problems
across ranks: no data-path collective exists (the problems share nothing), only
the timing/statistics reduction at the end (max of times over ranks, sums of
work).  torch.distributed is the plumbing (nccl on GPUs, gloo in CPU tests).
"""
from __future__ import annotations

import os


def world():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_items: int, rank: int, world_size: int) -> list:
    """Round-robin shard of item indices (problem i -> rank i mod P): balanced to
    within one item, deterministic, independent of timing."""
    if world_size < 1 or not (0 <= rank < world_size):
        raise ValueError("bad rank/world")
    return list(range(rank, n_items, world_size))


def reduce_stats(values, device=None):
    """Reduce per-rank statistics: returns (max, sum, min) tensors of `values`
    over all ranks (identity when not distributed).  The bench takes the max of
    device times (the job ends with its slowest rank) and sums the work."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t, t.clone(), t.clone()
    tmax, tsum, tmin = t.clone(), t.clone(), t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    dist.all_reduce(tmin, op=dist.ReduceOp.MIN)
    return tmax, tsum, tmin
