"""Host logic of the multi-GPU path (data divided into trunks that stay on
their processor; the per-iteration synchronisation of the centroid update is the only
communication).

Members are split into contiguous shards balanced by plan entries sum_k m*m_k (the work of
every B-ADMM iteration), not by member count.  The per-cluster partial sums of each shard are
all-reduced inside libad2 (NCCL); this module only decides the shard bounds and bootstraps the
communicator through torch.distributed.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(offsets: np.ndarray, world: int) -> np.ndarray:
    """Member index bounds [b_0=0, b_1, ..., b_world=N] of `world` contiguous shards whose point
    counts (hence plan entries) are as equal as possible: shard r ends at the first member whose
    cumulative point count reaches r/world of the total."""
    offsets = np.asarray(offsets, np.int64)
    N = len(offsets) - 1
    n = int(offsets[-1])
    bounds = np.zeros(world + 1, np.int64)
    for r in range(1, world):
        target = (n * r + world // 2) // world
        bounds[r] = int(np.searchsorted(offsets, target, side="left"))
    bounds[world] = N
    bounds = np.maximum.accumulate(np.clip(bounds, 0, N))
    return bounds


def shard_slice(b, r: int, bounds: np.ndarray):
    """The r-th shard of a workloads.Bundle (same K, m, d, centroids; its own members)."""
    return b.subset(np.arange(bounds[r], bounds[r + 1]))


def bootstrap_nccl(ctx, group=None):
    """Rank 0 draws an ncclUniqueId through libad2; torch.distributed broadcasts it; every rank
    then attaches its context to the communicator."""
    import torch.distributed as dist
    from . import ad2
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [ad2.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.attach_nccl(world, rank, obj[0])
    return rank, world
