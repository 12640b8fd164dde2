"""Factor sharding across GPUs.

Factors are independent given the poses (optimizer.cpp:53-56): each rank linearizes a contiguous
slice of the factor list in one launch, and the per-factor 121-double blocks are gathered to
rank 0 (the host solver) with a single collective — the only exchange step of the path. Works with
any torch.distributed backend (NCCL over NVLink on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Sequence

import numpy as np


def partition_factors(point_counts: Sequence[int], world: int) -> list[tuple[int, int]]:
    """Contiguous [begin, end) factor ranges, one per rank, balanced by Σ source points.

    Greedy prefix split at the world-quantiles of the cumulative point count; every rank gets a
    (possibly empty) range and the ranges tile [0, F) in order.
    """
    if world <= 0:
        raise ValueError("world size must be positive")
    w = np.asarray(point_counts, dtype=np.float64)
    F = len(w)
    if F == 0:
        return [(0, 0)] * world
    cum = np.cumsum(w)
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        b = int(np.searchsorted(cum, target, side="left"))
        # pick the closer of b and b+1 as the split point
        if b < F and b + 1 <= F and abs(cum[b] - target) < abs((cum[b - 1] if b > 0 else 0.0) - target):
            b = b + 1
        bounds.append(min(max(b, bounds[-1]), F))
    bounds.append(F)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def gather_blocks(local, counts: Sequence[int], dst: int = 0, group=None):
    """Gather per-rank [F_r, D] tensors to `dst` in rank order; returns the [ΣF_r, D] tensor on
    dst and None elsewhere. Pads to max F_r so one collective suffices."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    fmax = max(int(c) for c in counts)
    D = local.shape[1]
    send = torch.zeros((fmax, D), dtype=local.dtype, device=local.device)
    send[: local.shape[0]].copy_(local)
    bufs = [torch.zeros_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([bufs[r][: int(counts[r])] for r in range(world)], dim=0)
