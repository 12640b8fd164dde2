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


def all_gather_rows(local, counts: Sequence[int], group=None):
    """All-gather per-rank [F_r, D] tensors in rank order: every rank gets the [ΣF_r, D] tensor.
    Pads to max F_r so one collective suffices."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    fmax = max(int(c) for c in counts)
    D = local.shape[1]
    send = torch.zeros((fmax, D), dtype=local.dtype, device=local.device)
    send[: local.shape[0]].copy_(local)
    bufs = [torch.zeros_like(send) for _ in range(world)]
    dist.all_gather(bufs, send, group=group)
    return torch.cat([bufs[r][: int(counts[r])] for r in range(world)], dim=0)


class ShardedFactorGraph:
    """The LM's factor interface (linearize_all / total_error, optimizer.cpp:45-75) over a factor
    list split into contiguous, point-balanced ranges across ranks.

    Every rank owns a local graph for its range (a FactorGraph on its GPU; clouds and maps are
    replicated, so no data-path exchange is needed to build it) and runs the SAME LM
    (optimizer.optimize) on identical inputs: each linearization all-gathers the 121-double blocks
    and each error evaluation all-gathers the per-factor errors, summed in global factor order on
    every rank. The LM decisions are therefore identical everywhere (SPMD), and the collectives
    per LM step are exactly the blocks and the errors — poses never need a broadcast.
    """

    def __init__(self, local_graph, ij_all, counts: Sequence[int], num_poses: int, group=None, device="cpu"):
        self.local = local_graph
        self._ij = np.asarray(ij_all, np.int64).reshape(-1, 2)
        self.counts = [int(c) for c in counts]
        self.num_poses = int(num_poses)
        self.group = group
        self.device = device
        if sum(self.counts) != len(self._ij):
            raise ValueError("per-rank factor counts do not tile the factor list")

    def linearize_raw(self, poses):
        import torch

        raw, inl = self.local.linearize_raw(poses)
        local = torch.from_numpy(np.concatenate([np.asarray(raw, np.float64),
                                                 np.asarray(inl, np.float64)[:, None]], axis=1)).to(self.device)
        full = all_gather_rows(local, self.counts, self.group).cpu().numpy()
        return np.ascontiguousarray(full[:, :121]), full[:, 121].astype(np.int32)

    def total_error(self, poses) -> float:
        import torch

        err, _ = self.local.evaluate(poses)
        local = torch.from_numpy(np.asarray(err, np.float64).reshape(-1, 1)).to(self.device)
        full = all_gather_rows(local, self.counts, self.group).cpu().numpy().reshape(-1)
        return float(np.cumsum(full)[-1]) if len(full) else 0.0  # global factor order, sequential
