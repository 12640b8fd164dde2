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


# ------------------------------------------------------------------------------------------------
# One process per GPU (torchrun): rank r linearizes its share of ONE graph, rank 0 runs the LM.
# ------------------------------------------------------------------------------------------------
class RankShare:
    """This rank's share of a factor graph split across processes: factors [first, first + count)
    as a FactorGraph.create_range on the rank's GPU (the whole list's work decomposition, so its
    blocks are bit-identical to a single-GPU graph's). blocks(poses) returns the share's
    [count, 122] rows (121 block doubles + the inlier count) as a device tensor."""

    def __init__(self, graph, first: int, count: int, device):
        import torch

        self.graph, self.first, self.count, self.device = graph, int(first), int(count), device
        self._out = torch.empty((max(self.count, 1), 122), dtype=torch.float64, device=device)
        self._inl = torch.empty(max(self.count, 1), dtype=torch.int32, device=device)
        self._poses = None

    def blocks(self, poses):
        import torch

        if self._poses is None or self._poses.shape != poses.shape:
            self._poses = torch.empty_like(poses, device=self.device)
        self._poses.copy_(poses)
        torch.cuda.current_stream(self.device).synchronize()  # the context stream may differ from torch's
        blk = torch.empty((max(self.count, 1), 121), dtype=torch.float64, device=self.device)
        if self.count:
            self.graph.linearize_device(self._poses.data_ptr(), blk.data_ptr(), self._inl.data_ptr())
            self.graph.ctx.synchronize()
        self._out[:, :121].copy_(blk)
        self._out[:, 121].copy_(self._inl.to(torch.float64))
        return self._out[: self.count]


_CMD_STOP, _CMD_LINEARIZE = 0, 1


class GatheredGraph:
    """Rank 0's LM graph over a factor graph split across processes. Each
    linearization is ONE collective step: rank 0 broadcasts the command and the poses, every rank
    linearizes its share in one launch (RankShare), and the [F_r, 122] rows are gathered to rank 0 in
    factor order over one NCCL gather (NVLink). Rank 0 assembles the gathered blocks on its device
    (vgicp_graph_assemble_device with `root_graph`, a whole-list graph used only for planning,
    assembly and the damped solves) — the same kernel over the same blocks as a single-GPU run, so
    the assembled systems, errors and LM trace are bit-identical to it. The other ranks run serve()
    until rank 0 calls stop(). With root_graph=None (CPU tests) the assembly is the host restatement."""

    def __init__(self, share, counts, num_poses: int, ij_all, root_graph=None, group=None):
        import torch.distributed as dist

        self.share = share
        self.counts = [int(c) for c in counts]
        self.num_poses = int(num_poses)
        self._ij = np.asarray(ij_all, np.int64).reshape(-1, 2)
        self.root = root_graph
        self.group = group
        self.rank = dist.get_rank(group)
        self.ctx = root_graph.ctx if root_graph is not None else None
        self._last = None  # host copy of the last gathered rows (errors, inliers)
        if sum(self.counts) != len(self._ij):
            raise ValueError("per-rank factor counts do not tile the factor list")

    # ---- the collective step ----
    def _device(self):
        return self.share.device

    def _step(self, poses_np):
        """One distributed linearization at poses (rank 0: numpy n×12, others: None). Returns the
        [F, 122] gathered rows on rank 0's device (None elsewhere)."""
        import torch
        import torch.distributed as dist

        dev = self._device()
        cmd = torch.tensor([_CMD_LINEARIZE], dtype=torch.int64, device=dev)
        dist.broadcast(cmd, 0, group=self.group)
        poses = torch.empty((self.num_poses, 12), dtype=torch.float64, device=dev)
        if self.rank == 0:
            poses.copy_(torch.from_numpy(np.ascontiguousarray(poses_np)))
        dist.broadcast(poses, 0, group=self.group)
        local = self.share.blocks(poses)
        return gather_blocks(local, self.counts, dst=0, group=self.group)

    def serve(self) -> int:
        """Ranks != 0: answer linearization steps until rank 0 stops; returns the step count."""
        import torch
        import torch.distributed as dist

        dev = self._device()
        steps = 0
        while True:
            cmd = torch.empty(1, dtype=torch.int64, device=dev)
            dist.broadcast(cmd, 0, group=self.group)
            if int(cmd.item()) == _CMD_STOP:
                return steps
            poses = torch.empty((self.num_poses, 12), dtype=torch.float64, device=dev)
            dist.broadcast(poses, 0, group=self.group)
            gather_blocks(self.share.blocks(poses), self.counts, dst=0, group=self.group)
            steps += 1

    def stop(self) -> None:
        import torch
        import torch.distributed as dist

        dist.broadcast(torch.tensor([_CMD_STOP], dtype=torch.int64, device=self._device()), 0, group=self.group)

    # ---- the LM's graph interface (rank 0) ----
    def linearize_raw(self, poses):
        rows = self._step(poses_array_np(poses)).cpu().numpy()
        self._last = rows
        return np.ascontiguousarray(rows[:, :121]), rows[:, 121].astype(np.int32)

    def total_error(self, poses) -> float:
        raw, _ = self.linearize_raw(poses)  # the linearization's errors equal evaluate's bit for bit
        return float(np.cumsum(raw[:, 120])[-1]) if len(raw) else 0.0

    def linearized_errors(self):
        return np.ascontiguousarray(self._last[:, 120]), self._last[:, 121].astype(np.int32)

    def assembly_plan(self, fixed):
        return self.root.assembly_plan(fixed)

    def solver_plan(self):
        return self.root.solver_plan()

    def solve_damped(self, d_assembled: int, lam: float):
        return self.root.solve_damped(d_assembled, lam)

    def solve_damped_pair(self, d_assembled: int, lams):
        return self.root.solve_damped_pair(d_assembled, lams)

    def linearize_assembled_at(self, poses, d_assembled: int) -> None:
        """The optimizer's device-assembly step at host poses: one collective linearization, then
        the root's assembly kernel over the gathered blocks (factor order) into d_assembled."""
        import torch

        rows = self._step(poses_array_np(poses))
        self._last = rows.cpu().numpy()
        blocks = rows[:, :121].contiguous()
        torch.cuda.current_stream(self._device()).synchronize()
        self.root.assemble_device(blocks.data_ptr(), d_assembled)
        self.root.ctx.synchronize()


    def linearize_assembled(self, poses):
        """Host copy of the assembled system (diag S×6×6, offdiag P×6×6, rhs S×6) at host poses."""
        import torch

        plan = self.root._plan
        S, P = plan.num_slots, len(plan.pairs)
        d_asm = torch.empty((S + P) * 36 + S * 6 + 1, dtype=torch.float64, device=self._device())
        self.linearize_assembled_at(poses, d_asm.data_ptr())
        a = d_asm.cpu().numpy()
        return a[: S * 36].reshape(S, 6, 6), a[S * 36:(S + P) * 36].reshape(P, 6, 6), a[(S + P) * 36:(S + P) * 36 + S * 6].reshape(S, 6)


def poses_array_np(poses) -> np.ndarray:
    P = np.asarray(poses, np.float64)
    return np.ascontiguousarray(P.reshape(-1, 12))
