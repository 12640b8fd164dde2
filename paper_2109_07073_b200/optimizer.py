"""Levenberg–Marquardt over matching-cost factors with batched GPU linearization.

Host-side caller of the hot path, mirroring proj/src/optimizer.cpp:88-194 for graphs whose
factors are all VGICP matching-cost factors: every accepted estimate is re-linearized with ONE
launch for all factors (FactorGraph.linearize, the linearize_all of optimizer.cpp:45-62), every
candidate is scored with ONE error-only launch (total_error, optimizer.cpp:66-75, summed in factor
order on the host), Marquardt damping diag += λ·max(diag, 1e-10) (optimizer.cpp:119-123), step
acceptance iff the error decreases, λ ×0.1 / ×10, termination on relative decrease < 1e-6, step
norm < 1e-8, λ > 1e10 or max iterations. Gauge: the first pose of every connected component
without a fixed variable is anchored (optimizer.cpp:24-43). The reduced normal equations are
assembled on the device (block_solver.cpp:14-62, §8f #3) and solved with a banded host Cholesky
(chains) or a dense Cholesky on the GPU (loop-closing graphs); the reference's block Cholesky,
block_solver.cpp:64-123, is ~3% of the time per PAPER.md:410, and a failed factorization
escalates λ like the reference's failed pivot.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .vgicp import FactorGraph, poses_array

SMALL_ANGLE = 1e-8  # se3.cpp:10
ORTHONORMALIZE_EVERY = 50  # se3.cpp:11


def skew(v):
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def so3_exp(w):  # se3.cpp:46-55
    th = float(np.linalg.norm(w))
    W = skew(w)
    if th < SMALL_ANGLE:
        return np.eye(3) + W + 0.5 * (W @ W)
    return np.eye(3) + (np.sin(th) / th) * W + ((1.0 - np.cos(th)) / (th * th)) * (W @ W)


def so3_left_jacobian(w):  # se3.cpp:14-24
    th = float(np.linalg.norm(w))
    W = skew(w)
    if th < SMALL_ANGLE:
        return np.eye(3) + 0.5 * W + (W @ W) / 6.0
    t2 = th * th
    return np.eye(3) + ((1.0 - np.cos(th)) / t2) * W + ((th - np.sin(th)) / (t2 * th)) * (W @ W)


def se3_exp(xi) -> np.ndarray:  # se3.cpp:74-78, rotation part first
    xi = np.asarray(xi, np.float64)
    R = so3_exp(xi[:3])
    t = so3_left_jacobian(xi[:3]) @ xi[3:]
    return np.concatenate([R.reshape(9), t])


def se3_exp_batch(xi) -> np.ndarray:
    """se3_exp for n twists at once (n × 6 -> n × 12), same formulas and small-angle branch."""
    xi = np.asarray(xi, np.float64).reshape(-1, 6)
    w, v = xi[:, :3], xi[:, 3:]
    th = np.linalg.norm(w, axis=1)
    W = np.zeros((len(xi), 3, 3))
    W[:, 0, 1], W[:, 0, 2], W[:, 1, 0] = -w[:, 2], w[:, 1], w[:, 2]
    W[:, 1, 2], W[:, 2, 0], W[:, 2, 1] = -w[:, 0], -w[:, 1], w[:, 0]
    WW = W @ W
    small = th < SMALL_ANGLE
    ths = np.where(small, 1.0, th)
    a = np.where(small, 1.0, np.sin(ths) / ths)
    b = np.where(small, 0.5, (1.0 - np.cos(ths)) / (ths * ths))
    c = np.where(small, 1.0 / 6.0, (ths - np.sin(ths)) / (ths * ths * ths))
    I = np.eye(3)[None]
    R = I + a[:, None, None] * W + b[:, None, None] * WW
    J = I + b[:, None, None] * W + c[:, None, None] * WW
    t = np.einsum("nij,nj->ni", J, v)
    return np.concatenate([R.reshape(-1, 9), t], axis=1)


def compose_batch(A, B) -> np.ndarray:
    Ra, Rb = A[:, :9].reshape(-1, 3, 3), B[:, :9].reshape(-1, 3, 3)
    return np.concatenate([(Ra @ Rb).reshape(-1, 9), np.einsum("nij,nj->ni", Ra, B[:, 9:]) + A[:, 9:]], axis=1)


def compose(a, b) -> np.ndarray:  # se3.cpp:42-44
    Ra, Rb = a[:9].reshape(3, 3), b[:9].reshape(3, 3)
    return np.concatenate([(Ra @ Rb).reshape(9), Ra @ b[9:] + a[9:]])


def orthonormalized(T) -> np.ndarray:  # se3.cpp:80-91 (polar projection)
    U, _, Vt = np.linalg.svd(T[:9].reshape(3, 3))
    if np.linalg.det(U @ Vt) < 0:
        U[:, 2] = -U[:, 2]
    return np.concatenate([(U @ Vt).reshape(9), T[9:]])


@dataclass
class LmSettings:  # optimizer.hpp:12-21
    max_iterations: int = 50
    lambda_init: float = 1e-5
    lambda_increase: float = 10.0
    lambda_decrease: float = 0.1
    lambda_max: float = 1e10
    relative_error_decrease: float = 1e-6
    step_norm_tolerance: float = 1e-8


@dataclass
class IterationRecord:  # optimizer.hpp:33-39
    iteration: int
    error: float
    lam: float
    step_norm: float
    accepted: bool


@dataclass
class OptimizerReport:  # optimizer.hpp:41-50
    iterations: int = 0
    initial_error: float = 0.0
    final_error: float = 0.0
    trace: list = field(default_factory=list)
    reason: str = "max_iterations"
    wall_time_seconds: float = 0.0
    aborted: bool = False
    diagnostic: str = ""
    iteration_seconds: list = field(default_factory=list)  # wall time of each outer iteration


def effective_fixed_mask(num_poses: int, ij, fixed) -> np.ndarray:  # optimizer.cpp:24-43
    parent = list(range(num_poses))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for i, j in ij:
        parent[find(i)] = find(j)
    out = np.array(fixed, dtype=bool).copy()
    has = {}
    for v in range(num_poses):
        if out[v]:
            has[find(v)] = True
    for v in range(num_poses):
        r = find(v)
        if not has.get(r, False):
            out[v] = True
            has[r] = True
    return out


_ASM_CACHE: dict = {}


def _assembly_indices(ij: np.ndarray, num_poses: int):
    """Flat scatter indices of the 4 H blocks and 2 b segments of every factor (cached per graph)."""
    key = (ij.tobytes(), num_poses)
    hit = _ASM_CACHE.get(key)
    if hit is not None:
        return hit
    n6 = 6 * num_poses
    r6 = np.arange(6)
    rows = lambda v: 6 * v[:, None, None] + r6[None, :, None]  # noqa: E731
    cols = lambda v: 6 * v[:, None, None] + r6[None, None, :]  # noqa: E731
    i, j = ij[:, 0].astype(np.int64), ij[:, 1].astype(np.int64)
    idx_ii = (rows(i) * n6 + cols(i)).reshape(len(ij), 36)
    idx_ij = (rows(i) * n6 + cols(j)).reshape(len(ij), 36)
    idx_ji = (rows(j) * n6 + cols(i)).reshape(len(ij), 36)
    idx_jj = (rows(j) * n6 + cols(j)).reshape(len(ij), 36)
    hidx = np.concatenate([idx_ii, idx_ij, idx_ji, idx_jj], axis=1).ravel()
    bidx = np.concatenate([6 * i[:, None] + r6, 6 * j[:, None] + r6], axis=1).ravel()
    _ASM_CACHE.clear()
    _ASM_CACHE[key] = (hidx, bidx)
    return hidx, bidx


def assemble(raw: np.ndarray, ij: np.ndarray, num_poses: int):
    """Dense normal equations from 121-double factor blocks (block_solver.cpp:14-62 semantics):
    H[i,i] += H_ii, H[i,j] += H_ij, H[j,i] += H_ijᵀ, H[j,j] += H_jj, b[i] += b_i, b[j] += b_j."""
    n6 = 6 * num_poses
    hidx, bidx = _assembly_indices(np.asarray(ij), num_poses)
    F = len(raw)
    Hij = raw[:, 36:72].reshape(F, 6, 6)
    vals = np.concatenate([raw[:, 0:36], raw[:, 36:72], Hij.transpose(0, 2, 1).reshape(F, 36), raw[:, 72:108]], axis=1)
    H = np.bincount(hidx, weights=vals.ravel(), minlength=n6 * n6).reshape(n6, n6)
    b = np.bincount(bidx, weights=raw[:, 108:120].ravel(), minlength=n6)
    return H, b


def _cholesky_solve(Hr, br, lam, bandwidth=None):
    """Marquardt-damped Cholesky solve of a reduced system (optimizer.cpp:119-123); None when the
    damped system is not positive definite (escalates λ like a failed block pivot,
    block_solver.cpp:80-85). Banded LAPACK (pbtrf/pbtrs) when the bandwidth is small, else dense."""
    import scipy.linalg as sla

    m = Hr.shape[0]
    damp = lambda dg: dg + lam * np.maximum(dg, 1e-10)  # noqa: E731
    try:
        if bandwidth is not None and bandwidth < m // 4:
            ab = np.empty((bandwidth + 1, m))  # lower banded storage
            ab[0] = damp(np.diagonal(Hr))
            for k in range(1, bandwidth + 1):
                ab[k, : m - k] = np.diagonal(Hr, -k)
                ab[k, m - k:] = 0.0
            return sla.solveh_banded(ab, br, lower=True, check_finite=False)
        Hd = np.array(Hr, copy=True)
        Hd[np.diag_indices_from(Hd)] = damp(np.diagonal(Hr))
        c = sla.cho_factor(Hd, lower=True, overwrite_a=True, check_finite=False)
        return sla.cho_solve(c, br, check_finite=False)
    except np.linalg.LinAlgError:
        return None


class _ReducedSolver:
    """Damped solves of one device-assembled reduced system (slot order) for successive λ
    (optimizer.cpp:117-131): a banded LAPACK Cholesky on the host when the bandwidth is small
    (odometry chains; the band is filled straight from the blocks), otherwise a dense Cholesky —
    on the GPU (cuSOLVER potrf/potrs through torch; the S + P blocks are uploaded and scattered on
    the device once per linearization) when `device` is given, else on the host."""

    def __init__(self, diag, off, pairs, rhs, bandwidth=None, device=None, band=None):
        S = len(diag)
        m = 6 * S
        self.m, self.rhs = m, rhs.reshape(-1)
        self.band = band  # (graph, device address of the assembled system): GPU block-band Cholesky
        if band is not None:
            self.banded = self.gpu = False
            return
        if not isinstance(diag, np.ndarray) and (bandwidth is not None and bandwidth < m // 4 or device is None):
            diag, off, rhs = diag.cpu().numpy(), off.cpu().numpy(), rhs.cpu().numpy()  # host solvers
            self.rhs = rhs.reshape(-1)
        self.banded = bandwidth is not None and bandwidth < m // 4
        self.gpu = device is not None and not self.banded and m > 0
        if self.banded:
            bw = bandwidth
            ab = np.zeros((bw + 1, m))
            r = np.arange(6)
            rows = np.broadcast_to((6 * np.arange(S))[:, None, None] + r[None, :, None], (S, 6, 6))
            cols = np.broadcast_to((6 * np.arange(S))[:, None, None] + r[None, None, :], (S, 6, 6))
            lower = rows >= cols
            ab[(rows - cols)[lower], cols[lower]] = diag[lower]
            if len(pairs):
                a, b = pairs[:, 0].astype(np.int64), pairs[:, 1].astype(np.int64)
                R = np.broadcast_to((6 * a)[:, None, None] + r[None, :, None], off.shape)
                Cc = np.broadcast_to((6 * b)[:, None, None] + r[None, None, :], off.shape)
                k = (R - Cc).ravel()
                ok = k <= bw
                ab[k[ok], Cc.ravel()[ok]] = off.ravel()[ok]
            self.ab = ab
        elif self.gpu:
            import torch

            self.torch = torch
            tens = lambda x: x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x)).to(device)  # noqa: E731
            Hs = torch.zeros((S, 6, S, 6), dtype=torch.float64, device=device)
            s_idx = torch.arange(S, device=device)
            Hs[s_idx, :, s_idx, :] = tens(diag)
            if len(pairs):
                a = torch.from_numpy(pairs[:, 0].astype(np.int64)).to(device)
                b = torch.from_numpy(pairs[:, 1].astype(np.int64)).to(device)
                O = tens(off)
                Hs[a, :, b, :] = O
                Hs[b, :, a, :] = O.transpose(1, 2)
            self.Hd = Hs.reshape(m, m)
            self.bd = tens(rhs).reshape(-1, 1)
            self.dg = torch.diagonal(self.Hd).clone()
        else:
            self.Hr, _ = slot_system(diag, off, pairs, rhs)

    def solve(self, lam):
        if self.m == 0:
            return np.zeros(0)
        if self.band is not None:
            graph, addr = self.band
            return graph.solve_damped(addr, lam)
        if self.banded:
            import scipy.linalg as sla

            ab = self.ab.copy()
            ab[0] = ab[0] + lam * np.maximum(ab[0], 1e-10)  # optimizer.cpp:119-123
            try:
                return sla.solveh_banded(ab, self.rhs, lower=True, check_finite=False)
            except np.linalg.LinAlgError:
                return None
        if not self.gpu:
            return _cholesky_solve(self.Hr, self.rhs, lam, None)
        torch = self.torch
        A = self.Hd.clone()
        A.diagonal().copy_(self.dg + lam * torch.clamp(self.dg, min=1e-10))
        L, info = torch.linalg.cholesky_ex(A)
        if int(info.item()) != 0:
            return None
        return torch.cholesky_solve(self.bd, L).reshape(-1).cpu().numpy()


def solve_damped(H, b, active, lam, bandwidth=None):
    """Cholesky solve of the damped reduced system of a dense (all-variable) H; None when not
    positive definite."""
    act = np.flatnonzero(active)
    if len(act) == 0:
        return np.zeros_like(b)
    if act[-1] - act[0] + 1 == len(act):  # contiguous active range: a view, no gather
        s0, s1 = 6 * act[0], 6 * (act[-1] + 1)
        Hr, br, idx = H[s0:s1, s0:s1], b[s0:s1], slice(s0, s1)
    else:
        idx = np.flatnonzero(np.repeat(active, 6))
        Hr, br = H[np.ix_(idx, idx)], b[idx]
    x = _cholesky_solve(Hr, br, lam, bandwidth)
    if x is None:
        return None
    delta = np.zeros_like(b)
    delta[idx] = x
    return delta


def slot_system(diag, off, pairs, rhs):
    """Dense reduced system in slot order from the device-assembled blocks (BlockSystem layout:
    off[k] is the (row a, col b) block of pair k, a > b)."""
    S = len(diag)
    Hs = np.zeros((S, 6, S, 6))
    s = np.arange(S)
    Hs[s, :, s, :] = diag
    if len(pairs):
        a, b = pairs[:, 0], pairs[:, 1]
        Hs[a, :, b, :] = off
        Hs[b, :, a, :] = off.transpose(0, 2, 1)
    return Hs.reshape(6 * S, 6 * S), rhs.reshape(-1)


def scatter_slots(x, var_of_slot, num_poses):
    """Slot-space step -> delta_by_var (fixed variables stay zero)."""
    delta = np.zeros(6 * num_poses)
    if x is not None and len(var_of_slot):
        delta.reshape(-1, 6)[var_of_slot] = x.reshape(-1, 6)
    return delta


def _gpu_device(graph: FactorGraph):
    try:
        import torch

        return torch.device("cuda", graph.ctx.device) if torch.cuda.is_available() else None
    except Exception:
        return None


def graph_bandwidth(ij, active) -> int:
    """Scalar half-bandwidth of the reduced normal equations (6·max |rank(i) − rank(j)| + 5)."""
    rank = np.cumsum(active) - 1
    both = active[ij[:, 0]] & active[ij[:, 1]]
    if not both.any():
        return 5
    return int(6 * np.max(np.abs(rank[ij[both, 0]] - rank[ij[both, 1]])) + 5)


DENSE_SOLVE_MAX_UNKNOWNS = 2000  # above: the GPU block-band solver (vgicp_graph_solve_damped)


def _sequential_total(errors) -> float:
    """Σ errors in factor order, left to right (total_error, optimizer.cpp:66-75)."""
    return float(np.cumsum(errors)[-1]) if len(errors) else 0.0


def optimize(graph: FactorGraph, poses, fixed=None, settings: LmSettings | None = None, device_assembly: bool = True,
             gpu_solve: bool = True, speculative: bool = True, band_solve: bool | None = None, on_accept=None):
    """Run LM on `graph` from `poses` (num_poses × 12). Returns (poses, OptimizerReport).

    With device_assembly the normal equations are assembled on the GPU right after the
    linearization (vgicp_graph_linearize_assembled, block_solver.cpp:14-62) and only the S + P
    distinct blocks cross PCIe; otherwise the F factor blocks are downloaded and assembled here.
    With gpu_solve, systems too wide for the banded host solver are factorized on the GPU: with
    band_solve by the block-band Cholesky kernel over a reverse Cuthill-McKee order
    (vgicp_graph_solve_damped, solve_block_system of block_solver.cpp:64-122) when its envelope fits
    one thread-block cluster, else by a dense cuSOLVER Cholesky. band_solve=None picks the band
    kernel above DENSE_SOLVE_MAX_UNKNOWNS reduced unknowns (measured: 1.62 vs 1.84 ms at C3's 2,694
    unknowns, 3.8 vs 5.3 ms at C5's 5,994; dense memory and time grow as m² and m³).

    With speculative (device assembly only), every candidate is scored by LINEARIZING it instead of
    evaluating it: the linearization's per-factor errors equal evaluate_matching_cost's bit for
    bit (vgicp_graph_linearized_errors), so the accept/reject decisions and the trace are those of
    the reference loop (optimizer.cpp:113-186), and an accepted candidate's system is already
    assembled — one factor pass per accepted iteration instead of two (a rejected candidate costs
    the linearize/evaluate difference, ~10%)."""
    settings = settings or LmSettings()
    t_start = time.perf_counter()
    report = OptimizerReport()
    poses = poses_array(poses).copy()
    n = len(poses)
    ij = graph._ij
    fixed_mask = effective_fixed_mask(n, ij, np.zeros(n, bool) if fixed is None else fixed)
    active = ~fixed_mask
    bandwidth = graph_bandwidth(np.asarray(ij), active)
    updates = np.zeros(n, dtype=np.int64)

    if device_assembly:
        plan = graph.assembly_plan(fixed_mask.astype(np.uint8))

    spec = speculative and device_assembly and hasattr(graph, "linearized_errors")
    banded = bandwidth is not None and bandwidth < (6 * int(active.sum())) // 4
    dev = _gpu_device(graph) if (device_assembly and gpu_solve and not banded) else None
    if dev is not None:  # device-resident system: no PCIe round trip of the assembled blocks
        import torch

        S, P = plan.num_slots, len(plan.pairs)
        # two assembled-system buffers: the current system's solver keeps views into one while a
        # speculative candidate linearization fills the other
        d_asms = [torch.empty((S + P) * 36 + S * 6, dtype=torch.float64, device=dev) for _ in range(2 if spec else 1)]
        d_poses = torch.empty((n, 12), dtype=torch.float64, device=dev)
    if band_solve is None:
        band_solve = 6 * int(active.sum()) > DENSE_SOLVE_MAX_UNKNOWNS
    use_band = dev is not None and band_solve and hasattr(graph, "solver_plan") and graph.solver_plan()[1]
    buf = 0

    def linearize_system(at, which=0):
        if dev is not None:
            d_asm = d_asms[which]
            if hasattr(graph, "linearize_assembled_at"):  # a graph split across processes (sharding.py)
                graph.linearize_assembled_at(at, d_asm.data_ptr())
            else:
                d_poses.copy_(torch.from_numpy(np.ascontiguousarray(at)))
                graph.linearize_assembled_device(d_poses.data_ptr(), d_asm.data_ptr())
                graph.ctx.synchronize()  # the context stream may differ from torch's current stream
            return (d_asm[: S * 36].view(S, 6, 6), d_asm[S * 36:(S + P) * 36].view(P, 6, 6),
                    d_asm[(S + P) * 36:].view(S, 6))
        if device_assembly:
            diag, off, rhs = graph.linearize_assembled(at)
            return diag, off, rhs
        return assemble(graph.linearize_raw(at)[0], ij, n)

    system = linearize_system(poses)
    current = _sequential_total(graph.linearized_errors()[0]) if spec else graph.total_error(poses)
    report.initial_error = report.final_error = current
    lam = settings.lambda_init
    any_accepted = False
    for it in range(settings.max_iterations):
        t_it = time.perf_counter()
        if device_assembly:
            solver = _ReducedSolver(*system[:2], plan.pairs, system[2], bandwidth, dev,
                                    band=(graph, d_asms[buf].data_ptr()) if use_band else None)
        else:
            H, b = system
        accepted = False
        while True:
            if device_assembly:
                x = solver.solve(lam)
                delta = None if x is None else scatter_slots(x, plan.var_of_slot, n)
            else:
                delta = solve_damped(H, b, active, lam, bandwidth)
            if delta is None:
                lam *= settings.lambda_increase
                if lam > settings.lambda_max:
                    if not any_accepted:
                        report.aborted = True
                        report.reason = "solver_abort"
                        report.diagnostic = "linear solve failed at maximum damping; poses unchanged"
                    else:
                        report.reason = "lambda_limit"
                    break
                continue
            step_norm = float(np.linalg.norm(delta))
            if step_norm < settings.step_norm_tolerance:
                report.trace.append(IterationRecord(it, current, lam, step_norm, False))
                report.reason = "converged_step_norm"
                break
            cand = poses.copy()
            cand_updates = updates.copy()
            act = np.flatnonzero(active)
            # Pose::retract (se3.cpp:93-101): T · exp(δ), re-orthonormalised every 50 updates
            cand[act] = compose_batch(poses[act], se3_exp_batch(delta.reshape(-1, 6)[act]))
            cand_updates[act] += 1
            for v in act[cand_updates[act] >= ORTHONORMALIZE_EVERY]:
                cand[v] = orthonormalized(cand[v])
                cand_updates[v] = 0
            if spec:
                cand_system = linearize_system(cand, 1 - buf)
                cand_error = _sequential_total(graph.linearized_errors()[0])
            else:
                cand_error = graph.total_error(cand)
            if cand_error < current:
                if spec:
                    system, buf = cand_system, 1 - buf
                decrease = (current - cand_error) / max(current, 1e-300)
                poses, updates = cand, cand_updates
                any_accepted = accepted = True
                report.trace.append(IterationRecord(it, cand_error, lam, step_norm, True))
                if on_accept is not None:  # (iteration, accepted poses, damping used) — test / tooling hook
                    on_accept(it, poses.copy(), lam)
                current = cand_error
                lam = max(lam * settings.lambda_decrease, 1e-12)
                report.iterations += 1
                report.reason = "converged_relative_error" if decrease < settings.relative_error_decrease else report.reason
                break
            report.trace.append(IterationRecord(it, current, lam, step_norm, False))
            lam *= settings.lambda_increase
            if lam > settings.lambda_max:
                report.reason = "lambda_limit"
                break
        if not accepted or report.reason == "converged_relative_error":
            report.iteration_seconds.append(time.perf_counter() - t_it)
            break
        if not spec:
            system = linearize_system(poses)
        report.reason = "max_iterations"
        report.iteration_seconds.append(time.perf_counter() - t_it)
    if not report.aborted:
        report.final_error = current
    report.wall_time_seconds = time.perf_counter() - t_start
    return poses, report


def optimize_native(graph: FactorGraph, poses, fixed=None, settings: LmSettings | None = None, updates=None,
                    max_trace: int = 4096):
    """The same Levenberg-Marquardt run natively in the library (vgicp_graph_optimize): device
    linearization + assembly of every candidate (its errors are total_error), device block-band
    Cholesky (host Cholesky when the envelope is too wide), host retraction — no Python in the loop.
    Returns (poses, OptimizerReport); the graph's assembly plan is replaced by the effective mask's
    (call assembly_plan again before using linearize_assembled)."""
    import ctypes as C

    from . import _lib

    settings = settings or LmSettings()
    P = np.array(poses_array(poses), dtype=np.float64, copy=True)
    n = len(P)
    if n != graph.num_poses:
        raise ValueError("pose count does not match the graph")
    fx = None if fixed is None else np.ascontiguousarray(np.asarray(fixed, dtype=np.uint8).reshape(-1))
    upd = np.zeros(n, np.int32) if updates is None else np.ascontiguousarray(np.asarray(updates, np.int32))
    st = _lib.LmSettingsC(settings.max_iterations, settings.lambda_init, settings.lambda_increase,
                          settings.lambda_decrease, settings.lambda_max, settings.relative_error_decrease,
                          settings.step_norm_tolerance)
    rep = _lib.LmReportC()
    trace = np.zeros((max_trace, 5))
    its = np.zeros(max(1, settings.max_iterations))
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _lib.check(_lib.load().vgicp_graph_optimize(graph._h, ptr(P), ptr(fx) if fx is not None else None, ptr(upd),
                                                C.byref(st), C.byref(rep), ptr(trace), max_trace, ptr(its)))
    graph._plan = None  # the library now holds the effective mask's plan
    report = OptimizerReport(iterations=rep.iterations, initial_error=rep.initial_error, final_error=rep.final_error,
                             reason=_lib.LM_REASONS[rep.reason], wall_time_seconds=rep.wall_time_seconds,
                             aborted=bool(rep.aborted),
                             diagnostic="linear solve failed at maximum damping; poses unchanged" if rep.aborted else "")
    report.trace = [IterationRecord(int(r[0]), float(r[1]), float(r[2]), float(r[3]), bool(r[4]))
                    for r in trace[:min(rep.trace_length, max_trace)]]
    report.iteration_seconds = list(its[:rep.iteration_count_timed])
    report.solves, report.linearizations, report.band_solver = rep.solves, rep.linearizations, bool(rep.band_solver)
    if updates is not None:
        np.asarray(updates)[...] = upd
    return P, report
