"""LM integration: the batched GPU factors inside the reference's LM loop.

Ports the matching-cost optimizer tests of proj/tests/test_optimizer.cpp (two-pose registration,
non-increasing error trace, gauge invariance, determinism) plus CPU checks of the host-side
assembly / damping / solve against a dense oracle (oracles.hpp:86-127).
"""
import numpy as np
import pytest

import oracle_ctypes as O
from paper_2109_07073_b200 import optimizer as LM


def plane_cov(normal):
    n = np.asarray(normal, float) / np.linalg.norm(normal)
    a = np.array([1.0, 0, 0]) if abs(n[0]) < 0.9 else np.array([0, 1.0, 0])
    u = np.cross(n, a)
    u /= np.linalg.norm(u)
    v = np.cross(n, u)
    V = np.stack([n, u, v], axis=1)
    return V @ np.diag([1e-3, 1.0, 1.0]) @ V.T


def patch_cloud(rng: O.Rng, cells=8, wall=4):  # test_optimizer.cpp:27-44
    means, covs = [], []
    jit = lambda: rng.uniform(0.2, 0.8)  # noqa: E731
    for a in range(-cells, cells):
        for b in range(-cells, cells):
            means.append([a + jit(), b + jit(), 0.0])
            covs.append(plane_cov([0, 0, 1]))
        for h in range(wall):
            means.append([a + jit(), cells + 1.0, h + jit()])
            covs.append(plane_cov([0, 1, 0]))
            means.append([cells + 2.0, a + jit(), h + jit()])
            covs.append(plane_cov([1, 0, 0]))
    return np.array(means), np.array(covs)


# ------------------------------------------------------------------------------ CPU
def test_fixed_mask_anchors_each_component():  # optimizer.cpp:24-43
    m = LM.effective_fixed_mask(5, np.array([[0, 1], [3, 4]]), np.zeros(5, bool))
    assert m.tolist() == [True, False, True, True, False]
    m = LM.effective_fixed_mask(3, np.array([[0, 1], [1, 2]]), np.array([False, True, False]))
    assert m.tolist() == [False, True, False]


def test_assemble_and_solve_match_dense_oracle():  # test_optimizer.cpp:115-172
    rng = np.random.default_rng(62)
    for trial in range(10):
        n = int(rng.integers(2, 12))
        ij, raw = [], []
        for f in range(3 * n):
            i, j = (f, f + 1) if f < n - 1 else tuple(rng.choice(n, 2, replace=False))
            S = rng.uniform(-1, 1, (12, 12))
            Hf = S @ S.T + np.eye(12)
            r = np.zeros(121)
            r[0:36] = Hf[:6, :6].ravel()
            r[36:72] = Hf[:6, 6:].ravel()
            r[72:108] = Hf[6:, 6:].ravel()
            r[108:120] = rng.uniform(-1, 1, 12)
            ij.append((i, j))
            raw.append(r)
        ij, raw = np.array(ij), np.array(raw)
        H, b = LM.assemble(raw, ij, n)
        Hd = np.zeros((6 * n, 6 * n))
        bd = np.zeros(6 * n)
        for (i, j), r in zip(ij, raw):
            Hd[6 * i:6 * i + 6, 6 * i:6 * i + 6] += r[0:36].reshape(6, 6)
            Hd[6 * i:6 * i + 6, 6 * j:6 * j + 6] += r[36:72].reshape(6, 6)
            Hd[6 * j:6 * j + 6, 6 * i:6 * i + 6] += r[36:72].reshape(6, 6).T
            Hd[6 * j:6 * j + 6, 6 * j:6 * j + 6] += r[72:108].reshape(6, 6)
            bd[6 * i:6 * i + 6] += r[108:114]
            bd[6 * j:6 * j + 6] += r[114:120]
        assert np.abs(H - Hd).max() < 1e-12 and np.abs(b - bd).max() < 1e-12
        active = np.ones(n, bool)
        active[int(rng.integers(0, n))] = False
        x = LM.solve_damped(H, b, active, 0.0)
        idx = np.concatenate([np.arange(6 * v, 6 * v + 6) for v in np.flatnonzero(active)])
        assert np.linalg.norm(Hd[np.ix_(idx, idx)] @ x[idx] - bd[idx]) / np.linalg.norm(bd[idx]) < 1e-8


def test_singular_system_reports_failure():  # test_optimizer.cpp:174-186
    H = np.zeros((12, 12))
    H[:6, :6] = H[6:, 6:] = np.eye(6)
    H[:6, 6:] = H[6:, :6] = -np.eye(6)
    assert LM.solve_damped(H, np.zeros(12), np.array([True, True]), 0.0) is None


def test_se3_exp_matches_oracle():
    rng = np.random.default_rng(1)
    for _ in range(50):
        xi = rng.uniform(-1, 1, 6)
        assert np.allclose(LM.se3_exp(xi), O.se3_exp(xi), atol=1e-14)
    assert np.allclose(LM.se3_exp(np.full(6, 1e-10)), O.se3_exp(np.full(6, 1e-10)), atol=1e-18)


# ------------------------------------------------------------------------------ GPU
def registration_graph(seed, perturb_twist, G=None):
    import paper_2109_07073_b200 as V

    rng = O.Rng(seed)
    means, covs = patch_cloud(rng)
    means = O.to_f32_exact(means)
    ctx = V.default_context(0)
    target = V.PointCloud(means, covs, ctx)
    vmap = V.GaussianVoxelMap(target, 1.0)
    truth = LM.se3_exp(perturb_twist)
    # source points expressed in frame 1 == truth⁻¹ · map frame (test_optimizer.cpp:218-220)
    src_means = O.apply_pose(O.inverse(truth), means)
    R = truth[:9].reshape(3, 3)
    src_covs = np.einsum("ij,njk,lk->nil", R.T, covs, R.T)
    source = V.PointCloud(src_means, src_covs, ctx)
    factor = V.MatchingCostFactor(0, 1, source, vmap)
    graph = V.FactorGraph([factor], 2)
    return graph, truth, (target, vmap, source)


@pytest.mark.gpu
def test_two_pose_registration_recovers_relative_pose():  # test_optimizer.cpp:205-229
    twist = np.array([0.005, -0.004, 0.008, 0.3, -0.25, 0.1])
    graph, truth, keep = registration_graph(63, twist)
    start = LM.compose(truth, LM.se3_exp([0.01, 0.01, -0.02, 0.2, -0.15, 0.1]))
    poses, report = LM.optimize(graph, [O.IDENTITY, start], fixed=[True, False])
    assert report.final_error <= report.initial_error
    err = O.compose(O.inverse(truth), poses[1])
    assert np.linalg.norm(err[9:]) < 1e-4
    ang = np.arccos(np.clip((np.trace(err[:9].reshape(3, 3)) - 1) / 2, -1, 1))
    assert ang < 0.01 * np.pi / 180


@pytest.mark.gpu
def test_error_trace_non_increasing():  # test_optimizer.cpp:281-299
    graph, truth, keep = registration_graph(66, np.zeros(6))
    start = LM.se3_exp([0.02, 0.01, -0.03, 0.3, 0.2, -0.2])
    poses, report = LM.optimize(graph, [O.IDENTITY, start], fixed=[True, False])
    last = report.initial_error
    for rec in report.trace:
        if rec.accepted:
            assert rec.error <= last
            last = rec.error
    assert report.final_error <= report.initial_error


@pytest.mark.gpu
def test_gauge_invariance():  # test_optimizer.cpp:322-347
    graph, truth, keep = registration_graph(67, np.zeros(6))
    perturb = LM.se3_exp([0.01, -0.01, 0.02, 0.2, 0.1, -0.15])
    base, _ = LM.optimize(graph, [O.IDENTITY, perturb], fixed=[True, False])
    G = O.Rng(67).random_pose(0.7, 15.0)
    moved, _ = LM.optimize(graph, [G, O.compose(G, perturb)], fixed=[True, False])
    for v in range(2):
        expected = O.compose(G, base[v])
        assert np.abs(moved[v] - expected).max() < 1e-5  # fp32 per-point algebra (reference: 1e-6 in fp64)


@pytest.mark.gpu
def test_lm_deterministic():  # test_optimizer.cpp:349-372
    graph, truth, keep = registration_graph(68, np.zeros(6))
    start = LM.se3_exp([0.02, 0.01, -0.01, 0.25, -0.2, 0.1])
    a, _ = LM.optimize(graph, [O.IDENTITY, start], fixed=[True, False])
    b, _ = LM.optimize(graph, [O.IDENTITY, start], fixed=[True, False])
    assert np.array_equal(a, b)


@pytest.mark.gpu
def test_chain_lm_reduces_error_and_drift():
    """A short C2-style chain (circle, 3 links per frame): LM on the GPU factors lowers the total
    error and moves the drifted odometry toward ground truth."""
    import paper_2109_07073_b200 as V
    from bench_workloads import workloads as W

    spec = W.c2_spec(frames=12, points=5000)
    ctx = V.default_context(0)
    wl = W.build_graph_workload(ctx, spec, links=W.c2_links(12))
    poses, report = LM.optimize(wl.graph, wl.poses)
    assert report.final_error < report.initial_error
    assert report.iterations >= 1
    gt = wl.scans.gt

    def drift(P):
        rel = [O.compose(O.inverse(P[0]), P[k]) for k in range(len(P))]
        rel_gt = [O.compose(O.inverse(gt[0]), gt[k]) for k in range(len(gt))]
        return max(np.linalg.norm(a[9:] - b[9:]) for a, b in zip(rel, rel_gt))

    assert drift(poses) < drift(wl.poses)


def test_batched_se3_matches_scalar():
    rng = np.random.default_rng(3)
    xi = rng.uniform(-1, 1, (20, 6))
    xi[3] = 1e-10
    ref = np.stack([LM.se3_exp(x) for x in xi])
    assert np.allclose(LM.se3_exp_batch(xi), ref, atol=1e-14)
    A = LM.se3_exp_batch(rng.uniform(-1, 1, (20, 6)))
    assert np.allclose(LM.compose_batch(A, ref), np.stack([LM.compose(a, r) for a, r in zip(A, ref)]), atol=1e-14)


def test_banded_solve_matches_dense():
    rng = np.random.default_rng(5)
    from bench_workloads import workloads as W

    ij = np.array(W.c2_links(30))
    raw = np.zeros((len(ij), 121))
    for f in range(len(ij)):
        S = rng.uniform(-1, 1, (12, 12))
        Hf = S @ S.T + np.eye(12)
        raw[f, 0:36], raw[f, 36:72], raw[f, 72:108] = Hf[:6, :6].ravel(), Hf[:6, 6:].ravel(), Hf[6:, 6:].ravel()
        raw[f, 108:120] = rng.uniform(-1, 1, 12)
    H, b = LM.assemble(raw, ij, 30)
    active = np.ones(30, bool)
    active[0] = False
    bw = LM.graph_bandwidth(ij, active)
    assert bw == 6 * 3 + 5
    dense = LM.solve_damped(H, b, active, 1e-3, None)
    banded = LM.solve_damped(H, b, active, 1e-3, bw)
    assert np.allclose(dense, banded, rtol=1e-10, atol=1e-12)
    active[5] = False  # non-contiguous active set -> gather path
    assert np.allclose(LM.solve_damped(H, b, active, 1e-3, None), LM.solve_damped(H, b, active, 1e-3, LM.graph_bandwidth(ij, active)), rtol=1e-10, atol=1e-12)


def test_reduced_solver_banded_matches_dense():
    """Band filled straight from the device-assembled blocks == dense slot system (host)."""
    rng = np.random.default_rng(0)
    S = 12
    pairs = np.array([[a, b] for b in range(S) for a in range(b + 1, min(S, b + 3))], np.int32)
    diag = np.stack([(lambda M: M @ M.T + 6 * np.eye(6))(rng.standard_normal((6, 6))) for _ in range(S)])
    off = rng.standard_normal((len(pairs), 6, 6)) * 0.1
    rhs = rng.standard_normal((S, 6))
    banded = LM._ReducedSolver(diag, off, pairs, rhs, 6 * 2 + 5, None)
    dense = LM._ReducedSolver(diag, off, pairs, rhs, None, None)
    assert banded.banded and not dense.banded
    for lam in (0.0, 1e-3, 10.0):
        assert np.abs(banded.solve(lam) - dense.solve(lam)).max() < 1e-12
    H, b = LM.slot_system(diag, off, pairs, rhs)
    assert np.array_equal(H, H.T)
