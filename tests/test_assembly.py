"""Device-side normal-equation assembly: assemble_normal_equations
(block_solver.cpp:14-62) after the batched linearization, on the GPU.

CPU tests pin the restatement (tests/oracle_ctypes.assemble_normal_equations) to the reference's
assembly tests (test_optimizer.cpp:80-140). GPU tests require the device assembly to be
bit-identical to the restated assembly of the same (GPU-linearized) factor blocks — both sum each
block in factor order from zero — and the LM on the device-assembled system to match the host one.
"""
import numpy as np
import pytest

import oracle_ctypes as O


def random_se3_blocks(rng, n_vars, n_factors):  # test_optimizer.cpp:46-77 construction
    ij, blocks = [], []
    for f in range(n_factors):
        if f < n_vars - 1:
            i, j = f, f + 1
        else:
            i = int(rng.uniform(0, n_vars - 1))
            j = int(rng.uniform(0, n_vars))
            if j == i:
                j = (i + 1) % n_vars
        S = np.array([[rng.uniform(-1, 1) for _ in range(12)] for _ in range(12)])
        H = S @ S.T + np.eye(12)
        B = np.zeros(121)
        B[0:36] = H[:6, :6].ravel()
        B[36:72] = H[:6, 6:].ravel()
        B[72:108] = H[6:, 6:].ravel()
        B[108:120] = [rng.uniform(-1, 1) for _ in range(12)]
        ij.append((i, j))
        blocks.append(B)
    return np.array(ij), np.array(blocks)


def dense_assemble(blocks, ij, n):  # oracles.hpp dense_assemble
    H = np.zeros((6 * n, 6 * n))
    b = np.zeros(6 * n)
    for B, (i, j) in zip(blocks, ij):
        Hij = B[36:72].reshape(6, 6)
        H[6 * i:6 * i + 6, 6 * i:6 * i + 6] += B[0:36].reshape(6, 6)
        H[6 * i:6 * i + 6, 6 * j:6 * j + 6] += Hij
        H[6 * j:6 * j + 6, 6 * i:6 * i + 6] += Hij.T
        H[6 * j:6 * j + 6, 6 * j:6 * j + 6] += B[72:108].reshape(6, 6)
        b[6 * i:6 * i + 6] += B[108:114]
        b[6 * j:6 * j + 6] += B[114:120]
    return H, b


# ------------------------------------------------------------------------------ oracle (CPU)
def test_oracle_assembly_single_factor_against_fixed():  # test_optimizer.cpp:80-94
    ij, blocks = random_se3_blocks(O.Rng(60), 2, 1)
    slot_of, diag, off, rhs = O.assemble_normal_equations(blocks, [(0, 1)], [1, 0], 2)
    assert len(diag) == 1 and not off
    assert np.array_equal(diag[0], blocks[0, 72:108].reshape(6, 6))
    assert np.array_equal(rhs[0], blocks[0, 114:120])


def test_oracle_assembly_matches_dense():  # test_optimizer.cpp:118-140
    rng = O.Rng(61)
    for _ in range(10):
        n = 3 + int(rng.uniform(0, 17))
        ij, blocks = random_se3_blocks(rng, n, 2 * n)
        fixed = np.zeros(n, np.uint8)
        fixed[0] = 1
        Hd, bd = dense_assemble(blocks, ij, n)
        slot_of, diag, off, rhs = O.assemble_normal_equations(blocks, ij, fixed, n)
        var_of = {s: v for v, s in enumerate(slot_of) if s >= 0}
        for s, v in var_of.items():
            assert np.abs(rhs[s] - bd[6 * v:6 * v + 6]).max() < 1e-12
            assert np.abs(diag[s] - Hd[6 * v:6 * v + 6, 6 * v:6 * v + 6]).max() < 1e-12
        for (a, b), blk in off.items():
            va, vb = var_of[a], var_of[b]
            assert np.abs(blk - Hd[6 * va:6 * va + 6, 6 * vb:6 * vb + 6]).max() < 1e-12


# ------------------------------------------------------------------------------ GPU
gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    return pytest.importorskip("paper_2109_07073_b200")


def graph_case(V, nframes=8, n=3000, seed=70):
    rng = O.Rng(seed)
    clouds = []
    for _ in range(nframes):
        m, c = rng.gaussian_cloud(n, 10.0)
        clouds.append(V.PointCloud(m.astype(np.float32), V.cov6_from(c)))
    maps = V.GaussianVoxelMap.build_batch(clouds, 1.0)
    poses = np.stack([rng.random_pose(0.05, 0.5) for _ in range(nframes)])
    factors = [V.MatchingCostFactor(j - d, j, clouds[j], maps[j - d]) for j in range(nframes) for d in (1, 2, 5)
               if j - d >= 0]
    factors.append(V.MatchingCostFactor(nframes - 1, 0, clouds[0], maps[nframes - 1]))  # i > j orientation
    return V.FactorGraph(factors, nframes, chunk=2048), poses


@gpu
@pytest.mark.parametrize("fixed_vars", [(0,), (3,), (0, 4), ()])
def test_gpu_assembly_bit_exact(V, fixed_vars):
    graph, poses = graph_case(V)
    n = len(poses)
    fixed = np.zeros(n, np.uint8)
    fixed[list(fixed_vars)] = 1
    plan = graph.assembly_plan(fixed)
    diag, off, rhs = graph.linearize_assembled(poses)
    raw, _ = graph.linearize_raw(poses)
    slot_of, rdiag, roff, rrhs = O.assemble_normal_equations(raw, graph._ij, fixed, n)
    assert plan.num_slots == len(rdiag)
    assert [tuple(p) for p in plan.pairs] == sorted(roff, key=lambda ab: (ab[1], ab[0]))
    assert np.array_equal(diag, rdiag) and np.array_equal(rhs, rrhs)
    for k, (a, b) in enumerate(plan.pairs):
        assert np.array_equal(off[k], roff[(a, b)])
    assert [int(v) for v in plan.var_of_slot] == [int(np.flatnonzero(slot_of == s)[0]) for s in range(plan.num_slots)]


@gpu
def test_gpu_assembly_validation(V):
    graph, poses = graph_case(V, nframes=3, n=500)
    with pytest.raises(ValueError):
        graph.linearize_assembled(poses)  # no plan yet
    with pytest.raises(ValueError):
        graph.assembly_plan(np.zeros(2, np.uint8))


@gpu
def test_gpu_lm_device_assembly_matches_host(V):
    from paper_2109_07073_b200 import optimizer as LM

    graph, poses = graph_case(V, nframes=6, n=4000, seed=71)
    p_host, r_host = LM.optimize(graph, poses, device_assembly=False)
    p_dev, r_dev = LM.optimize(graph, poses, device_assembly=True)
    assert r_dev.iterations == r_host.iterations and r_dev.reason == r_host.reason
    assert abs(r_dev.final_error - r_host.final_error) <= 1e-9 * max(1.0, r_host.final_error)
    assert np.abs(p_dev - p_host).max() < 1e-9


@gpu
@pytest.mark.parametrize("seed", [70, 71, 72])
def test_gpu_linearized_errors_equal_evaluate(V, seed):
    """The error / inlier members of an assembled linearization equal evaluate() bit for bit (the
    speculative LM scores candidates with them)."""
    graph, poses = graph_case(V, seed=seed)
    graph.assembly_plan(np.zeros(len(poses), np.uint8))
    rng = O.Rng(seed + 100)
    for trial in range(3):
        P = poses if trial == 0 else np.stack([O.compose(p, rng.random_pose(0.02, 0.2)) for p in poses])
        graph.linearize_assembled(P)
        err, inl = graph.linearized_errors()
        e_ref, i_ref = graph.evaluate(P)
        assert np.array_equal(inl, i_ref)
        assert np.array_equal(err, e_ref), np.abs(err - e_ref).max()
        raw, rinl = graph.linearize_raw(P)
        assert np.array_equal(raw[:, 120], err) and np.array_equal(rinl, inl)


@gpu
@pytest.mark.parametrize("loop", [False, True])
def test_gpu_lm_speculative_matches_plain(V, loop):
    """Scoring candidates by linearization gives the reference loop's trace exactly (banded host
    solve for a chain, dense GPU solve with a loop closure)."""
    from paper_2109_07073_b200 import optimizer as LM

    rng = O.Rng(73)
    nframes = 8
    clouds = []
    for _ in range(nframes):
        m, c = rng.gaussian_cloud(3000, 10.0)
        clouds.append(V.PointCloud(m.astype(np.float32), V.cov6_from(c)))
    maps = V.GaussianVoxelMap.build_batch(clouds, 1.0)
    poses = np.stack([rng.random_pose(0.05, 0.5) for _ in range(nframes)])
    factors = [V.MatchingCostFactor(j - 1, j, clouds[j], maps[j - 1]) for j in range(1, nframes)]
    if loop:
        factors.append(V.MatchingCostFactor(nframes - 1, 0, clouds[0], maps[nframes - 1]))
    graph = V.FactorGraph(factors, nframes, chunk=2048)
    p0, r0 = LM.optimize(graph, poses, speculative=False)
    p1, r1 = LM.optimize(graph, poses, speculative=True)
    assert r1.iterations == r0.iterations and r1.reason == r0.reason
    assert r1.initial_error == r0.initial_error and r1.final_error == r0.final_error
    assert [(t.error, t.accepted, t.lam) for t in r1.trace] == [(t.error, t.accepted, t.lam) for t in r0.trace]
    assert np.array_equal(p1, p0)


@gpu
def test_gpu_linearize_zero_copy_pinned_buffers(V):
    """Page-locked caller buffers receive the blocks straight from the kernel (zero-copy); the
    result equals the staged path bit for bit, for linearize and evaluate."""
    import torch

    graph, poses = graph_case(V, seed=74)
    F = graph.num_factors()
    ref, ref_inl = graph.linearize_raw(poses)
    out = torch.full((F, 121), float("nan"), dtype=torch.float64).pin_memory().numpy()
    inl = torch.full((F,), -1, dtype=torch.int32).pin_memory().numpy()
    P = torch.from_numpy(np.ascontiguousarray(poses)).pin_memory().numpy()
    for _ in range(2):
        graph.linearize_raw(P, out, inl)
        assert np.array_equal(out, ref) and np.array_equal(inl, ref_inl)
    err, einl = graph.evaluate(poses)
    assert np.array_equal(err, ref[:, 120]) and np.array_equal(einl, ref_inl)


def _damped_dense(diag, off, pairs, rhs, lam):
    from paper_2109_07073_b200 import optimizer as LM

    H, b = LM.slot_system(diag, off, pairs, rhs)
    dg = np.diagonal(H).copy()
    H[np.diag_indices_from(H)] = dg + lam * np.maximum(dg, 1e-10)  # optimizer.cpp:119-123
    return H, b


@gpu
@pytest.mark.parametrize("seed", [70, 75])
def test_gpu_band_solver_matches_dense(V, seed):
    """Block-band Cholesky (RCM order, one cluster launch) vs a dense fp64 solve of the same
    damped system (solve_block_system semantics, block_solver.cpp:64-122)."""
    import torch

    graph, poses = graph_case(V, seed=seed)
    n = len(poses)
    fixed = np.zeros(n, np.uint8)
    fixed[0] = 1
    plan = graph.assembly_plan(fixed)
    bw, ok = graph.solver_plan()
    assert ok and 0 <= bw < plan.num_slots
    S, P = plan.num_slots, len(plan.pairs)
    d_asm = torch.empty((S + P) * 36 + S * 6, dtype=torch.float64, device="cuda")
    d_poses = torch.from_numpy(np.ascontiguousarray(poses)).cuda()
    graph.linearize_assembled_device(d_poses.data_ptr(), d_asm.data_ptr())
    graph.ctx.synchronize()
    a = d_asm.cpu().numpy()
    diag, off, rhs = a[: S * 36].reshape(S, 6, 6), a[S * 36:(S + P) * 36].reshape(P, 6, 6), a[(S + P) * 36:].reshape(S, 6)
    for lam in (1e-6, 1e-3, 1.0):
        x = graph.solve_damped(d_asm.data_ptr(), lam)
        H, b = _damped_dense(diag, off, plan.pairs, rhs, lam)
        ref = np.linalg.solve(H, b)
        assert x is not None
        assert np.abs(x - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max()), np.abs(x - ref).max()
        assert np.array_equal(x, graph.solve_damped(d_asm.data_ptr(), lam))  # deterministic


@gpu
def test_gpu_band_solver_pair_matches_single(V):
    """vgicp_graph_solve_damped_pair: both damping values bit-identical to two single solves, and a
    failing instance does not affect the other (the LM's next damping value rides along)."""
    import torch

    graph, poses = graph_case(V, seed=70)
    fixed = np.zeros(len(poses), np.uint8)
    fixed[0] = 1
    plan = graph.assembly_plan(fixed)
    assert graph.solver_plan()[1]
    S, P = plan.num_slots, len(plan.pairs)
    d_asm = torch.empty((S + P) * 36 + S * 6, dtype=torch.float64, device="cuda")
    graph.linearize_assembled_device(torch.from_numpy(np.ascontiguousarray(poses)).cuda().data_ptr(), d_asm.data_ptr())
    graph.ctx.synchronize()
    for lams in ((1e-6, 1e-5), (1e-3, 1e-2), (1.0, 1.0)):
        pair = graph.solve_damped_pair(d_asm.data_ptr(), lams)
        for lam, x in zip(lams, pair):
            assert x is not None and np.array_equal(x, graph.solve_damped(d_asm.data_ptr(), lam))
    # an indefinite system: negative damping breaks instance 0 only
    a = d_asm.cpu().numpy().copy()
    a[: S * 36].reshape(S, 6, 6)[S // 2] = -np.eye(6) * 1e-3
    bad = torch.from_numpy(a).cuda()
    x0, x1 = graph.solve_damped_pair(bad.data_ptr(), (0.0, 0.0))
    assert x0 is None and x1 is None
    # mixed outcome (what the LM's pair cache relies on): instance 0 fails, the damping rescues
    # instance 1 (the broken block becomes -1e-3 + 1e18·max(-1e-3, 1e-10) = 1e8, far above its
    # couplings), whose x and status stay its own
    x0, x1 = graph.solve_damped_pair(bad.data_ptr(), (0.0, 1e18))
    assert x0 is None and x1 is not None
    assert np.array_equal(x1, graph.solve_damped(bad.data_ptr(), 1e18))
    good = graph.solve_damped_pair(d_asm.data_ptr(), (1e-4, 1e-3))
    assert good[0] is not None and np.array_equal(good[1], graph.solve_damped(d_asm.data_ptr(), 1e-3))


@gpu
def test_gpu_band_solver_random_spd_and_failure(V):
    """Random SPD systems on a graph's block pattern (exact envelope handling incl. transposed
    pairs), and a non-positive-definite pivot block -> None (the reference's failed_slot)."""
    import torch

    graph, poses = graph_case(V, nframes=10, n=1500, seed=76)
    plan = graph.assembly_plan(np.zeros(len(poses), np.uint8))
    graph.solver_plan()
    S, P = plan.num_slots, len(plan.pairs)
    rng = np.random.default_rng(5)
    off = rng.standard_normal((P, 6, 6))
    H = np.zeros((6 * S, 6 * S))
    for k, (a_, b_) in enumerate(plan.pairs):
        H[6 * a_:6 * a_ + 6, 6 * b_:6 * b_ + 6] = off[k]
        H[6 * b_:6 * b_ + 6, 6 * a_:6 * a_ + 6] = off[k].T
    H += (np.abs(H).sum(1).max() + 1.0) * np.eye(6 * S)  # diagonally dominant -> SPD
    diag = np.stack([H[6 * s:6 * s + 6, 6 * s:6 * s + 6] for s in range(S)])
    rhs = rng.standard_normal((S, 6))
    buf = torch.from_numpy(np.concatenate([diag.ravel(), off.ravel(), rhs.ravel()])).cuda()
    x = graph.solve_damped(buf.data_ptr(), 0.0)
    ref = np.linalg.solve(H, rhs.ravel())
    assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()
    bad = diag.copy()
    bad[S // 2] = -np.eye(6)
    buf = torch.from_numpy(np.concatenate([bad.ravel(), off.ravel(), rhs.ravel()])).cuda()
    assert graph.solve_damped(buf.data_ptr(), 0.0) is None
    assert graph.solve_damped(torch.from_numpy(np.concatenate([diag.ravel(), off.ravel(), rhs.ravel()])).cuda()
                              .data_ptr(), 0.0) is not None  # the plan survives a failed solve


@gpu
def test_gpu_lm_band_solver_matches_dense_solver(V):
    from paper_2109_07073_b200 import optimizer as LM

    graph, poses = graph_case(V, nframes=8, n=3000, seed=77)
    p_d, r_d = LM.optimize(graph, poses, band_solve=False)
    p_b, r_b = LM.optimize(graph, poses, band_solve=True)
    assert r_b.iterations == r_d.iterations and r_b.reason == r_d.reason
    assert abs(r_b.final_error - r_d.final_error) <= 1e-9 * max(1.0, r_d.final_error)
    assert np.abs(p_b - p_d).max() < 1e-9


def _lm_graph(V, loop, seed=78, nframes=8):
    rng = O.Rng(seed)
    clouds = []
    for _ in range(nframes):
        m, c = rng.gaussian_cloud(3000, 10.0)
        clouds.append(V.PointCloud(m.astype(np.float32), V.cov6_from(c)))
    maps = V.GaussianVoxelMap.build_batch(clouds, 1.0)
    poses = np.stack([rng.random_pose(0.05, 0.5) for _ in range(nframes)])
    factors = [V.MatchingCostFactor(j - d, j, clouds[j], maps[j - d]) for j in range(1, nframes) for d in (1, 2)
               if j - d >= 0]
    if loop:
        factors.append(V.MatchingCostFactor(nframes - 1, 0, clouds[0], maps[nframes - 1]))
    return V.FactorGraph(factors, nframes, chunk=2048), poses


@gpu
@pytest.mark.parametrize("loop", [False, True])
@pytest.mark.parametrize("solver", ["host_band", "gpu_band", "host_rcm_band"])
def test_gpu_native_lm_matches_python_lm(V, monkeypatch, loop, solver):
    """vgicp_graph_optimize (the LM loop in the library) takes the reference loop's decisions: same
    accepted / rejected sequence, λ schedule, termination reason; errors and poses to 1e-9 (the
    solvers differ in rounding: host band in slot order / device band / host band in RCM order — the
    fallback when the envelope is too wide for the device kernel — vs the Python LM's)."""
    from paper_2109_07073_b200 import optimizer as LM

    if solver != "host_band":
        monkeypatch.setenv("VGICP_LM_NO_HOST_BAND", "1")
    if solver == "host_rcm_band":
        monkeypatch.setenv("VGICP_NO_BAND_SOLVER", "1")
    graph, poses = _lm_graph(V, loop)
    p_py, r_py = LM.optimize(graph, poses, band_solve=False)
    p_nat, r_nat = LM.optimize_native(graph, poses)
    assert r_nat.band_solver == (solver == "gpu_band")
    assert r_nat.iterations == r_py.iterations and r_nat.reason == r_py.reason
    assert [(t.accepted, t.lam) for t in r_nat.trace] == [(t.accepted, t.lam) for t in r_py.trace]
    for a, b in zip(r_nat.trace, r_py.trace):
        assert abs(a.error - b.error) <= 1e-9 * max(1.0, b.error)
    assert r_nat.initial_error == r_py.initial_error
    assert abs(r_nat.final_error - r_py.final_error) <= 1e-9 * max(1.0, r_py.final_error)
    assert np.abs(p_nat - p_py).max() < 1e-9
    assert r_nat.linearizations == len(r_nat.trace) + 1 - sum(1 for t in r_nat.trace if t.step_norm < 1e-8)


@gpu
@pytest.mark.parametrize("lambda_init", [1e-10, 1e-6])
def test_gpu_native_lm_pair_solve_identical(V, monkeypatch, lambda_init):
    """The device solver's pair launch (the next damping value solved alongside) changes nothing
    the LM computes: trace, solve count and poses equal the one-value-per-launch run bit for bit."""
    from paper_2109_07073_b200 import optimizer as LM

    monkeypatch.setenv("VGICP_LM_NO_HOST_BAND", "1")
    graph, poses = _lm_graph(V, True, seed=80)
    st = LM.LmSettings(lambda_init=lambda_init)
    p_pair, r_pair = LM.optimize_native(graph, poses, settings=st)
    monkeypatch.setenv("VGICP_LM_NO_PAIR_SOLVE", "1")
    p_one, r_one = LM.optimize_native(graph, poses, settings=st)
    assert r_pair.band_solver and r_one.band_solver
    assert [(t.accepted, t.lam, t.error) for t in r_pair.trace] == [(t.accepted, t.lam, t.error) for t in r_one.trace]
    assert r_pair.solves == r_one.solves and r_pair.reason == r_one.reason
    assert np.array_equal(p_pair, p_one)


@gpu
def test_gpu_native_lm_fixed_and_updates(V):
    """User-fixed poses stay put, updates_since_orthonormalization counts accepted retractions and
    wraps at 50 (se3.cpp:93-105), max_iterations bounds the run."""
    from paper_2109_07073_b200 import optimizer as LM

    graph, poses = _lm_graph(V, True, seed=79)
    fixed = np.zeros(len(poses), np.uint8)
    fixed[[0, 3]] = 1
    upd = np.full(len(poses), 48, np.int32)
    p, r = LM.optimize_native(graph, poses, fixed=fixed, settings=LM.LmSettings(max_iterations=3), updates=upd)
    assert r.iterations <= 3 and r.iterations >= 1
    assert np.array_equal(p[[0, 3]], poses[[0, 3]])
    moved = np.flatnonzero(fixed == 0)
    assert np.all(upd[[0, 3]] == 48)
    assert np.all(upd[moved] == (48 + r.iterations) % 50)
    R = p[moved, :9].reshape(-1, 3, 3)
    assert np.abs(R @ R.transpose(0, 2, 1) - np.eye(3)).max() < 1e-12  # orthonormalized on the wrap


@gpu
def test_gpu_native_lm_cuda_graph_identical(V, monkeypatch):
    """The native LM's candidate linearizations replayed as CUDA graphs (captured on the second use
    of each assembly buffer) change nothing: trace, solves and poses equal the per-call path."""
    from paper_2109_07073_b200 import optimizer as LM

    graph, poses = _lm_graph(V, True, seed=81)
    monkeypatch.setenv("VGICP_LM_CUDA_GRAPH", "1")
    p1, r1 = LM.optimize_native(graph, poses)
    monkeypatch.delenv("VGICP_LM_CUDA_GRAPH")
    p2, r2 = LM.optimize_native(graph, poses)
    assert [(t.accepted, t.lam, t.error) for t in r1.trace] == [(t.accepted, t.lam, t.error) for t in r2.trace]
    assert r1.linearizations == r2.linearizations and r1.linearizations >= 3
    assert np.array_equal(p1, p2)


@pytest.mark.gpu
@pytest.mark.parametrize("native", [True, False])
def test_zero_factor_graph_terminates_by_step_norm(native):
    """test_optimizer.cpp:301-320 with a matching-only graph: the only factor is a zero factor (disjoint
    clouds, 0 inliers), so the damped system solves to a zero step (damping floor) — the LM ends by
    step norm, not abort, and the free pose is left bit-for-bit unchanged."""
    import paper_2109_07073_b200 as V
    from paper_2109_07073_b200 import optimizer as LM

    ctx = V.default_context(0)
    rng = np.random.default_rng(5)
    tm = rng.normal(size=(500, 3)).astype(np.float32)
    sm = (rng.normal(size=(500, 3)) + [1000.0, 0, 0]).astype(np.float32)
    cov = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (500, 1))
    tgt, src = V.PointCloud(tm, cov, ctx), V.PointCloud(sm, cov, ctx)
    g = V.FactorGraph([V.MatchingCostFactor(0, 1, src, V.GaussianVoxelMap(tgt, 1.0))], 2)
    b = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 1.0, 0, 0])
    P = np.stack([np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0.0]), b])
    fixed = np.array([1, 0], np.uint8)
    run = LM.optimize_native if native else LM.optimize
    poses, rep = run(g, P, fixed=fixed)
    assert not rep.aborted
    assert rep.reason == "converged_step_norm"
    assert np.array_equal(np.asarray(poses)[1], b)


@pytest.mark.gpu
def test_native_lm_isolated_and_disconnected_components():
    """effective_fixed_mask (optimizer.cpp:24-43) on the native LM: a pose no factor touches and a
    second chain without a fixed pose are anchored at their first pose; anchored poses stay bit-for-
    bit, the rest move, and the native and Python LM agree (same trace; poses to 1e-9)."""
    import paper_2109_07073_b200 as V
    from paper_2109_07073_b200 import optimizer as LM

    ctx = V.default_context(0)
    rng = O.Rng(71)
    clouds = []
    for _ in range(5):
        m, c = rng.gaussian_cloud(3000, 6.0)
        m32 = np.asarray(m, np.float32)
        c6 = np.asarray(c).reshape(-1, 9)[:, [0, 1, 2, 4, 5, 8]].astype(np.float32)
        clouds.append(V.PointCloud(m32, c6, ctx))
    maps = V.GaussianVoxelMap.build_batch(clouds, 1.0)
    # chain A: 0-1 (0 fixed by the caller); chain B: 3-4 (no fixed pose); pose 2 isolated
    factors = [V.MatchingCostFactor(0, 1, clouds[1], maps[0]), V.MatchingCostFactor(3, 4, clouds[4], maps[3])]
    g = V.FactorGraph(factors, 5)
    P = np.stack([rng.random_pose(0.02, 0.1) for _ in range(5)])
    fixed = np.array([1, 0, 0, 0, 0], np.uint8)
    pn, rn = LM.optimize_native(g, P, fixed=fixed, settings=LM.LmSettings(max_iterations=5))
    pp, rp = LM.optimize(g, P, fixed=fixed, settings=LM.LmSettings(max_iterations=5))
    pn, pp = np.asarray(pn), np.asarray(pp)
    for v in (0, 2, 3):
        assert np.array_equal(pn[v], P[v]) and np.array_equal(pp[v], P[v])
    assert not np.array_equal(pn[1], P[1]) and not np.array_equal(pn[4], P[4])
    # same accept / reject sequence; poses and errors equal to the solvers' rounding (1e-9, as the
    # native-vs-Python test above)
    assert [(t.accepted, t.lam) for t in rn.trace] == [(t.accepted, t.lam) for t in rp.trace]
    assert np.abs(pn - pp).max() < 1e-9
    assert abs(rn.final_error - rp.final_error) <= 1e-9 * max(1.0, rp.final_error)
