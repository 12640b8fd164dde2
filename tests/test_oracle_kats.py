"""Pins the CPU oracle against the reference's own hot-path tests (CPU only, no GPU).

Each test ports a known-answer / brute-force test of /root/reference/proj/tests and cites it.
The reference holds no golden vector files and cannot be built here (no Eigen), so
these ported KATs are what pins the restatement.
"""
import numpy as np
import pytest

import oracle_ctypes as O


def test_single_point_voxel():  # test_voxelmap.cpp:23-34
    means = np.array([[0.2, 0.3, 0.4]])
    covs = np.diag([1.0, 1.0, 1e-3])[None]
    m = O.OracleMap(means, covs, 1.0)
    assert m.size() == 1
    keys, counts, vm, vc = m.export()
    assert m.lookup(means)[0] == keys[0]
    assert counts[0] == 1
    assert np.linalg.norm(vm[0] - means[0]) == 0.0
    assert np.linalg.norm(vc[0] - covs[0]) < 1e-15


def test_two_points_midpoint_and_spread():  # test_voxelmap.cpp:36-48
    m = O.OracleMap([[0.1, 0.1, 0.1], [0.3, 0.1, 0.1]], O.unit_covariances(2), 1.0)
    assert m.size() == 1
    _, counts, vm, vc = m.export()
    assert counts[0] == 2
    assert np.linalg.norm(vm[0] - [0.2, 0.1, 0.1]) < 1e-12
    expected = np.eye(3)
    expected[0, 0] += 0.01
    assert np.linalg.norm(vc[0] - expected) < 1e-12


def test_brute_force_bucketing_1000_points():  # test_voxelmap.cpp:50-69
    rng = O.Rng(10)
    pts = np.array([[rng.uniform(0, 10), rng.uniform(0, 10), rng.uniform(0, 10)] for _ in range(1000)])
    m = O.OracleMap(pts, O.unit_covariances(1000), 1.0)
    buckets = O.brute_force_buckets(pts, 1.0)
    assert m.size() == len(buckets)
    keys, counts, vm, _ = m.export()
    by_key = {int(k): i for i, k in enumerate(keys)}
    for coord, members in buckets.items():
        probe = np.array(coord, dtype=np.float64) + 0.5
        k = int(m.lookup(probe[None])[0])
        assert k != np.iinfo(np.uint64).max
        i = by_key[k]
        assert counts[i] == len(members)
        assert np.linalg.norm(vm[i] - pts[members].mean(axis=0)) < 1e-9


def test_floor_boundary_rule():  # test_voxelmap.cpp:71-82
    m = O.OracleMap([[0.5, 0.5, 0.5]], O.unit_covariances(1), 1.0)
    miss = np.iinfo(np.uint64).max
    got = m.lookup([[0.9, 0.9, 0.9], [5.0, 5.0, 5.0], [1.0, 0.5, 0.5], [0.0, 0.0, 0.0], [1.0 - 1e-12, 0.5, 0.5]])
    assert got[0] != miss and got[1] == miss and got[2] == miss and got[3] != miss and got[4] != miss


def test_total_count_equals_cloud_size():  # test_voxelmap.cpp:84-93
    rng = O.Rng(11)
    pts = np.array([rng.vector(20.0) for _ in range(5000)])
    m = O.OracleMap(pts, O.unit_covariances(5000), 0.7)
    _, counts, _, _ = m.export()
    assert counts.sum() == 5000 and m.total_points() == 5000


def test_order_independence():  # test_voxelmap.cpp:95-120
    rng = O.Rng(12)
    pts = np.array([rng.vector(15.0) for _ in range(3000)])
    perm = rng.shuffle(3000).astype(np.int64)
    a = O.OracleMap(pts, O.unit_covariances(3000), 1.0)
    b = O.OracleMap(pts[perm], O.unit_covariances(3000), 1.0)
    ka, ca, ma, va = a.export()
    kb, cb, mb, vb = b.export()
    assert np.array_equal(ka, kb) and np.array_equal(ca, cb)
    assert np.max(np.linalg.norm(ma - mb, axis=1)) < 1e-9
    assert np.max(np.linalg.norm((va - vb).reshape(-1, 9), axis=1)) < 1e-9


def test_thread_invariance_bitwise():  # test_voxelmap.cpp:122-136
    rng = O.Rng(13)
    pts = np.array([rng.vector(10.0) for _ in range(2000)])
    one = O.OracleMap(pts, O.unit_covariances(2000), 0.5, threads=1, deterministic=True)
    many = O.OracleMap(pts, O.unit_covariances(2000), 0.5, threads=4, deterministic=True)
    for x, y in zip(one.export(), many.export()):
        assert np.array_equal(x, y)


def test_overlap_self_and_far():  # test_voxelmap.cpp:138-149
    rng = O.Rng(14)
    pts = np.array([rng.vector(10.0) for _ in range(2000)])
    m = O.OracleMap(pts, O.unit_covariances(2000), 0.5)
    assert O.overlap_rate(pts, O.IDENTITY, m) == 1.0
    assert O.overlap_rate(pts, O.pose(t=(500, 0, 0)), m) == 0.0


def reference_overlap_scenes(seed=15, scenes=20):
    """test_voxelmap.cpp:151-169 scene stream (identical RNG draw order)."""
    rng = O.Rng(seed)
    out = []
    for _ in range(scenes):
        n_map = 200 + int(rng.uniform(0, 2000))
        n_cloud = 200 + int(rng.uniform(0, 2000))
        res = rng.uniform(0.2, 2.0)
        map_pts = np.array([rng.vector(12.0) for _ in range(n_map)])
        cloud_pts = np.array([rng.vector(12.0) for _ in range(n_cloud)])
        rel = rng.random_pose(0.5, 4.0)
        out.append((map_pts, cloud_pts, res, rel))
    return out


def test_overlap_equals_brute_force_20_scenes():  # test_voxelmap.cpp:151-169
    for map_pts, cloud_pts, res, rel in reference_overlap_scenes():
        m = O.OracleMap(map_pts, O.unit_covariances(len(map_pts)), res)
        got = O.overlap_rate(cloud_pts, rel, m)
        expected = O.brute_force_overlap_count(cloud_pts, rel, map_pts, res)
        assert got == expected / len(cloud_pts)


def test_overlap_37_of_100():  # test_voxelmap.cpp:171-183
    map_pts = [[x + 0.5, y + 0.5, 0.5] for x in range(5) for y in range(5)]
    cloud = [[0.5 + 0.1 * (i % 5), 0.5 + (i // 5 % 5), 0.5] for i in range(37)]
    cloud += [[100.0 + i, 0.0, 0.0] for i in range(63)]
    m = O.OracleMap(map_pts, O.unit_covariances(25), 1.0)
    assert O.overlap_rate(cloud, O.IDENTITY, m) == pytest.approx(0.37)


def test_range_limit_throws():  # test_voxelmap.cpp:185-188
    with pytest.raises(O.OracleOutOfRange):
        O.OracleMap([[2.0e6, 0, 0]], O.unit_covariances(1), 1.0)


def test_invalid_arguments():  # voxelmap.cpp:67-72, :121-123
    with pytest.raises(O.OracleInvalidArgument):
        O.OracleMap([[0.0, 0, 0]], O.unit_covariances(1), 0.0)
    m = O.OracleMap([[0.0, 0, 0]], O.unit_covariances(1), 1.0)
    with pytest.raises(O.OracleInvalidArgument):
        O.overlap_rate(np.zeros((0, 3)), O.IDENTITY, m)


def test_gicp_error_kat():  # test_factors.cpp:92-120
    mean = np.array([1.0, 2.0, 3.0])
    half = 0.5 * np.eye(3)
    err, _, _, _ = O.gicp_error(mean, half, mean, half, O.IDENTITY)
    assert err == 0.0
    err, _, info, valid = O.gicp_error(mean, half, mean + [1, 0, 0], half, O.IDENTITY)
    assert valid and err == pytest.approx(1.0, rel=1e-12)
    assert np.linalg.norm(info - np.eye(3)) < 1e-12
    rng = O.Rng(31)
    rz = O.pose(np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1]], dtype=np.float64))
    p2 = rng.vector(2.0)
    tgt = O.apply_pose(rz, p2)[0] + [0.3, -0.4, 0.2]
    err, res, _, _ = O.gicp_error(p2, half, tgt, half, rz)
    assert err == pytest.approx(res @ res, rel=1e-12)


def test_invert_covariance_singular_rejected():  # factors.cpp:38-46
    ok, _ = O.invert_covariance(np.zeros((3, 3)))
    assert not ok
    ok, _ = O.invert_covariance(np.diag([1.0, 1.0, 0.0]))
    assert not ok
    ok, inv = O.invert_covariance(np.diag([2.0, 4.0, 8.0]))
    assert ok and np.allclose(inv, np.diag([0.5, 0.25, 0.125]), rtol=0, atol=1e-15)
    M = np.array([[2.0, 0.3, 0.1], [0.3, 1.5, -0.2], [0.1, -0.2, 0.004 + 0.05]])
    ok, inv = O.invert_covariance(M)
    assert ok and np.linalg.norm(inv @ M - np.eye(3)) < 1e-12


def test_perfect_alignment():  # test_factors.cpp:122-162
    rng = O.Rng(32)
    means = np.array([rng.vector(5.0) for _ in range(100)])
    covs = np.array([rng.plane_covariance() for _ in range(100)])
    m = O.OracleMap(means, covs, 10.0)
    if m.size() != 100:
        means = np.array([[20.0 * (i % 10) + 5.0, 20.0 * (i // 10) + 5.0, 5.0] for i in range(100)])
        covs = np.array([rng.plane_covariance() for _ in range(100)])
        m = O.OracleMap(means, covs, 10.0)
        assert m.size() == 100
    T = rng.random_pose(0.5, 3.0)
    lin = O.linearize(means, covs, m, T, T)
    assert lin["error"] == pytest.approx(0.0, abs=1e-9)
    assert np.linalg.norm(lin["b_i"]) == pytest.approx(0.0, abs=1e-6)
    assert np.linalg.norm(lin["b_j"]) == pytest.approx(0.0, abs=1e-6)
    assert lin["inliers"] == 100
    H = np.block([[lin["H_ii"], lin["H_ij"]], [lin["H_ij"].T, lin["H_jj"]]])
    assert np.linalg.norm(lin["H_ii"] - lin["H_ii"].T) < 1e-9
    assert np.linalg.norm(lin["H_jj"] - lin["H_jj"].T) < 1e-9
    assert np.linalg.eigvalsh(H).min() > -1e-6


def fd_gradient(poses, cost, h=1e-6):  # oracles.hpp:131-148
    grad = np.zeros(6 * len(poses))
    for v in range(len(poses)):
        for d in range(6):
            delta = np.zeros(6)
            delta[d] = h
            plus = list(poses)
            minus = list(poses)
            plus[v] = O.compose(poses[v], O.se3_exp(delta))
            delta[d] = -h
            minus[v] = O.compose(poses[v], O.se3_exp(delta))
            grad[6 * v + d] = (cost(plus) - cost(minus)) / (2.0 * h)
    return grad


def test_gradient_matches_finite_differences():  # test_factors.cpp:164-181
    rng = O.Rng(33)
    for _ in range(5):
        s = rng.make_scene(200, 1.0)
        m = O.OracleMap(s["target_means"], s["target_covs"], 1.0)
        lin = O.linearize(s["source_means"], s["source_covs"], m, s["T_target"], s["T_source"])
        assert lin["inliers"] > 150
        fd = fd_gradient(
            [s["T_target"], s["T_source"]],
            lambda p: O.frozen_cost(s["source_means"], s["source_covs"], m, s["T_target"], s["T_source"], p[0], p[1]),
        )
        analytic = np.concatenate([-2.0 * lin["b_i"], -2.0 * lin["b_j"]])
        assert np.linalg.norm(analytic - fd) / np.linalg.norm(fd) < 1e-5


def test_quadratic_model_ratio():  # test_factors.cpp:183-222
    rng = O.Rng(34)
    s = rng.make_scene(300, 1.0)
    m = O.OracleMap(s["target_means"], s["target_covs"], 1.0)
    lin = O.linearize(s["source_means"], s["source_covs"], m, s["T_target"], s["T_source"])
    H = np.block([[lin["H_ii"], lin["H_ij"]], [lin["H_ij"].T, lin["H_jj"]]])
    b = np.concatenate([lin["b_i"], lin["b_j"]])
    dir_rng = O.Rng(35)
    direction = np.array([dir_rng.uniform(-1.0, 1.0) for _ in range(12)])
    direction /= np.linalg.norm(direction)
    diffs = []
    scales = [1e-2, 1e-3, 1e-4]
    for sc in scales:
        delta = sc * direction
        Ti = O.retract(s["T_target"], delta[:6])
        Tj = O.retract(s["T_source"], delta[6:])
        actual = O.frozen_cost(s["source_means"], s["source_covs"], m, s["T_target"], s["T_source"], Ti, Tj)
        model = lin["error"] - 2.0 * b @ delta + delta @ H @ delta
        diffs.append(abs(actual - model))
    k0 = diffs[0] / scales[0] ** 2
    for i in range(1, 3):
        assert diffs[i] / scales[i] ** 2 < 8.0 * k0 + 1e-6
    assert diffs[2] / scales[2] < 0.05 * (diffs[0] / scales[0]) + 1e-12


def test_disjoint_zero_factor():  # test_factors.cpp:224-241
    rng = O.Rng(36)
    sm, sc, tm, tc = [], [], [], []
    for _ in range(50):
        sm.append(rng.vector(2.0))
        sc.append(rng.plane_covariance())
        tm.append(rng.vector(2.0) + [1000, 0, 0])
        tc.append(rng.plane_covariance())
    m = O.OracleMap(tm, tc, 1.0)
    lin = O.linearize(sm, sc, m, O.IDENTITY, O.IDENTITY)
    assert lin["inliers"] == 0 and lin["error"] == 0.0
    assert not np.any(lin["raw"])


def test_gauge_invariance():  # test_factors.cpp:243-253
    rng = O.Rng(37)
    s = rng.make_scene(400, 1.0)
    m = O.OracleMap(s["target_means"], s["target_covs"], 1.0)
    base, _ = O.evaluate(s["source_means"], s["source_covs"], m, s["T_target"], s["T_source"])
    for _ in range(10):
        G = rng.random_pose(1.0, 50.0)
        e, _ = O.evaluate(s["source_means"], s["source_covs"], m, O.compose(G, s["T_target"]), O.compose(G, s["T_source"]))
        assert abs(e - base) < 1e-7 * max(1.0, base)


def test_deterministic_across_threads():  # test_factors.cpp:255-267
    rng = O.Rng(38)
    s = rng.make_scene(3000, 1.0)
    m = O.OracleMap(s["target_means"], s["target_covs"], 1.0)
    a = O.linearize(s["source_means"], s["source_covs"], m, s["T_target"], s["T_source"], threads=1, deterministic=True)
    b = O.linearize(s["source_means"], s["source_covs"], m, s["T_target"], s["T_source"], threads=4, deterministic=True)
    assert np.array_equal(a["raw"], b["raw"]) and a["inliers"] == b["inliers"]


def test_parallel_voxelmap_matches_serial():  # test_reference.cpp:43-57
    rng = O.Rng(81)
    means, covs = rng.gaussian_cloud(5000, 20.0)
    serial = O.OracleMap(means, covs, 0.8, serial=True)
    par = O.OracleMap(means, covs, 0.8, threads=2, deterministic=True)
    ks, cs, ms, vs = serial.export()
    kp, cp, mp, vp = par.export()
    assert np.array_equal(ks, kp) and np.array_equal(cs, cp)
    assert np.max(np.linalg.norm(ms - mp, axis=1)) < 1e-9
    assert np.max(np.linalg.norm((vs - vp).reshape(-1, 9), axis=1)) < 1e-9


def test_parallel_overlap_equals_serial():  # test_reference.cpp:59-69
    rng = O.Rng(82)
    mc, mcov = rng.gaussian_cloud(3000, 15.0)
    qc, _ = rng.gaussian_cloud(3000, 15.0)
    m = O.OracleMap(mc, mcov, 0.5)
    for _ in range(10):
        rel = rng.random_pose(0.3, 3.0)
        assert O.overlap_rate(qc, rel, m, threads=2) == O.overlap_rate(qc, rel, m, serial=True)


def test_parallel_linearization_matches_serial():  # test_reference.cpp:71-93
    rng = O.Rng(83)
    tm, tc = rng.gaussian_cloud(4000, 12.0)
    sm, sc = rng.gaussian_cloud(4000, 12.0)
    m = O.OracleMap(tm, tc, 1.0)
    Ti = rng.random_pose(0.1, 1.0)
    Tj = rng.random_pose(0.1, 1.0)
    serial = O.linearize(sm, sc, m, Ti, Tj, serial=True)
    for det in (False, True):
        par = O.linearize(sm, sc, m, Ti, Tj, threads=2, deterministic=det)
        assert par["inliers"] == serial["inliers"]
        scale = max(1.0, np.linalg.norm(serial["H_ii"]))
        for k in ("H_ii", "H_ij", "H_jj", "b_i", "b_j"):
            assert np.linalg.norm(par[k] - serial[k]) / scale < 1e-12
        assert abs(par["error"] - serial["error"]) / max(1.0, serial["error"]) < 1e-12


def test_adjoint_expansion_identity():
    """B = -A·Ad(T_ts) => H_ts = -H_tt·Ad, H_ss = AdᵀH_tt·Ad, b_s = -Adᵀb_t.

    The GPU accumulates only H_tt/b_t (29 scalars) and expands with Ad(T_ts) (se3.cpp:107-113);
    this checks the identity on the oracle's full 92-value accumulation.
    """
    rng = O.Rng(83)
    tm, tc = rng.gaussian_cloud(4000, 12.0)
    sm, sc = rng.gaussian_cloud(4000, 12.0)
    m = O.OracleMap(tm, tc, 1.0)
    Ti = rng.random_pose(0.1, 1.0)
    Tj = rng.random_pose(0.1, 1.0)
    lin = O.linearize(sm, sc, m, Ti, Tj)
    Ad = O.adjoint(O.compose(O.inverse(Ti), Tj))
    scale = max(1.0, np.linalg.norm(lin["H_ii"]))
    assert np.linalg.norm(-lin["H_ii"] @ Ad - lin["H_ij"]) / scale < 1e-12
    assert np.linalg.norm(Ad.T @ lin["H_ii"] @ Ad - lin["H_jj"]) / scale < 1e-12
    assert np.linalg.norm(-Ad.T @ lin["b_i"] - lin["b_j"]) / scale < 1e-12
