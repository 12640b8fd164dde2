"""GPU (sm_100a) parity against the CPU oracle, through the C ABI (paper_2109_07073_b200.vgicp).

Bar:
  - voxel keys, per-voxel counts, lookups, overlap hit counts, per-factor inlier counts: bit-exact;
  - voxel statistics (fp64 Kahan build): bit-exact;
  - H_ii, H_ij, H_jj, b_i, b_j: ‖Δ‖_F / max(1, ‖H_ii,ref‖_F) <= H_TOL (float32 per-point math vs
    the reference's double; normalisation of test_reference.cpp:85-91);
  - error: relative <= ERR_TOL (plane-regularised covariances, point_cloud.cpp:78); DEGENERATE_TOL
    for near-singular combined covariances, where fp32 Omega loses ~cond(M)·eps.
Inputs follow the GPU contract (float32 means and covariances); the oracle receives the same values.
"""
import numpy as np
import pytest

import oracle_ctypes as O
from helpers import contract_inputs, lin_dict, rel_block_error

V = pytest.importorskip("paper_2109_07073_b200")

pytestmark = pytest.mark.gpu

H_TOL = 1e-5
ERR_TOL = 1e-5
# near-singular combined covariances (zero or rank-deficient inputs): fp32 Omega loses ~cond(M)·eps
DEGENERATE_TOL = 1e-4
MISS = np.iinfo(np.uint64).max


@pytest.fixture(scope="module")
def ctx():
    return V.default_context(0)


def gpu_cloud(ctx, means, covs=None):
    m, c9, c6 = contract_inputs(means, covs)
    return V.PointCloud(m, c6, ctx), m, c9


def assert_map_parity(gmap: "V.GaussianVoxelMap", omap: O.OracleMap):
    gk, gc, gm, gv = gmap.export()
    ok, oc, om, ov = omap.export()
    assert gmap.size() == omap.size()
    assert np.array_equal(gk, ok)
    assert np.array_equal(gc, oc)
    assert np.array_equal(gm, om), np.max(np.abs(gm - om))
    assert np.array_equal(gv, ov), np.max(np.abs(gv - ov))


# ------------------------------------------------------------------------------ voxel map
def test_single_point_voxel(ctx):  # test_voxelmap.cpp:23-34
    cloud, m, c9 = gpu_cloud(ctx, [[0.2, 0.3, 0.4]], np.diag([1.0, 1.0, 1e-3])[None])
    g = V.GaussianVoxelMap(cloud, 1.0)
    assert g.size() == 1 and g.total_points() == 1
    keys, counts, means, covs = g.export()
    assert counts[0] == 1 and np.array_equal(means[0], m[0])
    assert np.linalg.norm(covs[0] - c9[0].reshape(3, 3)) < 1e-15
    assert g.lookup(m)[0] == keys[0]


def test_two_point_voxel(ctx):  # test_voxelmap.cpp:36-48
    cloud, m, c9 = gpu_cloud(ctx, [[0.1, 0.1, 0.1], [0.3, 0.1, 0.1]], O.unit_covariances(2))
    g = V.GaussianVoxelMap(cloud, 1.0)
    assert_map_parity(g, O.OracleMap(m, c9, 1.0))
    _, counts, means, covs = g.export()
    assert counts[0] == 2
    assert np.linalg.norm(means[0] - m.mean(axis=0)) < 1e-9


@pytest.mark.parametrize("seed,n,scale,res", [(10, 1000, 10.0, 1.0), (11, 5000, 20.0, 0.7), (13, 2000, 10.0, 0.5), (81, 5000, 20.0, 0.8)])
def test_voxelmap_bit_exact(ctx, seed, n, scale, res):  # test_voxelmap.cpp:50-136, test_reference.cpp:43-57
    rng = O.Rng(seed)
    means, covs = rng.gaussian_cloud(n, scale)
    cloud, m, c9 = gpu_cloud(ctx, means, covs)
    g = V.GaussianVoxelMap(cloud, res)
    omap = O.OracleMap(m, c9, res, threads=4, deterministic=True)
    assert_map_parity(g, omap)
    assert g.total_points() == n
    _, counts, _, _ = g.export()
    assert counts.sum() == n
    # brute-force bucketing (oracles.hpp:45-61)
    assert g.size() == len(O.brute_force_buckets(m, res))


def test_voxelmap_order_independence(ctx):  # test_voxelmap.cpp:95-120
    rng = O.Rng(12)
    pts = np.array([rng.vector(15.0) for _ in range(3000)])
    perm = rng.shuffle(3000).astype(np.int64)
    a, _, _ = gpu_cloud(ctx, pts, O.unit_covariances(3000))
    b, _, _ = gpu_cloud(ctx, pts[perm], O.unit_covariances(3000))
    ka, ca, ma, va = V.GaussianVoxelMap(a, 1.0).export()
    kb, cb, mb, vb = V.GaussianVoxelMap(b, 1.0).export()
    assert np.array_equal(ka, kb) and np.array_equal(ca, cb)
    assert np.max(np.abs(ma - mb)) < 1e-9 and np.max(np.abs(va - vb)) < 1e-9


def test_voxelmap_batch_equals_single(ctx):
    rng = O.Rng(90)
    clouds, singles = [], []
    for k in range(5):
        means, covs = rng.gaussian_cloud(500 + 300 * k, 10.0)
        c, m, c9 = gpu_cloud(ctx, means, covs)
        clouds.append(c)
    res = [0.5, 1.0, 2.0, 0.7, 1.3]
    batch = V.GaussianVoxelMap.build_batch(clouds, res)
    for c, r, b in zip(clouds, res, batch):
        s = V.GaussianVoxelMap(c, r)
        for x, y in zip(s.export(), b.export()):
            assert np.array_equal(x, y)


def test_floor_boundary_lookup(ctx):  # test_voxelmap.cpp:71-82
    cloud, _, _ = gpu_cloud(ctx, [[0.5, 0.5, 0.5]], O.unit_covariances(1))
    g = V.GaussianVoxelMap(cloud, 1.0)
    got = g.lookup([[0.9, 0.9, 0.9], [5.0, 5.0, 5.0], [1.0, 0.5, 0.5], [0.0, 0.0, 0.0], [1.0 - 1e-12, 0.5, 0.5], [np.nan, 0, 0], [3e6, 0, 0]])
    assert got[0] != MISS and got[1] == MISS and got[2] == MISS and got[3] != MISS and got[4] != MISS
    assert got[5] == MISS and got[6] == MISS


@pytest.mark.parametrize("res", [0.3, 0.25, 1.0])
def test_lookup_matches_oracle_near_faces(ctx, res):
    """Points and probes within a few ulps of voxel faces (and exactly on them): the exact-floor
    fast path and its IEEE-division fallback must agree with floor(p / r) bit for bit."""
    rng = np.random.default_rng(5)
    base = rng.integers(-50, 50, size=(2000, 3)).astype(np.float64) * res
    b32 = base.astype(np.float32)
    ulp32 = np.spacing(np.abs(b32) + np.float32(res)).astype(np.float32)
    pts = (b32 + rng.integers(-3, 4, size=(2000, 3)).astype(np.float32) * ulp32).astype(np.float64)
    pts = np.concatenate([pts, b32.astype(np.float64)])
    cloud, m, c9 = gpu_cloud(ctx, pts, O.unit_covariances(len(pts)))
    g = V.GaussianVoxelMap(cloud, res)
    omap = O.OracleMap(m, c9, res)
    assert_map_parity(g, omap)
    eps = rng.integers(-4, 5, size=base.shape) * np.spacing(np.abs(base) + res)
    probes = np.concatenate([pts, base, base + eps, base + res * 0.5, -base + eps])
    assert np.array_equal(g.lookup(probes), omap.lookup(probes))


def test_single_point_lookup_and_voxel_coord(ctx):  # voxelmap.cpp:45-55, 106-117
    rng = O.Rng(92)
    means, covs = rng.gaussian_cloud(2000, 6.0)
    c, m, c9 = gpu_cloud(ctx, means, covs)
    g = V.GaussianVoxelMap(c, 0.5)
    om = O.OracleMap(m, c9, 0.5)
    ok, ocnt, omean, ocov = om.export()
    index = {int(k): i for i, k in enumerate(ok)}
    for p in list(m[:50]) + [rng.vector(10.0) for _ in range(50)] + [np.array([1e7, 0.0, 0.0])]:
        v = g.lookup_voxel(p)
        key = int(O.OracleMap.lookup(om, p[None])[0])
        if key == int(MISS):
            assert v is None
        else:
            i = index[key]
            assert np.array_equal(v[0], omean[i]) and np.array_equal(v[1], ocov[i]) and v[2] == ocnt[i]
        if abs(p[0]) < 1e5:
            assert g.voxel_coord(p) == tuple(int(np.floor(x / 0.5)) for x in p)


def test_range_and_invalid(ctx):  # test_voxelmap.cpp:185-188, voxelmap.cpp:67-72
    cloud, _, _ = gpu_cloud(ctx, [[2.0e6, 0, 0]], O.unit_covariances(1))
    with pytest.raises(IndexError):
        V.GaussianVoxelMap(cloud, 1.0)
    ok, _, _ = gpu_cloud(ctx, [[0.0, 0, 0]], O.unit_covariances(1))
    with pytest.raises(ValueError):
        V.GaussianVoxelMap(ok, 0.0)
    with pytest.raises(ValueError):
        V.GaussianVoxelMap(ok, -1.0)
    # NaN passes the reference's `resolution <= 0` check and fails voxel_coord's range test
    with pytest.raises(O.OracleOutOfRange):
        O.OracleMap([[0.0, 0, 0]], O.unit_covariances(1), float("nan"))
    with pytest.raises(IndexError):
        V.GaussianVoxelMap(ok, float("nan"))
    with pytest.raises(IndexError):
        V.GaussianVoxelMap.build_batch([ok, ok], [1.0, float("nan")])
    with pytest.raises(ValueError):  # documented deviation: +inf (every point in voxel 0) is rejected
        V.GaussianVoxelMap(ok, float("inf"))
    raw = V.PointCloud(np.zeros((3, 3), np.float32), None, ctx)
    with pytest.raises(ValueError):
        V.GaussianVoxelMap(raw, 1.0)
    empty = V.PointCloud(np.zeros((0, 3), np.float32), None, ctx)
    g = V.GaussianVoxelMap(ok, 1.0)
    with pytest.raises(ValueError):
        V.overlap_rate(empty, O.IDENTITY, g)
    # an empty cloud has no covariances (point_cloud.hpp:28): no map (voxelmap.cpp:69-71), no factor
    # source (factors.cpp:58-63)
    empty_cov = V.PointCloud(np.zeros((0, 3), np.float32), np.zeros((0, 6), np.float32), ctx)
    with pytest.raises(ValueError):
        V.GaussianVoxelMap(empty_cov, 1.0)
    with pytest.raises(ValueError):
        V.MatchingCostFactor(0, 1, empty_cov, g)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_map_points_are_out_of_range(ctx, monkeypatch, bad):
    """A NaN / Inf point in a map's cloud fails the reference's range test (voxelmap.cpp:45-55:
    !(c >= -2^20 && c < 2^20) holds for NaN) -> out_of_range, no map — for the hand-written build,
    the sort-based build, a batch (the whole batch fails, as the oracle fails on that cloud), and
    float64 clouds."""
    rng = np.random.default_rng(5)
    pts = rng.uniform(-5, 5, size=(500, 3))
    pts[137, 1] = bad
    cov = O.unit_covariances(len(pts))
    with pytest.raises(O.OracleOutOfRange):
        O.OracleMap(np.asarray(pts, np.float32).astype(np.float64), cov, 1.0)
    cloud, _, _ = gpu_cloud(ctx, pts, cov)
    good, _, _ = gpu_cloud(ctx, rng.uniform(-5, 5, size=(300, 3)), O.unit_covariances(300))
    with pytest.raises(IndexError):
        V.GaussianVoxelMap(cloud, 1.0)
    with pytest.raises(IndexError):
        V.GaussianVoxelMap.build_batch([good, cloud], [1.0, 0.5])
    monkeypatch.setenv("VGICP_SORTED_BUILD", "1")
    with pytest.raises(IndexError):
        V.GaussianVoxelMap(cloud, 1.0)
    monkeypatch.delenv("VGICP_SORTED_BUILD")
    p64 = pts + 1e-9
    c64 = V.PointCloud(p64, cov.reshape(-1, 3, 3), ctx)
    assert c64.is_f64()
    with pytest.raises(IndexError):
        V.GaussianVoxelMap(c64, 1.0)
    assert V.GaussianVoxelMap(good, 1.0).size() > 0  # the context stays usable


# ------------------------------------------------------------------------------ overlap
def test_overlap_self_and_far(ctx):  # test_voxelmap.cpp:138-149
    rng = O.Rng(14)
    pts = np.array([rng.vector(10.0) for _ in range(2000)])
    cloud, _, _ = gpu_cloud(ctx, pts, O.unit_covariances(2000))
    g = V.GaussianVoxelMap(cloud, 0.5)
    assert V.overlap_rate(cloud, O.IDENTITY, g) == 1.0
    assert V.overlap_rate(cloud, O.pose(t=(500, 0, 0)), g) == 0.0


def test_overlap_20_scenes_exact(ctx):  # test_voxelmap.cpp:151-169
    from test_oracle_kats import reference_overlap_scenes

    for map_pts, cloud_pts, res, rel in reference_overlap_scenes():
        mc, mm, mc9 = gpu_cloud(ctx, map_pts, O.unit_covariances(len(map_pts)))
        qc, qm, _ = gpu_cloud(ctx, cloud_pts)
        g = V.GaussianVoxelMap(mc, res)
        got = V.overlap_rate(qc, rel, g)
        expected = O.brute_force_overlap_count(qm, rel, mm, res)
        assert got == expected / len(qm)
        assert got == O.overlap_rate(qm, rel, O.OracleMap(mm, mc9, res))


def test_overlap_37_of_100(ctx):  # test_voxelmap.cpp:171-183
    map_pts = [[x + 0.5, y + 0.5, 0.5] for x in range(5) for y in range(5)]
    cloud = [[0.5 + 0.1 * (i % 5), 0.5 + (i // 5 % 5), 0.5] for i in range(37)] + [[100.0 + i, 0.0, 0.0] for i in range(63)]
    mc, _, _ = gpu_cloud(ctx, map_pts, O.unit_covariances(25))
    qc, _, _ = gpu_cloud(ctx, cloud)
    assert V.overlap_hits(qc, [O.IDENTITY], [V.GaussianVoxelMap(mc, 1.0)])[0] == 37


def test_overlap_culling_is_exact(ctx):
    """Probes whose transformed cloud box misses the map's occupied region are culled on the host
    (hits exactly 0); near, far and grazing probes all match the oracle."""
    rng = O.Rng(91)
    means, covs = rng.gaussian_cloud(3000, 10.0)
    c, m, c9 = gpu_cloud(ctx, means, covs)
    g = V.GaussianVoxelMap(c, 1.0)
    omap = O.OracleMap(m, c9, 1.0)
    rels = [rng.random_pose(0.3, 3.0) for _ in range(20)]
    for shift in (25.0, 29.0, 31.0, 35.0, 60.0, 1e4):  # around and beyond the map's extent
        T = rng.random_pose(0.2, 0.0)
        T[9] = shift
        rels.append(T)
    hits = V.overlap_hits([c] * len(rels), rels, [g] * len(rels))
    for T, h in zip(rels, hits):
        assert h == O.overlap_hits(m, T, omap)
    assert hits[-1] == 0


def test_overlap_batch_matches_serial(ctx):  # test_reference.cpp:59-69
    rng = O.Rng(82)
    mcl, mcov = rng.gaussian_cloud(3000, 15.0)
    qcl, _ = rng.gaussian_cloud(3000, 15.0)
    mc, mm, mc9 = gpu_cloud(ctx, mcl, mcov)
    qc, qm, _ = gpu_cloud(ctx, qcl)
    g = V.GaussianVoxelMap(mc, 0.5)
    omap = O.OracleMap(mm, mc9, 0.5)
    rels = [rng.random_pose(0.3, 3.0) for _ in range(10)]
    rates = V.overlap_rates(qc, rels, [g] * 10)
    for rel, r in zip(rels, rates):
        assert r == O.overlap_rate(qm, rel, omap, serial=True)
    assert np.array_equal(V.overlap_rates(qc, rels, V.MapSet([g] * 10)), rates)  # device map set


@pytest.mark.parametrize("res", [0.25, 1.0, 2.0])
def test_overlap_occupancy_bitmap_equals_hash_probe(ctx, monkeypatch, res):
    """Overlap through the maps' occupancy bitmaps (default) vs through the cuckoo-hash probes
    (maps built with VGICP_NO_OCCUPANCY=1) vs the oracle: identical hit counts, including points
    on brick / box faces, outside the occupied box and beyond the ±2^20 key range."""
    rng = O.Rng(93)
    means, covs = rng.gaussian_cloud(5000, 12.0)
    means[:50] = np.round(means[:50] / res) * res  # exactly on voxel faces
    c, m, c9 = gpu_cloud(ctx, means, covs)
    g_occ = V.GaussianVoxelMap(c, res)
    monkeypatch.setenv("VGICP_NO_OCCUPANCY", "1")
    g_hash = V.GaussianVoxelMap(c, res)
    monkeypatch.delenv("VGICP_NO_OCCUPANCY")
    q, qm, _ = gpu_cloud(ctx, np.concatenate([rng.gaussian_cloud(3000, 14.0)[0], [[1e7, 0.0, 0.0], [-3e6, 1.0, 2.0]]]))
    omap = O.OracleMap(m, c9, res)
    rels = [rng.random_pose(0.3, 2.0) for _ in range(12)] + [O.IDENTITY]
    h_occ = V.overlap_hits([q] * len(rels), rels, [g_occ] * len(rels))
    h_hash = V.overlap_hits([q] * len(rels), rels, [g_hash] * len(rels))
    assert list(h_occ) == list(h_hash)
    for T, h in zip(rels, h_occ):
        assert h == O.overlap_hits(qm, T, omap)


@pytest.mark.parametrize("res,shift", [(1.0, 0.0), (0.25, 1500.0), (2.0, -8000.0), (0.1, 300.0)])
def test_overlap_fp32_screen_near_faces(ctx, res, shift):
    """The occupancy kernel's fp32 screen must reproduce the reference's fp64 floor exactly: query
    points are placed so that their transformed positions sit at 0, 1e-9 .. 1e-3 voxel from voxel
    faces (large translations included), against a checkerboard map where any floor error flips
    the occupancy of the point. Counts must equal the oracle's for every pose."""
    rng = np.random.default_rng(int(res * 100) + int(abs(shift)))
    # checkerboard map: voxel centres with (x + y + z) even, around the origin
    g = np.arange(-12, 12)
    cx, cy, cz = np.meshgrid(g, g, np.arange(-3, 3), indexing="ij")
    even = ((cx + cy + cz) % 2) == 0
    centres = (np.stack([cx[even], cy[even], cz[even]], 1) + 0.5) * res
    map_pts = np.asarray(centres, np.float32).astype(np.float64)
    mc, mm, mc9 = gpu_cloud(ctx, map_pts, O.unit_covariances(len(map_pts)))
    gmap = V.GaussianVoxelMap(mc, res)
    omap = O.OracleMap(mm, mc9, res)
    eps = np.array([0.0, 1e-9, -1e-9, 1e-7, -1e-7, 1e-6, -1e-6, 1e-5, -1e-5, 1e-4, -1e-4, 1e-3, -1e-3])
    rels, clouds, qms = [], [], []
    for trial in range(6):
        ang = rng.normal(size=3) * 0.4
        th = np.linalg.norm(ang)
        K = np.array([[0, -ang[2], ang[1]], [ang[2], 0, -ang[0]], [-ang[1], ang[0], 0]]) / max(th, 1e-12)
        R = np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K
        t = rng.normal(size=3) * 5.0 + np.array([shift, -0.5 * shift, 0.0])
        T = np.concatenate([R.ravel(), t])
        # targets in the map frame: near faces on one, two or three axes
        k = rng.integers(-11, 11, size=(4000, 3)).astype(np.float64)
        k[:, 2] = rng.integers(-3, 3, size=4000)
        frac = rng.uniform(0.05, 0.95, size=(4000, 3))
        on = rng.integers(0, 2, size=(4000, 3)).astype(bool)
        frac[on] = rng.choice(eps, size=on.sum())
        q = (k + frac) * res
        p = (q - t) @ R  # R^T (q - t)
        qm = np.asarray(p, np.float32).astype(np.float64)
        c, qmm, _ = gpu_cloud(ctx, qm)
        rels.append(T)
        clouds.append(c)
        qms.append(qmm)
    hits = V.overlap_hits(clouds, rels, [gmap] * len(rels))
    for T, qm, h in zip(rels, qms, hits):
        ref = O.overlap_hits(qm, T, omap)
        assert h == ref, (h, ref)
        assert 0 < ref < len(qm)


def test_overlap_mapset_sweep_matches_batch(ctx, monkeypatch):
    """vgicp_overlap_mapset (items built and culled on the device) equals vgicp_overlap_batch and the
    oracle: near, far (culled), grazing poses, maps of three resolutions, a map set without bitmaps."""
    rng = O.Rng(95)
    maps, omaps = [], []
    for k, res in enumerate([0.5, 1.0, 2.0, 1.0, 0.5]):
        means, covs = rng.gaussian_cloud(2500, 10.0 + 3 * k)
        c, m, c9 = gpu_cloud(ctx, means, covs)
        maps.append(V.GaussianVoxelMap(c, res))
        omaps.append(O.OracleMap(m, c9, res))
    q, qm, _ = gpu_cloud(ctx, rng.gaussian_cloud(4000, 12.0)[0])
    rels = []
    for k in range(len(maps)):
        T = rng.random_pose(0.3, 2.0)
        if k == 2:
            T[9] = 1e4  # far: culled on the device
        rels.append(T)
    rels_all = rels * 8  # 40 probes: two chunks of 32
    maps_all = maps * 8
    ms = V.MapSet(maps_all)
    h_set = V.overlap_hits(q, rels_all, ms)
    h_batch = V.overlap_hits(q, rels_all, maps_all)
    assert list(h_set) == list(h_batch)
    for T, om, h in zip(rels_all, omaps * 8, h_set):
        assert h == O.overlap_hits(qm, T, om)
    assert h_set[2] == 0
    monkeypatch.setenv("VGICP_NO_OCCUPANCY", "1")  # maps without bitmaps: the generic path
    g_hash = V.GaussianVoxelMap(gpu_cloud(ctx, *rng.gaussian_cloud(2000, 9.0))[0], 1.0)
    monkeypatch.delenv("VGICP_NO_OCCUPANCY")
    mixed = V.MapSet([g_hash] + maps)
    hm = V.overlap_hits(q, [rels[0]] + rels, mixed)
    assert list(hm[1:]) == list(h_batch[:5])


# ------------------------------------------------------------------------------ factors
def factor_case(ctx, sm, sc, tm, tc, res):
    src, smm, sc9 = gpu_cloud(ctx, sm, sc)
    tgt, tmm, tc9 = gpu_cloud(ctx, tm, tc)
    g = V.GaussianVoxelMap(tgt, res)
    omap = O.OracleMap(tmm, tc9, res)
    return V.MatchingCostFactor(0, 1, src, g), smm, sc9, omap


def check_factor(fac, smm, sc9, omap, Tt, Ts, h_tol=H_TOL, e_tol=ERR_TOL):
    lin = V.linearize_matching_cost(fac, Tt, Ts)
    ref = O.linearize(smm, sc9, omap, Tt, Ts)
    assert lin.inliers == ref["inliers"]
    errs = rel_block_error(lin_dict(lin), ref)
    for k, v in errs.items():
        assert v <= (e_tol if k == "error" else h_tol), (k, v, errs)
    err, inl = V.evaluate_matching_cost(fac, Tt, Ts)
    ref_err, ref_inl = O.evaluate(smm, sc9, omap, Tt, Ts)
    assert inl == ref_inl
    assert err == lin.error  # same per-point arithmetic and reduction order in both kernels
    assert abs(err - ref_err) <= e_tol * max(1.0, abs(ref_err))
    assert np.array_equal(lin.H_ii, lin.H_ii.T) and np.array_equal(lin.H_jj, lin.H_jj.T)
    return lin, ref, errs


def test_linearize_reference_scene_83(ctx):  # test_reference.cpp:71-93
    rng = O.Rng(83)
    tm, tc = rng.gaussian_cloud(4000, 12.0)
    sm, sc = rng.gaussian_cloud(4000, 12.0)
    fac, smm, sc9, omap = factor_case(ctx, sm, sc, tm, tc, 1.0)
    Ti = rng.random_pose(0.1, 1.0)
    Tj = rng.random_pose(0.1, 1.0)
    check_factor(fac, smm, sc9, omap, Ti, Tj)


@pytest.mark.parametrize("seed,points", [(33, 200), (34, 300), (37, 400), (38, 3000)])
def test_linearize_make_scene(ctx, seed, points):  # test_factors.cpp:33-68 scenes
    rng = O.Rng(seed)
    s = rng.make_scene(points, 1.0)
    fac, smm, sc9, omap = factor_case(ctx, s["source_means"], s["source_covs"], s["target_means"], s["target_covs"], 1.0)
    lin, ref, _ = check_factor(fac, smm, sc9, omap, s["T_target"], s["T_source"])
    assert lin.inliers > 0.75 * points


def test_gauge_invariance(ctx):  # test_factors.cpp:243-253
    rng = O.Rng(37)
    s = rng.make_scene(400, 1.0)
    fac, smm, sc9, omap = factor_case(ctx, s["source_means"], s["source_covs"], s["target_means"], s["target_covs"], 1.0)
    base, _ = V.evaluate_matching_cost(fac, s["T_target"], s["T_source"])
    for _ in range(10):
        G = rng.random_pose(1.0, 50.0)
        e, _ = V.evaluate_matching_cost(fac, O.compose(G, s["T_target"]), O.compose(G, s["T_source"]))
        assert abs(e - base) < 1e-5 * max(1.0, base)


def test_disjoint_zero_factor(ctx):  # test_factors.cpp:224-241
    rng = O.Rng(36)
    sm, sc, tm, tc = [], [], [], []
    for _ in range(50):
        sm.append(rng.vector(2.0))
        sc.append(rng.plane_covariance())
        tm.append(rng.vector(2.0) + [1000, 0, 0])
        tc.append(rng.plane_covariance())
    fac, _, _, _ = factor_case(ctx, sm, sc, tm, tc, 1.0)
    lin = V.linearize_matching_cost(fac, O.IDENTITY, O.IDENTITY)
    assert lin.inliers == 0 and lin.error == 0.0
    assert not np.any(lin.H_ii) and not np.any(lin.H_ij) and not np.any(lin.H_jj)
    assert not np.any(lin.b_i) and not np.any(lin.b_j)


def test_perfect_alignment(ctx):  # test_factors.cpp:122-162
    rng = O.Rng(32)
    means = np.array([[20.0 * (i % 10) + 5.0, 20.0 * (i // 10) + 5.0, 5.0] for i in range(100)])
    covs = np.array([rng.plane_covariance() for _ in range(100)])
    fac, smm, sc9, omap = factor_case(ctx, means, covs, means, covs, 10.0)
    T = rng.random_pose(0.5, 3.0)
    lin = V.linearize_matching_cost(fac, T, T)
    assert lin.inliers == 100
    assert lin.error < 1e-6
    H = np.block([[lin.H_ii, lin.H_ij], [lin.H_ij.T, lin.H_jj]])
    assert np.linalg.eigvalsh(H).min() > -1e-6 * max(1.0, np.abs(H).max())


def test_singular_combined_covariance_skipped(ctx):  # factors.cpp:108-110, :39-41
    """Zero covariances make M singular: the fp64 LDLT path must skip exactly like the oracle."""
    rng = O.Rng(44)
    n = 300
    sm = np.array([rng.vector(3.0) for _ in range(n)])
    tm = sm + 0.01 * np.array([rng.vector(1.0) for _ in range(n)])
    sc = np.zeros((n, 3, 3))
    tc = np.zeros((n, 3, 3))
    sc[: n // 2] = [rng.plane_covariance() for _ in range(n // 2)]  # half the points regular
    tc[::3] = [rng.plane_covariance() for _ in range(len(tc[::3]))]
    fac, smm, sc9, omap = factor_case(ctx, sm, sc, tm, tc, 0.5)
    T = O.IDENTITY
    lin, ref, _ = check_factor(fac, smm, sc9, omap, T, T, h_tol=1e-5, e_tol=DEGENERATE_TOL)
    assert 0 < ref["inliers"] < n


def test_factor_with_nonfinite_and_out_of_range_source_points(ctx):
    """Source points that are NaN / Inf or land beyond ±2^20 voxels miss (lookup returns null,
    voxelmap.cpp:110-112) and are skipped exactly like the oracle — no exception on this path."""
    rng = O.Rng(93)
    tm, tc = rng.gaussian_cloud(2000, 5.0)
    sm, sc = rng.gaussian_cloud(2000, 5.0)
    sm = sm.copy()
    sm[::97] = np.nan
    sm[5::101, 1] = np.inf
    sm[7::103, 0] = 3.0e6  # beyond 2^20 voxels at 1 m
    fac, smm, sc9, omap = factor_case(ctx, sm, sc, tm, tc, 1.0)
    T = O.IDENTITY
    lin = V.linearize_matching_cost(fac, T, T)
    ref = O.linearize(smm, sc9, omap, T, T)
    assert lin.inliers == ref["inliers"] and 0 < lin.inliers < len(sm)
    d = rel_block_error(lin_dict(lin), ref)
    assert max(d.values()) <= H_TOL, d
    err, inl = V.evaluate_matching_cost(fac, T, T)
    assert inl == ref["inliers"]


def test_gicp_error_kat(ctx):  # test_factors.cpp:92-120 (fp64 kernel: bit-exact vs oracle)
    mean = np.array([1.0, 2.0, 3.0])
    half = 0.5 * np.eye(3)
    r = V.gicp_error(mean, half, mean, half, O.IDENTITY)
    assert r.error == 0.0 and r.valid
    r = V.gicp_error(mean, half, mean + [1, 0, 0], half, O.IDENTITY)
    assert r.error == pytest.approx(1.0, rel=1e-12)
    assert np.linalg.norm(r.information - np.eye(3)) < 1e-12
    rng = O.Rng(31)
    for _ in range(20):
        sm, tm = rng.vector(5.0), rng.vector(5.0)
        sc, tc = rng.plane_covariance(), rng.plane_covariance()
        T = rng.random_pose(0.5, 2.0)
        g = V.gicp_error(sm, sc, tm, tc, T)
        e, res, info, valid = O.gicp_error(sm, sc, tm, tc, T)
        assert g.valid == valid and g.error == e
        assert np.array_equal(g.residual, res) and np.array_equal(g.information, info)
    bad = V.gicp_error(mean, np.zeros((3, 3)), mean + 1, np.zeros((3, 3)), O.IDENTITY)
    assert not bad.valid and bad.error == 0.0


def test_factor_validation(ctx):  # factors.cpp:57-66
    rng = O.Rng(50)
    means, covs = rng.gaussian_cloud(100, 5.0)
    c, _, _ = gpu_cloud(ctx, means, covs)
    g = V.GaussianVoxelMap(c, 1.0)
    with pytest.raises(ValueError):
        V.MatchingCostFactor(1, 1, c, g)
    raw = V.PointCloud(np.zeros((5, 3), np.float32), None, ctx)
    with pytest.raises(ValueError):
        V.MatchingCostFactor(0, 1, raw, g)


# ------------------------------------------------------------------------------ batched graph
def build_graph_case(ctx, nframes=6, n=3000, seed=60, res=1.0):
    rng = O.Rng(seed)
    clouds, frames = [], []
    for _ in range(nframes):
        means, covs = rng.gaussian_cloud(n, 10.0)
        c, m, c9 = gpu_cloud(ctx, means, covs)
        clouds.append(c)
        frames.append((m, c9))
    maps = V.GaussianVoxelMap.build_batch(clouds, res)
    omaps = [O.OracleMap(m, c9, res) for m, c9 in frames]
    poses = [rng.random_pose(0.05, 0.5) for _ in range(nframes)]
    factors = []
    for j in range(nframes):
        for d in (1, 2):
            i = j - d
            if i >= 0:
                factors.append(V.MatchingCostFactor(i, j, clouds[j], maps[i]))
    return factors, frames, omaps, poses


def test_graph_batch_matches_oracle(ctx):
    factors, frames, omaps, poses = build_graph_case(ctx)
    graph = V.FactorGraph(factors, len(poses), chunk=1024)
    lins = graph.linearize(poses)
    errs, inls = graph.evaluate(poses)
    for f, lin, e, inl in zip(factors, lins, errs, inls):
        m, c9 = frames[f.source_index]
        ref = O.linearize(m, c9, omaps[f.target_index], poses[f.target_index], poses[f.source_index])
        assert lin.inliers == ref["inliers"] == inl
        assert lin.i == f.target_index and lin.j == f.source_index
        d = rel_block_error(lin_dict(lin), ref)
        assert max(d.values()) <= H_TOL, d
        assert abs(e - ref["error"]) <= ERR_TOL * max(1.0, ref["error"])


def test_graph_deterministic_and_chunk_invariant_counts(ctx):
    factors, _, _, poses = build_graph_case(ctx, nframes=4, n=5000, seed=61)
    g1 = V.FactorGraph(factors, len(poses), chunk=512)
    a, ia = g1.linearize_raw(poses)
    b, ib = g1.linearize_raw(poses)
    assert np.array_equal(a, b) and np.array_equal(ia, ib)  # bitwise run-to-run
    g2 = V.FactorGraph(factors, len(poses), chunk=4096)
    c, ic = g2.linearize_raw(poses)
    assert np.array_equal(ia, ic)
    scale = np.maximum(1.0, np.linalg.norm(a[:, :36], axis=1))
    assert np.max(np.linalg.norm(a - c, axis=1) / scale) < 1e-6  # fp32 per-thread order changes with chunking


def test_graph_multiresolution_matches_oracle(ctx):
    """C5 shape: one graph whose factors use 0.5 / 1 / 2 m maps round-robin (one launch)."""
    rng = O.Rng(63)
    res = (0.5, 1.0, 2.0)
    clouds, frames = [], []
    for _ in range(5):
        means, covs = rng.gaussian_cloud(3000, 8.0)
        c, m, c9 = gpu_cloud(ctx, means, covs)
        clouds.append(c)
        frames.append((m, c9))
    maps = {r: V.GaussianVoxelMap.build_batch(clouds, r) for r in res}
    omaps = {r: [O.OracleMap(m, c9, r) for m, c9 in frames] for r in res}
    poses = [rng.random_pose(0.05, 0.5) for _ in range(5)]
    links = [(i, j) for j in range(5) for i in range(j)]
    factors = [V.MatchingCostFactor(i, j, clouds[j], maps[res[k % 3]][i]) for k, (i, j) in enumerate(links)]
    graph = V.FactorGraph(factors, 5)
    for k, ((i, j), lin) in enumerate(zip(links, graph.linearize(poses))):
        m, c9 = frames[j]
        ref = O.linearize(m, c9, omaps[res[k % 3]][i], poses[i], poses[j])
        assert lin.inliers == ref["inliers"]
        d = rel_block_error(lin_dict(lin), ref)
        assert max(d.values()) <= H_TOL, (res[k % 3], d)


def test_graph_preallocated_and_pinned_outputs(ctx):
    """linearize_raw into caller buffers: pageable (staged) and page-locked (direct D2H)."""
    import torch

    factors, _, _, poses = build_graph_case(ctx, nframes=4, n=2000, seed=62)
    g = V.FactorGraph(factors, len(poses))
    a, ia = g.linearize_raw(poses)
    F = len(factors)
    b, ib = np.empty((F, 121)), np.empty(F, np.int32)
    g.linearize_raw(poses, b, ib)
    pc = torch.empty((F, 121), dtype=torch.float64).pin_memory().numpy()
    pi = torch.empty(F, dtype=torch.int32).pin_memory().numpy()
    g.linearize_raw(poses, pc, pi)
    assert np.array_equal(a, b) and np.array_equal(a, pc) and np.array_equal(ia, ib) and np.array_equal(ia, pi)
    with pytest.raises(ValueError):
        g.linearize_raw(poses, np.empty((F, 120)), ib)


def test_graph_validation(ctx):
    factors, _, _, poses = build_graph_case(ctx, nframes=3, n=500, seed=62)
    with pytest.raises(ValueError):
        V.FactorGraph(factors, 2)  # index out of range
    g = V.FactorGraph(factors, 3)
    with pytest.raises(ValueError):
        g.linearize(poses[:2])


# ------------------------------------------------------------------------------ hand-written build
def _sorted_build(monkeypatch, clouds, res):
    monkeypatch.setenv("VGICP_SORTED_BUILD", "1")
    try:
        return V.GaussianVoxelMap.build_batch(clouds, res)
    finally:
        monkeypatch.delenv("VGICP_SORTED_BUILD")


def test_handwritten_build_equals_sorted_build(ctx, monkeypatch):
    """The rank-numbered hand-written build (build.cu: bitmap + stable counting sort + Kahan) and the
    sort-based build give bit-identical exports (keys, counts, fp64 means / covariances) and
    bit-identical factor results, overlap hits and lookups — on a batch of mixed sizes and
    resolutions, dense voxels (hundreds of points), and a map whose voxel count exceeds the
    shared-memory cursor array (global-cursor variant)."""
    rng = O.Rng(401)
    clouds, res = [], []
    for k in range(6):
        means, covs = rng.gaussian_cloud(800 + 700 * k, 4.0 + 6 * k)
        clouds.append(gpu_cloud(ctx, means, covs)[0])
        res.append([0.25, 0.5, 1.0, 2.0, 0.7, 1.3][k])
    dense = np.repeat(np.array([rng.vector(0.4) for _ in range(20)]), 150, axis=0)  # 150 points per voxel
    dense = dense + np.random.default_rng(3).uniform(-0.01, 0.01, dense.shape)
    clouds.append(gpu_cloud(ctx, dense, O.unit_covariances(len(dense)))[0])
    res.append(1.0)
    big = np.random.default_rng(4).uniform(-60, 60, size=(70000, 3))  # V ~ 70k > smem cursors
    clouds.append(gpu_cloud(ctx, big, O.unit_covariances(len(big)))[0])
    res.append(0.5)
    fast = V.GaussianVoxelMap.build_batch(clouds, res)
    slow = _sorted_build(monkeypatch, clouds, res)
    monkeypatch.setenv("VGICP_BUILD_SCATTER", "1")  # warp-serial scatter instead of the shared-memory radix sort
    scatter = V.GaussianVoxelMap.build_batch(clouds, res)
    monkeypatch.delenv("VGICP_BUILD_SCATTER")
    monkeypatch.setenv("VGICP_SORT_5BIT", "1")  # 5-bit digits (3 passes) instead of 4-bit
    four = V.GaussianVoxelMap.build_batch(clouds, res)
    monkeypatch.delenv("VGICP_SORT_5BIT")
    for f, s, w, q in zip(fast, slow, scatter, four):
        assert f.size() == s.size() and f.total_points() == s.total_points()
        for x, y, z, u in zip(f.export(), s.export(), w.export(), q.export()):
            assert np.array_equal(x, y) and np.array_equal(x, z) and np.array_equal(x, u)
    # factors: target maps from each build, same sources / poses -> identical blocks
    poses = np.stack([rng.random_pose(0.05, 0.5) for _ in range(len(clouds))])
    def graph(maps):
        fs = [V.MatchingCostFactor(k, k + 1, clouds[k + 1], maps[k]) for k in range(5)]
        return V.FactorGraph(fs, len(clouds))
    ra, ia = graph(fast).linearize_raw(poses)
    rb, ib = graph(slow).linearize_raw(poses)
    assert np.array_equal(ia, ib) and np.array_equal(ra, rb)
    rels = [O.compose(O.inverse(poses[k]), poses[k + 1]) for k in range(5)]
    assert np.array_equal(V.overlap_hits([clouds[k + 1] for k in range(5)], rels, fast[:5]),
                          V.overlap_hits([clouds[k + 1] for k in range(5)], rels, slow[:5]))
    probes = np.concatenate([big[:3000], big[:3000] + 0.3])
    assert np.array_equal(fast[-1].lookup(probes), slow[-1].lookup(probes))  # on-demand hash table


def test_handwritten_build_hash_mode_equals_rank_mode(ctx, monkeypatch):
    """VGICP_NO_RANK=1 makes the factor kernels probe the on-demand cuckoo table of hand-built maps:
    the same blocks as the rank lookups, bit for bit."""
    rng = O.Rng(402)
    clouds = [gpu_cloud(ctx, *rng.gaussian_cloud(3000, 10.0))[0] for _ in range(3)]
    maps = V.GaussianVoxelMap.build_batch(clouds, [1.0, 1.0, 1.0])
    poses = np.stack([rng.random_pose(0.05, 0.5) for _ in range(3)])
    fs = [V.MatchingCostFactor(0, 1, clouds[1], maps[0]), V.MatchingCostFactor(1, 2, clouds[2], maps[1])]
    ra, ia = V.FactorGraph(fs, 3).linearize_raw(poses)
    monkeypatch.setenv("VGICP_NO_RANK", "1")
    rb, ib = V.FactorGraph(fs, 3).linearize_raw(poses)
    assert np.array_equal(ia, ib) and np.array_equal(ra, rb)


def test_upload_batch_equals_single_uploads(ctx):
    """vgicp_cloud_upload_batch (one staged copy, one segmented sort for all Morton orders) gives the
    same device layout as one vgicp_cloud_upload per cloud: bit-identical factor blocks, overlap hits
    and maps; raw (covariance-free) and empty clouds included."""
    rng = O.Rng(403)
    ms, cs = [], []
    for k in range(5):
        m, c = rng.gaussian_cloud(700 + 900 * k, 8.0)
        m32, _, c6 = contract_inputs(m, c)
        ms.append(m32)
        cs.append(c6)
    raw = rng.gaussian_cloud(500, 8.0)[0].astype(np.float32)
    batch = V.PointCloud.upload_batch(ms + [raw, np.zeros((0, 3), np.float32)], cs + [None, None], ctx)
    single = [V.PointCloud(m, c, ctx) for m, c in zip(ms, cs)]
    assert [len(b) for b in batch] == [len(m) for m in ms] + [500, 0]
    assert not batch[5].has_covariances() and batch[0].has_covariances()
    poses = np.stack([rng.random_pose(0.05, 0.5) for _ in range(5)])
    def run(clouds):
        maps = V.GaussianVoxelMap.build_batch(clouds[:5], [1.0] * 5)
        fs = [V.MatchingCostFactor(k, k + 1, clouds[k + 1], maps[k]) for k in range(4)]
        raw_out, inl = V.FactorGraph(fs, 5).linearize_raw(poses)
        rels = [O.compose(O.inverse(poses[k]), poses[k + 1]) for k in range(4)]
        hits = V.overlap_hits([clouds[k + 1] for k in range(4)], rels, maps[:4])
        return raw_out, inl, hits, [m.export() for m in maps]
    a, b = run(batch), run(single)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    for x, y in zip(a[3], b[3]):
        for u, w in zip(x, y):
            assert np.array_equal(u, w)
    rel = O.compose(O.inverse(poses[0]), poses[1])
    maps = V.GaussianVoxelMap.build_batch(batch[:1], [1.0])
    assert V.overlap_hits([batch[5]], [rel], maps)[0] == V.overlap_hits([V.PointCloud(raw, None, ctx)], [rel], maps)[0]


def test_sprawling_map_in_a_batch_and_graph(ctx):
    """A cloud whose occupied box is too large for an occupancy bitmap (two clusters ~4e5 voxels
    apart) takes the sort-based build inside a batch of hand-built maps; every map still exports the
    oracle's statistics, and a graph over both kinds falls back to hash probes for all its factors
    (rank lookups need every target to carry bricks) with oracle-exact inliers."""
    rng = O.Rng(77)
    clouds, frames = [], []
    for k in range(4):
        means, covs = rng.gaussian_cloud(2500, 8.0)
        means = np.asarray(means)
        if k == 1:  # second cluster far away on every axis
            means[1250:] += np.array([2.0e5, -1.9e5, 1.8e5])
        c, m, c9 = gpu_cloud(ctx, means, covs)
        clouds.append(c)
        frames.append((m, c9))
    maps = V.GaussianVoxelMap.build_batch(clouds, [0.5, 0.5, 1.0, 1.0])
    omaps = [O.OracleMap(m, c9, r) for (m, c9), r in zip(frames, [0.5, 0.5, 1.0, 1.0])]
    for g, o in zip(maps, omaps):
        assert_map_parity(g, o)
    poses = [rng.random_pose(0.03, 0.3) for _ in range(4)]
    factors = [V.MatchingCostFactor(i, j, clouds[j], maps[i]) for i, j in ((0, 1), (1, 2), (1, 3), (2, 3), (0, 3))]
    graph = V.FactorGraph(factors, 4)
    raw, inl = graph.linearize_raw(np.stack(poses))
    for k, f in enumerate(factors):
        m, c9 = frames[f.source_index]
        ref = O.linearize(m, c9, omaps[f.target_index], poses[f.target_index], poses[f.source_index])
        assert int(inl[k]) == ref["inliers"]
        d = rel_block_error(O.unpack121(raw[k]), ref)
        assert max(d.values()) <= H_TOL, d
    rel = O.compose(O.inverse(poses[1]), poses[2])
    assert V.overlap_hits(clouds[2], [rel], [maps[1]])[0] == O.overlap_hits(frames[2][0], rel, omaps[1])


@pytest.mark.parametrize("n,res", [(70000, 1000.0), (30000, 0.5)])
def test_extreme_voxel_occupancy(ctx, n, res):
    """One voxel holding every point (70k points, 1 km voxels: one lane folds them all in input order),
    and 30k identical points: exports equal the oracle's Kahan merge bit for bit; a factor over the
    one-voxel map matches the oracle."""
    rng = np.random.default_rng(11)
    if res > 1.0:
        pts = rng.uniform(1.0, 900.0, size=(n, 3))
    else:
        pts = np.repeat(np.array([[3.3, -7.1, 0.26]]), n, axis=0)
    covs = np.repeat(np.diag([0.3, 0.2, 1e-3])[None], n, axis=0)
    cloud, m, c9 = gpu_cloud(ctx, pts, covs)
    gmap = V.GaussianVoxelMap(cloud, res)
    omap = O.OracleMap(m, c9, res)
    assert gmap.size() == 1
    assert_map_parity(gmap, omap)
    src, sm, sc9 = gpu_cloud(ctx, pts[:5000] + 0.01, covs[:5000])
    fac = V.MatchingCostFactor(0, 1, src, gmap)
    check_factor(fac, sm, sc9, omap, O.IDENTITY, O.IDENTITY)


def test_mapset_append_matches_batch(ctx):
    """A keyframe database grown one map at a time (vgicp_mapset_append, geometric growth of the
    device block) sweeps exactly like vgicp_overlap_batch and like a set created in one call; a map
    without an occupancy bitmap (sprawling box) moves the set to the generic path, still exact."""
    rng = O.Rng(91)
    clouds, frames, maps = [], [], []
    for k in range(40):
        means, covs = rng.gaussian_cloud(800, 6.0)
        c, m, c9 = gpu_cloud(ctx, means, covs)
        clouds.append(c)
        frames.append((m, c9))
    maps = V.GaussianVoxelMap.build_batch(clouds, [0.5 + 0.05 * (k % 7) for k in range(40)])
    probe = clouds[0]
    grown = V.MapSet([], ctx=ctx)
    for k, mp in enumerate(maps):
        grown.append(mp)
        if k in (0, 1, 4, 17, 39):
            rels = [rng.random_pose(0.05, 0.4) for _ in range(k + 1)]
            a = V.overlap_hits(probe, rels, grown)
            b = V.overlap_hits([probe] * (k + 1), rels, maps[:k + 1])
            c = V.overlap_hits(probe, rels, V.MapSet(maps[:k + 1]))
            assert np.array_equal(a, b) and np.array_equal(a, c)
    far = np.asarray(rng.gaussian_cloud(800, 6.0)[0])
    far[400:] += np.array([2.0e5, 1.5e5, -2.5e5])
    fc, fm, fc9 = gpu_cloud(ctx, far, O.unit_covariances(len(far)))
    sprawl = V.GaussianVoxelMap(fc, 0.5)
    grown.append([sprawl])
    rels = [rng.random_pose(0.05, 0.4) for _ in range(41)]
    a = V.overlap_hits(probe, rels, grown)
    assert np.array_equal(a, V.overlap_hits([probe] * 41, rels, maps + [sprawl]))
    assert a[40] == O.overlap_hits(frames[0][0], rels[40], O.OracleMap(fm, fc9, 0.5))


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_nonfinite_pose_gives_zero_factor(ctx, bad):
    """A non-finite pose transforms every point to NaN / Inf: no lookup hits (voxelmap.cpp:110-112), so
    the reference's accumulators stay zero (factors.cpp:97-146) — an all-zero block with 0 inliers,
    not the NaN an Ad(T) expansion of zeros would give; the graph's other factors are unaffected."""
    factors, frames, omaps, poses = build_graph_case(ctx, nframes=4, n=2000, seed=63)
    P = np.stack(poses)
    P[2, 9] = bad
    raw, inl = V.FactorGraph(factors, 4).linearize_raw(P)
    err, inl2 = V.FactorGraph(factors, 4).evaluate(P)
    for k, f in enumerate(factors):
        m, c9 = frames[f.source_index]
        ref = O.linearize(m, c9, omaps[f.target_index], P[f.target_index], P[f.source_index])
        if 2 in (f.target_index, f.source_index):
            assert inl[k] == 0 == ref["inliers"] and inl2[k] == 0
            assert not np.any(raw[k]) and not np.any(ref["raw"]) and err[k] == 0.0
        else:
            assert inl[k] == ref["inliers"] > 0
            assert max(rel_block_error(O.unpack121(raw[k]), ref).values()) <= H_TOL


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_overlap_nonfinite_pose_and_points(ctx, monkeypatch, bad):
    """overlap_rate (voxelmap.cpp:119-135) with a non-finite pose counts no hit; non-finite probe points
    never hit — on the occupancy path (batch and map set) and on the hash-probe path, equal to the
    oracle."""
    rng = O.Rng(95)
    tm, tc = rng.gaussian_cloud(3000, 6.0)
    sm, sc = rng.gaussian_cloud(3000, 6.0)
    sm = np.asarray(sm)
    sm[::37] = bad
    tgt, tmm, tc9 = gpu_cloud(ctx, tm, tc)
    src, smm, _ = gpu_cloud(ctx, sm, sc)
    gmap = V.GaussianVoxelMap(tgt, 0.5)
    omap = O.OracleMap(tmm, tc9, 0.5)
    good = rng.random_pose(0.05, 0.3)
    badpose = np.array(good)
    badpose[4] = bad
    poses = [good, badpose]
    want = [O.overlap_hits(smm, p, omap) for p in poses]
    assert want[1] == 0 and want[0] > 0
    assert list(V.overlap_hits([src, src], poses, [gmap, gmap])) == want
    assert list(V.overlap_hits(src, poses, V.MapSet([gmap, gmap]))) == want
    monkeypatch.setenv("VGICP_OVERLAP_PERITEM", "1")  # the generic per-item kernel
    assert list(V.overlap_hits([src, src], poses, [gmap, gmap])) == want
    monkeypatch.delenv("VGICP_OVERLAP_PERITEM")


def test_signed_zero_subnormal_and_face_coordinates(ctx):
    """Coordinates -0.0, float32 subnormals and exact voxel faces (x = k·r) take the reference's floor
    (voxelmap.cpp:48: floor(x / r)); the same cloud twice in one batch at two resolutions gives two
    independent maps — exports, lookups and overlap hits equal the oracle's."""
    tiny = np.float32(1e-40)  # subnormal in float32, exact in float64
    pts = np.array([[-0.0, 0.0, -0.0], [tiny, -tiny, 0.0], [1.0, -1.0, 2.0], [0.5, 0.25, -0.75],
                    [-0.5, 3.0, -2.0], [2.0, 2.0, 2.0], [-tiny, 1.0, -1.0]], np.float32)
    pts = np.concatenate([pts, np.random.default_rng(8).uniform(-3, 3, size=(200, 3)).astype(np.float32)])
    cloud, m, c9 = gpu_cloud(ctx, pts, O.unit_covariances(len(pts)))
    maps = V.GaussianVoxelMap.build_batch([cloud, cloud], [1.0, 0.25])
    for g, r in zip(maps, [1.0, 0.25]):
        omap = O.OracleMap(m, c9, r)
        assert_map_parity(g, omap)
        probe = np.concatenate([m, -m, m + 0.5 * r])
        assert np.array_equal(g.lookup(probe), omap.lookup(probe))
        rel = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0.25 * r, 0, 0.0])
        assert V.overlap_hits(cloud, [rel], [g])[0] == O.overlap_hits(m, rel, omap)


def test_tile_boundary_source_sizes(ctx):
    """Source clouds of 1 .. 4,097 points around the 32-lane / 64-point tile / 512-point item
    boundaries, together in one graph with one 20k-point factor: inliers exact, blocks within
    tolerance, errors equal to linearize's."""
    rng = O.Rng(97)
    tm, tc = rng.gaussian_cloud(20000, 8.0)
    tgt, tmm, tc9 = gpu_cloud(ctx, tm, tc)
    gmap = V.GaussianVoxelMap(tgt, 1.0)
    omap = O.OracleMap(tmm, tc9, 1.0)
    sizes = [1, 2, 31, 32, 33, 63, 64, 65, 127, 129, 511, 512, 513, 4097, 20000]
    srcs, frames = [], []
    for n in sizes:
        sm, sc = rng.gaussian_cloud(n, 8.0)
        c, m, c9 = gpu_cloud(ctx, sm, sc)
        srcs.append(c)
        frames.append((m, c9))
    factors = [V.MatchingCostFactor(0, k + 1, s, gmap) for k, s in enumerate(srcs)]
    poses = np.stack([O.IDENTITY] + [rng.random_pose(0.01, 0.1) for _ in sizes])
    for chunk in (0, 512):
        g = V.FactorGraph(factors, len(poses), chunk=chunk)
        raw, inl = g.linearize_raw(poses)
        err, inl2 = g.evaluate(poses)
        assert np.array_equal(inl, inl2) and np.array_equal(err, raw[:, 120])
        for k, (m, c9) in enumerate(frames):
            ref = O.linearize(m, c9, omap, poses[0], poses[k + 1])
            assert int(inl[k]) == ref["inliers"], (sizes[k], chunk)
            d = rel_block_error(O.unpack121(raw[k]), ref)
            assert max(d.values()) <= H_TOL, (sizes[k], d)


def test_overlap_probe_sizes(ctx, monkeypatch):
    """Overlap probes of 1 .. 4,097 points (4 points per lane, 32 maps per chunk boundaries) against
    33 maps: exact hits on the batched, map-set and per-item paths."""
    rng = O.Rng(98)
    maps, omaps = [], []
    for k in range(33):
        tm, tc = rng.gaussian_cloud(1500, 5.0)
        c, m, c9 = gpu_cloud(ctx, tm, tc)
        maps.append(V.GaussianVoxelMap(c, 0.5 + 0.1 * (k % 4)))
        omaps.append(O.OracleMap(m, c9, 0.5 + 0.1 * (k % 4)))
    mset = V.MapSet(maps)
    for n in (1, 3, 4, 5, 127, 128, 129, 4097):
        sm, sc = rng.gaussian_cloud(n, 5.0)
        probe, smm, _ = gpu_cloud(ctx, sm, sc)
        rels = [rng.random_pose(0.05, 0.5) for _ in maps]
        want = [O.overlap_hits(smm, r, o) for r, o in zip(rels, omaps)]
        assert list(V.overlap_hits([probe] * len(maps), rels, maps)) == want, n
        assert list(V.overlap_hits(probe, rels, mset)) == want, n
        monkeypatch.setenv("VGICP_OVERLAP_PERITEM", "1")
        assert list(V.overlap_hits([probe] * len(maps), rels, maps)) == want, n
        monkeypatch.delenv("VGICP_OVERLAP_PERITEM")


def test_build_path_thresholds(ctx):
    """Clouds straddling every switch of the hand-written build on this device (B200: 227 KB of
    opt-in shared memory): the shared-memory radix sort's point limit (24,896 / 24,897 points), the
    shared-memory bitmap's brick limit (28,928 / 28,929 bricks: a one-brick-wide box 4·28,928 voxels
    long) and the counting kernel's shared-memory cursor limit (57,855 / 57,856 voxels in a
    60,000-point cloud) — one batch and singly, exports equal to the oracle."""
    import torch

    optin = torch.cuda.get_device_properties(0).shared_memory_per_block_optin
    sort_max = (optin - 32768 - 512) // 8
    bricks = (optin - 1024) // 8
    cursors = (optin - 1024) // 4 - 1
    rng = np.random.default_rng(21)
    clouds = []
    for n in (sort_max, sort_max + 1):
        clouds.append(rng.uniform(-40, 40, size=(n, 3)))
    for w in (bricks, bricks + 1):  # a line of voxels x in [0, 4w), y = z = 0, both ends occupied
        x = np.concatenate([[0.5, 4 * w - 0.5], rng.uniform(0, 4 * w, size=3000)])
        clouds.append(np.stack([x, np.full_like(x, 0.5), np.full_like(x, 0.5)], 1))
    for v in (cursors, cursors + 1):  # v distinct voxel centres, then repeats up to 60,000 points
        cells = rng.permutation(80 * 80 * 80)[:v]
        centres = np.stack([cells % 80, (cells // 80) % 80, cells // 6400], 1) + 0.5
        pts = np.concatenate([centres, centres[rng.integers(0, v, size=60000 - v)] + 0.1])
        clouds.append(pts)
    gclouds, frames = [], []
    for pts in clouds:
        c, m, c9 = gpu_cloud(ctx, pts, O.unit_covariances(len(pts)))
        gclouds.append(c)
        frames.append((m, c9))
    batch = V.GaussianVoxelMap.build_batch(gclouds, 1.0)
    for k, (m, c9) in enumerate(frames):
        omap = O.OracleMap(m, c9, 1.0)
        assert_map_parity(batch[k], omap)
        assert_map_parity(V.GaussianVoxelMap(gclouds[k], 1.0), omap)
    assert batch[4].size() == cursors and batch[5].size() == cursors + 1
