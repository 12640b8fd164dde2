"""Float64 source clouds: the reference's global graph uses submap clouds —
transform_cloud + voxel_downsample output, float64 and not float32-exact (pipeline.cpp:100-111) — as
factor sources (:141) and overlap probes (:139). Such clouds keep their float64 means on the device;
keys, correspondences, overlap hits, inlier counts and map statistics must equal the oracle fed the
SAME float64 values, bit for bit, including points within 1e-9 m of voxel faces where a float32
rounding of the cloud would flip the voxel. H / b / error keep the float32-algebra tolerance.
"""
import numpy as np
import pytest

import oracle_ctypes as O
from helpers import lin_dict, rel_block_error

V = pytest.importorskip("paper_2109_07073_b200")

pytestmark = pytest.mark.gpu

H_TOL = 1e-5
ERR_TOL = 1e-5
EPS = np.array([1e-12, -1e-12, 1e-9, -1e-9, 3e-8, -3e-8, 1e-7, -1e-7, 1e-6, -1e-6])


@pytest.fixture(scope="module")
def ctx():
    return V.default_context(0)


def checkerboard_map(ctx, res, base=(64, -40, 0)):
    """Voxels with (x + y + z) even in a block at ~60-100 m (fp32 ulp 7.6e-6 m there): any floor
    error flips the occupancy of a point."""
    g = np.arange(0, 24)
    cx, cy, cz = np.meshgrid(g + base[0], g + base[1], np.arange(0, 6) + base[2], indexing="ij")
    even = ((cx + cy + cz) % 2) == 0
    centres = (np.stack([cx[even], cy[even], cz[even]], 1) + 0.5) * res
    m = np.asarray(centres, np.float32).astype(np.float64)
    c9 = O.unit_covariances(len(m))
    return V.GaussianVoxelMap(V.PointCloud(m, O.cov9(c9)[:, [0, 1, 2, 4, 5, 8]].astype(np.float32), ctx), res), \
        O.OracleMap(m, c9, res)


def near_face_points(rng, n, res, base=(64, -40, 0)):
    """float64 points (in the map frame) at EPS-sized offsets from voxel faces on 1-3 axes."""
    k = np.stack([rng.integers(0, 24, n) + base[0], rng.integers(0, 24, n) + base[1],
                  rng.integers(0, 6, n) + base[2]], 1).astype(np.float64)
    frac = rng.uniform(0.05, 0.95, size=(n, 3))
    on = rng.integers(0, 2, size=(n, 3)).astype(bool)
    on[:, 0] |= ~on.any(1)
    frac[on] = rng.choice(EPS, size=on.sum())
    return (k + frac) * res


def plane_covs64(rng, n):
    """float64 plane-like covariances with tiny asymmetries (as R·C·Rᵀ produces)."""
    out = np.empty((n, 3, 3))
    for i in range(n):
        a = rng.normal(size=3)
        Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        out[i] = Q @ np.diag([1e-3, 1.0, 1.0]) @ Q.T
        out[i, 0, 1] += 1e-17 * a[0]
    return out


def test_f64_upload_kept_and_f32_exact_inputs_unchanged(ctx):
    rng = np.random.default_rng(1)
    p = rng.normal(size=(500, 3)) * 30
    assert V.PointCloud(p, None, ctx).is_f64()
    assert not V.PointCloud(p.astype(np.float32).astype(np.float64), None, ctx).is_f64()
    assert not V.PointCloud(p.astype(np.float32), None, ctx).is_f64()
    c = plane_covs64(rng, 500)
    assert V.PointCloud(p.astype(np.float32).astype(np.float64), c, ctx).is_f64()  # inexact covariances


@pytest.mark.parametrize("res", [1.0, 0.5])
def test_f64_overlap_near_faces_exact(ctx, res):
    """Overlap hits of float64 probes equal the oracle's on the same float64 values, through the
    occupancy kernel (batch), the map-set sweep and the hash-probe kernel; a float32 rounding of
    the same cloud would have given different counts (the test has teeth)."""
    gmap, omap = checkerboard_map(ctx, res)
    rng = np.random.default_rng(int(res * 10))
    clouds, rels, p64s = [], [], []
    differs = 0
    for trial in range(4):
        q = near_face_points(rng, 6000, res)
        if trial == 0:
            T = O.IDENTITY.copy()
            p = q
        else:  # a rotated / translated probe: p = Rᵀ(q - t), evaluated in float64
            T = np.asarray(O.Rng(100 + trial).random_pose(0.05, 0.5))
            R, t = T[:9].reshape(3, 3), T[9:]
            p = (q - t) @ R
        c = V.PointCloud(p, None, ctx)
        assert c.is_f64()
        clouds.append(c)
        rels.append(T)
        p64s.append(p)
        p32 = p.astype(np.float32).astype(np.float64)
        differs += O.overlap_hits(p32, T, omap) != O.overlap_hits(p, T, omap)
    assert differs > 0
    hits = V.overlap_hits(clouds, rels, [gmap] * len(rels))
    for T, p, h in zip(rels, p64s, hits):
        ref = O.overlap_hits(p, T, omap)
        assert int(h) == ref and 0 < ref < len(p)
    ms = V.MapSet([gmap, gmap])
    for T, c, p in zip(rels, clouds, p64s):
        got = V.overlap_hits(c, [T, T], ms)
        assert list(map(int, got)) == [O.overlap_hits(p, T, omap)] * 2


def test_f64_overlap_hash_path_exact(ctx, monkeypatch):
    """The hash-probe overlap kernels (maps without occupancy bitmaps / the per-item kernel) read the
    float64 means too."""
    monkeypatch.setenv("VGICP_OVERLAP_PERITEM", "1")
    gmap, omap = checkerboard_map(ctx, 1.0)
    rng = np.random.default_rng(5)
    p = near_face_points(rng, 5000, 1.0)
    c = V.PointCloud(p, None, ctx)
    assert int(V.overlap_hits([c], [O.IDENTITY], [gmap])[0]) == O.overlap_hits(p, O.IDENTITY, omap)
    monkeypatch.delenv("VGICP_OVERLAP_PERITEM")
    monkeypatch.setenv("VGICP_NO_OCCUPANCY", "1")
    gmap2 = V.GaussianVoxelMap(V.PointCloud(omap_points(omap), np.tile([1.0, 0, 0, 1, 0, 1], (omap.size(), 1)), ctx), 1.0)
    assert int(V.overlap_hits([c], [O.IDENTITY], [gmap2])[0]) == O.overlap_hits(p, O.IDENTITY, omap)


def omap_points(omap):
    _, _, m, _ = omap.export()
    return m


@pytest.mark.parametrize("res", [1.0, 0.5])
def test_f64_map_build_near_faces_bit_exact(ctx, res):
    """GaussianVoxelMap over a float64 device cloud accumulates its exact float64 means and all 9
    covariance entries: export (keys, counts, means, covariances) equals the oracle bit for bit."""
    rng = np.random.default_rng(7)
    p = near_face_points(rng, 20000, res)
    c = plane_covs64(rng, len(p))
    cloud = V.PointCloud(p, c, ctx)
    assert cloud.is_f64()
    gk, gcnt, gm, gc = V.GaussianVoxelMap(cloud, res).export()
    ok_, ocnt, om, oc = O.OracleMap(p, c.reshape(-1, 9), res).export()
    assert np.array_equal(gk, ok_) and np.array_equal(gcnt, ocnt)
    assert np.array_equal(gm, om) and np.array_equal(gc, oc)
    # batched build mixing float32 and float64 clouds
    p32 = p.astype(np.float32).astype(np.float64)
    c32 = V.PointCloud(p32, c.reshape(-1, 9)[:, [0, 1, 2, 4, 5, 8]].astype(np.float32), ctx)
    m64, m32 = V.GaussianVoxelMap.build_batch([cloud, c32], [res, res])
    assert np.array_equal(m64.export()[0], ok_)
    c6 = c.reshape(-1, 9)[:, [0, 1, 2, 4, 5, 8]].astype(np.float32).astype(np.float64)
    assert np.array_equal(m32.export()[0], O.OracleMap(p32, O.cov9(c6), res).export()[0])


@pytest.mark.parametrize("res", [1.0, 0.5])
def test_f64_factor_near_faces(ctx, res):
    """linearize / evaluate with a float64 source cloud whose points sit within 1e-12..1e-6 m of voxel
    faces: inliers equal the oracle's on the same float64 cloud; blocks within H_TOL."""
    rng = np.random.default_rng(11)
    # target map: checkerboard with plane covariances
    g = np.arange(0, 24)
    cx, cy, cz = np.meshgrid(g + 64, g - 40, np.arange(0, 6), indexing="ij")
    even = ((cx + cy + cz) % 2) == 0
    tm = np.asarray((np.stack([cx[even], cy[even], cz[even]], 1) + 0.5) * res, np.float32).astype(np.float64)
    tm = np.repeat(tm, 3, 0) + np.asarray(rng.uniform(-0.3, 0.3, size=(3 * len(tm), 3)) * res, np.float32)
    orng = O.Rng(3)
    tc6 = np.stack([orng.plane_covariance() for _ in range(len(tm))]).reshape(-1, 9)[:, [0, 1, 2, 4, 5, 8]]
    tc6 = tc6.astype(np.float32)
    tgt = V.PointCloud(tm, tc6, ctx)
    gmap = V.GaussianVoxelMap(tgt, res)
    omap = O.OracleMap(tm, O.cov9(tc6.astype(np.float64)), res)
    sp = near_face_points(rng, 12000, res)
    sc = plane_covs64(rng, len(sp))
    src = V.PointCloud(sp, sc, ctx)
    assert src.is_f64()
    fac = V.MatchingCostFactor(0, 1, src, gmap)
    differs = 0
    for trial in range(3):
        Ti = O.IDENTITY.copy() if trial == 0 else np.asarray(O.Rng(200 + trial).random_pose(0.02, 0.2))
        Tj = O.IDENTITY.copy() if trial == 0 else np.asarray(O.Rng(300 + trial).random_pose(0.02, 0.2))
        lin = V.linearize_matching_cost(fac, Ti, Tj)
        err, inl = V.evaluate_matching_cost(fac, Ti, Tj)
        ref = O.linearize(sp, sc.reshape(-1, 9), omap, Ti, Tj)
        ref_err, ref_inl = O.evaluate(sp, sc.reshape(-1, 9), omap, Ti, Tj)
        assert lin.inliers == ref["inliers"] == inl == ref_inl and ref_inl > 0
        e = rel_block_error(lin_dict(lin), ref)
        assert max(e[k] for k in ("H_ii", "H_ij", "H_jj", "b_i", "b_j")) <= H_TOL, e
        assert e["error"] <= ERR_TOL and abs(err - ref_err) <= ERR_TOL * max(1.0, ref_err)
        sp32 = sp.astype(np.float32).astype(np.float64)
        differs += O.evaluate(sp32, sc.reshape(-1, 9), omap, Ti, Tj)[1] != ref_inl
    assert differs > 0


def test_f64_mixed_graph(ctx):
    """A graph mixing float32 and float64 source clouds (two launches per pass): every factor equals
    its single-factor evaluation bit for bit, and inliers equal the oracle's."""
    rng = O.Rng(41)
    factors, oracle = [], []
    maps = []
    for k in range(4):
        m, c = rng.gaussian_cloud(3000, 10.0)
        m32 = np.asarray(m, np.float32).astype(np.float64)
        c6 = V.cov6_from(c)
        maps.append((V.GaussianVoxelMap(V.PointCloud(m32, c6, ctx), 1.0), O.OracleMap(m32, O.cov9(c6.astype(np.float64)), 1.0)))
    for k in range(6):
        m, c = rng.gaussian_cloud(2500 + 300 * k, 10.0)
        if k % 2:
            m = np.asarray(m, np.float32).astype(np.float64)
            c = O.cov9(V.cov6_from(c).astype(np.float64))
        src = V.PointCloud(m, c, ctx)
        assert src.is_f64() == (k % 2 == 0)
        t = k % 4
        factors.append(V.MatchingCostFactor(t, 4 + k % 2, src, maps[t][0]))
        oracle.append((m, np.asarray(c).reshape(-1, 9), maps[t][1], t, 4 + k % 2))
    poses = [np.asarray(rng.random_pose(0.05, 0.3)) for _ in range(6)]
    graph = V.FactorGraph(factors, 6)
    raw, inl = graph.linearize_raw(poses)
    errs, einl = graph.evaluate(poses)
    for f, (fac, (m, c, om, i, j)) in enumerate(zip(factors, oracle)):
        single = V.linearize_matching_cost(fac, poses[i], poses[j])
        ref = O.linearize(m, c, om, poses[i], poses[j])
        assert inl[f] == single.inliers == ref["inliers"] == einl[f]
        assert raw[f][120] == single.error
        e = rel_block_error(lin_dict(single), ref)
        assert max(e.values()) <= H_TOL, e
