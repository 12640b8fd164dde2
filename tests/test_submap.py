"""Submap creation path: transform_cloud (point_cloud.cpp:26-42),
voxel_downsample (voxelmap.cpp:137-169) and the submap's voxel map (pipeline.cpp:92-114).

CPU tests pin the oracle restatement to the reference's own cases (test_point_cloud.cpp:136-173,
test_voxelmap.cpp:190-204); GPU tests require bit-exact agreement with the oracle: the fp64
transform uses the reference's op order, and the fp64 voxel statistics (all 9 covariance sums,
Kahan) are bit-identical, so downsampled clouds and submap maps match exactly.
"""
import numpy as np
import pytest

import oracle_ctypes as O

IDENT = np.array([1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0, 0, 0, 0])


def random_points(rng: O.Rng, n: int, scale: float) -> np.ndarray:
    return np.stack([rng.vector(scale) for _ in range(n)])


def plane_covs(rng: O.Rng, n: int) -> np.ndarray:
    return np.stack([rng.plane_covariance() for _ in range(n)])


def pose_rz(theta, t=(0.0, 0.0, 0.0)):
    c, s = np.cos(theta), np.sin(theta)
    return np.array([c, -s, 0, s, c, 0, 0, 0, 1.0, *t])


# ------------------------------------------------------------------------------ oracle (CPU)
def test_oracle_transform_identity_translation_rotation():  # test_point_cloud.cpp:136-160
    rng = O.Rng(7)
    m = random_points(rng, 50, 3.0)
    c = O.estimate_covariances(m, 8)
    sm, sc = O.transform_cloud(m, c, IDENT)
    assert np.array_equal(sm, m) and np.array_equal(sc, c)
    tm, tc = O.transform_cloud(m, c, np.array([1.0, 0, 0, 0, 1, 0, 0, 0, 1, 1, 2, 3]))
    assert np.array_equal(tc, c)
    np.testing.assert_allclose(tm - m, np.tile([1.0, 2.0, 3.0], (50, 1)), atol=1e-12)
    _, rc = O.transform_cloud(np.zeros((1, 3)), np.diag([2.0, 5.0, 9.0])[None], pose_rz(np.pi / 2))
    assert np.abs(rc[0] - np.diag([5.0, 2.0, 9.0])).max() < 1e-12


def test_oracle_transform_roundtrip():  # test_point_cloud.cpp:162-173
    rng = O.Rng(8)
    m = random_points(rng, 100, 10.0)
    c = O.estimate_covariances(m, 8)
    T = rng.random_pose(1.0, 5.0)
    tm, tc = O.transform_cloud(m, c, T)
    bm, bc = O.transform_cloud(tm, tc, O.inverse(T))
    assert np.abs(bm - m).max() < 1e-9 and np.abs(bc - c).max() < 1e-9


def test_oracle_voxel_downsample_one_point_per_voxel():  # test_voxelmap.cpp:190-204
    rng = O.Rng(16)
    m = random_points(rng, 4000, 8.0)
    c = O.unit_covariances(4000)
    dm, dc = O.voxel_downsample(m, c, 1.0)
    assert len(dm) == O.OracleMap(m, c, 1.0).size()
    dm2, _ = O.voxel_downsample(m, c, 1.0)
    assert np.array_equal(dm, dm2)
    keys = [O.voxel_key(1.0, p) for p in dm]  # the voxel mean lies in its voxel -> ascending keys
    assert keys == sorted(keys)


# ------------------------------------------------------------------------------ GPU parity
gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    return pytest.importorskip("paper_2109_07073_b200")


def assert_export_equal(gmap, omap):
    gk, gc, gm, gv = gmap.export()
    ok, oc, om, ov = omap.export()
    assert np.array_equal(gk, ok) and np.array_equal(gc, oc)
    assert np.array_equal(gm, om), np.abs(gm - om).max()
    assert np.array_equal(gv, ov), np.abs(gv - ov).max()


@gpu
def test_gpu_transform_bit_exact(V):
    rng = O.Rng(21)
    m = random_points(rng, 5000, 60.0)
    c = plane_covs(rng, 5000)
    for _ in range(4):
        T = rng.random_pose(1.0, 30.0)
        gm, gc = V.transform_cloud(m, c, T)
        om, oc = O.transform_cloud(m, c, T)
        assert np.array_equal(gm, om) and np.array_equal(gc, oc)
    gm, gc = V.transform_cloud(m, None, T)
    assert gc is None and np.array_equal(gm, O.transform_cloud(m, None, T)[0])


@gpu
@pytest.mark.parametrize("res", [0.5, 1.0, 2.0])
def test_gpu_build_f64_bit_exact(V, res):
    """fp64 cloud with full, slightly asymmetric (transformed) covariances."""
    rng = O.Rng(22)
    m = random_points(rng, 8000, 15.0)
    c = plane_covs(rng, 8000)
    T = rng.random_pose(0.7, 5.0)
    tm, tc = O.transform_cloud(m, c, T)
    assert not np.array_equal(tc, tc.transpose(0, 2, 1))  # R·C·Rᵀ is not exactly symmetric
    assert_export_equal(V.GaussianVoxelMap.from_arrays(tm, tc, res), O.OracleMap(tm, tc, res))


@gpu
def test_gpu_voxel_downsample_matches_oracle(V):
    rng = O.Rng(16)
    m = random_points(rng, 4000, 8.0)
    c = O.unit_covariances(4000)
    gm, gc = V.voxel_downsample(m, c, 1.0)
    om, oc = O.voxel_downsample(m, c, 1.0)
    assert np.array_equal(gm, om) and np.array_equal(gc, oc)


@gpu
def test_gpu_build_f64_validation(V):
    m = np.zeros((4, 3))
    c = np.tile(np.eye(3), (4, 1, 1))
    with pytest.raises(ValueError):
        V.GaussianVoxelMap.from_arrays(m, c, 0.0)
    with pytest.raises(ValueError):
        V.GaussianVoxelMap.from_arrays(m, None, 1.0)
    with pytest.raises(IndexError):
        V.GaussianVoxelMap.from_arrays(np.array([[2.0e6, 0, 0]]), np.eye(3)[None], 1.0)


def submap_case(V, nframes=5, n=3000, seed=30):
    rng = O.Rng(seed)
    frames64, poses = [], []
    for k in range(nframes):
        m = random_points(rng, n, 20.0).astype(np.float32).astype(np.float64)
        c = plane_covs(rng, n).astype(np.float32).astype(np.float64)
        frames64.append((m, c))
        poses.append(rng.random_pose(0.3, 4.0))
    clouds = [V.PointCloud(m, c) for m, c in frames64]
    return frames64, poses, clouds


@gpu
@pytest.mark.parametrize("ds_res", [0.25, 0.5, 0.0])
def test_gpu_submap_build_bit_exact(V, ds_res):
    frames64, poses, clouds = submap_case(V)
    sub = V.build_submap(clouds, poses, ds_res, 1.0)
    om, oc, omap = O.submap(frames64, poses, ds_res, 1.0)
    assert_export_equal(sub.voxels, omap)
    if ds_res > 0:
        gk, gcnt, gm, gc = sub.downsampled.export()
        assert np.array_equal(gm, om) and np.array_equal(gc, oc)
    else:
        assert sub.downsampled is None
    assert sub.cloud.size() == len(om) and sub.cloud.has_covariances()
    assert sub.voxels.total_points() == len(om)


@gpu
def test_gpu_submap_cloud_as_factor_source(V):
    """The submap cloud is a float64 device cloud (its means are transform_cloud + voxel_downsample
    output, not float32-exact: pipeline.cpp:100-111) and a factor source / overlap probe exactly as
    the reference uses it (:139, :141): inliers and overlap hits equal the oracle fed the float64
    submap cloud `om` itself, blocks within the float32-algebra tolerance."""
    from helpers import lin_dict, rel_block_error

    frames64, poses, clouds = submap_case(V, nframes=3, n=4000, seed=31)
    sub_a = V.build_submap(clouds, poses, 0.25, 1.0)
    sub_b = V.build_submap(clouds[1:], poses[1:], 0.25, 1.0)
    om, oc, _ = O.submap(frames64[1:], poses[1:], 0.25, 1.0)
    oc9 = np.asarray(oc).reshape(-1, 9)
    assert sub_b.cloud.is_f64() and sub_b.cloud.size() == len(om)
    assert not np.array_equal(om, om.astype(np.float32).astype(np.float64))
    _, _, omap_a = O.submap(frames64, poses, 0.25, 1.0)
    fac = V.MatchingCostFactor(0, 1, sub_b.cloud, sub_a.voxels)
    rng = O.Rng(77)
    for Ta, Tb in [(IDENT, O.IDENTITY), (rng.random_pose(0.01, 0.1), rng.random_pose(0.01, 0.1))]:
        lin = V.linearize_matching_cost(fac, Ta, Tb)
        err, inl = V.evaluate_matching_cost(fac, Ta, Tb)
        ref = O.linearize(om, oc9, omap_a, Ta, Tb)
        assert lin.inliers == ref["inliers"] == inl and lin.inliers > 0
        e = rel_block_error(lin_dict(lin), ref)
        assert max(e.values()) <= 1e-5, e
        rel = O.compose(O.inverse(Ta), Tb)
        assert int(V.overlap_hits([sub_b.cloud], [rel], [sub_a.voxels])[0]) == O.overlap_hits(om, rel, omap_a)
    # a map built from the submap cloud equals the reference's GaussianVoxelMap(submap cloud)
    gk, gcnt, gm, gc = V.GaussianVoxelMap(sub_b.cloud, 0.5).export()
    ok_, ocnt, omm, occ = O.OracleMap(om, oc9, 0.5).export()
    assert np.array_equal(gk, ok_) and np.array_equal(gcnt, ocnt) and np.array_equal(gm, omm) and np.array_equal(gc, occ)
    # the submap cloud as a frame of another submap transforms its exact float64 values
    sub_c = V.build_submap([sub_b.cloud], [poses[0]], 0.0, 1.0)
    _, _, omap_c = O.submap([(om, oc9)], [poses[0]], 0.0, 1.0)
    assert_export_equal(sub_c.voxels, omap_c)


@gpu
def test_gpu_submap_validation(V):
    frames64, poses, clouds = submap_case(V, nframes=2, n=100)
    with pytest.raises(ValueError):
        V.build_submap([], [], 0.5, 1.0)
    with pytest.raises(ValueError):
        V.build_submap(clouds, poses, 0.5, 0.0)
    raw = V.PointCloud(frames64[0][0])
    with pytest.raises(ValueError):
        V.build_submap([raw], poses[:1], 0.5, 1.0)


@gpu
def test_gpu_submap_nonfinite_pose_is_out_of_range(V):
    """A non-finite frame pose makes NaN submap points; voxel_downsample / the map build then raise
    out_of_range (voxelmap.cpp:45-55) in the oracle and on the GPU alike (with and without downsampling);
    the context stays usable."""
    frames64, poses, clouds = submap_case(V, nframes=2, n=200)
    bad = np.array(poses, dtype=np.float64)
    bad[1, 9] = np.nan
    with pytest.raises(O.OracleOutOfRange):
        O.submap(frames64, bad, 0.5, 1.0)
    for ds in (0.5, 0.0):
        with pytest.raises(IndexError):
            V.build_submap(clouds, bad, ds, 1.0)
    assert V.build_submap(clouds, poses, 0.5, 1.0) is not None
