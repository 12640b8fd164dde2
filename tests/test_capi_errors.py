"""Error behaviour of the C ABI entry points (include/vgicp_b200.h) on a GPU: every call returns a
status instead of throwing, with the reference's exception classes mapped to
VGICP_E_INVALID_ARGUMENT (std::invalid_argument) and VGICP_E_OUT_OF_RANGE (std::out_of_range)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

V = pytest.importorskip("paper_2109_07073_b200")
from paper_2109_07073_b200 import _lib  # noqa: E402

OK, INVALID, OUT_OF_RANGE = 0, 1, 2


@pytest.fixture(scope="module")
def env():
    ctx = V.default_context(0)
    rng = np.random.default_rng(5)
    m = rng.uniform(-5, 5, (500, 3)).astype(np.float32)
    c = np.tile(np.array([1, 0, 0, 1, 0, 1e-3], np.float32), (500, 1))
    cloud = V.PointCloud(m, c, ctx)
    vmap = V.GaussianVoxelMap(cloud, 1.0)
    return ctx, cloud, vmap, m


def ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def test_null_arguments_are_invalid(env):
    ctx, cloud, vmap, m = env
    lib = _lib.load()
    out = C.c_void_p()
    assert lib.vgicp_voxelmap_build(None, cloud.handle, 1.0, C.byref(out)) == INVALID
    assert lib.vgicp_voxelmap_build(ctx.handle, cloud.handle, 1.0, None) == INVALID
    assert lib.vgicp_transform_cloud(ctx.handle, None, None, 5, None, None, None) == INVALID
    assert lib.vgicp_submap_build(ctx.handle, None, None, 1, 0.5, 1.0, None, None, C.byref(out)) == INVALID
    assert lib.vgicp_graph_assembly_plan(None, None, None, None, None) == INVALID
    assert lib.vgicp_estimate_covariances(ctx.handle, None, 100, 10, 1e-3, None) == INVALID
    assert lib.vgicp_last_error()  # a message is always set


def test_status_mapping_of_reference_exceptions(env):
    ctx, cloud, vmap, m = env
    lib = _lib.load()
    out = C.c_void_p()
    # resolution <= 0 -> invalid_argument (voxelmap.cpp:67-69)
    assert lib.vgicp_voxelmap_build(ctx.handle, cloud.handle, 0.0, C.byref(out)) == INVALID
    # beyond ±2^20 voxels -> out_of_range (voxelmap.cpp:49-51), no map returned
    far = np.array([[2.0e6, 0, 0]], np.float64)
    cov = np.eye(3)[None].copy()
    assert lib.vgicp_voxelmap_build_f64(ctx.handle, ptr(far), ptr(cov), 1, 1.0, C.byref(out)) == OUT_OF_RANGE
    assert not out.value
    # too few points for k -> invalid_argument (point_cloud.cpp:47-53)
    few = np.zeros((5, 3), np.float32)
    cov6 = np.zeros((5, 6), np.float32)
    assert lib.vgicp_estimate_covariances(ctx.handle, ptr(few), 5, 10, 1e-3, ptr(cov6)) == INVALID
    # k > 32 is outside the GPU kernel's range
    pts = np.random.default_rng(0).uniform(size=(100, 3)).astype(np.float32)
    cov6 = np.zeros((100, 6), np.float32)
    assert lib.vgicp_estimate_covariances(ctx.handle, ptr(pts), 100, 33, 1e-3, ptr(cov6)) == INVALID


def test_assembly_requires_plan_and_matching_mask(env):
    ctx, cloud, vmap, m = env
    g = V.FactorGraph([V.MatchingCostFactor(0, 1, cloud, vmap)], 2)
    lib = _lib.load()
    poses = np.tile(np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0.0]), (2, 1))
    d = np.zeros(36)
    assert lib.vgicp_graph_linearize_assembled(g.handle, ptr(poses), ptr(d), ptr(d), ptr(d)) == INVALID
    fixed = np.array([1, 1], np.uint8)  # everything fixed: no slots, no pairs
    plan = g.assembly_plan(fixed)
    assert plan.num_slots == 0 and len(plan.pairs) == 0
    diag, off, rhs = g.linearize_assembled(poses)
    assert diag.shape == (0, 6, 6) and off.shape == (0, 6, 6) and rhs.shape == (0, 6)


def test_single_frame_submap_without_downsampling(env):
    ctx, cloud, vmap, m = env
    ident = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0.0])
    sub = V.build_submap([cloud], [ident], 0.0, 1.0)
    # identity transform of float data: the submap map equals the frame's own map
    gk, gc, gm, gv = sub.voxels.export()
    rk, rc, rm, rv = vmap.export()
    assert np.array_equal(gk, rk) and np.array_equal(gc, rc)
    assert np.array_equal(gm, rm) and np.array_equal(gv, rv)
    assert sub.downsampled is None and sub.cloud.size() == len(m)
