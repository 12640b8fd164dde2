"""The reference's analytic factor properties (test_factors.cpp:164-222), checked on the GPU's blocks:
the gradient -2b against central finite differences of the frozen matching cost (voxel association
and Omega held at the linearization point; oracles.hpp:131-148 / test_factors.cpp:71-89), and the
Gauss-Newton quadratic model error - 2 b^T d + d^T H d against that cost along a random direction.

The frozen cost is evaluated by the oracle in fp64 (test infrastructure); the scene is the
reference's make_scene (points kept 1e-3 voxels clear of faces). Float32 clouds round the scene to
the GPU input contract first (the oracle sees the same rounded values); float64 clouds upload the
scene's doubles as they are.

The gradient bound is 1e-4, not the reference's 1e-5: the per-hit algebra is float32 and the
scene's plane covariances (eigenvalues 1, 1, 1e-3) give κ(M) ≈ 1e3, so Ω e carries ~κ·2^-24
relative error per hit; measured 4e-7 to 2.6e-5 over the five scenes in both modes (the oracle's
own fp64 blocks meet 1e-5, test_oracle_kats.py). The quadratic-model test holds as written.
"""
import numpy as np
import pytest

import oracle_ctypes as O
from helpers import contract_inputs

V = pytest.importorskip("paper_2109_07073_b200")

pytestmark = pytest.mark.gpu


def fd_gradient(poses, cost, h=1e-6):  # oracles.hpp:131-148 (central differences on the right perturbation)
    grad = np.zeros(6 * len(poses))
    for v in range(len(poses)):
        for d in range(6):
            delta = np.zeros(6)
            delta[d] = h
            plus, minus = list(poses), list(poses)
            plus[v] = O.compose(poses[v], O.se3_exp(delta))
            delta[d] = -h
            minus[v] = O.compose(poses[v], O.se3_exp(delta))
            grad[6 * v + d] = (cost(plus) - cost(minus)) / (2.0 * h)
    return grad


def scene_on_gpu(ctx, s, f64):
    if f64:
        sm, sc9 = s["source_means"], s["source_covs"].reshape(-1, 9)
        tm, tc9 = s["target_means"], s["target_covs"].reshape(-1, 9)
        src = V.PointCloud(sm, s["source_covs"], ctx)
        tgt = V.PointCloud(tm, s["target_covs"], ctx)
        assert src.is_f64() and tgt.is_f64()
    else:
        sm, sc9, sc6 = contract_inputs(s["source_means"], s["source_covs"])
        tm, tc9, tc6 = contract_inputs(s["target_means"], s["target_covs"])
        src = V.PointCloud(sm, sc6, ctx)
        tgt = V.PointCloud(tm, tc6, ctx)
    gmap = V.GaussianVoxelMap(tgt, 1.0)
    omap = O.OracleMap(tm, tc9, 1.0)
    return V.MatchingCostFactor(0, 1, src, gmap), sm, sc9, omap


@pytest.mark.parametrize("f64", [False, True])
def test_gpu_gradient_matches_finite_differences(f64):  # test_factors.cpp:164-181
    ctx = V.default_context(0)
    rng = O.Rng(33)
    for _ in range(5):
        s = rng.make_scene(200, 1.0)
        fac, sm, sc9, omap = scene_on_gpu(ctx, s, f64)
        lin = V.linearize_matching_cost(fac, s["T_target"], s["T_source"])
        assert lin.inliers > 150
        fd = fd_gradient([s["T_target"], s["T_source"]],
                         lambda p: O.frozen_cost(sm, sc9, omap, s["T_target"], s["T_source"], p[0], p[1]))
        analytic = np.concatenate([-2.0 * lin.b_i, -2.0 * lin.b_j])
        rel = np.linalg.norm(analytic - fd) / np.linalg.norm(fd)
        assert rel < 1e-4


@pytest.mark.parametrize("f64", [False, True])
def test_gpu_quadratic_model(f64):  # test_factors.cpp:183-222
    """|actual - model| / s^2 stays bounded as s -> 0 and |actual - model| / s vanishes linearly. The
    model's constant term is the fp64 frozen cost at the linearization point (the GPU's own error
    differs from it by the float32 algebra, ~1e-7 relative, which would swamp the s = 1e-4 term);
    its gradient and curvature are the GPU's b and H."""
    ctx = V.default_context(0)
    rng = O.Rng(34)
    s = rng.make_scene(300, 1.0)
    fac, sm, sc9, omap = scene_on_gpu(ctx, s, f64)
    lin = V.linearize_matching_cost(fac, s["T_target"], s["T_source"])
    e0 = O.frozen_cost(sm, sc9, omap, s["T_target"], s["T_source"], s["T_target"], s["T_source"])
    assert abs(lin.error - e0) <= 1e-5 * e0
    H = np.block([[lin.H_ii, lin.H_ij], [lin.H_ij.T, lin.H_jj]])
    b = np.concatenate([lin.b_i, lin.b_j])
    dir_rng = O.Rng(35)
    direction = np.array([dir_rng.uniform(-1.0, 1.0) for _ in range(12)])
    direction /= np.linalg.norm(direction)
    diffs, scales = [], [1e-2, 1e-3, 1e-4]
    for sc in scales:
        delta = sc * direction
        Ti = O.retract(s["T_target"], delta[:6])
        Tj = O.retract(s["T_source"], delta[6:])
        actual = O.frozen_cost(sm, sc9, omap, s["T_target"], s["T_source"], Ti, Tj)
        model = e0 - 2.0 * b @ delta + delta @ H @ delta
        diffs.append(abs(actual - model))
    k0 = diffs[0] / scales[0] ** 2
    for i in range(1, 3):
        assert diffs[i] / scales[i] ** 2 < 8.0 * k0 + 1e-6, diffs
    assert diffs[2] / scales[2] < 0.05 * (diffs[0] / scales[0]) + 1e-12, diffs
