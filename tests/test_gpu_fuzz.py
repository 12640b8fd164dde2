"""Randomised parity sweep (GPU vs oracle) over scene shapes, resolutions, poses and covariance
kinds — including rank-deficient ones where the skip decision is made by the fp64 LDLT path.

Every case: bit-exact voxel map export, exact inlier counts (the skip decisions of near-singular M
included: float64 clouds decide on their float64 covariances) and overlap hits; blocks within the
tolerances below. Odd seeds upload target and source as float64 clouds whose values
are not float32-exact (submap clouds, pipeline.cpp:100-111), fed to the oracle unrounded; every
fourth seed also checks the sort-based build (VGICP_SORTED_BUILD) exports the same map bit for bit.
"""
import os

import numpy as np
import pytest

import oracle_ctypes as O
from helpers import contract_inputs, lin_dict, rel_block_error

V = pytest.importorskip("paper_2109_07073_b200")

pytestmark = pytest.mark.gpu

# The per-hit algebra is float32 (the reference's is double): its error grows with κ(M), M = C_t +
# R C_s Rᵀ, and random scenes reach far larger κ than the fixed parity scenes. Tolerances from the
# measured distribution over 3,000 seeds (tools/fuzz_errors.py, profiles/fuzz_errors_r02.log):
# regular covariances max 1.5e-5 (median 2.8e-7); rank-deficient ones ("line" / "zero", κ up to
# ~1e4 on the float32 path) max 2.5e-4 (median 1.4e-6). float64 clouds show the same distribution.
H_TOL = 2e-5
ERR_TOL = 2e-5
DEGENERATE_TOL = 3e-4


def covariances(rng: np.random.Generator, n: int, kind: str) -> np.ndarray:
    if kind == "plane":
        v = rng.normal(size=(n, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        return np.eye(3)[None] - (1 - 1e-3) * v[:, :, None] * v[:, None, :]
    if kind == "random":
        A = rng.normal(size=(n, 3, 3)) * 0.3
        return A @ A.transpose(0, 2, 1) + 1e-4 * np.eye(3)
    if kind == "line":  # rank 1: the combined covariance is near singular for many pairs
        v = rng.normal(size=(n, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        return 0.05 * v[:, :, None] * v[:, None, :]
    return np.zeros((n, 3, 3))  # "zero": only the target covariance regularises


def random_pose(rng, rot, trans):
    w = rng.normal(size=3) * rot
    th = np.linalg.norm(w)
    K = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    R = np.eye(3) if th == 0 else np.eye(3) + np.sin(th) / th * K + (1 - np.cos(th)) / th**2 * K @ K
    return np.concatenate([R.reshape(9), rng.normal(size=3) * trans])


def run_case(seed, sorted_build_env=None):
    """One random scene: exact parts asserted here; returns (kinds, f64, degenerate, block errors)."""
    rng = np.random.default_rng(1000 + seed)
    ctx = V.default_context(0)
    n = int(rng.integers(300, 4000))
    scale = float(rng.choice([2.0, 10.0, 60.0]))
    res = float(rng.choice([0.25, 0.5, 1.0, 2.0]))
    kind_t, kind_s = rng.choice(["plane", "random", "line", "zero"], size=2)
    if kind_t == "zero" and kind_s == "zero":
        kind_t = "plane"
    tm = rng.normal(size=(n, 3)) * scale
    sm = tm[rng.permutation(n)] + rng.normal(size=(n, 3)) * 0.05 * res
    f64 = seed % 2 == 1
    if f64:  # float64 device clouds: the oracle sees the very same (non-float32-exact) values
        tmf, tcov = tm + 1e-9, covariances(rng, n, kind_t)
        smf, scov = sm + 1e-9, covariances(rng, n, kind_s)
        tc9, sc9 = tcov.reshape(-1, 9), scov.reshape(-1, 9)
        tgt = V.PointCloud(tmf, tcov, ctx)
        src = V.PointCloud(smf, scov, ctx)
        assert tgt.is_f64() and src.is_f64()
    else:
        tmf, tc9, tc6 = contract_inputs(tm, covariances(rng, n, kind_t))
        smf, sc9, sc6 = contract_inputs(sm, covariances(rng, n, kind_s))
        tgt = V.PointCloud(tmf, tc6, ctx)
        src = V.PointCloud(smf, sc6, ctx)
    gmap = V.GaussianVoxelMap(tgt, res)
    omap = O.OracleMap(tmf, tc9, res)
    gk, gc, gm, gv = gmap.export()
    ok, oc, om, ov = omap.export()
    assert np.array_equal(gk, ok) and np.array_equal(gc, oc)
    assert np.array_equal(gm, om) and np.array_equal(gv, ov)
    if sorted_build_env is not None and seed % 4 == 0:
        sorted_build_env.setenv("VGICP_SORTED_BUILD", "1")
        sorted_map = V.GaussianVoxelMap(tgt, res)
        sorted_build_env.delenv("VGICP_SORTED_BUILD")
        for x, y in zip(sorted_map.export(), (gk, gc, gm, gv)):
            assert np.array_equal(x, y)

    Tt = random_pose(rng, 0.2, 1.0)
    Ts = O.compose(Tt, random_pose(rng, 0.02, 0.1 * res))
    fac = V.MatchingCostFactor(0, 1, src, gmap)
    lin = V.linearize_matching_cost(fac, Tt, Ts)
    ref = O.linearize(smf, sc9, omap, Tt, Ts)
    assert lin.inliers == ref["inliers"], (kind_t, kind_s, res)
    rel = O.compose(O.inverse(Tt), Ts)
    assert V.overlap_hits(src, [rel], [gmap])[0] == O.overlap_hits(smf, rel, omap)
    degenerate = "line" in (kind_t, kind_s) or "zero" in (kind_t, kind_s)
    return (str(kind_t), str(kind_s), res, scale), f64, degenerate, rel_block_error(lin_dict(lin), ref)


@pytest.mark.parametrize("seed", range(int(os.environ.get("VGICP_FUZZ_SEEDS", "24"))))
def test_random_scene_parity(seed, monkeypatch):
    kinds, f64, degenerate, d = run_case(seed, monkeypatch)
    assert max(v for k, v in d.items() if k != "error") <= (DEGENERATE_TOL if degenerate else H_TOL), (kinds, f64, d)
    assert d["error"] <= (DEGENERATE_TOL if degenerate else ERR_TOL), (kinds, f64, d)
