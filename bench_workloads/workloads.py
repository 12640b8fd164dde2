"""Measured configurations of BASELINE.json, built on the product path.

  C1 single factor: two ~20k-point line scans, 1 m voxels
  C2 odometry chain: 100-frame circle, factors (k-d -> k) for d = 1..3 (294 factors)
  C3 KITTI-00-shaped dense graph: 450-frame figure-eight, every frame linked to its (up to) 10
     highest-overlap predecessors with overlap > 0.025 (pipeline.cpp:135-141 rule), ~4,500 factors
  C4 overlap sweep: one new frame against many keyframe maps
  C5 multi-resolution loop-closing graph: 1,000-frame figure-eight, up to 10 links per frame by
     the overlap rule, factors assigned round-robin to 0.5 / 1 / 2 m maps (3 maps per frame),
     ~10,000 factors
Factor direction follows the reference: target = older frame (owns the map), source = newer frame
(pipeline.cpp:46-48, 141). Factor selection runs the GPU overlap query (the keyframe / factor
creation path, voxelmap.cpp:119-135).
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import synthetic as S

# The product package is imported lazily (only by the builders that upload to a device), so the
# reference bench arm — scans, host covariances, link selection on the oracle — never loads it.


def pose_inv(T):
    T = np.asarray(T, np.float64)
    R = T[:9].reshape(3, 3)
    Rt = R.T
    return np.concatenate([Rt.reshape(9), -(Rt @ T[9:])])


def relative_poses(poses, pairs) -> np.ndarray:
    """T_i⁻¹·T_j for every (i, j) pair, vectorised (12-double poses)."""
    P = np.asarray(poses, np.float64)
    I = np.fromiter((p[0] for p in pairs), dtype=np.int64, count=len(pairs))
    J = np.fromiter((p[1] for p in pairs), dtype=np.int64, count=len(pairs))
    Rs = P[:, :9].reshape(-1, 3, 3)
    R = np.einsum("kba,kbc->kac", Rs[I], Rs[J])  # R_iᵀ R_j
    t = np.einsum("kba,kb->ka", Rs[I], P[J, 9:] - P[I, 9:])  # R_iᵀ (t_j - t_i)
    return np.ascontiguousarray(np.concatenate([R.reshape(-1, 9), t], axis=1))


def pose_mul(A, B):
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    Ra, Rb = A[:9].reshape(3, 3), B[:9].reshape(3, 3)
    return np.concatenate([(Ra @ Rb).reshape(9), Ra @ B[9:] + A[9:]])


@dataclass
class Scans:
    means: list  # float32 n×3
    cov6: list  # float32 n×6
    gt: np.ndarray
    odom: np.ndarray


def make_scans(spec: S.SceneSpec, frames_needed=None, threads: int = 0, ctx=None) -> Scans:
    """Generate the scans and their plane-regularised covariances (k=10, eps=1e-3, as
    run_pipeline.cpp:131). With a context the covariances come from the batched GPU kernel
    (estimate_covariances_batch), otherwise from the host preprocessing (synthetic.cpp)."""
    seq = S.generate(spec)
    idx = list(range(len(seq.scans)) if frames_needed is None else frames_needed)
    covs = [None] * len(seq.scans)
    if ctx is not None:
        from paper_2109_07073_b200.vgicp import estimate_covariances_batch

        for k, c in zip(idx, estimate_covariances_batch([seq.scans[k] for k in idx], 10, 1e-3, ctx)):
            covs[k] = c
    else:
        for k in idx:
            covs[k] = S.estimate_covariances(seq.scans[k], 10, 1e-3, threads)
    return Scans(seq.scans, covs, seq.ground_truth, seq.odometry)


def c3_spec(frames=450, points=20000, seed=1) -> S.SceneSpec:
    # drift bias of the initial guesses: 0.1 deg yaw + 1 cm per frame
    return S.SceneSpec(shape="figure_eight", frames=frames, radius=50.0, points_per_scan=points, seed=seed,
                       drift=(0.0, 0.0, np.deg2rad(0.1), 0.01, 0.0, 0.0))


def c2_spec(frames=100, points=20000, seed=2) -> S.SceneSpec:
    return S.SceneSpec(shape="circle", frames=frames, radius=50.0, points_per_scan=points, seed=seed,
                       drift=(0.0, 0.0, np.deg2rad(0.1), 0.0, 0.0, 0.0))


def c1_spec(points=20000, seed=3) -> S.SceneSpec:
    return S.SceneSpec(shape="line", frames=2, spacing=1.0, points_per_scan=points, seed=seed)


def select_links(overlaps: dict, frames: int, max_links: int = 10, min_overlap: float = 0.025):
    """For each frame j, its up-to-max_links predecessors i with overlap > min_overlap (strict,
    pipeline.cpp:140), highest overlap first; returns [(i, j)] sorted by (j, i)."""
    by_j: dict = {}
    for (i, j), ov in overlaps.items():
        if ov > min_overlap:
            by_j.setdefault(j, []).append((-ov, i))
    links = []
    for j in range(1, frames):
        cands = sorted(by_j.get(j, []))[:max_links]
        links.extend(sorted((i, j) for _, i in cands))
    return links


@dataclass
class GraphWorkload:
    ctx: object  # paper_2109_07073_b200.Context
    scans: Scans
    clouds: list
    maps: list
    links: list  # (target i, source j)
    factors: list
    graph: object  # paper_2109_07073_b200.FactorGraph
    poses: np.ndarray  # num_poses × 12 (initial guesses: drifted odometry)
    resolution: float
    build_seconds: dict = field(default_factory=dict)

    @property
    def num_factors(self) -> int:
        return len(self.factors)

    def num_points(self) -> int:
        return self.graph.num_points()


def build_graph_workload(ctx, spec: S.SceneSpec, resolution: float = 1.0, max_links: int = 10,
                         min_overlap: float = 0.025, links=None, chunk: int = 0, threads: int = 0,
                         gpu_covariances: bool = True) -> GraphWorkload:
    from paper_2109_07073_b200.vgicp import FactorGraph, GaussianVoxelMap, MatchingCostFactor, PointCloud, overlap_hits

    t0 = time.perf_counter()
    scans = make_scans(spec, threads=threads, ctx=ctx if gpu_covariances else None)
    t1 = time.perf_counter()
    clouds = PointCloud.upload_batch(scans.means, scans.cov6, ctx)
    maps = GaussianVoxelMap.build_batch(clouds, resolution)
    ctx.synchronize()
    t2 = time.perf_counter()
    n = len(clouds)
    if links is None:
        pairs = [(i, j) for j in range(1, n) for i in range(j)]
        rels = relative_poses(scans.gt, pairs)  # T_i⁻¹·T_j, pipeline.cpp:138
        hits = overlap_hits([clouds[j] for _, j in pairs], rels, [maps[i] for i, _ in pairs])
        overlaps = {p: float(h) / len(scans.means[p[1]]) for p, h in zip(pairs, hits)}
        links = select_links(overlaps, n, max_links, min_overlap)
    t3 = time.perf_counter()
    factors = [MatchingCostFactor(i, j, clouds[j], maps[i]) for i, j in links]
    graph = FactorGraph(factors, n, chunk=chunk, ctx=ctx)
    t4 = time.perf_counter()
    return GraphWorkload(ctx, scans, clouds, maps, list(links), factors, graph, np.ascontiguousarray(scans.odom), resolution,
                         dict(scans=t1 - t0, upload_and_maps=t2 - t1, overlap_selection=t3 - t2, graph=t4 - t3))


def c2_links(frames: int = 100, depth: int = 3):
    return [(k - d, k) for k in range(1, frames) for d in range(1, depth + 1) if k - d >= 0]


C5_RESOLUTIONS = (0.5, 1.0, 2.0)


def c5_spec(frames=1000, points=20000, seed=5) -> S.SceneSpec:
    return S.SceneSpec(shape="figure_eight", frames=frames, radius=50.0, points_per_scan=points, seed=seed,
                       drift=(0.0, 0.0, np.deg2rad(0.1), 0.01, 0.0, 0.0))


def build_c5_workload(ctx, spec: S.SceneSpec | None = None, max_links: int = 10, min_overlap: float = 0.025,
                      chunk: int = 0) -> GraphWorkload:
    """C5: every frame gets 0.5 / 1 / 2 m maps; links by the overlap rule on the 1 m maps; link k
    uses the map of resolution C5_RESOLUTIONS[k % 3]."""
    from paper_2109_07073_b200.vgicp import FactorGraph, GaussianVoxelMap, MatchingCostFactor, PointCloud, overlap_hits

    spec = spec or c5_spec()
    t0 = time.perf_counter()
    scans = make_scans(spec, ctx=ctx)
    t1 = time.perf_counter()
    clouds = PointCloud.upload_batch(scans.means, scans.cov6, ctx)
    maps = {r: GaussianVoxelMap.build_batch(clouds, r) for r in C5_RESOLUTIONS}
    ctx.synchronize()
    t2 = time.perf_counter()
    n = len(clouds)
    pairs = [(i, j) for j in range(1, n) for i in range(j)]
    rels = relative_poses(scans.gt, pairs)
    hits = overlap_hits([clouds[j] for _, j in pairs], rels, [maps[1.0][i] for i, _ in pairs])
    overlaps = {p: float(h) / len(scans.means[p[1]]) for p, h in zip(pairs, hits)}
    links = select_links(overlaps, n, max_links, min_overlap)
    t3 = time.perf_counter()
    factors = [MatchingCostFactor(i, j, clouds[j], maps[C5_RESOLUTIONS[k % 3]][i]) for k, (i, j) in enumerate(links)]
    graph = FactorGraph(factors, n, chunk=chunk, ctx=ctx)
    t4 = time.perf_counter()
    return GraphWorkload(ctx, scans, clouds, [m for r in C5_RESOLUTIONS for m in maps[r]], list(links), factors, graph,
                         np.ascontiguousarray(scans.odom), 1.0,
                         dict(scans=t1 - t0, upload_and_maps=t2 - t1, overlap_selection=t3 - t2, graph=t4 - t3))
