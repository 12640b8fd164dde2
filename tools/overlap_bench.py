"""Overlap kernel timing: the C3 factor-selection sweep shape (all pairs of 120 frames), device-timed."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2109_07073_b200 as V
from bench_workloads import workloads as W
ctx = V.default_context()
sc = W.make_scans(W.c3_spec(frames=120), ctx=ctx)
clouds = [V.PointCloud(m, c, ctx) for m, c in zip(sc.means, sc.cov6)]
maps = V.GaussianVoxelMap.build_batch(clouds, 1.0)
pairs = [(i, j) for j in range(1, 120) for i in range(j)]
rels = np.stack([W.pose_mul(W.pose_inv(sc.gt[i]), sc.gt[j]) for i, j in pairs])
cl = [clouds[j] for _, j in pairs]
mp = [maps[i] for i, _ in pairs]
V.overlap_hits(cl, rels, mp)
ctx.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    V.overlap_hits(cl, rels, mp)
dt = (time.perf_counter() - t0) / 5
probes = len(pairs) * 20000
print(f"overlap sweep {len(pairs)} pairs: {1e3*dt:.2f} ms, {probes/dt/1e9:.1f} G probes/s")
