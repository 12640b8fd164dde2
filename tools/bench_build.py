"""Time the graph-construction stages of the C3 workload (not part of the bench line)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2109_07073_b200 as V
from bench_workloads import workloads as W

ctx = V.Context(0)
t = time.perf_counter()
sc = W.make_scans(W.c3_spec())
print(f"scans+covariances {time.perf_counter() - t:.2f} s")
t = time.perf_counter()
clouds = [V.PointCloud(m, c, ctx) for m, c in zip(sc.means, sc.cov6)]
ctx.synchronize()
print(f"upload 450 clouds {time.perf_counter() - t:.3f} s")
for rep in range(3):
    t = time.perf_counter()
    maps = V.GaussianVoxelMap.build_batch(clouds, 1.0)
    ctx.synchronize()
    print(f"build_batch 450 maps {time.perf_counter() - t:.3f} s, voxels {sum(m.size() for m in maps)}")
t = time.perf_counter()
one = V.GaussianVoxelMap(clouds[0], 1.0)
ctx.synchronize()
print(f"single map {1e3 * (time.perf_counter() - t):.2f} ms")
pairs = [(i, j) for j in range(1, 450) for i in range(j)]
rels = [W.pose_mul(W.pose_inv(sc.gt[i]), sc.gt[j]) for i, j in pairs]
for rep in range(2):
    t = time.perf_counter()
    hits = V.overlap_hits([clouds[j] for _, j in pairs], rels, [maps[i] for i, _ in pairs])
    print(f"overlap {len(pairs)} pairs {time.perf_counter() - t:.3f} s")
