"""Stage timing of the submap path on the C3 workload's first 20 frames (diagnostic)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2109_07073_b200 as V
from bench_workloads import workloads as W

ctx = V.default_context()
sc = W.make_scans(W.c3_spec(frames=20), ctx=ctx)
clouds = [V.PointCloud(m, c, ctx) for m, c in zip(sc.means, sc.cov6)]
poses = np.stack([W.pose_mul(W.pose_inv(sc.gt[0]), sc.gt[k]) for k in range(20)])


def t(label, fn, reps=5):
    fn()
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    ctx.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0) / reps:8.2f} ms")


t("submap full (cloud)", lambda: V.build_submap(clouds, poses, 0.25, 1.0))
t("submap no cloud", lambda: V.build_submap(clouds, poses, 0.25, 1.0, want_cloud=False))
t("submap no downsample, no cloud", lambda: V.build_submap(clouds, poses, 0.0, 1.0, want_cloud=False))
t("build_batch 20 frames @1.0", lambda: V.GaussianVoxelMap.build_batch(clouds, 1.0))
m = np.concatenate(sc.means).astype(np.float64)
c = np.repeat(np.eye(3)[None], len(m), 0)
t("build_f64 400k (host arrays)", lambda: V.GaussianVoxelMap.from_arrays(m, c, 0.25))
