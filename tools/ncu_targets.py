"""Small driver that launches each profiled kernel family once on C3-shaped data (for ncu):
linearize + evaluate (factor_kernel), device assembly, covariance kNN, submap transform + fp64 build."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2109_07073_b200 as V
from bench_workloads import workloads as W

ctx = V.default_context()
wl = W.build_graph_workload(ctx, W.c3_spec())
g = wl.graph
g.linearize_raw(wl.poses)
g.evaluate(wl.poses)
fixed = np.zeros(len(wl.poses), np.uint8)
fixed[0] = 1
g.assembly_plan(fixed)
g.linearize_assembled(wl.poses)
V.estimate_covariances_batch(wl.scans.means[:50], 10, 1e-3, ctx)
poses = np.stack([W.pose_mul(W.pose_inv(wl.scans.gt[0]), wl.scans.gt[k]) for k in range(20)])
V.build_submap(wl.clouds[:20], poses, 0.25, 1.0)
ctx.synchronize()
print("ncu targets done")
