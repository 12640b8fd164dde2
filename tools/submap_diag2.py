"""Bench-order diagnostic for the submap leg: C3 workload, C1, C4, covariance legs, then submap."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import bench as B
import paper_2109_07073_b200 as V
from paper_2109_07073_b200 import workloads as W
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = V.Context(0, stream=stream.cuda_stream)
wl = W.build_graph_workload(ctx, W.c3_spec())
poses = np.stack([W.pose_mul(W.pose_inv(wl.scans.gt[0]), wl.scans.gt[k]) for k in range(20)])
def tm(label):
    t0 = time.perf_counter()
    for _ in range(3):
        V.build_submap(wl.clouds[:20], poses, 0.25, 1.0)
    print(label, 1e3 * (time.perf_counter() - t0) / 3, "ms", flush=True)
tm("start")
B.run_c1(ctx, 16); tm("after c1")
B.run_c4(ctx); tm("after c4")
B.run_covariances(ctx, wl.scans.means); tm("after cov")
os.environ["VGICP_VERBOSE"] = "1"
for _ in range(2):
    t0 = time.perf_counter(); V.build_submap(wl.clouds[:20], poses, 0.25, 1.0); print("one", 1e3*(time.perf_counter()-t0), flush=True)
