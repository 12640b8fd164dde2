"""Per-call submap timings from a cold context (diagnostic)."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2109_07073_b200 as V
from paper_2109_07073_b200 import workloads as W
ctx = V.default_context()
sc = W.make_scans(W.c3_spec(frames=20), ctx=ctx)
clouds = [V.PointCloud(m, c, ctx) for m, c in zip(sc.means, sc.cov6)]
poses = np.stack([W.pose_mul(W.pose_inv(sc.gt[0]), sc.gt[k]) for k in range(20)])
os.environ["VGICP_VERBOSE"] = "1"
for k in range(8):
    t0 = time.perf_counter()
    sub = V.build_submap(clouds, poses, 0.25, 1.0)
    print("call", k, round(1e3 * (time.perf_counter() - t0), 2), "ms", flush=True)
