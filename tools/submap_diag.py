"""Reproduces the bench order (C3 workload resident, C4 maps built) before timing the submap leg."""
import sys, time, os
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2109_07073_b200 as V
from paper_2109_07073_b200 import workloads as W, synthetic as S
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = V.Context(0, stream=stream.cuda_stream)
wl = W.build_graph_workload(ctx, W.c3_spec())
poses = np.stack([W.pose_mul(W.pose_inv(wl.scans.gt[0]), wl.scans.gt[k]) for k in range(20)])
def tm(label):
    V.build_submap(wl.clouds[:20], poses, 0.25, 1.0)
    t0 = time.perf_counter()
    for _ in range(3):
        V.build_submap(wl.clouds[:20], poses, 0.25, 1.0)
    print(label, 1e3 * (time.perf_counter() - t0) / 3, "ms", flush=True)
tm("after C3 build")
seq = S.generate(S.SceneSpec(shape="figure_eight", frames=4001, radius=50.0, points_per_scan=20000, seed=4))
unit = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (20000, 1))
clouds = [V.PointCloud(m, unit[: len(m)], ctx) for m in seq.scans]
maps = V.GaussianVoxelMap.build_batch(clouds[:4000], 1.0)
tm("with C4 maps resident")
del maps, clouds
import gc; gc.collect()
tm("after C4 freed")
os.environ["VGICP_VERBOSE"] = "1"
V.build_submap(wl.clouds[:20], poses, 0.25, 1.0)
