"""C4 sweep breakdown: Python marshalling vs C ABI call vs kernel (diagnostic)."""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2109_07073_b200 as V
from bench_workloads import workloads as W, synthetic as S
from paper_2109_07073_b200 import _lib
ctx = V.default_context()
n_maps = 4000
seq = S.generate(S.SceneSpec(shape="figure_eight", frames=n_maps + 1, radius=50.0, points_per_scan=20000, seed=4))
unit = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (20000, 1))
clouds = [V.PointCloud(m, unit[: len(m)], ctx) for m in seq.scans]
maps = V.GaussianVoxelMap.build_batch(clouds[:n_maps], 1.0)
new = clouds[n_maps]
rels = np.stack([W.pose_mul(W.pose_inv(seq.ground_truth[i]), seq.ground_truth[n_maps]) for i in range(n_maps)])
def t(label, fn, reps=10):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    print(f"{label:32s} {1e3*(time.perf_counter()-t0)/reps:7.3f} ms", flush=True)
t("overlap_hits (python API)", lambda: V.overlap_hits(new, rels, maps))
m = n_maps
ch = (C.c_void_p * m)(*[new.handle] * m)
mh = (C.c_void_p * m)(*[x.handle for x in maps])
P = np.ascontiguousarray(rels)
hits = np.zeros(m, np.uint64)
t("vgicp_overlap_batch (C ABI only)", lambda: _lib.load().vgicp_overlap_batch(ctx.handle, ch, P.ctypes.data_as(C.c_void_p), mh, m, hits.ctypes.data_as(C.c_void_p)))
t("marshalling only", lambda: ((C.c_void_p * m)(*[new.handle] * m), (C.c_void_p * m)(*[x.handle for x in maps])))
