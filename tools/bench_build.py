"""Time the C3 map build (450 float32 clouds, 1.0 m): the hand-written build (build.cu) vs the
sort-based one (VGICP_SORTED_BUILD=1), wall clock through vgicp_voxelmap_build_batch (each call ends
in a stream synchronisation). `--profile`: only the hand-written build, for ncu."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2109_07073_b200 as V  # noqa: E402
from bench_workloads import workloads as W  # noqa: E402

profile = "--profile" in sys.argv
ctx = V.Context(0)
t = time.perf_counter()
sc = W.make_scans(W.c3_spec(), ctx=ctx)
print(f"scans+covariances {time.perf_counter() - t:.2f} s")
t = time.perf_counter()
clouds = V.PointCloud.upload_batch(sc.means, sc.cov6, ctx)
ctx.synchronize()
print(f"upload 450 clouds {time.perf_counter() - t:.3f} s")
for mode in (["fast"] if profile else ["fast", "sorted", "fast"]):
    if mode == "sorted":
        os.environ["VGICP_SORTED_BUILD"] = "1"
    ts = []
    for rep in range(1 if profile else 5):
        t = time.perf_counter()
        maps = V.GaussianVoxelMap.build_batch(clouds, 1.0)
        ctx.synchronize()
        ts.append(time.perf_counter() - t)
    os.environ.pop("VGICP_SORTED_BUILD", None)
    print(f"{mode:6s} build_batch 450 maps: min {1e3 * min(ts):.3f} ms median {1e3 * sorted(ts)[len(ts) // 2]:.3f} ms, "
          f"voxels {sum(m.size() for m in maps)}")
