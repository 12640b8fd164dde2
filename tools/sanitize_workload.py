"""Small workload touching every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): batched upload, hand-written map build (shared-memory mark+rank, radix sort,
scatter and global-cursor variants, accumulate, export, on-demand hash table), the sort-based build,
float64 clouds and the submap path, overlap (occupancy, hash, map set), factor kernels (rank + hash
lookups, float64 sources), device assembly, band solver (single + pair), native LM, sharded graph over
two contexts, covariance preprocessing. Sizes are kept small (the tools slow kernels ~100x)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle_ctypes as O  # noqa: E402
import paper_2109_07073_b200 as V  # noqa: E402
from paper_2109_07073_b200 import optimizer as LM  # noqa: E402

rng = O.Rng(91)
ctx = V.default_context(0)
frames = []
for k in range(5):
    m, c = rng.gaussian_cloud(1500 + 300 * k, 8.0)
    frames.append((m.astype(np.float32), V.cov6_from(c).astype(np.float32)))
clouds = V.PointCloud.upload_batch([f[0] for f in frames], [f[1] for f in frames], ctx)
maps = V.GaussianVoxelMap.build_batch(clouds, [1.0, 0.5, 1.0, 2.0, 1.0])
for env in ("VGICP_BUILD_SCATTER", "VGICP_SORTED_BUILD"):
    os.environ[env] = "1"
    alt = V.GaussianVoxelMap.build_batch(clouds[:2], [1.0, 0.5])
    assert all(np.array_equal(a, b) for a, b in zip(alt[0].export(), maps[0].export()))
    del os.environ[env]
big = np.random.default_rng(4).uniform(-60, 60, size=(60000, 3)).astype(np.float32)
bmap = V.GaussianVoxelMap(V.PointCloud(big, np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (len(big), 1)), ctx), 0.5)
print("big map voxels", bmap.size(), "lookup", int((bmap.lookup(big[:100].astype(np.float64)) != V.KEY_MISS).sum()))
poses = np.stack([rng.random_pose(0.05, 0.5) for _ in range(5)])
links = [(0, 1), (1, 2), (2, 3), (3, 4), (0, 2), (4, 0)]
graph = V.FactorGraph([V.MatchingCostFactor(i, j, clouds[j], maps[i]) for i, j in links], 5, chunk=1024)
raw, inl = graph.linearize_raw(poses)
err, _ = graph.evaluate(poses)
os.environ["VGICP_NO_RANK"] = "1"
hraw, _ = V.FactorGraph([V.MatchingCostFactor(i, j, clouds[j], maps[i]) for i, j in links], 5).linearize_raw(poses)
del os.environ["VGICP_NO_RANK"]
rels = [O.compose(O.inverse(poses[i]), poses[j]) for i, j in links]
hits = V.overlap_hits([clouds[j] for _, j in links], rels, [maps[i] for i, _ in links])
ms = V.MapSet(maps)
mhits = V.overlap_hits(clouds[1], [O.compose(O.inverse(poses[k]), poses[1]) for k in range(5)], ms)
os.environ["VGICP_LM_NO_HOST_BAND"] = "1"
p_opt, rep = LM.optimize_native(graph, poses, settings=LM.LmSettings(max_iterations=3))
del os.environ["VGICP_LM_NO_HOST_BAND"]
ctx2 = V.Context(0)
c2 = V.PointCloud.upload_batch([f[0] for f in frames], [f[1] for f in frames], ctx2)
m2 = V.GaussianVoxelMap.build_batch(c2, [1.0, 0.5, 1.0, 2.0, 1.0])
sh = V.FactorGraph.sharded([[V.MatchingCostFactor(i, j, clouds[j], maps[i]) for i, j in links],
                            [V.MatchingCostFactor(i, j, c2[j], m2[i]) for i, j in links]], 5)
sraw, _ = sh.linearize_raw(poses)
assert np.array_equal(sraw, raw)
sub = V.build_submap(clouds[:3], poses[:3], 0.25, 1.0)
sf = V.MatchingCostFactor(0, 1, sub.cloud, maps[0])
V.FactorGraph([sf], 2).linearize_raw(poses[:2])
cov = V.estimate_covariances(frames[0][0][:800], 10, 1e-3, ctx)
print("ok", int(inl.sum()), float(err.sum()), int(hits.sum()), int(mhits.sum()), rep.reason, sub.voxels.size(), cov.shape)
