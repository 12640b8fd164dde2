"""Small single-factor linearize/evaluate run (for compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import oracle_ctypes as O
import paper_2109_07073_b200 as V

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
rng = O.Rng(83)
tm, tc = rng.gaussian_cloud(n, 12.0)
sm, sc = rng.gaussian_cloud(n, 12.0)
ctx = V.default_context(0)
tgt = V.PointCloud(tm, tc, ctx)
src = V.PointCloud(sm, sc, ctx)
vmap = V.GaussianVoxelMap(tgt, 1.0)
f = V.MatchingCostFactor(0, 1, src, vmap)
Ti, Tj = rng.random_pose(0.1, 1.0), rng.random_pose(0.1, 1.0)
lin = V.linearize_matching_cost(f, Ti, Tj)
print("inliers", lin.inliers, "error", lin.error)
print("eval", V.evaluate_matching_cost(f, Ti, Tj))
