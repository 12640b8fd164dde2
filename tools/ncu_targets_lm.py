"""Launches the LM-side kernels once on C3 data for ncu (diagnostic): device assembly, the band
solver (damped solve), and a C4-style map-set overlap sweep."""
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2109_07073_b200 as V  # noqa: E402
from paper_2109_07073_b200 import optimizer as LM  # noqa: E402
from bench_workloads import workloads as W  # noqa: E402

ctx = V.default_context()
wl = W.build_graph_workload(ctx, W.c3_spec())
g = wl.graph
n = len(wl.poses)
fixed = LM.effective_fixed_mask(n, g._ij, np.zeros(n, bool))
plan = g.assembly_plan(fixed.astype(np.uint8))
S, P = plan.num_slots, len(plan.pairs)
d_asm = torch.empty((S + P) * 36 + S * 6, dtype=torch.float64, device="cuda")
d_poses = torch.from_numpy(np.ascontiguousarray(wl.poses)).cuda()
g.linearize_assembled_device(d_poses.data_ptr(), d_asm.data_ptr())
ctx.synchronize()
g.solver_plan()
g.solve_damped(d_asm.data_ptr(), 1e-5)
ms = V.MapSet(wl.maps[:400])
rels = np.stack([W.pose_mul(W.pose_inv(wl.scans.gt[i]), wl.scans.gt[400]) for i in range(400)])
V.overlap_hits(wl.clouds[400], rels, ms)
ctx.synchronize()
print("lm ncu targets done")
