"""Timing breakdown of one C3 LM iteration's pieces (diagnostic)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2109_07073_b200 as V
from bench_workloads import workloads as W
from paper_2109_07073_b200 import optimizer as LM
ctx = V.default_context()
wl = W.build_graph_workload(ctx, W.c3_spec())
g, poses = wl.graph, wl.poses
n = len(poses)
fixed = LM.effective_fixed_mask(n, g._ij, np.zeros(n, bool))
plan = g.assembly_plan(fixed.astype(np.uint8))
dev = torch.device("cuda", 0)
S, P = plan.num_slots, len(plan.pairs)
d_asm = torch.empty((S + P) * 36 + S * 6, dtype=torch.float64, device=dev)
d_poses = torch.from_numpy(np.ascontiguousarray(poses)).to(dev)
def t(label, fn, reps=10):
    fn(); torch.cuda.synchronize(); ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); ctx.synchronize()
    print(f"{label:36s} {1e3*(time.perf_counter()-t0)/reps:7.3f} ms", flush=True)
t("linearize_assembled_device", lambda: (g.linearize_assembled_device(d_poses.data_ptr(), d_asm.data_ptr()), ctx.synchronize()))
sysv = (d_asm[: S * 36].view(S, 6, 6), d_asm[S * 36:(S + P) * 36].view(P, 6, 6), d_asm[(S + P) * 36:].view(S, 6))
bw = LM.graph_bandwidth(np.asarray(g._ij), ~fixed)
t("build dense system on GPU", lambda: LM._ReducedSolver(*sysv[:2], plan.pairs, sysv[2], bw, dev))
sol = LM._ReducedSolver(*sysv[:2], plan.pairs, sysv[2], bw, dev)
t("cholesky + solve (GPU)", lambda: sol.solve(1e-5))
t("total_error (evaluate + D2H)", lambda: g.total_error(poses))
delta = np.random.default_rng(0).standard_normal(6 * n) * 1e-4
act = np.flatnonzero(~fixed)
t("retract (host)", lambda: LM.compose_batch(poses[act], LM.se3_exp_batch(delta.reshape(-1, 6)[act])))
