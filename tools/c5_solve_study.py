"""C5 LM damped-solve study (diagnostic): dense cuSOLVER vs the GPU block-band solver on the
1,000-pose multi-resolution graph, and the full LM both ways."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2109_07073_b200 as V  # noqa: E402
from paper_2109_07073_b200 import optimizer as LM  # noqa: E402
from bench_workloads import workloads as W  # noqa: E402

ctx = V.default_context()
wl = W.build_c5_workload(ctx)
g, poses = wl.graph, wl.poses
n = len(poses)
fixed = LM.effective_fixed_mask(n, g._ij, np.zeros(n, bool))
plan = g.assembly_plan(fixed.astype(np.uint8))
dev = torch.device("cuda", 0)
S, P = plan.num_slots, len(plan.pairs)
d_asm = torch.empty((S + P) * 36 + S * 6, dtype=torch.float64, device=dev)
d_poses = torch.from_numpy(np.ascontiguousarray(poses)).to(dev)
g.linearize_assembled_device(d_poses.data_ptr(), d_asm.data_ptr())
ctx.synchronize()
sysv = (d_asm[: S * 36].view(S, 6, 6), d_asm[S * 36:(S + P) * 36].view(P, 6, 6), d_asm[(S + P) * 36:].view(S, 6))
bw = LM.graph_bandwidth(np.asarray(g._ij), ~fixed)
sol = LM._ReducedSolver(*sysv[:2], plan.pairs, sysv[2], bw, dev)
print(f"factors {len(g._ij)} slots {S} pairs {P} m {sol.m}")


def t(label, fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{label:44s} {1e3 * (time.perf_counter() - t0) / reps:8.3f} ms", flush=True)


lam = 1e-5
t("dense solve (cuSOLVER potrf/potrs)", lambda: sol.solve(lam))
bwp, ok = g.solver_plan()
print("band plan: bandwidth", bwp, "supported", ok)
if ok:
    t("band solve", lambda: g.solve_damped(d_asm.data_ptr(), lam))
    print("band vs dense max rel diff",
          float(np.abs(g.solve_damped(d_asm.data_ptr(), lam) - sol.solve(lam)).max() / np.abs(sol.solve(lam)).max()))
for band in (False, True):
    LM.optimize(g, poses, settings=LM.LmSettings(max_iterations=1), band_solve=band)
    _, rep = LM.optimize(g, poses, settings=LM.LmSettings(max_iterations=10), band_solve=band)
    its = sorted(rep.iteration_seconds)
    print(f"LM band={band}: {rep.iterations} its, median {1e3 * its[len(its) // 2]:.2f} ms/it, final {rep.final_error:.6f}")
