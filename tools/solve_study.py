"""C3 LM damped-solve study (diagnostic): timing of the dense GPU Cholesky variants and the
sparsity of the reduced system under reverse Cuthill-McKee ordering."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import scipy.sparse as sp  # noqa: E402
import scipy.sparse.csgraph as csg  # noqa: E402
import torch  # noqa: E402

import paper_2109_07073_b200 as V  # noqa: E402
from paper_2109_07073_b200 import optimizer as LM  # noqa: E402
from bench_workloads import workloads as W  # noqa: E402

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
g.linearize_assembled_device(d_poses.data_ptr(), d_asm.data_ptr())
ctx.synchronize()
sysv = (d_asm[: S * 36].view(S, 6, 6), d_asm[S * 36:(S + P) * 36].view(P, 6, 6), d_asm[(S + P) * 36:].view(S, 6))
bw = LM.graph_bandwidth(np.asarray(g._ij), ~fixed)
sol = LM._ReducedSolver(*sysv[:2], plan.pairs, sysv[2], bw, dev)
m = sol.m
print(f"slots {S} pairs {P} m {m} bandwidth {bw}")


def t(label, fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{label:44s} {1e3 * (time.perf_counter() - t0) / reps:8.3f} ms", flush=True)


lam = 1e-5
A = sol.Hd.clone()
A.diagonal().copy_(sol.dg + lam * torch.clamp(sol.dg, min=1e-10))
t("solve() (current: clone, potrf, info, potrs, D2H)", lambda: sol.solve(lam))
t("cholesky_ex only (+sync)", lambda: torch.linalg.cholesky_ex(A))
L, _ = torch.linalg.cholesky_ex(A)
t("cholesky_solve only", lambda: torch.cholesky_solve(sol.bd, L))
A32 = A.float()
t("cholesky_ex fp32", lambda: torch.linalg.cholesky_ex(A32))
# CUDA-graph-captured damped solve (static shapes)
static_lam = torch.zeros((), dtype=torch.float64, device=dev)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        B = sol.Hd.clone()
        B.diagonal().copy_(sol.dg + static_lam * torch.clamp(sol.dg, min=1e-10))
        Lg, infog = torch.linalg.cholesky_ex(B)
        xg = torch.cholesky_solve(sol.bd, Lg)
torch.cuda.current_stream().wait_stream(s)
graph = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(graph):
        B = sol.Hd.clone()
        B.diagonal().copy_(sol.dg + static_lam * torch.clamp(sol.dg, min=1e-10))
        Lg, infog = torch.linalg.cholesky_ex(B)
        xg = torch.cholesky_solve(sol.bd, Lg)

    def run_graph():
        static_lam.fill_(lam)
        graph.replay()
        return int(infog.item()), xg.cpu()

    t("CUDA graph: damp + potrf + potrs (+info, D2H)", run_graph)
    ref = sol.solve(lam)
    print("graph result max |diff|", float(np.abs(run_graph()[1].numpy().reshape(-1) - ref).max()))
except Exception as e:  # noqa: BLE001
    print("graph capture failed:", repr(e))

# sparsity under RCM (block level)
ij = np.asarray(g._ij)
act_slots = {int(v): s_ for s_, v in enumerate(plan.var_of_slot)}
rows, cols = [], []
for a, b in plan.pairs:
    rows += [a, b]
    cols += [b, a]
Ab = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(S, S))
perm = csg.reverse_cuthill_mckee(Ab, symmetric_mode=True)
inv = np.empty_like(perm)
inv[perm] = np.arange(S)
pa, pb = inv[plan.pairs[:, 0]], inv[plan.pairs[:, 1]]
print("block bandwidth: slot order", int(np.abs(plan.pairs[:, 0] - plan.pairs[:, 1]).max()),
      "RCM", int(np.abs(pa - pb).max()))
prof = np.zeros(S, np.int64)
for a, b in zip(pa, pb):
    hi, lo = max(a, b), min(a, b)
    prof[hi] = max(prof[hi], hi - lo)
print("RCM envelope (blocks)", int(prof.sum()), "of dense", S * (S - 1) // 2,
      "-> factor flops ratio ~", float((prof.astype(float) ** 2).sum() / (S ** 3 / 3)))

# GPU block-band Cholesky (vgicp_graph_solve_damped)
bwp, okp = g.solver_plan()
print("band solver plan: bandwidth", bwp, "supported", okp)
if okp:
    t("band solve (RCM block Cholesky, x to host)", lambda: g.solve_damped(d_asm.data_ptr(), lam))
    t("band solve pair (lam, 10·lam: two clusters, one launch)",
      lambda: g.solve_damped_pair(d_asm.data_ptr(), (lam, 10 * lam)))
    xb = g.solve_damped(d_asm.data_ptr(), lam)
    ref = sol.solve(lam)
    print("band vs dense max rel diff", float(np.abs(xb - ref).max() / np.abs(ref).max()))
