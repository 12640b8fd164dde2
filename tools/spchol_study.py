"""C3 LM damped-solve study, part 2 (diagnostic): cuSOLVER's sparse Cholesky (csrchol low-level
API: analysis once per sparsity pattern, numeric factor + solve per damping value) under several
fill-reducing orderings, against the dense cuSOLVER potrf path the LM uses."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import scipy.sparse as sp  # noqa: E402
import torch  # noqa: E402

import paper_2109_07073_b200 as V  # noqa: E402
from paper_2109_07073_b200 import optimizer as LM  # noqa: E402
from bench_workloads import workloads as W  # noqa: E402

cus = C.CDLL("libcusolver.so.11")
csp = C.CDLL("libcusparse.so.12")


def ok(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed: {rc}")


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
lam = 1e-5
ref = sol.solve(lam)
A = sol.Hd.clone()
A.diagonal().copy_(sol.dg + lam * torch.clamp(sol.dg, min=1e-10))
Ah = A.cpu().numpy()
b = sol.bd.reshape(-1).cpu().numpy()
m = Ah.shape[0]
Asp = sp.csr_matrix(Ah)
Asp.eliminate_zeros()
print(f"m {m} nnz {Asp.nnz} ({Asp.nnz / m / m:.3%} dense)")

h = C.c_void_p()
ok(cus.cusolverSpCreate(C.byref(h)), "cusolverSpCreate")
descr = C.c_void_p()
ok(csp.cusparseCreateMatDescr(C.byref(descr)), "cusparseCreateMatDescr")
stream = torch.cuda.current_stream().cuda_stream
ok(cus.cusolverSpSetStream(h, C.c_void_p(stream)), "setStream")


def host_perm(kind):
    rp = np.ascontiguousarray(Asp.indptr.astype(np.int32))
    ci = np.ascontiguousarray(Asp.indices.astype(np.int32))
    p = np.zeros(m, np.int32)
    ip = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    if kind == "none":
        return np.arange(m, dtype=np.int32)
    if kind == "symrcm":
        ok(cus.cusolverSpXcsrsymrcmHost(h, m, Asp.nnz, descr, ip(rp), ip(ci), ip(p)), kind)
    elif kind == "symamd":
        ok(cus.cusolverSpXcsrsymamdHost(h, m, Asp.nnz, descr, ip(rp), ip(ci), ip(p)), kind)
    elif kind == "metisnd":
        ok(cus.cusolverSpXcsrmetisndHost(h, m, Asp.nnz, descr, ip(rp), ip(ci), None, ip(p)), kind)
    return p


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / reps


print(f"dense potrf+potrs (current solve())        {timeit(lambda: sol.solve(lam)):8.3f} ms")
for kind in ("none", "symrcm", "symamd", "metisnd"):
    try:
        p = host_perm(kind)
        Ap = Asp[p][:, p].tocsr()
        Ap.sort_indices()
        rp = torch.from_numpy(Ap.indptr.astype(np.int32)).to(dev)
        ci = torch.from_numpy(Ap.indices.astype(np.int32)).to(dev)
        vals = torch.from_numpy(Ap.data.astype(np.float64)).to(dev)
        bp = torch.from_numpy(b[p].copy()).to(dev)
        x = torch.empty(m, dtype=torch.float64, device=dev)
        info = C.c_void_p()
        ok(cus.cusolverSpCreateCsrcholInfo(C.byref(info)), "createInfo")
        t0 = time.perf_counter()
        ok(cus.cusolverSpXcsrcholAnalysis(h, m, Ap.nnz, descr, C.c_void_p(rp.data_ptr()), C.c_void_p(ci.data_ptr()),
                                          info), "analysis")
        internal, work = C.c_size_t(), C.c_size_t()
        ok(cus.cusolverSpDcsrcholBufferInfo(h, m, Ap.nnz, descr, C.c_void_p(vals.data_ptr()),
                                            C.c_void_p(rp.data_ptr()), C.c_void_p(ci.data_ptr()), info,
                                            C.byref(internal), C.byref(work)), "bufferInfo")
        torch.cuda.synchronize()
        t_an = 1e3 * (time.perf_counter() - t0)
        buf = torch.empty(max(work.value, 1), dtype=torch.uint8, device=dev)
        pos = C.c_int()

        def run():
            ok(cus.cusolverSpDcsrcholFactor(h, m, Ap.nnz, descr, C.c_void_p(vals.data_ptr()),
                                            C.c_void_p(rp.data_ptr()), C.c_void_p(ci.data_ptr()), info,
                                            C.c_void_p(buf.data_ptr())), "factor")
            ok(cus.cusolverSpDcsrcholZeroPivot(h, info, C.c_double(0.0), C.byref(pos)), "zeroPivot")
            ok(cus.cusolverSpDcsrcholSolve(h, m, C.c_void_p(bp.data_ptr()), C.c_void_p(x.data_ptr()), info,
                                           C.c_void_p(buf.data_ptr())), "solve")
            return x.cpu()

        def factor_only():
            ok(cus.cusolverSpDcsrcholFactor(h, m, Ap.nnz, descr, C.c_void_p(vals.data_ptr()),
                                            C.c_void_p(rp.data_ptr()), C.c_void_p(ci.data_ptr()), info,
                                            C.c_void_p(buf.data_ptr())), "factor")

        tt = timeit(run)
        tf = timeit(factor_only)
        xs = np.empty(m)
        xs[p] = run().numpy()
        err = float(np.abs(xs - ref).max() / max(1e-300, np.abs(ref).max()))
        print(f"csrchol {kind:8s} analysis {t_an:8.2f} ms  internal {internal.value / 1e6:6.1f} MB  "
              f"factor {tf:7.3f} ms  factor+pivot+solve+D2H {tt:7.3f} ms  rel diff {err:.2e} pivot {pos.value}",
              flush=True)
        cus.cusolverSpDestroyCsrcholInfo(info)
    except Exception as e:  # noqa: BLE001
        print(kind, "failed:", repr(e), flush=True)
