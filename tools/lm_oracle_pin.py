"""Native GPU LM (vgicp_graph_optimize) vs the same LM driven by the CPU oracle's factors (the
reference's double-precision arithmetic) on C2 and a 60-frame C3 slice: trace lengths, final errors,
pose differences, for the default and a tight convergence tolerance."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_2109_07073_b200 as V  # noqa: E402
from bench import _OracleGraph  # noqa: E402
from bench_workloads import workloads as W  # noqa: E402
from paper_2109_07073_b200 import optimizer as LM  # noqa: E402


def pose_diff(A, B):
    dt = np.abs(A[:, 9:] - B[:, 9:]).max()
    dr = 0.0
    for a, b in zip(A, B):
        R = a[:9].reshape(3, 3).T @ b[:9].reshape(3, 3)
        dr = max(dr, np.arccos(np.clip((np.trace(R) - 1) / 2, -1, 1)))
    return dt, dr


ctx = V.default_context(0)
threads = os.cpu_count() or 1
cases = {"C2": (W.c2_spec(), W.c2_links(100)), "C3-60": (W.c3_spec(frames=60), None)}
for name, (spec, links) in cases.items():
    wl = W.build_graph_workload(ctx, spec, links=links, threads=threads)
    og = _OracleGraph(wl, threads)
    for tol in (1e-6, 1e-10):
        st = LM.LmSettings(relative_error_decrease=tol, max_iterations=50)
        t = time.perf_counter()
        pg, rg = LM.optimize_native(wl.graph, wl.poses, settings=st)
        tg = time.perf_counter() - t
        t = time.perf_counter()
        po, ro = LM.optimize(og, wl.poses, settings=st, device_assembly=False, gpu_solve=False)
        to = time.perf_counter() - t
        dt, dr = pose_diff(pg, po)
        print(f"{name} F={wl.num_factors} tol={tol:g}: gpu its={rg.iterations} err={rg.final_error:.6f} ({rg.reason}, {tg:.2f}s) | "
              f"oracle its={ro.iterations} err={ro.final_error:.6f} ({ro.reason}, {to:.2f}s) | rel err diff "
              f"{abs(rg.final_error - ro.final_error) / ro.final_error:.3e} | max dt {dt:.3e} m, max dr {dr:.3e} rad", flush=True)
        print("   gpu trace", [(round(t.error, 3), t.accepted) for t in rg.trace][:12])
        print("   ora trace", [(round(t.error, 3), t.accepted) for t in ro.trace][:12])
