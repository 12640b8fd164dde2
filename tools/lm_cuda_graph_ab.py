"""Native LM per-iteration wall time with and without CUDA-graph replay of the candidate
linearization (VGICP_LM_CUDA_GRAPH=1 vs the default per-call path), on C2, C3 and C5."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2109_07073_b200 as V  # noqa: E402
from bench_workloads import workloads as W  # noqa: E402
from paper_2109_07073_b200 import optimizer as LM  # noqa: E402

ctx = V.default_context(0)
cases = [("C2", lambda: W.build_graph_workload(ctx, W.c2_spec(), links=W.c2_links(100))),
         ("C3", lambda: W.build_graph_workload(ctx, W.c3_spec())), ("C5", lambda: W.build_c5_workload(ctx))]
for name, mk in cases:
    wl = mk()
    st = LM.LmSettings(max_iterations=30 if name != "C5" else 10)
    for mode in ("graph", "plain", "graph", "plain"):
        if mode == "graph":
            os.environ["VGICP_LM_CUDA_GRAPH"] = "1"
        LM.optimize_native(wl.graph, wl.poses, settings=LM.LmSettings(max_iterations=2))
        _, r = LM.optimize_native(wl.graph, wl.poses, settings=st)
        os.environ.pop("VGICP_LM_CUDA_GRAPH", None)
        its = sorted(r.iteration_seconds)
        print(f"{name} {mode:5s}: its={r.iterations} total {1e3 * r.wall_time_seconds:.2f} ms, mean "
              f"{1e3 * sum(its) / len(its):.3f} ms, median {1e3 * its[len(its) // 2]:.3f} ms", flush=True)
    del wl
