"""Per-phase wall-clock profile of the speculative C3 LM (diagnostic): monkeypatches the pieces
optimize() calls and accumulates their time."""
import sys
import time
from collections import defaultdict

import numpy as np

sys.path.insert(0, ".")
import paper_2109_07073_b200 as V  # noqa: E402
from paper_2109_07073_b200 import optimizer as LM  # noqa: E402
from bench_workloads import workloads as W  # noqa: E402

ctx = V.default_context()
wl = W.build_graph_workload(ctx, W.c3_spec())
acc = defaultdict(float)
cnt = defaultdict(int)


def wrap(obj, name, label):
    fn = getattr(obj, name)

    def inner(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        acc[label] += time.perf_counter() - t0
        cnt[label] += 1
        return r

    setattr(obj, name, inner)


g = wl.graph
wrap(g, "linearize_assembled_device", "linearize+assemble (enqueue)")
wrap(g.ctx, "synchronize", "ctx.synchronize (kernel wait)")
wrap(g, "linearized_errors", "linearized_errors D2H")
wrap(LM._ReducedSolver, "solve", "solve")
wrap(LM, "compose_batch", "retract compose")
wrap(LM, "se3_exp_batch", "retract exp")
orig_init = LM._ReducedSolver.__init__


def init(self, *a, **k):
    t0 = time.perf_counter()
    orig_init(self, *a, **k)
    acc["solver init (dense scatter)"] += time.perf_counter() - t0
    cnt["solver init (dense scatter)"] += 1


LM._ReducedSolver.__init__ = init
LM.optimize(g, wl.poses, settings=LM.LmSettings(max_iterations=2))
acc.clear()
cnt.clear()
t0 = time.perf_counter()
_, rep = LM.optimize(g, wl.poses)
total = time.perf_counter() - t0
print(f"iterations {rep.iterations}, total {1e3 * total:.2f} ms, per iteration {1e3 * total / max(1, rep.iterations):.3f} ms")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:34s} {1e3 * v / max(1, rep.iterations):7.3f} ms/it  ({cnt[k]} calls)")
print(f"  {'other (python)':34s} {1e3 * (total - sum(acc.values())) / max(1, rep.iterations):7.3f} ms/it")
