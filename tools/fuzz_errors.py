"""Distribution of the float32-algebra block errors over the randomised parity sweep
(tests/test_gpu_fuzz.py scenes; needs a GPU): per category (float32 / float64 clouds x regular /
degenerate covariances) the median, p99 and max of max(H, b blocks) and of the error term, plus the
worst seeds. Usage: python tools/fuzz_errors.py [num_seeds]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import test_gpu_fuzz as F  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    rows = []
    for seed in range(n):
        kinds, f64, degenerate, d = F.run_case(seed)
        rows.append((seed, kinds, f64, degenerate, max(v for k, v in d.items() if k != "error"), d["error"]))
    print(f"{n} seeds; exact parts (map export, inliers, overlap hits) equal the oracle on all of them")
    for f64 in (False, True):
        for deg in (False, True):
            sel = [r for r in rows if r[2] == f64 and r[3] == deg]
            if not sel:
                continue
            h = np.array([r[4] for r in sel])
            e = np.array([r[5] for r in sel])
            name = f"{'float64' if f64 else 'float32'} clouds, {'degenerate' if deg else 'regular'} covariances"
            print(f"{name:48s} n={len(sel):4d}  blocks median {np.median(h):.2e} p99 {np.quantile(h, .99):.2e} "
                  f"max {h.max():.2e} | error median {np.median(e):.2e} p99 {np.quantile(e, .99):.2e} max {e.max():.2e}")
    print("worst 10 seeds (blocks):")
    for r in sorted(rows, key=lambda r: -r[4])[:10]:
        print(f"  seed {r[0]:5d} {r[1]} f64={r[2]} blocks {r[4]:.2e} error {r[5]:.2e}")


if __name__ == "__main__":
    main()
