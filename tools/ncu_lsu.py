"""Per-source-line LSU attribution (shared wavefronts, excess from bank conflicts, global L1 tag
requests) of a kernel in an .ncu-rep."""
import csv, subprocess, sys
from collections import defaultdict

rep, kernel = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "factor_kernel")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{kernel}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
src = {}
idx = None
cur_file = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        idx = (r.index("L1 Wavefronts Shared"), r.index("L1 Wavefronts Shared Excessive"), r.index("L1 Tag Requests Global"))
        continue
    if r[0] != "":
        cur = (cur_file, r[0])
        src[cur] = r[1]
        continue
    if idx is None:
        continue
    for k, i in enumerate(idx):
        try:
            agg[cur][k] += float(r[i] or 0)
        except (ValueError, IndexError):
            pass
tot = [sum(v[k] for v in agg.values()) for k in range(3)]
print(f"shared wavefronts {tot[0]:.3e}  excessive {tot[1]:.3e}  global tag requests {tot[2]:.3e}")
for key, v in sorted(agg.items(), key=lambda kv: -(kv[1][0] + kv[1][2]))[:25]:
    print(f"{v[0]:10.3e} {v[1]:10.3e} {v[2]:10.3e}  {key[0]}:{key[1]} {src[key].strip()[:90]}")
