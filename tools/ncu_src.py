"""Summarise an ncu report's source page (CUDA lines with SASS metrics) by stall samples."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kernel = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "factor_kernel")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{kernel}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = cur_line = None
stall = defaultdict(float); inst = defaultdict(float); src = {}
wi = ii = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        wi = r.index("Warp Stall Sampling (All Samples)"); ii = r.index("Instructions Executed"); continue
    if r[0] != "":
        cur_line = (cur_file, r[0]); src[cur_line] = r[1]; continue
    try:
        stall[cur_line] += float(r[wi] or 0); inst[cur_line] += float(r[ii] or 0)
    except (ValueError, TypeError, IndexError):
        pass
ts = sum(stall.values()) or 1; ti = sum(inst.values()) or 1
print(f"samples {ts:.0f} warp-inst {ti:.3e}")
for k in sorted(stall, key=lambda k: -stall[k])[:top]:
    print(f"{100*stall[k]/ts:5.1f}% st {100*inst[k]/ti:5.1f}% in {k[0]}:{k[1]:>4} {src[k].strip()[:100]}")
