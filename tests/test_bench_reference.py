"""The --impl reference bench arm (CPU, no GPU): runs the oracle port on a small C3-shaped graph
through bench.py, prints the contract's JSON line, and maps no product library — only oracle/."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_small_graph():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--frames", "12", "--points",
                        "3000", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "factors/s"
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["factors"] > 0
    libs = line["native_libraries"]
    assert libs and all(x.startswith("oracle/") for x in libs), libs
