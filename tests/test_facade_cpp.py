"""The header-only C++ façade (include/vgicp_b200.hpp) compiles against the C ABI and, on a GPU,
runs the reference-facing C++ API end to end (tests/cpp/test_facade.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tests" / "cpp" / "_build" / "test_facade"


def build():
    import os

    env = dict(os.environ)
    env.pop("CXX", None)
    env.pop("CC", None)
    subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")], check=True, env=env)


def test_facade_compiles():
    build()
    assert BIN.exists()


@pytest.mark.gpu
def test_facade_runs_on_gpu():
    build()
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade ok" in r.stdout
