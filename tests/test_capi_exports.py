"""CPU-only checks of the C-ABI boundary: the library loads, exports every symbol that
include/vgicp_b200.h declares (and the Python binding declares no extra), and fails loudly
instead of falling back when no device is usable."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "vgicp_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vgicp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_api():
    syms = declared_symbols()
    for must in ("vgicp_voxelmap_build", "vgicp_overlap_rate", "vgicp_linearize_matching_cost",
                 "vgicp_evaluate_matching_cost", "vgicp_gicp_error", "vgicp_graph_linearize"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2109_07073_b200 import _lib

    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_no_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2109_07073_b200 as V

    with pytest.raises(V.NoDeviceError):
        V.Context(0)


def test_host_voxel_key_matches_oracle():
    import numpy as np

    import oracle_ctypes as O
    from paper_2109_07073_b200 import GaussianVoxelMap

    rng = np.random.default_rng(3)
    for _ in range(500):
        p = rng.normal(0, 50, 3)
        r = float(rng.uniform(0.1, 3))
        assert GaussianVoxelMap.pack_key(r, p) == O.voxel_key(r, p)
    with pytest.raises(IndexError):
        GaussianVoxelMap.pack_key(1.0, [2.0e6, 0, 0])


def test_package_has_no_oracle_dependency():
    """The product path never imports, includes or links the checker (oracle/) or the benchmark
    input generator that lives beside it (bench_workloads/, oracle/synthetic.cpp)."""
    pkg = ROOT / "paper_2109_07073_b200"
    bad = re.compile(r"(import\s+oracle|oracle_ctypes|vgicp_oracle|liboracle|oracle/_build|bench_workloads|libvgicp_synth|#include\s+[<\"].*oracle)")
    for f in [*pkg.rglob("*.py"), *pkg.rglob("*.cu"), *pkg.rglob("*.cuh"), *pkg.rglob("*.h"), *pkg.rglob("Makefile")]:
        assert not bad.search(f.read_text()), f
