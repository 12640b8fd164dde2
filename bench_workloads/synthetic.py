"""Benchmark input pipeline: seeded synthetic KITTI-shaped scans + covariance preprocessing.

Thin ctypes wrapper over oracle/_build/libvgicp_synth.so (oracle/synthetic.cpp), the oracle's
restatement of the reference's generate_synthetic_sequence (proj/src/synthetic.cpp:121-213) and
estimate_covariances (proj/src/point_cloud.cpp:44-83), SURVEY.md §8(c). Benchmark / test input
generation only, outside every timed region: the product package never imports it, and both bench
arms (ours and --impl reference) generate identical scans with it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from pathlib import Path

LIB_PATH = Path(__file__).resolve().parents[1] / "oracle" / "_build" / "libvgicp_synth.so"

SHAPES = {"line": 0, "circle": 1, "figure_eight": 2, "figure-eight": 2}


class _Spec(C.Structure):
    _fields_ = [
        ("shape", C.c_int),
        ("frames", C.c_int),
        ("radius", C.c_double),
        ("spacing", C.c_double),
        ("points_per_scan", C.c_int),
        ("max_range", C.c_double),
        ("noise_sigma", C.c_double),
        ("drift", C.c_double * 6),
        ("seed", C.c_uint64),
        ("box_count", C.c_int),
        ("sensor_height", C.c_double),
    ]


@dataclass
class SceneSpec:
    """SyntheticSceneSpec (include/vgicp/synthetic.hpp:20-33) with the §8(d) benchmark defaults."""

    shape: str = "circle"
    frames: int = 100
    radius: float = 50.0
    spacing: float = 2.0
    points_per_scan: int = 20000
    max_range: float = 80.0
    noise_sigma: float = 0.02
    drift: tuple = (0.0, 0.0, 0.0, 0.0, 0.0, 0.0)
    seed: int = 1
    box_count: int = 400
    sensor_height: float = 1.73


@dataclass
class Sequence:
    scans: list = field(default_factory=list)  # float32 n×3 local-frame points
    ground_truth: np.ndarray = None  # frames × 12
    odometry: np.ndarray = None  # frames × 12


_LIB = None


def _load():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle` (or __graft_entry__.build())")
        lib = C.CDLL(str(LIB_PATH))
        lib.vs_generate.restype = C.c_int
        lib.vs_generate.argtypes = [C.POINTER(_Spec), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.vs_estimate_covariances.restype = C.c_int
        lib.vs_estimate_covariances.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int]
        _LIB = lib
    return _LIB


def generate(spec: SceneSpec) -> Sequence:
    s = _Spec()
    s.shape = SHAPES[spec.shape]
    s.frames = spec.frames
    s.radius = spec.radius
    s.spacing = spec.spacing
    s.points_per_scan = spec.points_per_scan
    s.max_range = spec.max_range
    s.noise_sigma = spec.noise_sigma
    for k in range(6):
        s.drift[k] = spec.drift[k]
    s.seed = spec.seed
    s.box_count = spec.box_count
    s.sensor_height = spec.sensor_height
    pts = np.zeros((spec.frames, spec.points_per_scan, 3), np.float32)
    counts = np.zeros(spec.frames, np.int32)
    gt = np.zeros((spec.frames, 12))
    odom = np.zeros((spec.frames, 12))
    rc = _load().vs_generate(C.byref(s), pts.ctypes.data, counts.ctypes.data, gt.ctypes.data, odom.ctypes.data)
    if rc != 0:
        raise ValueError("invalid synthetic scene spec")
    return Sequence([np.ascontiguousarray(pts[k, : counts[k]]) for k in range(spec.frames)], gt, odom)


def estimate_covariances(points: np.ndarray, k: int = 10, plane_epsilon: float = 1e-3, threads: int = 0) -> np.ndarray:
    """Per-point plane-regularised covariances, n×6 float32 (xx xy xz yy yz zz)."""
    p = np.ascontiguousarray(points, dtype=np.float32)
    out = np.zeros((len(p), 6), np.float32)
    rc = _load().vs_estimate_covariances(p.ctypes.data, len(p), int(k), float(plane_epsilon), out.ctypes.data, int(threads or os.cpu_count() or 1))
    if rc != 0:
        raise ValueError("covariance estimation requires k >= 4 and more than k points")
    return out
