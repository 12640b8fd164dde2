"""ctypes loader for the product library lib/libvgicp_b200.so (C ABI: include/vgicp_b200.h).

There is no CPU fallback: if the CUDA library is missing, or no sm_100 device is visible when a
context is created, the calls raise.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
import os as _os

LIB_PATH = Path(_os.environ["VGICP_LIB"]) if _os.environ.get("VGICP_LIB") else PKG / "lib" / "libvgicp_b200.so"
HEADER = PKG.parent / "include" / "vgicp_b200.h"

LINEARIZED_DOUBLES = 121
KEY_MISS = (1 << 64) - 1

OK = 0
E_INVALID_ARGUMENT = 1
E_OUT_OF_RANGE = 2
E_CUDA = 3
E_NO_DEVICE = 4
E_OUT_OF_MEMORY = 5


class VgicpError(RuntimeError):
    """A CUDA / device failure inside the library."""


class NoDeviceError(VgicpError):
    pass


class LmSettingsC(C.Structure):  # vgicp_lm_settings
    _fields_ = [("max_iterations", C.c_int), ("lambda_init", C.c_double), ("lambda_increase", C.c_double),
                ("lambda_decrease", C.c_double), ("lambda_max", C.c_double),
                ("relative_error_decrease", C.c_double), ("step_norm_tolerance", C.c_double)]


class LmReportC(C.Structure):  # vgicp_lm_report
    _fields_ = [("iterations", C.c_int), ("initial_error", C.c_double), ("final_error", C.c_double),
                ("reason", C.c_int), ("aborted", C.c_int), ("wall_time_seconds", C.c_double),
                ("trace_length", C.c_int), ("iteration_count_timed", C.c_int), ("solves", C.c_int),
                ("linearizations", C.c_int), ("band_solver", C.c_int)]


LM_REASONS = ["converged_relative_error", "converged_step_norm", "max_iterations", "lambda_limit", "solver_abort"]


class FactorDesc(C.Structure):
    _fields_ = [
        ("target_index", C.c_int32),
        ("source_index", C.c_int32),
        ("source", C.c_void_p),
        ("target", C.c_void_p),
    ]


_vp = C.c_void_p
_sz = C.c_size_t
_d = C.c_double
_i = C.c_int
_PD = C.POINTER(C.c_double)

# name -> (restype, argtypes); every entry point declared in include/vgicp_b200.h
SIGNATURES = {
    "vgicp_last_error": (C.c_char_p, []),
    "vgicp_version": (C.c_char_p, []),
    "vgicp_device_count": (_i, [C.POINTER(_i)]),
    "vgicp_ctx_create": (_i, [_i, _vp, C.POINTER(_vp)]),
    "vgicp_ctx_destroy": (_i, [_vp]),
    "vgicp_ctx_stream": (_i, [_vp, C.POINTER(_vp)]),
    "vgicp_ctx_synchronize": (_i, [_vp]),
    "vgicp_ctx_launch_count": (_i, [_vp, C.POINTER(C.c_uint64)]),
    "vgicp_cloud_upload": (_i, [_vp, _vp, _vp, _sz, C.POINTER(_vp)]),
    "vgicp_cloud_upload_f64": (_i, [_vp, _vp, _vp, _sz, C.POINTER(_vp)]),
    "vgicp_cloud_upload_batch": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "vgicp_cloud_replicate": (_i, [_vp, _vp, C.POINTER(_vp)]),
    "vgicp_voxelmap_replicate": (_i, [_vp, _vp, C.POINTER(_vp)]),
    "vgicp_ctx_create_multi": (_i, [_vp, _i, _vp]),
    "vgicp_cloud_is_f64": (_i, [_vp, C.POINTER(_i)]),
    "vgicp_cloud_size": (_i, [_vp, C.POINTER(_sz)]),
    "vgicp_cloud_has_covariances": (_i, [_vp, C.POINTER(_i)]),
    "vgicp_cloud_destroy": (_i, [_vp]),
    "vgicp_voxelmap_build": (_i, [_vp, _vp, _d, C.POINTER(_vp)]),
    "vgicp_voxelmap_build_batch": (_i, [_vp, _vp, _vp, _i, _vp]),
    "vgicp_voxelmap_destroy": (_i, [_vp]),
    "vgicp_voxelmap_size": (_i, [_vp, C.POINTER(_sz)]),
    "vgicp_voxelmap_resolution": (_i, [_vp, _PD]),
    "vgicp_voxelmap_total_points": (_i, [_vp, C.POINTER(_sz)]),
    "vgicp_voxelmap_export": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "vgicp_voxelmap_lookup": (_i, [_vp, _vp, _sz, _vp]),
    "vgicp_voxel_key": (_i, [_d, _vp, C.POINTER(C.c_uint64)]),
    "vgicp_overlap_rate": (_i, [_vp, _vp, _vp, _vp, _PD]),
    "vgicp_overlap_batch": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "vgicp_linearize_matching_cost": (_i, [_vp, C.POINTER(FactorDesc), _vp, _vp, _vp, C.POINTER(C.c_int32)]),
    "vgicp_evaluate_matching_cost": (_i, [_vp, C.POINTER(FactorDesc), _vp, _vp, _PD, C.POINTER(C.c_int32)]),
    "vgicp_gicp_error": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _PD, _vp, _vp, C.POINTER(_i)]),
    "vgicp_graph_create": (_i, [_vp, _vp, _i, _i, _i, C.POINTER(_vp)]),
    "vgicp_graph_destroy": (_i, [_vp]),
    "vgicp_graph_create_range": (_i, [_vp, _vp, _i, _i, _i, _i, _i, C.POINTER(_vp)]),
    "vgicp_graph_create_sharded": (_i, [_vp, _i, _vp, _i, _i, _i, C.POINTER(_vp)]),
    "vgicp_graph_num_shards": (_i, [_vp, C.POINTER(_i)]),
    "vgicp_graph_shard_range": (_i, [_vp, _i, C.POINTER(_i), C.POINTER(_i)]),
    "vgicp_graph_assemble_device": (_i, [_vp, _vp, _vp]),
    "vgicp_graph_num_factors": (_i, [_vp, C.POINTER(_i)]),
    "vgicp_graph_num_points": (_i, [_vp, C.POINTER(C.c_uint64)]),
    "vgicp_graph_linearize": (_i, [_vp, _vp, _vp, _vp]),
    "vgicp_graph_evaluate": (_i, [_vp, _vp, _vp, _vp]),
    "vgicp_graph_linearize_device": (_i, [_vp, _vp, _vp, _vp]),
    "vgicp_graph_evaluate_device": (_i, [_vp, _vp, _vp, _vp]),
    "vgicp_estimate_covariances": (_i, [_vp, _vp, _sz, _i, _d, _vp]),
    "vgicp_voxelmap_build_f64": (_i, [_vp, _vp, _vp, _sz, _d, _vp]),
    "vgicp_graph_assembly_plan": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "vgicp_graph_linearize_assembled": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "vgicp_graph_linearize_assembled_device": (_i, [_vp, _vp, _vp]),
    "vgicp_graph_linearized_errors": (_i, [_vp, _vp, _vp]),
    "vgicp_graph_solver_plan": (_i, [_vp, _vp, _vp]),
    "vgicp_graph_solve_damped": (_i, [_vp, _vp, C.c_double, _vp, _vp]),
    "vgicp_graph_solve_damped_pair": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "vgicp_graph_optimize": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int, _vp]),
    "vgicp_mapset_create": (_i, [_vp, _vp, C.c_int, _vp]),
    "vgicp_mapset_destroy": (_i, [_vp]),
    "vgicp_mapset_append": (_i, [_vp, _vp, C.c_int]),
    "vgicp_mapset_size": (_i, [_vp, _vp]),
    "vgicp_overlap_mapset": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "vgicp_transform_cloud": (_i, [_vp, _vp, _vp, _sz, _vp, _vp, _vp]),
    "vgicp_submap_build": (_i, [_vp, _vp, _vp, _i, _d, _d, _vp, _vp, _vp]),
    "vgicp_estimate_covariances_batch": (_i, [_vp, _vp, _vp, _i, _i, _d, _vp]),
}

_LIB = None


def load() -> C.CDLL:
    """Load the in-tree CUDA library (built by __graft_entry__.build()); raise if absent."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(vgicp_b200 has no CPU fallback)"
            )
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def last_error() -> str:
    return load().vgicp_last_error().decode()


def check(rc: int) -> None:
    """Map a vgicp_status onto the exception the reference would raise."""
    if rc == OK:
        return
    msg = last_error()
    if rc == E_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc == E_OUT_OF_RANGE:
        raise IndexError(msg)  # std::out_of_range
    if rc == E_NO_DEVICE:
        raise NoDeviceError(msg)
    if rc == E_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise VgicpError(msg)
