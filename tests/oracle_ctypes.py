"""ctypes binding of the CPU oracle (oracle/vgicp_oracle.h) — TEST INFRASTRUCTURE ONLY.

The oracle is the checker: tests call it on the same inputs as the GPU path and compare.
Nothing in paper_2109_07073_b200/ imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
LIB_PATH = ORACLE_DIR / "_build" / "libvgicp_oracle.so"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build_oracle() -> Path:
    if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < max(
        (ORACLE_DIR / f).stat().st_mtime for f in ("vgicp_oracle.cpp", "vgicp_oracle.h", "Makefile")
    ):
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)
    return LIB_PATH


def _load():
    lib = C.CDLL(str(build_oracle()))
    vp = C.c_void_p
    sz = C.c_size_t
    d = C.c_double
    i = C.c_int
    sig = {
        "or_last_error": (C.c_char_p, []),
        "or_voxelmap_build": (i, [_dp, _dp, sz, d, i, i, C.POINTER(vp)]),
        "or_voxelmap_build_serial": (i, [_dp, _dp, sz, d, C.POINTER(vp)]),
        "or_voxelmap_destroy": (None, [vp]),
        "or_voxelmap_size": (sz, [vp]),
        "or_voxelmap_total_points": (sz, [vp]),
        "or_voxelmap_export": (None, [vp, vp, vp, vp, vp]),
        "or_voxelmap_lookup": (None, [vp, _dp, sz, _u64p]),
        "or_voxel_key": (i, [d, _dp, C.POINTER(C.c_uint64)]),
        "or_overlap_rate": (i, [_dp, sz, _dp, vp, i, i, C.POINTER(d), C.POINTER(C.c_uint64)]),
        "or_overlap_rate_serial": (i, [_dp, sz, _dp, vp, C.POINTER(d)]),
        "or_linearize": (i, [_dp, _dp, sz, vp, _dp, _dp, i, i, _dp, C.POINTER(C.c_int32)]),
        "or_linearize_serial": (i, [_dp, _dp, sz, vp, _dp, _dp, _dp, C.POINTER(C.c_int32)]),
        "or_evaluate": (i, [_dp, _dp, sz, vp, _dp, _dp, i, i, C.POINTER(d), C.POINTER(C.c_int32)]),
        "or_gicp_error": (None, [_dp, _dp, _dp, _dp, _dp, C.POINTER(d), _dp, _dp, C.POINTER(i)]),
        "or_invert_covariance": (i, [_dp, _dp]),
        "or_frozen_cost": (d, [_dp, _dp, sz, vp, _dp, _dp, _dp, _dp]),
        "or_se3_exp": (None, [_dp, _dp]),
        "or_compose": (None, [_dp, _dp, _dp]),
        "or_inverse": (None, [_dp, _dp]),
        "or_retract": (None, [_dp, _dp, _dp]),
        "or_adjoint": (None, [_dp, _dp]),
        "or_rng_create": (vp, [C.c_uint64]),
        "or_rng_destroy": (None, [vp]),
        "or_rng_uniform": (d, [vp, d, d]),
        "or_rng_vector": (None, [vp, d, _dp]),
        "or_random_pose": (None, [vp, d, d, _dp]),
        "or_random_plane_covariance": (None, [vp, _dp]),
        "or_random_gaussian_cloud": (None, [vp, i, d, _dp, _dp]),
        "or_make_scene": (None, [vp, i, d, d, _dp, _dp, _dp, _dp, _dp, _dp]),
        "or_rng_shuffle": (None, [vp, _u64p, sz]),
        "or_estimate_covariances": (i, [_dp, sz, i, d, _dp]),
        "or_transform_cloud": (None, [_dp, vp, sz, _dp, _dp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = _load()
    return _LIB


class OracleError(Exception):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


class OracleOutOfRange(OracleError, IndexError):
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().or_last_error().decode()
    if rc == 1:
        raise OracleInvalidArgument(msg)
    if rc == 2:
        raise OracleOutOfRange(msg)
    raise OracleError(msg)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def cov9(covs) -> np.ndarray:
    """Accept n×3×3, n×9 or n×6 (xx,xy,xz,yy,yz,zz) covariances; return n×9."""
    c = np.asarray(covs, dtype=np.float64)
    if c.ndim == 3:
        return _f64(c.reshape(-1, 9))
    if c.shape[-1] == 9:
        return _f64(c)
    if c.shape[-1] == 6:
        xx, xy, xz, yy, yz, zz = (c[:, k] for k in range(6))
        return _f64(np.stack([xx, xy, xz, xy, yy, yz, xz, yz, zz], axis=1))
    raise ValueError("covariances must be n×3×3, n×9 or n×6")


class OracleMap:
    """GaussianVoxelMap restatement (voxelmap.cpp:65-135)."""

    def __init__(self, means, covs, resolution, threads=0, deterministic=False, serial=False):
        means = _f64(means, (-1, 3))
        covs9 = cov9(covs) if len(means) else np.zeros((0, 9))
        h = C.c_void_p()
        if serial:
            _check(lib().or_voxelmap_build_serial(means, covs9, len(means), float(resolution), C.byref(h)))
        else:
            _check(
                lib().or_voxelmap_build(
                    means, covs9, len(means), float(resolution), int(threads), int(deterministic), C.byref(h)
                )
            )
        self._h = h
        self.resolution = float(resolution)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_voxelmap_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def size(self) -> int:
        return int(lib().or_voxelmap_size(self._h))

    def total_points(self) -> int:
        return int(lib().or_voxelmap_total_points(self._h))

    def export(self):
        v = self.size()
        keys = np.zeros(v, np.uint64)
        counts = np.zeros(v, np.int32)
        means = np.zeros((v, 3))
        covs = np.zeros((v, 9))
        lib().or_voxelmap_export(
            self._h, keys.ctypes.data, counts.ctypes.data, means.ctypes.data, covs.ctypes.data
        )
        return keys, counts, means, covs.reshape(v, 3, 3)

    def lookup(self, points) -> np.ndarray:
        p = _f64(points, (-1, 3))
        out = np.zeros(len(p), np.uint64)
        lib().or_voxelmap_lookup(self._h, p, len(p), out)
        return out


def voxel_key(resolution, p) -> int:
    k = C.c_uint64()
    _check(lib().or_voxel_key(float(resolution), _f64(p, (3,)), C.byref(k)))
    return int(k.value)


def overlap_rate(means, pose12, omap: OracleMap, threads=0, deterministic=False, serial=False):
    m = _f64(means, (-1, 3))
    rate = C.c_double()
    if serial:
        _check(lib().or_overlap_rate_serial(m, len(m), _f64(pose12, (12,)), omap.handle, C.byref(rate)))
        return rate.value
    hits = C.c_uint64()
    _check(
        lib().or_overlap_rate(
            m, len(m), _f64(pose12, (12,)), omap.handle, int(threads), int(deterministic), C.byref(rate), C.byref(hits)
        )
    )
    return rate.value


def overlap_hits(means, pose12, omap: OracleMap, threads=0) -> int:
    m = _f64(means, (-1, 3))
    rate = C.c_double()
    hits = C.c_uint64()
    _check(lib().or_overlap_rate(m, len(m), _f64(pose12, (12,)), omap.handle, int(threads), 0, C.byref(rate), C.byref(hits)))
    return int(hits.value)


def unpack121(out: np.ndarray):
    return dict(
        H_ii=out[0:36].reshape(6, 6),
        H_ij=out[36:72].reshape(6, 6),
        H_jj=out[72:108].reshape(6, 6),
        b_i=out[108:114],
        b_j=out[114:120],
        error=float(out[120]),
    )


def linearize(src_means, src_covs, omap: OracleMap, T_target, T_source, threads=0, deterministic=False, serial=False):
    m = _f64(src_means, (-1, 3))
    c = cov9(src_covs)
    out = np.zeros(121)
    inl = C.c_int32()
    if serial:
        _check(lib().or_linearize_serial(m, c, len(m), omap.handle, _f64(T_target, (12,)), _f64(T_source, (12,)), out, C.byref(inl)))
    else:
        _check(
            lib().or_linearize(
                m, c, len(m), omap.handle, _f64(T_target, (12,)), _f64(T_source, (12,)), int(threads), int(deterministic), out, C.byref(inl)
            )
        )
    r = unpack121(out)
    r["inliers"] = int(inl.value)
    r["raw"] = out
    return r


def evaluate(src_means, src_covs, omap: OracleMap, T_target, T_source, threads=0, deterministic=False):
    m = _f64(src_means, (-1, 3))
    c = cov9(src_covs)
    err = C.c_double()
    inl = C.c_int32()
    _check(
        lib().or_evaluate(
            m, c, len(m), omap.handle, _f64(T_target, (12,)), _f64(T_source, (12,)), int(threads), int(deterministic), C.byref(err), C.byref(inl)
        )
    )
    return err.value, int(inl.value)


def gicp_error(src_mean, src_cov, tgt_mean, tgt_cov, T):
    err = C.c_double()
    res = np.zeros(3)
    info = np.zeros(9)
    valid = C.c_int()
    lib().or_gicp_error(
        _f64(src_mean, (3,)), _f64(src_cov, (9,)), _f64(tgt_mean, (3,)), _f64(tgt_cov, (9,)), _f64(T, (12,)),
        C.byref(err), res, info, C.byref(valid),
    )
    return err.value, res, info.reshape(3, 3), bool(valid.value)


def invert_covariance(M):
    out = np.zeros(9)
    ok = lib().or_invert_covariance(_f64(M, (9,)), out)
    return bool(ok), out.reshape(3, 3)


def frozen_cost(src_means, src_covs, omap, lin_t, lin_s, T_t, T_s) -> float:
    m = _f64(src_means, (-1, 3))
    return float(
        lib().or_frozen_cost(m, cov9(src_covs), len(m), omap.handle, _f64(lin_t, (12,)), _f64(lin_s, (12,)), _f64(T_t, (12,)), _f64(T_s, (12,)))
    )


# --- SE3 helpers -------------------------------------------------------------------------------
IDENTITY = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], dtype=np.float64)


def se3_exp(twist) -> np.ndarray:
    out = np.zeros(12)
    lib().or_se3_exp(_f64(twist, (6,)), out)
    return out


def compose(a, b) -> np.ndarray:
    out = np.zeros(12)
    lib().or_compose(_f64(a, (12,)), _f64(b, (12,)), out)
    return out


def inverse(a) -> np.ndarray:
    out = np.zeros(12)
    lib().or_inverse(_f64(a, (12,)), out)
    return out


def retract(a, twist) -> np.ndarray:
    out = np.zeros(12)
    lib().or_retract(_f64(a, (12,)), _f64(twist, (6,)), out)
    return out


def adjoint(a) -> np.ndarray:
    out = np.zeros(36)
    lib().or_adjoint(_f64(a, (12,)), out)
    return out.reshape(6, 6)


def pose(R=None, t=(0.0, 0.0, 0.0)) -> np.ndarray:
    R = np.eye(3) if R is None else np.asarray(R, dtype=np.float64)
    return np.concatenate([R.reshape(9), np.asarray(t, dtype=np.float64)])


def apply_pose(T, p) -> np.ndarray:
    """Pose::apply with the oracle's stated op order ((R0*p0 + R1*p1) + R2*p2) + t (no FMA)."""
    T = np.asarray(T, dtype=np.float64)
    p = np.asarray(p, dtype=np.float64).reshape(-1, 3)
    R = T[:9].reshape(3, 3)
    out = np.empty_like(p)
    for i in range(3):
        out[:, i] = ((R[i, 0] * p[:, 0] + R[i, 1] * p[:, 1]) + R[i, 2] * p[:, 2]) + T[9 + i]
    return out


# --- Test RNG (oracles.hpp:151-168) ------------------------------------------------------------
class Rng:
    def __init__(self, seed: int):
        self._h = lib().or_rng_create(C.c_uint64(seed))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_rng_destroy(self._h)
            self._h = None

    def uniform(self, lo, hi) -> float:
        return float(lib().or_rng_uniform(self._h, float(lo), float(hi)))

    def vector(self, scale) -> np.ndarray:
        out = np.zeros(3)
        lib().or_rng_vector(self._h, float(scale), out)
        return out

    def random_pose(self, rot_scale, trans_scale) -> np.ndarray:
        out = np.zeros(12)
        lib().or_random_pose(self._h, float(rot_scale), float(trans_scale), out)
        return out

    def plane_covariance(self) -> np.ndarray:
        out = np.zeros(9)
        lib().or_random_plane_covariance(self._h, out)
        return out.reshape(3, 3)

    def gaussian_cloud(self, n, scale):
        means = np.zeros((n, 3))
        covs = np.zeros((n, 9))
        lib().or_random_gaussian_cloud(self._h, int(n), float(scale), means, covs)
        return means, covs.reshape(n, 3, 3)

    def make_scene(self, points, resolution, margin=1e-3):
        Tt = np.zeros(12)
        Ts = np.zeros(12)
        sm = np.zeros((points, 3))
        sc = np.zeros((points, 9))
        tm = np.zeros((points, 3))
        tc = np.zeros((points, 9))
        lib().or_make_scene(self._h, int(points), float(resolution), float(margin), Tt, Ts, sm, sc, tm, tc)
        return dict(T_target=Tt, T_source=Ts, source_means=sm, source_covs=sc.reshape(-1, 3, 3),
                    target_means=tm, target_covs=tc.reshape(-1, 3, 3))

    def shuffle(self, n) -> np.ndarray:
        perm = np.arange(n, dtype=np.uint64)
        lib().or_rng_shuffle(self._h, perm, n)
        return perm


# --- Brute-force oracles (oracles.hpp:37-82), hash-free -----------------------------------------
def bucket_coord(p, resolution) -> np.ndarray:
    p = np.asarray(p, dtype=np.float64).reshape(-1, 3)
    return np.floor(p / resolution).astype(np.int64)


def brute_force_buckets(points, resolution):
    """dict coord-tuple -> member indices, first-seen order (oracles.hpp:45-61)."""
    coords = bucket_coord(points, resolution)
    buckets: dict = {}
    for i, c in enumerate(map(tuple, coords)):
        buckets.setdefault(c, []).append(i)
    return buckets


def brute_force_overlap_count(cloud, rel, map_points, resolution) -> int:
    """Sorted-cell binary search membership (oracles.hpp:65-82)."""
    cells = np.unique(bucket_coord(map_points, resolution), axis=0)
    q = bucket_coord(apply_pose(rel, cloud), resolution)
    cells_v = cells.view([("x", np.int64), ("y", np.int64), ("z", np.int64)]).ravel()
    q_v = np.ascontiguousarray(q).view([("x", np.int64), ("y", np.int64), ("z", np.int64)]).ravel()
    idx = np.searchsorted(cells_v, q_v)
    idx = np.clip(idx, 0, len(cells_v) - 1)
    return int(np.sum(cells_v[idx] == q_v))


def estimate_covariances(means, k=10, plane_epsilon=1e-3) -> np.ndarray:
    """reference::estimate_covariances restatement (brute-force kNN); n×3×3."""
    m = _f64(means, (-1, 3))
    out = np.zeros((len(m), 9))
    _check(lib().or_estimate_covariances(m, len(m), int(k), float(plane_epsilon), out))
    return out.reshape(-1, 3, 3)


def transform_cloud(means, covs, pose12):
    """transform_cloud (point_cloud.cpp:26-42) restatement; returns (n×3, n×3×3 or None)."""
    m = _f64(means, (-1, 3))
    c = None if covs is None else cov9(covs)
    om = np.zeros_like(m)
    oc = None if c is None else np.zeros_like(c)
    lib().or_transform_cloud(m, None if c is None else c.ctypes.data, len(m), _f64(pose12, (12,)), om,
                             None if oc is None else oc.ctypes.data)
    return om, (None if oc is None else oc.reshape(-1, 3, 3))


def voxel_downsample(means, covs, resolution):
    """voxel_downsample (voxelmap.cpp:137-169) restatement: the voxel statistics of the (Kahan)
    GaussianVoxelMap in ascending packed-key order (intensities are not on this path)."""
    _, _, vm, vc = OracleMap(means, covs, resolution).export()
    return vm, vc


def submap(frames, poses12, downsample_resolution, map_resolution):
    """emit_submap's data path (pipeline.cpp:92-114): transform each frame into the submap frame,
    merge in frame order, voxel_downsample, build the submap's voxel map. frames: [(means, covs)]."""
    ms, cs = [], []
    for (m, c), T in zip(frames, poses12):
        tm, tc = transform_cloud(m, c, T)
        ms.append(tm)
        cs.append(tc)
    m = np.concatenate(ms)
    c = np.concatenate(cs)
    if downsample_resolution > 0:
        m, c = voxel_downsample(m, c, downsample_resolution)
    return m, c, OracleMap(m, c, map_resolution)


def assemble_normal_equations(blocks121, ij, fixed, num_variables):
    """assemble_normal_equations (block_solver.cpp:14-62), restated with the reference's loop order:
    slots in reverse insertion order of the active variables; for each factor in order
    block(si,si) += H_ii, rhs[si] += b_i, block(sj,sj) += H_jj, rhs[sj] += b_j, and the off-diagonal
    H_ij (or H_ijᵀ) into the lower-triangle block. Returns (slot_of_var, diag, {(a, b): block}, rhs)."""
    fixed = np.asarray(fixed, bool)
    active = int((~fixed).sum())
    slot_of = -np.ones(num_variables, int)
    rank = 0
    for v in range(num_variables):
        if not fixed[v]:
            slot_of[v] = active - 1 - rank
            rank += 1
    diag = np.zeros((active, 6, 6))
    rhs = np.zeros((active, 6))
    off = {}
    for f, (i, j) in enumerate(np.asarray(ij)):
        B = np.asarray(blocks121[f], np.float64)
        Hii, Hij, Hjj = B[0:36].reshape(6, 6), B[36:72].reshape(6, 6), B[72:108].reshape(6, 6)
        si, sj = slot_of[i], slot_of[j]
        if si >= 0:
            diag[si] += Hii
            rhs[si] += B[108:114]
        if sj >= 0:
            diag[sj] += Hjj
            rhs[sj] += B[114:120]
        if si >= 0 and sj >= 0:
            if si >= sj:
                off[(si, sj)] = off.get((si, sj), np.zeros((6, 6))) + Hij
            else:
                off[(sj, si)] = off.get((sj, si), np.zeros((6, 6))) + Hij.T
    return slot_of, diag, off, rhs


def unit_covariances(n) -> np.ndarray:
    return np.broadcast_to(np.eye(3), (n, 3, 3)).copy()


def to_f32_exact(a) -> np.ndarray:
    """Round to float32 and back: the GPU input contract (KITTI .bin precision, io.cpp:50)."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def num_threads_env() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", "0") or 0)
