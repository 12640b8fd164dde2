"""Python mirror of the reference's VGICP operator API over the C ABI (include/vgicp_b200.h).

Names, argument meaning and error behaviour follow /root/reference/proj:
  GaussianVoxelMap            include/vgicp/voxelmap.hpp:28-56   (ValueError ~ std::invalid_argument,
  overlap_rate                include/vgicp/voxelmap.hpp:60-61    IndexError ~ std::out_of_range)
  MatchingCostFactor          include/vgicp/factors.hpp:36-45
  LinearizedFactor            include/vgicp/factors.hpp:19-29
  linearize_matching_cost     include/vgicp/factors.hpp:76-77
  evaluate_matching_cost      include/vgicp/factors.hpp:80-81
  gicp_error                  include/vgicp/factors.hpp:62-70
Batch entry points (FactorGraph.linearize / .evaluate, overlap_rates) issue one launch for all
factors / probes — the integration point of linearize_all / total_error (optimizer.cpp:45-75).

All compute runs in the sm_100a kernels of lib/libvgicp_b200.so; this module only marshals.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from ._lib import FactorDesc, check

__all__ = [
    "Context",
    "default_context",
    "PointCloud",
    "GaussianVoxelMap",
    "overlap_rate",
    "overlap_rates",
    "overlap_hits",
    "MapSet",
    "MatchingCostFactor",
    "LinearizedFactor",
    "GicpErrorResult",
    "linearize_matching_cost",
    "evaluate_matching_cost",
    "gicp_error",
    "FactorGraph",
    "AssemblyPlan",
    "as_pose12",
    "cov6_from",
    "estimate_covariances",
    "estimate_covariances_batch",
    "transform_cloud",
    "voxel_downsample",
    "build_submap",
    "Submap",
]


# ------------------------------------------------------------------------------------ helpers
def as_pose12(T) -> np.ndarray:
    """Pose as 12 doubles (row-major R, then t). Accepts 12-vectors, 4×4 / 3×4 matrices, (R, t)."""
    if isinstance(T, tuple) and len(T) == 2:
        R, t = T
        return np.ascontiguousarray(np.concatenate([np.asarray(R, np.float64).reshape(9), np.asarray(t, np.float64).reshape(3)]))
    a = np.asarray(T, dtype=np.float64)
    if a.shape == (12,):
        return np.ascontiguousarray(a)
    if a.shape in ((4, 4), (3, 4)):
        return np.ascontiguousarray(np.concatenate([a[:3, :3].reshape(9), a[:3, 3]]))
    raise ValueError(f"cannot interpret pose of shape {a.shape}")


def poses_array(poses) -> np.ndarray:
    a = np.asarray(poses, dtype=np.float64)
    if a.ndim == 2 and a.shape[1] == 12:
        return np.ascontiguousarray(a)
    return np.ascontiguousarray(np.stack([as_pose12(p) for p in poses]))


def cov6_from(covs) -> np.ndarray:
    """Six unique entries (xx, xy, xz, yy, yz, zz) as float32 from n×3×3, n×9 or n×6."""
    c = np.asarray(covs)
    if c.ndim == 3:
        c = c.reshape(len(c), 9)
    if c.shape[-1] == 9:
        c = c[:, [0, 1, 2, 4, 5, 8]]
    elif c.shape[-1] != 6:
        raise ValueError("covariances must be n×3×3, n×9 or n×6")
    return np.ascontiguousarray(c, dtype=np.float32)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------------------------ context
class Context:
    """One CUDA device + stream (vgicp_ctx). Not reentrant, like the reference optimizer."""

    def __init__(self, device: int = 0, stream: int | None = None):
        lib = _lib.load()
        h = C.c_void_p()
        check(lib.vgicp_ctx_create(int(device), C.c_void_p(stream) if stream else None, C.byref(h)))
        self._h = h
        self.device = int(device)

    @property
    def handle(self):
        return self._h

    def stream(self) -> int:
        s = C.c_void_p()
        check(_lib.load().vgicp_ctx_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def synchronize(self) -> None:
        check(_lib.load().vgicp_ctx_synchronize(self._h))

    def launch_count(self) -> int:
        n = C.c_uint64()
        check(_lib.load().vgicp_ctx_launch_count(self._h, C.byref(n)))
        return int(n.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().vgicp_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_DEFAULT: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _DEFAULT:
        _DEFAULT[device] = Context(device)
    return _DEFAULT[device]


class _Handle:
    _destroy = ""

    def __init__(self, ctx: Context, h: C.c_void_p):
        self.ctx = ctx
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            getattr(_lib.load(), self._destroy)(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------------------------ clouds
class PointCloud(_Handle):
    """Device-resident PointCloud (point_cloud.hpp:21-37).

    float32 means + the 6 unique float32 covariance entries (KITTI precision, io.cpp:50). Means or
    covariances given as float64 values that are not float32-exact (submap clouds: transform_cloud +
    voxel_downsample output, pipeline.cpp:100-111) make a float64 cloud (vgicp_cloud_upload_f64): its
    exact values drive every key, correspondence, overlap hit and map statistic, as in the reference.
    """

    _destroy = "vgicp_cloud_destroy"

    def __init__(self, means, covariances=None, ctx: Context | None = None):
        ctx = ctx or default_context()
        m64 = np.asarray(means)
        m64 = m64.reshape(-1, 3) if m64.size else m64.reshape(0, 3)
        c64 = None if covariances is None else np.asarray(covariances)
        if c64 is not None and (c64.ndim == 0 or c64.shape[0] != len(m64)):
            raise ValueError("covariance count does not match point count")
        h = C.c_void_p()
        if self._needs_f64(m64, c64):
            mm = np.ascontiguousarray(m64, dtype=np.float64)
            cc = None
            if c64 is not None:
                cc = np.asarray(c64, np.float64)
                if cc.ndim == 3:
                    cc = cc.reshape(len(cc), 9)
                elif cc.shape[-1] == 6:  # unique entries -> full symmetric matrix
                    cc = cc[:, [0, 1, 2, 1, 3, 4, 2, 4, 5]]
                cc = np.ascontiguousarray(cc)
            check(_lib.load().vgicp_cloud_upload_f64(ctx.handle, _ptr(mm), _ptr(cc) if cc is not None else None,
                                                     len(mm), C.byref(h)))
            super().__init__(ctx, h)
            self.means, self.cov6 = mm, (None if cc is None else cov6_from(cc))
            return
        m = np.ascontiguousarray(m64, dtype=np.float32)
        c = None if c64 is None else cov6_from(c64)
        check(_lib.load().vgicp_cloud_upload(ctx.handle, _ptr(m), _ptr(c) if c is not None else None, len(m), C.byref(h)))
        super().__init__(ctx, h)
        self.means = m
        self.cov6 = c

    @staticmethod
    def _needs_f64(means: np.ndarray, covs) -> bool:
        """True when a float64 input does not survive the float32 round trip (or a 3×3 covariance is
        not exactly symmetric): such clouds keep their float64 values on the device."""
        def inexact(a):
            a = np.asarray(a)
            if a.dtype != np.float64 or a.size == 0:
                return False
            with np.errstate(over="ignore", invalid="ignore"):
                r = a.astype(np.float32).astype(np.float64)
            return not np.array_equal(r, a, equal_nan=True)
        if inexact(means):
            return True
        if covs is None:
            return False
        c = np.asarray(covs)
        if inexact(c):
            return True
        if c.dtype == np.float64 and c.size and (c.ndim == 3 or c.shape[-1] == 9):
            f = c.reshape(len(c), 9)
            return not (np.array_equal(f[:, 1], f[:, 3]) and np.array_equal(f[:, 2], f[:, 6])
                        and np.array_equal(f[:, 5], f[:, 7]))
        return False

    @classmethod
    def upload_batch(cls, means_list, covariances_list=None, ctx: Context | None = None) -> list["PointCloud"]:
        """Many float32 clouds in one vgicp_cloud_upload_batch call (one staged copy, one launch per
        layout stage for the batch); identical to PointCloud(m, c) per cloud. Clouds that need float64
        storage (see _needs_f64) are uploaded one by one."""
        ctx = ctx or default_context()
        covs = list(covariances_list) if covariances_list is not None else [None] * len(means_list)
        if len(covs) != len(means_list):
            raise ValueError("one covariance array per cloud")
        out: list = [None] * len(means_list)
        batch = []
        for k, (m, c) in enumerate(zip(means_list, covs)):
            m64 = np.asarray(m)
            m64 = m64.reshape(-1, 3) if m64.size else m64.reshape(0, 3)
            c64 = None if c is None else np.asarray(c)
            if c64 is not None and len(c64.reshape(len(c64), -1)) != len(m64):
                raise ValueError("covariance count does not match point count")
            if cls._needs_f64(m64, c64):
                out[k] = cls(m64, c64, ctx)
            else:
                batch.append((k, np.ascontiguousarray(m64, dtype=np.float32), None if c64 is None else cov6_from(c64)))
        if batch:
            nb = len(batch)
            xyz = (C.c_void_p * nb)(*[b[1].ctypes.data for b in batch])
            cv = (C.c_void_p * nb)(*[b[2].ctypes.data if b[2] is not None else None for b in batch])
            ns = (C.c_size_t * nb)(*[len(b[1]) for b in batch])
            hs = (C.c_void_p * nb)()
            check(_lib.load().vgicp_cloud_upload_batch(ctx.handle, xyz, cv, ns, nb, hs))
            for (k, m, c), h in zip(batch, hs):
                cloud = cls.__new__(cls)
                _Handle.__init__(cloud, ctx, C.c_void_p(h))
                cloud.means, cloud.cov6 = m, c
                out[k] = cloud
        return out

    def replicate(self, ctx: "Context") -> "PointCloud":
        """vgicp_cloud_replicate: this cloud's device layout copied to ctx's device (bit-identical)."""
        h = C.c_void_p()
        check(_lib.load().vgicp_cloud_replicate(self._h, ctx.handle, C.byref(h)))
        cloud = PointCloud.adopt(ctx, h)
        cloud.means, cloud.cov6 = self.means, self.cov6
        return cloud

    def is_f64(self) -> bool:
        v = C.c_int()
        check(_lib.load().vgicp_cloud_is_f64(self._h, C.byref(v)))
        return bool(v.value)

    @classmethod
    def adopt(cls, ctx: Context, handle: C.c_void_p) -> "PointCloud":
        """Wrap a device-only cloud handle returned by the C ABI (e.g. the submap cloud)."""
        cloud = cls.__new__(cls)
        _Handle.__init__(cloud, ctx, handle)
        cloud.means = None
        cloud.cov6 = None
        return cloud

    def size(self) -> int:
        if self.means is not None:
            return len(self.means)
        n = C.c_size_t()
        check(_lib.load().vgicp_cloud_size(self._h, C.byref(n)))
        return int(n.value)

    def __len__(self) -> int:
        return self.size()

    def empty(self) -> bool:
        return self.size() == 0

    def has_covariances(self) -> bool:
        h = C.c_int()
        check(_lib.load().vgicp_cloud_has_covariances(self._h, C.byref(h)))
        return bool(h.value) and self.size() > 0


def estimate_covariances(points, k: int = 10, plane_epsilon: float = 1e-3, ctx: Context | None = None) -> np.ndarray:
    """estimate_covariances (point_cloud.cpp:44-83) on the GPU -> n×6 float32 (xx xy xz yy yz zz)."""
    return estimate_covariances_batch([points], k, plane_epsilon, ctx)[0]


def estimate_covariances_batch(clouds, k: int = 10, plane_epsilon: float = 1e-3, ctx: Context | None = None) -> list:
    """Covariances of many clouds in one batched GPU pass."""
    ctx = ctx or default_context()
    pts = [np.ascontiguousarray(np.asarray(p, dtype=np.float32).reshape(-1, 3)) for p in clouds]
    outs = [np.empty((len(p), 6), np.float32) for p in pts]
    m = len(pts)
    if m == 0:
        return []
    xp = (C.c_void_p * m)(*[p.ctypes.data for p in pts])
    ns = (C.c_size_t * m)(*[len(p) for p in pts])
    op = (C.c_void_p * m)(*[o.ctypes.data for o in outs])
    check(_lib.load().vgicp_estimate_covariances_batch(ctx.handle, xp, ns, m, int(k), float(plane_epsilon), op))
    return outs


# ------------------------------------------------------------------------------------ submap path
def transform_cloud(means, covariances, pose, ctx: Context | None = None):
    """transform_cloud (point_cloud.cpp:26-42) in float64 on the GPU: (T·means, R·C·Rᵀ)."""
    ctx = ctx or default_context()
    m = np.ascontiguousarray(np.asarray(means, np.float64).reshape(-1, 3))
    c = None if covariances is None else np.ascontiguousarray(np.asarray(covariances, np.float64).reshape(-1, 9))
    om = np.zeros_like(m)
    oc = None if c is None else np.zeros_like(c)
    T = as_pose12(pose)
    check(_lib.load().vgicp_transform_cloud(ctx.handle, _ptr(m), _ptr(c) if c is not None else None, len(m), _ptr(T),
                                            _ptr(om), _ptr(oc) if oc is not None else None))
    return om, (None if oc is None else oc.reshape(-1, 3, 3))


def voxel_downsample(means, covariances, resolution: float, ctx: Context | None = None):
    """voxel_downsample (voxelmap.cpp:137-169): one (mean, covariance) per voxel in ascending packed
    key order — the float64 voxel statistics of the map built at `resolution`."""
    _, _, vm, vc = GaussianVoxelMap.from_arrays(means, covariances, resolution, ctx).export()
    return vm, vc


@dataclass
class Submap:
    cloud: "PointCloud | None"         # float32 device cloud of the (downsampled) merged points
    voxels: "GaussianVoxelMap"         # the submap's voxel map (global resolution)
    downsampled: "GaussianVoxelMap | None"  # export() = the float64 submap cloud


def build_submap(frames: Sequence[PointCloud], poses, downsample_resolution: float, map_resolution: float,
                 want_cloud: bool = True) -> Submap:
    """MappingPipeline::emit_submap's data path (pipeline.cpp:92-114) on the GPU: frames transformed
    into the submap frame by `poses` (frame -> submap), merged, voxel-downsampled and mapped."""
    if not frames:
        raise ValueError("submap requires at least one frame")
    ctx = frames[0].ctx
    m = len(frames)
    P = poses_array(poses)
    if len(P) != m:
        raise ValueError("one pose per frame")
    hs = (C.c_void_p * m)(*[f.handle for f in frames])
    ds, cl, mp = C.c_void_p(), C.c_void_p(), C.c_void_p()
    check(_lib.load().vgicp_submap_build(ctx.handle, hs, _ptr(P), m, float(downsample_resolution), float(map_resolution),
                                         C.byref(ds), C.byref(cl) if want_cloud else None, C.byref(mp)))
    cloud = PointCloud.adopt(ctx, cl) if want_cloud and cl.value else None
    downs = GaussianVoxelMap(None, downsample_resolution, _handle=ds, _ctx=ctx) if ds.value else None
    return Submap(cloud, GaussianVoxelMap(None, map_resolution, _handle=mp, _ctx=ctx), downs)


# ------------------------------------------------------------------------------------ voxel maps
class GaussianVoxelMap(_Handle):
    """GaussianVoxelMap(cloud, resolution) — voxelmap.cpp:65-104, built on the GPU."""

    _destroy = "vgicp_voxelmap_destroy"

    def __init__(self, cloud: PointCloud | None, resolution: float, _handle=None, _ctx: Context | None = None):
        if _handle is None:
            h = C.c_void_p()
            check(_lib.load().vgicp_voxelmap_build(cloud.ctx.handle, cloud.handle, float(resolution), C.byref(h)))
        else:
            h = _handle
        super().__init__(cloud.ctx if cloud is not None else _ctx, h)
        self.cloud = cloud  # keeps the source alive for callers that re-derive stats
        self._resolution = float(resolution)

    def replicate(self, ctx: "Context", cloud: "PointCloud | None" = None) -> "GaussianVoxelMap":
        """vgicp_voxelmap_replicate: the map copied to ctx's device (one transfer, bit-identical
        statistics) instead of a rebuild there."""
        h = C.c_void_p()
        check(_lib.load().vgicp_voxelmap_replicate(self._h, ctx.handle, C.byref(h)))
        return GaussianVoxelMap(None, self._resolution, _handle=h, _ctx=ctx)

    @staticmethod
    def from_arrays(means, covariances, resolution: float, ctx: Context | None = None) -> "GaussianVoxelMap":
        """GaussianVoxelMap over a float64 cloud in the reference layout (n×3 means, n×3×3 / n×9
        covariances, all 9 entries accumulated) — voxelmap.cpp:65-104."""
        ctx = ctx or default_context()
        m = np.ascontiguousarray(np.asarray(means, np.float64).reshape(-1, 3))
        c = None if covariances is None else np.ascontiguousarray(np.asarray(covariances, np.float64).reshape(-1, 9))
        if c is not None and len(c) != len(m):
            raise ValueError("covariance count does not match point count")
        h = C.c_void_p()
        check(_lib.load().vgicp_voxelmap_build_f64(ctx.handle, _ptr(m), _ptr(c) if c is not None else None, len(m),
                                                   float(resolution), C.byref(h)))
        return GaussianVoxelMap(None, resolution, _handle=h, _ctx=ctx)

    @staticmethod
    def build_batch(clouds: Sequence[PointCloud], resolutions) -> list["GaussianVoxelMap"]:
        """Build m maps in one batched pass (all-or-nothing)."""
        m = len(clouds)
        if m == 0:
            return []
        ctx = clouds[0].ctx
        res = np.ascontiguousarray(np.broadcast_to(np.asarray(resolutions, np.float64), (m,)))
        hs = (C.c_void_p * m)(*[c.handle for c in clouds])
        outs = (C.c_void_p * m)()
        check(_lib.load().vgicp_voxelmap_build_batch(ctx.handle, hs, _ptr(res), m, outs))
        return [GaussianVoxelMap(clouds[k], res[k], _handle=C.c_void_p(outs[k])) for k in range(m)]

    def resolution(self) -> float:
        return self._resolution

    def size(self) -> int:
        n = C.c_size_t()
        check(_lib.load().vgicp_voxelmap_size(self._h, C.byref(n)))
        return int(n.value)

    def __len__(self) -> int:
        return self.size()

    def total_points(self) -> int:
        n = C.c_size_t()
        check(_lib.load().vgicp_voxelmap_total_points(self._h, C.byref(n)))
        return int(n.value)

    def export(self):
        """voxels() in ascending key order: (keys u64[V], counts i32[V], means f64[V,3], covs f64[V,3,3])."""
        v = self.size()
        keys = np.zeros(v, np.uint64)
        counts = np.zeros(v, np.int32)
        means = np.zeros((v, 3))
        covs = np.zeros((v, 9))
        check(_lib.load().vgicp_voxelmap_export(self._h, _ptr(keys), _ptr(counts), _ptr(means), _ptr(covs)))
        return keys, counts, means, covs.reshape(v, 3, 3)

    def voxels(self) -> dict:
        keys, counts, means, covs = self.export()
        return {int(k): (means[i], covs[i], int(counts[i])) for i, k in enumerate(keys)}

    def lookup(self, points) -> np.ndarray:
        """Packed key of the voxel containing each point, or KEY_MISS (voxelmap.cpp:106-117)."""
        p = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
        out = np.zeros(len(p), np.uint64)
        check(_lib.load().vgicp_voxelmap_lookup(self._h, _ptr(p), len(p), _ptr(out)))
        return out

    def lookup_voxel(self, point):
        """GaussianVoxelMap::lookup (voxelmap.cpp:106-117) of one point: (mean, covariance, count)
        of the populated voxel containing it, or None (out-of-range and NaN points miss)."""
        key = int(self.lookup(point)[0])
        if key == _lib.KEY_MISS:
            return None
        keys, counts, means, covs = self._exported()
        i = int(np.searchsorted(keys, np.uint64(key)))
        return means[i], covs[i], int(counts[i])

    def _exported(self):
        if getattr(self, "_export_cache", None) is None:
            self._export_cache = self.export()  # immutable after construction (voxelmap.hpp:27)
        return self._export_cache

    def voxel_coord(self, point) -> tuple[int, int, int]:
        """voxel_coord (voxelmap.cpp:45-55): floor(p / r) per axis; IndexError beyond ±2^20."""
        k = GaussianVoxelMap.pack_key(self._resolution, point)
        return tuple(int(((k >> sh) & 0x1FFFFF) - (1 << 20)) for sh in (42, 21, 0))

    @staticmethod
    def pack_key(resolution: float, point) -> int:
        """voxel_coord + pack_key (voxelmap.cpp:45-63); IndexError beyond ±2^20 voxels."""
        p = np.ascontiguousarray(np.asarray(point, dtype=np.float64).reshape(3))
        k = C.c_uint64()
        check(_lib.load().vgicp_voxel_key(float(resolution), _ptr(p), C.byref(k)))
        return int(k.value)


def overlap_rate(cloud: PointCloud, pose_rel, voxelmap: GaussianVoxelMap) -> float:
    """Exact hits / N (voxelmap.cpp:119-135); ValueError on an empty cloud."""
    T = as_pose12(pose_rel)
    r = C.c_double()
    check(_lib.load().vgicp_overlap_rate(cloud.ctx.handle, cloud.handle, _ptr(T), voxelmap.handle, C.byref(r)))
    return r.value


class MapSet:
    """A fixed sequence of voxel maps with its handle array built once (e.g. the keyframe maps a new
    frame is swept against, pipeline.cpp:135-150): overlap_hits(cloud, poses, map_set) then skips
    the per-call marshalling of thousands of handles."""

    def __init__(self, maps, ctx: Context | None = None):
        self.maps = list(maps)
        self.handles = np.fromiter((x.handle.value for x in self.maps), dtype=np.uint64, count=len(self.maps))
        self.ctx = self.maps[0].ctx if self.maps else ctx
        self._h = None
        if self.ctx is not None:  # device-resident copy (vgicp_mapset): single-cloud sweeps build their items on the GPU
            h = C.c_void_p()
            check(_lib.load().vgicp_mapset_create(self.ctx.handle, _ptr(self.handles), len(self.maps), C.byref(h)))
            self._h = h

    def append(self, maps) -> "MapSet":
        """Add maps at the end (a new keyframe's map): vgicp_mapset_append, amortised O(1) per map."""
        new = [maps] if isinstance(maps, GaussianVoxelMap) else list(maps)
        if not new:
            return self
        if self._h is None:  # an empty set made without a context: adopt the first map's
            self.ctx = new[0].ctx
            h = C.c_void_p()
            check(_lib.load().vgicp_mapset_create(self.ctx.handle, None, 0, C.byref(h)))
            self._h = h
        handles = np.fromiter((x.handle.value for x in new), dtype=np.uint64, count=len(new))
        check(_lib.load().vgicp_mapset_append(self._h, _ptr(handles), len(new)))
        self.maps.extend(new)
        self.handles = np.concatenate([self.handles, handles])
        return self

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().vgicp_mapset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self) -> int:
        return len(self.maps)

    def __iter__(self):
        return iter(self.maps)


def overlap_hits(clouds, poses, maps) -> np.ndarray:
    """Exact hit counts of m (cloud, pose, map) probes in one launch. `maps` may be a MapSet."""
    map_set = maps if isinstance(maps, MapSet) else None
    maps = map_set.maps if map_set is not None else list(maps)
    m = len(maps)
    single_cloud = isinstance(clouds, PointCloud)
    if single_cloud:
        clouds = [clouds] * m
    clouds = list(clouds)
    if len(clouds) != m:
        raise ValueError("clouds and maps differ in length")
    P = poses_array(poses)
    if len(P) != m:
        raise ValueError("poses and maps differ in length")
    hits = np.zeros(m, np.uint64)
    if m == 0:
        return hits
    ctx = maps[0].ctx
    if map_set is not None and single_cloud and map_set._h is not None:
        check(_lib.load().vgicp_overlap_mapset(ctx.handle, clouds[0].handle, _ptr(P), map_set._h, _ptr(hits)))
        return hits
    # handle arrays as uint64 (pointer-sized) numpy arrays: cheap to build for thousands of maps
    if single_cloud:
        ch = np.full(m, clouds[0].handle.value, np.uint64)
    else:
        ch = np.fromiter((c.handle.value for c in clouds), dtype=np.uint64, count=m)
    mh = map_set.handles if map_set is not None else np.fromiter((x.handle.value for x in maps), dtype=np.uint64,
                                                                  count=m)
    check(_lib.load().vgicp_overlap_batch(ctx.handle, _ptr(ch), _ptr(P), _ptr(mh), m, _ptr(hits)))
    return hits


def overlap_rates(clouds, poses, maps) -> np.ndarray:
    maps = maps if isinstance(maps, MapSet) else list(maps)
    hits = overlap_hits(clouds, poses, maps)
    sizes = np.array([c.size() for c in ([clouds] * len(maps) if isinstance(clouds, PointCloud) else clouds)], np.float64)
    return hits.astype(np.float64) / sizes


# ------------------------------------------------------------------------------------ factors
@dataclass
class LinearizedFactor:
    """LinearizedFactor (factors.hpp:19-29); b = -ΣJᵀΩe, gradient = -2[b_i; b_j]."""

    i: int = -1
    j: int = -1
    H_ii: np.ndarray = field(default_factory=lambda: np.zeros((6, 6)))
    H_ij: np.ndarray = field(default_factory=lambda: np.zeros((6, 6)))
    H_jj: np.ndarray = field(default_factory=lambda: np.zeros((6, 6)))
    b_i: np.ndarray = field(default_factory=lambda: np.zeros(6))
    b_j: np.ndarray = field(default_factory=lambda: np.zeros(6))
    error: float = 0.0
    inliers: int = 0

    @staticmethod
    def from_raw(raw: np.ndarray, i: int, j: int, inliers: int) -> "LinearizedFactor":
        return LinearizedFactor(
            i=i, j=j, H_ii=raw[0:36].reshape(6, 6), H_ij=raw[36:72].reshape(6, 6), H_jj=raw[72:108].reshape(6, 6),
            b_i=raw[108:114], b_j=raw[114:120], error=float(raw[120]), inliers=int(inliers),
        )


class MatchingCostFactor:
    """MatchingCostFactor (factors.cpp:50-67): target owns the map, source supplies the points."""

    def __init__(self, target_index: int, source_index: int, source_points: PointCloud, target_voxels: GaussianVoxelMap):
        if target_index == source_index:
            raise ValueError("matching cost factor requires distinct variables")
        if source_points is None or source_points.empty():
            raise ValueError("matching cost factor requires a nonempty source cloud")
        if not source_points.has_covariances():
            raise ValueError("matching cost factor requires source covariances")
        if target_voxels is None or target_voxels.size() == 0:
            raise ValueError("matching cost factor requires a nonempty target voxel map")
        self.target_index = int(target_index)
        self.source_index = int(source_index)
        self.source_points = source_points
        self.target_voxels = target_voxels

    def desc(self) -> FactorDesc:
        return FactorDesc(self.target_index, self.source_index, self.source_points.handle, self.target_voxels.handle)


def linearize_matching_cost(factor: MatchingCostFactor, T_target, T_source) -> LinearizedFactor:
    out = np.zeros(_lib.LINEARIZED_DOUBLES)
    inl = C.c_int32()
    d = factor.desc()
    check(
        _lib.load().vgicp_linearize_matching_cost(
            factor.source_points.ctx.handle, C.byref(d), _ptr(as_pose12(T_target)), _ptr(as_pose12(T_source)), _ptr(out), C.byref(inl)
        )
    )
    return LinearizedFactor.from_raw(out, factor.target_index, factor.source_index, inl.value)


def evaluate_matching_cost(factor: MatchingCostFactor, T_target, T_source) -> tuple[float, int]:
    err = C.c_double()
    inl = C.c_int32()
    d = factor.desc()
    check(
        _lib.load().vgicp_evaluate_matching_cost(
            factor.source_points.ctx.handle, C.byref(d), _ptr(as_pose12(T_target)), _ptr(as_pose12(T_source)), C.byref(err), C.byref(inl)
        )
    )
    return err.value, int(inl.value)


@dataclass
class GicpErrorResult:
    """GicpErrorResult (factors.hpp:62-67)."""

    error: float
    residual: np.ndarray
    information: np.ndarray
    valid: bool


def gicp_error(source_mean, source_cov, target_mean, target_cov, T, ctx: Context | None = None) -> GicpErrorResult:
    ctx = ctx or default_context()
    f = lambda a, n: np.ascontiguousarray(np.asarray(a, np.float64).reshape(n))  # noqa: E731
    sm, sc, tm, tc = f(source_mean, 3), f(source_cov, 9), f(target_mean, 3), f(target_cov, 9)
    err = C.c_double()
    res = np.zeros(3)
    info = np.zeros(9)
    valid = C.c_int()
    check(
        _lib.load().vgicp_gicp_error(
            ctx.handle, _ptr(sm), _ptr(sc), _ptr(tm), _ptr(tc), _ptr(as_pose12(T)), C.byref(err), _ptr(res), _ptr(info), C.byref(valid)
        )
    )
    return GicpErrorResult(err.value, res, info.reshape(3, 3), bool(valid.value))


@dataclass
class AssemblyPlan:
    num_slots: int
    pairs: np.ndarray        # P×2 (row slot a, column slot b), a > b, ascending (b, a)
    var_of_slot: np.ndarray  # S variable indices


class FactorGraph(_Handle):
    """A fixed set of matching-cost factors linearized / evaluated in one launch per pass."""

    _destroy = "vgicp_graph_destroy"

    def __init__(self, factors: Iterable[MatchingCostFactor], num_poses: int, chunk: int = 0, ctx: Context | None = None):
        self.factors = list(factors)
        ctx = ctx or (self.factors[0].source_points.ctx if self.factors else default_context())
        n = len(self.factors)
        descs = (FactorDesc * max(n, 1))(*[f.desc() for f in self.factors])
        h = C.c_void_p()
        check(_lib.load().vgicp_graph_create(ctx.handle, descs, n, int(num_poses), int(chunk), C.byref(h)))
        super().__init__(ctx, h)
        self.num_poses = int(num_poses)
        self._ij = np.array([[f.target_index, f.source_index] for f in self.factors], np.int64).reshape(-1, 2)

    @classmethod
    def _adopt(cls, ctx: "Context", handle: C.c_void_p, factors, num_poses: int, keep=()) -> "FactorGraph":
        g = cls.__new__(cls)
        _Handle.__init__(g, ctx, handle)
        g.factors = list(factors)
        g.num_poses = int(num_poses)
        g._ij = np.array([[f.target_index, f.source_index] for f in g.factors], np.int64).reshape(-1, 2)
        g._keep = keep  # handles the C graph references (replicated clouds / maps of other shards)
        return g

    @classmethod
    def create_range(cls, factors: Sequence[MatchingCostFactor], num_poses: int, first: int, count: int,
                     chunk: int = 0, ctx: "Context | None" = None) -> "FactorGraph":
        """vgicp_graph_create_range: factors [first, first + count) of the list under the WHOLE list's
        work decomposition (per-factor blocks bit-identical to FactorGraph(factors)); one rank's share
        of a graph split across processes. Its blocks are indexed 0..count-1."""
        factors = list(factors)
        ctx = ctx or (factors[0].source_points.ctx if factors else default_context())
        descs = (FactorDesc * max(len(factors), 1))(*[f.desc() for f in factors])
        h = C.c_void_p()
        check(_lib.load().vgicp_graph_create_range(ctx.handle, descs, len(factors), int(num_poses), int(chunk),
                                                   int(first), int(count), C.byref(h)))
        return cls._adopt(ctx, h, factors[first:first + count], num_poses, keep=(factors,))

    @classmethod
    def sharded(cls, factor_lists: Sequence[Sequence[MatchingCostFactor]], num_poses: int,
                chunk: int = 0) -> "FactorGraph":
        """vgicp_graph_create_sharded: ONE graph split over several contexts (devices).
        factor_lists[r] holds the same factors with context r's handles (clouds / maps replicated);
        context 0 is the root. Every method works as on a single-context graph, with bit-identical
        results (the root's assembly reads the shards' blocks over peer memory)."""
        lists = [list(fl) for fl in factor_lists]
        if not lists or any(len(fl) != len(lists[0]) for fl in lists):
            raise ValueError("one factor list of equal length per shard")
        ctxs = [fl[0].source_points.ctx if fl else default_context() for fl in lists]
        n = len(lists[0])
        arrays = [(FactorDesc * max(n, 1))(*[f.desc() for f in fl]) for fl in lists]
        ptrs = (C.c_void_p * len(lists))(*[C.cast(a, C.c_void_p) for a in arrays])
        hs = (C.c_void_p * len(lists))(*[c.handle for c in ctxs])
        h = C.c_void_p()
        check(_lib.load().vgicp_graph_create_sharded(hs, len(lists), ptrs, n, int(num_poses), int(chunk), C.byref(h)))
        return cls._adopt(ctxs[0], h, lists[0], num_poses, keep=(lists, ctxs))

    @classmethod
    def sharded_replicas(cls, factors: Sequence[MatchingCostFactor], num_poses: int, contexts: Sequence["Context"],
                         chunk: int = 0) -> "FactorGraph":
        """The factors' clouds and maps replicated (vgicp_cloud_replicate / vgicp_voxelmap_replicate,
        each shared handle once) from contexts[0] onto the other contexts, then ONE sharded graph."""
        factors = list(factors)
        lists = [factors]
        for ctx in contexts[1:]:
            clouds, maps = {}, {}
            rep = []
            for f in factors:
                c, m = f.source_points, f.target_voxels
                if id(c) not in clouds:
                    clouds[id(c)] = c.replicate(ctx)
                if id(m) not in maps:
                    maps[id(m)] = m.replicate(ctx)
                rep.append(MatchingCostFactor(f.target_index, f.source_index, clouds[id(c)], maps[id(m)]))
            lists.append(rep)
        return cls.sharded(lists, num_poses, chunk=chunk)

    def num_shards(self) -> int:
        v = C.c_int()
        check(_lib.load().vgicp_graph_num_shards(self._h, C.byref(v)))
        return int(v.value)

    def shard_range(self, shard: int) -> tuple[int, int]:
        a, b = C.c_int(), C.c_int()
        check(_lib.load().vgicp_graph_shard_range(self._h, int(shard), C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def assemble_device(self, d_blocks: int, d_assembled: int) -> None:
        """vgicp_graph_assemble_device: assemble F×121 blocks given in device memory (factor order)."""
        check(_lib.load().vgicp_graph_assemble_device(self._h, C.c_void_p(d_blocks), C.c_void_p(d_assembled)))

    def num_factors(self) -> int:
        return len(self.factors)

    def num_points(self) -> int:
        n = C.c_uint64()
        check(_lib.load().vgicp_graph_num_points(self._h, C.byref(n)))
        return int(n.value)

    def linearize_raw(self, poses, out: np.ndarray | None = None, inliers: np.ndarray | None = None):
        """F×121 blocks + F inliers. `out` / `inliers` may be preallocated; page-locked buffers (e.g.
        from torch pin_memory) are written by the kernel's epilogue directly over PCIe (zero-copy:
        the result transfer overlaps the launch), others through a staging copy."""
        P = poses_array(poses)
        if len(P) != self.num_poses:
            raise ValueError("pose count does not match the graph")
        F = self.num_factors()
        if out is None:
            out = np.empty((F, _lib.LINEARIZED_DOUBLES))
        if inliers is None:
            inliers = np.empty(F, np.int32)
        if out.shape != (F, _lib.LINEARIZED_DOUBLES) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float64 F×121 array")
        if inliers.shape != (F,) or inliers.dtype != np.int32 or not inliers.flags.c_contiguous:
            raise ValueError("inliers must be a C-contiguous int32 array of length F")
        inl = inliers
        check(_lib.load().vgicp_graph_linearize(self._h, _ptr(P), _ptr(out), _ptr(inl)))
        return out, inl

    def linearize(self, poses) -> list[LinearizedFactor]:
        out, inl = self.linearize_raw(poses)
        return [LinearizedFactor.from_raw(out[k], int(self._ij[k, 0]), int(self._ij[k, 1]), inl[k]) for k in range(len(out))]

    def evaluate(self, poses) -> tuple[np.ndarray, np.ndarray]:
        P = poses_array(poses)
        if len(P) != self.num_poses:
            raise ValueError("pose count does not match the graph")
        err = np.zeros(self.num_factors())
        inl = np.zeros(self.num_factors(), np.int32)
        check(_lib.load().vgicp_graph_evaluate(self._h, _ptr(P), _ptr(err), _ptr(inl)))
        return err, inl

    def total_error(self, poses) -> float:
        """Σ factor errors in factor order (total_error, optimizer.cpp:66-75, matching part)."""
        err, _ = self.evaluate(poses)
        return float(np.cumsum(err)[-1]) if len(err) else 0.0  # sequential (not pairwise) summation

    # ---- device-side normal-equation assembly (block_solver.cpp:14-62) ----
    def assembly_plan(self, fixed) -> "AssemblyPlan":
        """Fix the variable mask; returns the slot numbering and the off-diagonal block pairs."""
        fx = np.ascontiguousarray(np.asarray(fixed, dtype=np.uint8).reshape(-1))
        if len(fx) != self.num_poses:
            raise ValueError("fixed mask length does not match the graph")
        S, P = C.c_int(), C.c_int()
        check(_lib.load().vgicp_graph_assembly_plan(self._h, _ptr(fx), C.byref(S), C.byref(P), None))
        pairs = np.zeros((P.value, 2), np.int32)
        check(_lib.load().vgicp_graph_assembly_plan(self._h, _ptr(fx), C.byref(S), C.byref(P), _ptr(pairs)))
        active = np.flatnonzero(fx == 0)
        var_of_slot = active[::-1].copy()  # slot 0 = last active variable (block_solver.cpp:26-34)
        self._plan = AssemblyPlan(int(S.value), pairs, var_of_slot)
        return self._plan

    def linearize_assembled(self, poses):
        """One linearization pass assembled on the device: (diag S×6×6, offdiag P×6×6, rhs S×6)."""
        plan = getattr(self, "_plan", None)
        if plan is None:
            raise ValueError("no assembly plan (call assembly_plan first)")
        P = poses_array(poses)
        if len(P) != self.num_poses:
            raise ValueError("pose count does not match the graph")
        S, Np = plan.num_slots, len(plan.pairs)
        diag = np.zeros((S, 36))
        off = np.zeros((Np, 36))
        rhs = np.zeros((S, 6))
        check(_lib.load().vgicp_graph_linearize_assembled(self._h, _ptr(P), _ptr(diag), _ptr(off), _ptr(rhs)))
        return diag.reshape(S, 6, 6), off.reshape(Np, 6, 6), rhs

    # device-resident variants (pointers are device addresses, e.g. torch tensor data_ptr())
    def linearize_assembled_device(self, d_poses: int, d_assembled: int) -> None:
        """[diag S×36 | offdiag P×36 | rhs S×6] into device memory (enqueued, not synchronised)."""
        if getattr(self, "_plan", None) is None:
            raise ValueError("no assembly plan (call assembly_plan first)")
        check(_lib.load().vgicp_graph_linearize_assembled_device(self._h, C.c_void_p(d_poses), C.c_void_p(d_assembled)))

    def linearized_errors(self):
        """(errors[F] float64, inliers[F] int32) of the latest assembled linearization — equal to
        evaluate() at the same poses."""
        err = np.zeros(self.num_factors())
        inl = np.zeros(self.num_factors(), np.int32)
        check(_lib.load().vgicp_graph_linearized_errors(self._h, _ptr(err), _ptr(inl)))
        return err, inl

    def solver_plan(self) -> tuple[int, bool]:
        """Band solver plan for the current assembly plan: (block bandwidth after reverse
        Cuthill-McKee, whether the GPU band solver supports it)."""
        bw, ok = C.c_int(), C.c_int()
        check(_lib.load().vgicp_graph_solver_plan(self._h, C.byref(bw), C.byref(ok)))
        self._band = bool(ok.value)
        return int(bw.value), self._band

    def solve_damped(self, d_assembled: int, lam: float):
        """x (S×6, slot order) of the damped assembled system at device address `d_assembled`, or
        None when a pivot block is not positive definite (block_solver.cpp:78-82)."""
        S = self._plan.num_slots
        x = np.empty(6 * S)
        ok = C.c_int()
        check(_lib.load().vgicp_graph_solve_damped(self._h, C.c_void_p(d_assembled), C.c_double(lam), _ptr(x),
                                                   C.byref(ok)))
        return x if ok.value else None

    def solve_damped_pair(self, d_assembled: int, lams):
        """solve_damped at two damping values in one launch (two clusters run concurrently):
        a list of two results, each x or None."""
        S = self._plan.num_slots
        x = np.empty(12 * S)
        lam = np.ascontiguousarray(lams, dtype=np.float64)
        ok = (C.c_int * 2)()
        check(_lib.load().vgicp_graph_solve_damped_pair(self._h, C.c_void_p(d_assembled), _ptr(lam), _ptr(x), ok))
        return [x[6 * S * i:6 * S * (i + 1)].copy() if ok[i] else None for i in range(2)]

    def linearize_device(self, d_poses: int, d_out: int, d_inliers: int) -> None:
        check(_lib.load().vgicp_graph_linearize_device(self._h, C.c_void_p(d_poses), C.c_void_p(d_out), C.c_void_p(d_inliers)))

    def evaluate_device(self, d_poses: int, d_errors: int, d_inliers: int) -> None:
        check(_lib.load().vgicp_graph_evaluate_device(self._h, C.c_void_p(d_poses), C.c_void_p(d_errors), C.c_void_p(d_inliers)))
