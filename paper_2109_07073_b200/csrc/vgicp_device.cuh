// Device-side data layout and exact-arithmetic helpers shared by the sm_100a kernels.
//
// HBM layout:
//  - source cloud, SoA, 36 B/point: pa[i] = (x, y, z, c_xx) float4, pb[i] = (c_xy, c_xz, c_yy, c_yz)
//    float4, pc[i] = c_zz float. Means are float32 (KITTI precision), so the fp64 transform below
//    sees exactly the values the oracle sees.
//  - voxel map: open-addressing hash table of 48-B records (key + voxel-local fp32 statistics),
//    capacity a power of two >= 2V (load factor <= 0.5, linear probing), plus cold fp64 arrays in
//    ascending key order (keys, counts, means, covariances) for export and the rare fp64 path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace vgicp {

constexpr unsigned long long kEmptyKey = ~0ull;  // valid keys use 63 bits (voxelmap.cpp:57-63)
constexpr int kKeyBits = 21;                     // voxelmap.cpp:12
constexpr double kKeyBias = 1048576.0;           // 2^20, voxelmap.cpp:13

// 48-byte hash-table record. The first 16 B (key + 2 mean floats) is all a probe reads.
struct __align__(16) VoxelRec {
  unsigned long long key;
  float mx, my;                 // voxel-local mean: mean - coord * resolution (fp32)
  float mz, cxx, cxy, cxz;      // covariance (fp32), symmetric
  float cyy, cyz, czz;
  int vid;                      // index into the cold fp64 arrays (ascending key order)
};
static_assert(sizeof(VoxelRec) == 48, "VoxelRec must be 48 bytes");

struct MapDev {
  const VoxelRec* table;
  const double* cov64;  // V×9 row-major fp64 covariances (cold)
  double res;
  double inv_res;
  unsigned shift;       // 64 - log2(capacity)
  unsigned mask;        // capacity - 1
};

// ------------------------------------------------------------------------------------------
// Exact fp64 helpers: explicit round-to-nearest intrinsics are never contracted into FMAs,
// so these reproduce the oracle's (and x86-64 SSE2's) separately rounded operations.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ double dot3_rn(double a0, double a1, double a2, double b0, double b1, double b2) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1)), __dmul_rn(a2, b2));
}

// Pose::apply (se3.hpp:43): ((R_i0 p0 + R_i1 p1) + R_i2 p2) + t_i.
__device__ __forceinline__ void apply_pose_rn(const double* T, double p0, double p1, double p2, double& q0,
                                              double& q1, double& q2) {
  q0 = __dadd_rn(dot3_rn(T[0], T[1], T[2], p0, p1, p2), T[9]);
  q1 = __dadd_rn(dot3_rn(T[3], T[4], T[5], p0, p1, p2), T[10]);
  q2 = __dadd_rn(dot3_rn(T[6], T[7], T[8], p0, p1, p2), T[11]);
}

// floor(x / r) exactly as std::floor(point[a] / resolution_) (voxelmap.cpp:48, :109), i.e. the
// floor of the correctly rounded IEEE quotient. Fast path: y = x * fl(1/r) is within 3.4e-16|y|
// of fl(x/r); when no integer lies within 8e-16|y| of y both have the same floor. Otherwise
// (points within ~1e-15 relative of a voxel face, zero, NaN) take the IEEE division.
__device__ __forceinline__ double voxel_floor(double x, double r, double inv_r) {
  const double y = __dmul_rn(x, inv_r);
  const double tol = fmax(fabs(y) * 8.0e-16, 1.0e-300);
  const double lo = floor(__dsub_rn(y, tol));
  const double hi = floor(__dadd_rn(y, tol));
  if (lo == hi) return lo;
  return floor(__ddiv_rn(x, r));
}

__device__ __forceinline__ bool in_key_range(double c) { return c >= -kKeyBias && c < kKeyBias; }

// pack_key (voxelmap.cpp:57-63) for in-range integral coordinates.
__device__ __forceinline__ unsigned long long pack_key(double c0, double c1, double c2) {
  const unsigned long long k0 = static_cast<unsigned long long>(static_cast<long long>(c0) + (1ll << 20));
  const unsigned long long k1 = static_cast<unsigned long long>(static_cast<long long>(c1) + (1ll << 20));
  const unsigned long long k2 = static_cast<unsigned long long>(static_cast<long long>(c2) + (1ll << 20));
  return (((k0 << kKeyBits) | k1) << kKeyBits) | k2;
}

__device__ __forceinline__ double key_coord(unsigned long long key, int axis) {
  const int sh = (2 - axis) * kKeyBits;
  return static_cast<double>(static_cast<long long>((key >> sh) & 0x1FFFFFull) - (1ll << 20));
}

// Voxel key of point q under resolution r; false when any axis is outside ±2^20 (or NaN).
__device__ __forceinline__ bool voxel_key(double q0, double q1, double q2, double r, double inv_r,
                                          unsigned long long& key, double& c0, double& c1, double& c2) {
  c0 = voxel_floor(q0, r, inv_r);
  c1 = voxel_floor(q1, r, inv_r);
  c2 = voxel_floor(q2, r, inv_r);
  if (!(in_key_range(c0) && in_key_range(c1) && in_key_range(c2))) return false;
  key = pack_key(c0, c1, c2);
  return true;
}

// Fibonacci hashing into a power-of-two table.
__device__ __forceinline__ unsigned hash_slot(unsigned long long key, unsigned shift) {
  return static_cast<unsigned>((key * 0x9E3779B97F4A7C15ull) >> shift);
}

// Linear probe. Returns the slot of `key` or -1. Also returns the record's first 16 B
// (mx, my) through the out-params to save one load on a hit.
__device__ __forceinline__ int probe(const VoxelRec* __restrict__ table, unsigned shift, unsigned mask,
                                     unsigned long long key, float& mx, float& my) {
  unsigned slot = hash_slot(key, shift);
  while (true) {
    const uint4 h = __ldg(reinterpret_cast<const uint4*>(table + slot));
    const unsigned long long k = (static_cast<unsigned long long>(h.y) << 32) | h.x;
    if (k == key) {
      mx = __uint_as_float(h.z);
      my = __uint_as_float(h.w);
      return static_cast<int>(slot);
    }
    if (k == kEmptyKey) return -1;
    slot = (slot + 1) & mask;
  }
}

__device__ __forceinline__ bool probe_hit(const VoxelRec* __restrict__ table, unsigned shift, unsigned mask,
                                          unsigned long long key) {
  unsigned slot = hash_slot(key, shift);
  while (true) {
    const unsigned long long k = __ldg(&table[slot].key);
    if (k == key) return true;
    if (k == kEmptyKey) return false;
    slot = (slot + 1) & mask;
  }
}

}  // namespace vgicp
