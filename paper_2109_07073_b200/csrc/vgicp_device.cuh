// Device-side data layout and exact-arithmetic helpers shared by the sm_100a kernels.
//
// HBM layout:
//  - source cloud, SoA, 36 B/point: pa[i] = (x, y, z, c_xx) float4, pb[i] = (c_xy, c_xz, c_yy, c_yz)
//    float4, pc[i] = c_zz float. Means are float32 (KITTI precision), so the fp64 transform below
//    sees exactly the values the oracle sees.
//  - voxel map: two-choice bucketed hash table (buckets of 4 keys = 32 B, load <= 0.5, every
//    lookup = two independent sector loads), 48-B voxel-local fp32 statistics per slot, plus cold
//    fp64 arrays in ascending key order (keys, counts, means, covariances) for export and the
//    rare fp64 path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace vgicp {

constexpr unsigned long long kEmptyKey = ~0ull;  // valid keys use 63 bits (voxelmap.cpp:57-63)
constexpr int kKeyBits = 21;                     // voxelmap.cpp:12
constexpr double kKeyBias = 1048576.0;           // 2^20, voxelmap.cpp:13

// Two-choice bucketed hash table. Keys live in buckets of kBucket = 4 slots (32 B = one L2
// sector); a key is stored in one of two buckets chosen by independent hashes, so every lookup
// is exactly two independent sector loads (no probe chains). Per-slot statistics live in a
// parallel array indexed by slot.
constexpr int kBucket = 4;

struct __align__(16) VoxelStats {  // compact build-time record (by voxel id)
  float mx, my, mz, cxx;        // voxel-local mean (mean - coord * resolution) and covariance, fp32
  float cxy, cxz, cyy, cyz;
  float czz;
  int vid;                      // index into the cold fp64 arrays (ascending key order)
  int pad0, pad1;
};
static_assert(sizeof(VoxelStats) == 48, "VoxelStats must be 48 bytes");

// Per-slot statistics in the table, split so a hit costs one 32-B and one 8-B gather.
struct __align__(32) SlotStatsA {
  float mx, my, mz, cxx, cxy, cxz, cyy, cyz;
};
struct __align__(8) SlotStatsB {
  float czz;
  int vid;
};

struct MapDev {
  const unsigned long long* keys;  // capacity = kBucket * num_buckets, kEmptyKey when free
  const SlotStatsA* sa;            // per slot
  const SlotStatsB* sb;            // per slot
  const double* cov64;             // V×9 row-major fp64 covariances (cold)
  double res;
  double inv_res;
  unsigned shift;                  // 32 - log2(num_buckets)
  unsigned pad;
};

// 256-bit read-only global load (sm_100: LDG.E.ENL2.256).
__device__ __forceinline__ void ldg256(const void* p, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3,
                                       unsigned& r4, unsigned& r5, unsigned& r6, unsigned& r7) {
  asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
      : "l"(p));
}

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

// One axis of voxel_coord (voxelmap.cpp:45-55): floor(x / r) exactly as
// std::floor(point[a] / resolution_) — the floor of the correctly rounded IEEE quotient — and
// the ±2^20 range check. Fast path: y = x·fl(1/r) differs from fl(x/r) by < 3.4e-16|y| (< 7.2e-10
// for |y| < 2^21), so when frac(y) lies in (2e-9, 1 - 2e-9) both have the same floor. Points
// within ~1e-9 voxel of a face, zeros, infinities and NaN take the IEEE division. On success
// returns the biased 21-bit coordinate k = c + 2^20 and frac_r ≈ x - c·r (voxel-local offset).
// Exact path (out of line, returns by value so the fast path keeps everything in registers):
// (c, x - c·r) with c = floor(fl(x / r)); c is NaN for NaN input.
static __device__ __noinline__ double2 voxel_axis_exact(double x, double r) {
  const double c = floor(__ddiv_rn(x, r));
  return make_double2(c, __dsub_rn(x, __dmul_rn(c, r)));
}

__device__ __forceinline__ bool voxel_axis(double x, double r, double inv_r, unsigned& k, double& local) {
  const double y = __dmul_rn(x, inv_r);
  double c = floor(y);
  const double f = __dsub_rn(y, c);
  if (f > 2.0e-9 && f < 1.0 - 2.0e-9) {
    local = __dmul_rn(f, r);
  } else {
    const double2 e = voxel_axis_exact(x, r);
    c = e.x;
    local = e.y;
  }
  const bool in = c >= -kKeyBias && c < kKeyBias;  // false for NaN
  k = static_cast<unsigned>((in ? __double2int_rz(c) : 0) + (1 << 20));
  return in;
}

__device__ __forceinline__ bool in_key_range(double c) { return c >= -kKeyBias && c < kKeyBias; }

// pack_key (voxelmap.cpp:57-63) as (hi, lo) 32-bit halves of ((k0 << 42) | (k1 << 21) | k2).
__device__ __forceinline__ void pack_key32(unsigned k0, unsigned k1, unsigned k2, unsigned& hi, unsigned& lo) {
  lo = k2 | (k1 << 21);
  hi = (k1 >> 11) | (k0 << 10);
}

__device__ __forceinline__ unsigned long long key64(unsigned hi, unsigned lo) {
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}

__device__ __forceinline__ void unpack_key(unsigned long long key, unsigned& k0, unsigned& k1, unsigned& k2) {
  k0 = static_cast<unsigned>(key >> 42) & 0x1FFFFFu;
  k1 = static_cast<unsigned>(key >> 21) & 0x1FFFFFu;
  k2 = static_cast<unsigned>(key) & 0x1FFFFFu;
}

__device__ __forceinline__ double key_coord(unsigned long long key, int axis) {
  const int sh = (2 - axis) * kKeyBits;
  return static_cast<double>(static_cast<long long>((key >> sh) & 0x1FFFFFull) - (1ll << 20));
}

// Two independent spatial hashes of the biased voxel coordinates -> bucket index (32-bit ops).
__device__ __forceinline__ unsigned bucket1(unsigned k0, unsigned k1, unsigned k2, unsigned shift) {
  const unsigned h = (k0 * 73856093u) ^ (k1 * 19349663u) ^ (k2 * 83492791u);
  return (h * 0x9E3779B1u) >> shift;
}
__device__ __forceinline__ unsigned bucket2(unsigned k0, unsigned k1, unsigned k2, unsigned shift) {
  const unsigned h = (k0 * 2654435761u) ^ (k1 * 2246822519u) ^ (k2 * 3266489917u) ^ 0x5bd1e995u;
  return ((h ^ (h >> 15)) * 0x85EBCA6Bu) >> shift;
}

// Voxel key of q under resolution r; false when any axis is outside ±2^20 (or NaN).
__device__ __forceinline__ bool voxel_key(double q0, double q1, double q2, double r, double inv_r, unsigned& k0,
                                          unsigned& k1, unsigned& k2, double& l0, double& l1, double& l2) {
  return voxel_axis(q0, r, inv_r, k0, l0) & voxel_axis(q1, r, inv_r, k1, l1) & voxel_axis(q2, r, inv_r, k2, l2);
}

// Issue the two bucket loads (2 × 32 B, independent) for a key.
struct BucketPair {
  unsigned a[8];
  unsigned b[8];
};
__device__ __forceinline__ BucketPair load_buckets(const unsigned long long* __restrict__ keys, unsigned b1,
                                                   unsigned b2) {
  BucketPair r;
  ldg256(keys + kBucket * b1, r.a[0], r.a[1], r.a[2], r.a[3], r.a[4], r.a[5], r.a[6], r.a[7]);
  ldg256(keys + kBucket * b2, r.b[0], r.b[1], r.b[2], r.b[3], r.b[4], r.b[5], r.b[6], r.b[7]);
  return r;
}

// Slot of (hi, lo) among the 8 loaded candidates, or -1.
__device__ __forceinline__ int match_buckets(const BucketPair& p, unsigned b1, unsigned b2, unsigned hi, unsigned lo) {
  int s = -1;
#pragma unroll
  for (int q = 0; q < kBucket; ++q) {
    s = (p.a[2 * q] == lo && p.a[2 * q + 1] == hi) ? static_cast<int>(kBucket * b1 + q) : s;
    s = (p.b[2 * q] == lo && p.b[2 * q + 1] == hi) ? static_cast<int>(kBucket * b2 + q) : s;
  }
  return s;
}

__device__ __forceinline__ int find_slot(const MapDev& map, unsigned k0, unsigned k1, unsigned k2) {
  unsigned hi, lo;
  pack_key32(k0, k1, k2, hi, lo);
  const unsigned b1 = bucket1(k0, k1, k2, map.shift), b2 = bucket2(k0, k1, k2, map.shift);
  return match_buckets(load_buckets(map.keys, b1, b2), b1, b2, hi, lo);
}

}  // namespace vgicp
