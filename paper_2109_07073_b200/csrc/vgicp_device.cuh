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

// Device-side bounds checks of the debug build (make -C paper_2109_07073_b200/csrc debug, loaded with
// VGICP_LIB=.../lib_debug/libvgicp_b200.so): a violated index invariant prints its site and traps the
// kernel (the launch then fails with cudaErrorLaunchFailure / illegal instruction instead of reading
// or writing out of bounds). Compiled out of the product build.
#ifdef VGICP_DEBUG_BOUNDS
#define VG_CHECK(cond)                                                                                  \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("VG_CHECK failed %s:%d block (%d,%d) thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, blockIdx.y, \
             threadIdx.x, #cond);                                                                       \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define VG_CHECK(cond) \
  do {                 \
  } while (0)
#endif

constexpr unsigned long long kEmptyKey = ~0ull;  // valid keys use 63 bits (voxelmap.cpp:57-63)
constexpr int kKeyBits = 21;                     // voxelmap.cpp:12
constexpr double kKeyBias = 1048576.0;           // 2^20, voxelmap.cpp:13

// Two-choice bucketed (cuckoo) hash table. Keys live in buckets of kBucket = 2 slots (16 B); a key
// is stored in one of two buckets chosen by independent hashes, so every lookup is exactly two
// independent 16-B loads (no probe chains) and 4 key compares. Per-slot statistics live in
// parallel arrays indexed by slot.
constexpr int kBucket = 2;  // slots per bucket (16 B of keys: one LDG.128)

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

// Occupancy bitmap of a map's occupied voxel box: one 16-B record per 4×4×4 brick of voxels
// (bricks row-major, z fastest; bit (x&3)<<4 | (y&3)<<2 | (z&3) of the box-relative coordinate)
// holding the brick's 64 occupancy bits and the rank of its first occupied voxel. The overlap query
// needs only the bits; the factor kernels turn a hit into the voxel's rank (brick rank + popcount
// of the lower bits), which indexes rank-ordered statistics — one coherent 16-B load per probe
// instead of two hash-bucket loads. occ == nullptr: probe the hash table.
struct __align__(16) OccWord {
  unsigned long long bits;  // brick occupancy
  unsigned rank;            // occupied voxels in all earlier bricks (rank of the brick's first voxel)
  unsigned pad;
};
struct OccDev {
  const OccWord* occ;
  unsigned kx0, ky0, kz0;  // biased (key) coordinates of the box's lower corner
  unsigned ex, ey, ez;     // box extent in voxels
  unsigned nby, nbz;       // bricks along y and z
};
// Word index / bit of biased voxel coordinates; false outside the occupied box (= a miss).
__device__ __forceinline__ bool occ_locate(const OccDev& o, unsigned k0, unsigned k1, unsigned k2, unsigned& word,
                                           unsigned& bit) {
  const unsigned rx = k0 - o.kx0, ry = k1 - o.ky0, rz = k2 - o.kz0;  // wraps to huge values below the box
  word = ((rx >> 2) * o.nby + (ry >> 2)) * o.nbz + (rz >> 2);
  bit = ((rx & 3u) << 4) | ((ry & 3u) << 2) | (rz & 3u);
  return (rx < o.ex) & (ry < o.ey) & (rz < o.ez);
}

struct MapDev {
  const unsigned long long* keys;  // capacity = kBucket * num_buckets, kEmptyKey when free
  const SlotStatsA* sa;            // per slot
  const SlotStatsB* sb;            // per slot
  const double* cov64;             // fp64 covariances by voxel id (cold): V×9 row-major, or V×6 unique
                                   // entries (xx xy xz yy yz zz) when bit 0 is set — see cov_row
  double res;
  double inv_res;
  unsigned shift;                  // 32 - log2(num_buckets)
  unsigned pad;
  OccDev occ;                      // occupancy bitmap; factor graphs in rank mode index sa / sb by rank
};

// The fp64 covariance of voxel `vid` as 9 row-major entries from a (possibly 6-wide, tagged) array.
__device__ __forceinline__ void cov_row(const double* tagged, int vid, double* C) {
  const uintptr_t b = reinterpret_cast<uintptr_t>(tagged);
  if (b & 1u) {
    const double* c = reinterpret_cast<const double*>(b & ~uintptr_t(1)) + 6 * static_cast<size_t>(vid);
    C[0] = c[0], C[1] = c[1], C[2] = c[2], C[3] = c[1], C[4] = c[3], C[5] = c[4], C[6] = c[2], C[7] = c[4], C[8] = c[5];
  } else {
    const double* c = tagged + 9 * static_cast<size_t>(vid);
#pragma unroll
    for (int e = 0; e < 9; ++e) C[e] = c[e];
  }
}

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

// Fast path of one axis: y = x·fl(1/r), c = floor(y), f = y - c. Returns whether the fast path
// is certain (f within (2e-9, 1 - 2e-9), i.e. |f - 0.5| < 0.5 - 2e-9; false for inf / NaN).
__device__ __forceinline__ bool voxel_axis_fast(double x, double r, double inv_r, int& c_int, double& local) {
  const double y = __dmul_rn(x, inv_r);
  const double c = floor(y);
  const double f = __dsub_rn(y, c);
  c_int = __double2int_rz(c);  // saturates: out-of-range values fail the range test below
  local = __dmul_rn(f, r);
  return fabs(__dsub_rn(f, 0.5)) < 0.5 - 2.0e-9;
}

__device__ __forceinline__ bool voxel_axis(double x, double r, double inv_r, unsigned& k, double& local) {
  int c;
  if (!voxel_axis_fast(x, r, inv_r, c, local)) {
    const double2 e = voxel_axis_exact(x, r);
    if (!(e.x >= -kKeyBias && e.x < kKeyBias)) return false;  // also rejects NaN
    c = __double2int_rz(e.x);
    local = e.y;
  }
  k = static_cast<unsigned>(c + (1 << 20));
  return k < (1u << 21);
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
// bucket1 is locality-preserving: the 8 voxels of an aligned 2×2×2 block share one hashed group of
// 8 consecutive buckets (8 × 16 B = one 128-B line), so spatially ordered probes (source clouds are
// streamed in Morton order) hit few lines and mostly L1. bucket2 is a plain spatial hash.
__device__ __forceinline__ unsigned bucket1(unsigned k0, unsigned k1, unsigned k2, unsigned shift) {
  const unsigned h = ((k0 >> 1) * 73856093u) ^ ((k1 >> 1) * 19349663u) ^ ((k2 >> 1) * 83492791u);
  const unsigned group = (h * 0x9E3779B1u) >> (shift + 3);
  return (group << 3) | (k0 & 1u) | ((k1 & 1u) << 1) | ((k2 & 1u) << 2);
}
#ifndef VG_B2_LOCAL
#define VG_B2_LOCAL 0
#endif
__device__ __forceinline__ unsigned bucket2(unsigned k0, unsigned k1, unsigned k2, unsigned shift) {
  const unsigned h = (k0 * 2654435761u) ^ (k1 * 2246822519u) ^ (k2 * 3266489917u) ^ 0x5bd1e995u;
#if VG_B2_LOCAL
  // the alternative bucket lives in bucket1's 8-bucket group (same 128-B line), never bucket1 itself
  const unsigned b1 = bucket1(k0, k1, k2, shift);
  const unsigned r = 1u + ((h ^ (h >> 15)) * 0x85EBCA6Bu >> 29) % 7u;
  return (b1 & ~7u) | ((b1 + r) & 7u);
#else
  return ((h ^ (h >> 15)) * 0x85EBCA6Bu) >> shift;
#endif
}

// Voxel key of q under resolution r; false when any axis is outside ±2^20 (or NaN). The three
// axes share one branch to the exact path.
__device__ __forceinline__ bool voxel_key(double q0, double q1, double q2, double r, double inv_r, unsigned& k0,
                                          unsigned& k1, unsigned& k2, double& l0, double& l1, double& l2) {
  int c0, c1, c2;
  const bool f0 = voxel_axis_fast(q0, r, inv_r, c0, l0);
  const bool f1 = voxel_axis_fast(q1, r, inv_r, c1, l1);
  const bool f2 = voxel_axis_fast(q2, r, inv_r, c2, l2);
  if (!(f0 && f1 && f2)) {
    bool ok = true;
    if (!f0) ok &= voxel_axis(q0, r, inv_r, k0, l0), c0 = static_cast<int>(k0) - (1 << 20);
    if (!f1) ok &= voxel_axis(q1, r, inv_r, k1, l1), c1 = static_cast<int>(k1) - (1 << 20);
    if (!f2) ok &= voxel_axis(q2, r, inv_r, k2, l2), c2 = static_cast<int>(k2) - (1 << 20);
    if (!ok) return false;
  }
  k0 = static_cast<unsigned>(c0 + (1 << 20));
  k1 = static_cast<unsigned>(c1 + (1 << 20));
  k2 = static_cast<unsigned>(c2 + (1 << 20));
  return (k0 < (1u << 21)) & (k1 < (1u << 21)) & (k2 < (1u << 21));
}

// Issue the two bucket loads (2 × 16 B, independent) for a key.
struct BucketPair {
  uint4 a;
  uint4 b;
};
#ifndef VG_B2_HINT
#if VG_B2_LOCAL
#define VG_B2_HINT 0
#else
#define VG_B2_HINT 2
#endif
#endif
// bucket2 is a random probe: optionally keep it out of L1 so that the spatially coherent bucket1
// lines and slot statistics stay resident there.
__device__ __forceinline__ uint4 ldg_bucket2(const void* p) {
#if VG_B2_HINT == 1
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
#elif VG_B2_HINT == 2
  return __ldcg(reinterpret_cast<const uint4*>(p));
#else
  return __ldg(reinterpret_cast<const uint4*>(p));
#endif
}
__device__ __forceinline__ BucketPair load_buckets(const unsigned long long* __restrict__ keys, unsigned b1,
                                                   unsigned b2) {
  BucketPair r;
  r.a = __ldg(reinterpret_cast<const uint4*>(keys + kBucket * b1));
  r.b = ldg_bucket2(keys + kBucket * b2);
  return r;
}

// Slot of (hi, lo) among the 4 loaded candidates, or -1.
__device__ __forceinline__ int match_buckets(const BucketPair& p, unsigned b1, unsigned b2, unsigned hi, unsigned lo) {
  int s = -1;
  s = (p.a.x == lo && p.a.y == hi) ? static_cast<int>(kBucket * b1) : s;
  s = (p.a.z == lo && p.a.w == hi) ? static_cast<int>(kBucket * b1 + 1) : s;
  s = (p.b.x == lo && p.b.y == hi) ? static_cast<int>(kBucket * b2) : s;
  s = (p.b.z == lo && p.b.w == hi) ? static_cast<int>(kBucket * b2 + 1) : s;
  return s;
}

__device__ __forceinline__ int find_slot(const MapDev& map, unsigned k0, unsigned k1, unsigned k2) {
  unsigned hi, lo;
  pack_key32(k0, k1, k2, hi, lo);
  const unsigned b1 = bucket1(k0, k1, k2, map.shift), b2 = bucket2(k0, k1, k2, map.shift);
  return match_buckets(load_buckets(map.keys, b1, b2), b1, b2, hi, lo);
}

}  // namespace vgicp
