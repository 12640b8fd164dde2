// Batched VGICP matching-cost factor kernels (sm_100a): linearize (factors.cpp:90-148) and
// evaluate (factors.cpp:150-181) for every factor of a graph in ONE launch.
//
// Grid: one CTA per work item (factor, chunk of source points); every warp streams its own 64-point
// Morton tiles with TMA bulk copies. Per source point:
//   fp64  q = T_ts·mu (reference op order), exact voxel key, brick-record lookup of the target map's
//         occupancy bitmap (rank = the voxel's statistics index; cuckoo-hash probes for maps without)
//   hits  are queued per warp; the math below runs on full batches of 32 queued hits
//   fp32  e = voxel-local mean - (q - corner), M = C_t + R C_s Rᵀ, Omega = M⁻¹ (cofactor),
//         H_tt = AᵀΩA with A = [-[q]x | I] as Q = -[q]xΩ[q]x (6), P = [q]xΩ (9), Ω (6),
//         b_t = [-q×Ωe; -Ωe] (6), error eᵀΩe  -> 28 fp32 accumulators + int inliers
//   near-singular M (fp32 Sylvester test without margin) -> the oracle-identical fp64 LDLT path
// Reduction without float atomics: per-thread fp32 -> warp butterfly in fp64 -> one
// partial per warp; the last warp of a factor (integer arrival counter) sums the factor's partials in
// (item, warp) order and expands, in fp64,
//   H_ts = -H_tt·Ad,  H_ss = AdᵀH_tt·Ad,  b_s = -Adᵀb_t,  Ad = Ad(T_ts) (se3.cpp:107-113),
// which is exact algebra because B = -A·Ad(T_ts). Fixed orders everywhere => deterministic.
#include <atomic>

#include "exact_math.cuh"
#include "internal.h"

namespace vgicp {

namespace {

constexpr int kWarps = kFactorThreads / 32;

// T_ts = T_target⁻¹ · T_source (factors.cpp:94), entry k of the 12-double pose, computed with
// the oracle's op order: inverse (se3.hpp:45) then compose (se3.cpp:42-44).
__device__ __forceinline__ double relative_pose_entry(const double* Tt, const double* Ts, int k) {
  if (k < 9) {
    const int i = k / 3, j = k % 3;
    return dot3_rn(Tt[i], Tt[3 + i], Tt[6 + i], Ts[j], Ts[3 + j], Ts[6 + j]);
  }
  const int i = k - 9;
  const double inv_t = -dot3_rn(Tt[i], Tt[3 + i], Tt[6 + i], Tt[9], Tt[10], Tt[11]);
  return __dadd_rn(dot3_rn(Tt[i], Tt[3 + i], Tt[6 + i], Ts[9], Ts[10], Ts[11]), inv_t);
}

// Rare path: M near singular in fp32 -> recompute M and the LDLT decision in fp64 exactly as
// the oracle (factors.cpp:38-46, :107) and return Omega as fp32.
__device__ __noinline__ bool omega_fp64(const double* T, float sxx, float sxy, float sxz, float syy, float syz,
                                        float szz, const double* cov_tagged, int vid, float* om) {
  const double Cs[9] = {sxx, sxy, sxz, sxy, syy, syz, sxz, syz, szz};
  double Ct[9], M[9], O[9];
  cov_row(cov_tagged, vid, Ct);
  combined_cov_rn(T, Cs, Ct, M);
  if (!invert_covariance_rn(M, O)) return false;
  om[0] = (float)O[0];
  om[1] = (float)O[1];
  om[2] = (float)O[2];
  om[3] = (float)O[4];
  om[4] = (float)O[5];
  om[5] = (float)O[8];
  return true;
}

// The same decision for a float64 source cloud: its exact float64 covariance (all 9 entries, as the
// oracle / reference hold it) instead of the float32 tile copy, so a near-singular M is skipped or
// kept exactly as the reference's double LDLT decides.
__device__ __noinline__ bool omega_fp64_c9(const double* T, const double* Cs, const double* cov_tagged, int vid,
                                           float* om) {
  double Ct[9], M[9], O[9];
  cov_row(cov_tagged, vid, Ct);
  combined_cov_rn(T, Cs, Ct, M);
  if (!invert_covariance_rn(M, O)) return false;
  om[0] = (float)O[0];
  om[1] = (float)O[1];
  om[2] = (float)O[2];
  om[3] = (float)O[4];
  om[4] = (float)O[5];
  om[5] = (float)O[8];
  return true;
}

#ifndef VG_ILP
#define VG_ILP 2
#endif
#ifndef VG_B2_LAZY
#define VG_B2_LAZY 0  // read bucket2 only when bucket1 is full and misses
#endif
#ifndef VG_PREFETCH
#define VG_PREFETCH 2  // rank lookups: L1 prefetch of a hit's statistics at append time (1: 32-B part, 2: both)
#endif
#ifndef VG_STAGES
#define VG_STAGES 2
#endif
constexpr int kILP = VG_ILP;                        // points per lane per tile (independent probes in flight)
constexpr int kWarpTile = 32 * kILP;           // points per warp per tile
static_assert(kFactorTile % kPointBlock == 0, "work items must start on a point block");

// ---- TMA (cp.async.bulk) + mbarrier helpers --------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Per-hit math of the linearization (factors.cpp:99-134) in fp32, accumulated into the 28 sums
// (or the error only): l = (q - voxel corner, q.x), qy/qz the rest of q, C_s = (cxx, cs = (xy xz yy
// yz), szz), v0/v1/v2 the voxel's slot statistics. Near-singular M -> the fp64 LDLT decision
// (kF64: on the float64 covariance of source point `pos`, Morton position in the cloud).
template <bool kLinearize, bool kF64>
__device__ __forceinline__ void hit_math(const float* Rf, const double* T, const MapDev& map, float4 l, float qy,
                                         float qz, float cxx, float4 cs, float szz, float4 v0, float4 v1, float2 v2,
                                         float* acc, int& inl, const FactorDev* fp, int pos) {
  const float sxx = cxx, sxy = cs.x, sxz = cs.y, syy = cs.z, syz = cs.w;

  // residual e = mu' - q in voxel-local coordinates
  const float e0 = v0.x - l.x;
  const float e1 = v0.y - l.y;
  const float e2 = v0.z - l.z;

  // M = C_t + R C_s Rᵀ (fp32)
  const float r00 = Rf[0], r01 = Rf[1], r02 = Rf[2];
  const float r10 = Rf[3], r11 = Rf[4], r12 = Rf[5];
  const float r20 = Rf[6], r21 = Rf[7], r22 = Rf[8];
  const float t00 = r00 * sxx + r01 * sxy + r02 * sxz;
  const float t01 = r00 * sxy + r01 * syy + r02 * syz;
  const float t02 = r00 * sxz + r01 * syz + r02 * szz;
  const float t10 = r10 * sxx + r11 * sxy + r12 * sxz;
  const float t11 = r10 * sxy + r11 * syy + r12 * syz;
  const float t12 = r10 * sxz + r11 * syz + r12 * szz;
  const float t20 = r20 * sxx + r21 * sxy + r22 * sxz;
  const float t21 = r20 * sxy + r21 * syy + r22 * syz;
  const float t22 = r20 * sxz + r21 * syz + r22 * szz;
  const float m00 = v0.w + (t00 * r00 + t01 * r01 + t02 * r02);
  const float m01 = v1.x + (t00 * r10 + t01 * r11 + t02 * r12);
  const float m02 = v1.y + (t00 * r20 + t01 * r21 + t02 * r22);
  const float m11 = v1.z + (t10 * r10 + t11 * r11 + t12 * r12);
  const float m12 = v1.w + (t10 * r20 + t11 * r21 + t12 * r22);
  const float m22 = v2.x + (t20 * r20 + t21 * r21 + t22 * r22);

  // Omega = M⁻¹ by cofactors; Sylvester test with margins decides the fast path
  const float a00 = m11 * m22 - m12 * m12;
  const float a01 = m02 * m12 - m01 * m22;
  const float a02 = m01 * m12 - m02 * m11;
  const float a11 = m00 * m22 - m02 * m02;
  const float a12 = m01 * m02 - m00 * m12;
  const float a22 = m00 * m11 - m01 * m01;
  const float det = m00 * a00 + m01 * a01 + m02 * a02;
  const float tr = m00 + m11 + m22;
  float o00, o01, o02, o11, o12, o22;
  if (tr > 0.f && m00 > 1e-6f * tr && a22 > 1e-6f * tr * tr && det > 1e-5f * tr * tr * tr) {
    float inv;  // MUFU reciprocal + one Newton step (~1 ulp; the fp32 algebra sets the tolerance)
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(det));
    inv = inv * (2.0f - det * inv);
    o00 = a00 * inv;
    o01 = a01 * inv;
    o02 = a02 * inv;
    o11 = a11 * inv;
    o12 = a12 * inv;
    o22 = a22 * inv;
  } else {
    float om[6];
    const int vid = __float_as_int(v2.y);
    if constexpr (kF64) {
      VG_CHECK(pos >= 0 && pos < fp->n);
      const unsigned src_i = fp->blk64[pos / kPointBlock].idx[pos % kPointBlock];
      VG_CHECK(src_i < static_cast<unsigned>(fp->n));
      if (!omega_fp64_c9(T, fp->c64 + 9 * static_cast<size_t>(src_i), map.cov64, vid, om)) return;
    } else {
      if (!omega_fp64(T, sxx, sxy, sxz, syy, syz, szz, map.cov64, vid, om)) return;
    }
    o00 = om[0], o01 = om[1], o02 = om[2], o11 = om[3], o12 = om[4], o22 = om[5];
  }
  const float w0 = o00 * e0 + o01 * e1 + o02 * e2;
  const float w1 = o01 * e0 + o11 * e1 + o12 * e2;
  const float w2 = o02 * e0 + o12 * e1 + o22 * e2;
  ++inl;
  if constexpr (!kLinearize) {
    acc[0] += e0 * w0 + e1 * w1 + e2 * w2;
  } else {
    const float qf0 = l.w, qf1 = qy, qf2 = qz;
    // P = [q]x Ω
    const float p00 = qf1 * o02 - qf2 * o01, p01 = qf1 * o12 - qf2 * o11, p02 = qf1 * o22 - qf2 * o12;
    const float p10 = qf2 * o00 - qf0 * o02, p11 = qf2 * o01 - qf0 * o12, p12 = qf2 * o02 - qf0 * o22;
    const float p20 = qf0 * o01 - qf1 * o00, p21 = qf0 * o11 - qf1 * o01, p22 = qf0 * o12 - qf1 * o02;
    // Q = -P [q]x  (symmetric)
    acc[0] += p02 * qf1 - p01 * qf2;   // Q00
    acc[1] += p00 * qf2 - p02 * qf0;   // Q01
    acc[2] += p01 * qf0 - p00 * qf1;   // Q02
    acc[3] += p10 * qf2 - p12 * qf0;   // Q11
    acc[4] += p11 * qf0 - p10 * qf1;   // Q12
    acc[5] += p21 * qf0 - p20 * qf1;   // Q22
    acc[6] += p00;
    acc[7] += p01;
    acc[8] += p02;
    acc[9] += p10;
    acc[10] += p11;
    acc[11] += p12;
    acc[12] += p20;
    acc[13] += p21;
    acc[14] += p22;
    acc[15] += o00;
    acc[16] += o01;
    acc[17] += o02;
    acc[18] += o11;
    acc[19] += o12;
    acc[20] += o22;
    // b_t = -AᵀΩe = [-(q × w); -w]
    acc[21] -= qf1 * w2 - qf2 * w1;
    acc[22] -= qf2 * w0 - qf0 * w2;
    acc[23] -= qf0 * w1 - qf1 * w0;
    acc[24] -= w0;
    acc[25] -= w1;
    acc[26] -= w2;
    acc[27] += e0 * w0 + e1 * w1 + e2 * w2;
  }
}

// End of a warp's share of a work item: fp64 butterfly over the 32 lanes in a fixed order, one
// partial per warp (no float atomics; once per ~2,500 points per warp). An integer arrival counter
// elects the last warp of the factor, which sums the factor's partials in (item, warp) order and
// expands in fp64. `gw` = this warp's partial slot, `parts` = partial slots per work item, `ws` =
// 180 doubles of per-warp shared scratch.
template <bool kLinearize>
__device__ __forceinline__ void finish_factor(const float* acc, int inl, int lane, size_t gw, int parts,
                                              const WorkItem& w, const FactorDev* __restrict__ fp, const double* T,
                                              double* ws, double* __restrict__ partials, int* __restrict__ part_inl,
                                              unsigned* __restrict__ counters, double* __restrict__ out,
                                              int* __restrict__ out_inl) {
  constexpr int kAcc = kLinearize ? kLinAcc : 1;
  // ---- warp reduction: fp64 butterfly over the 32 lanes, fixed order; one partial per warp
  //      (no float atomics). Once per ~2,500 points per warp, so its cost is negligible. ----
#pragma unroll
  for (int k = 0; k < kAcc; ++k) {
    double v = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) partials[gw * kPartialStride + k] = v;
  }
  inl = __reduce_add_sync(0xffffffffu, inl);
  if (lane == 0) part_inl[gw] = inl;
  __threadfence();
  __syncwarp();
  // Integer arrival counter; the electing warp clears it for the next launch. (A launch that fails to
  // start leaves it untouched; launch_factor clears the counters after any launch error.)
  unsigned last = 0;
  if (lane == 0) {
    const unsigned arrived = atomicAdd(&counters[w.factor], 1u) + 1u;
    VG_CHECK(arrived <= static_cast<unsigned>(fp->item_count * parts));
    last = arrived == static_cast<unsigned>(fp->item_count * parts) ? 1u : 0u;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();

  // ---- last warp of this factor: (item, warp)-ordered sum of the partials, fp64 epilogue ----
  double* tot = ws;           // 28
  double* H = ws + 32;        // 36
  double* Ad = ws + 72;       // 36
  double* HA = ws + 108;      // 36
  double* Hss = ws + 144;     // 36
  const size_t gb = (size_t)fp->item_begin * parts;
  const int gc = fp->item_count * parts;
  if (lane < kAcc) {
    double sum = 0.0;
    for (int g = 0; g < gc; ++g) sum += __ldcg(&partials[(gb + g) * kPartialStride + lane]);
    tot[lane] = sum;
  }
  int tinl = 0;
  if (lane == 0) {
    for (int g = 0; g < gc; ++g) tinl += __ldcg(&part_inl[gb + g]);
    counters[w.factor] = 0u;  // ready for the next launch
  }
  __syncwarp();

  if constexpr (!kLinearize) {
    if (lane == 0) {
      out[w.factor] = tot[0];
      out_inl[w.factor] = tinl;
    }
    return;
  } else {
    const int f = w.factor;
    double* o = out + (size_t)f * VGICP_LINEARIZED_DOUBLES;
    if (__shfl_sync(0xffffffffu, tinl, 0) == 0) {
      // no hit: the reference's accumulators stay zero (factors.cpp:97-146) — also when T_ts is not
      // finite, where the Ad(T_ts) expansion below would turn 0 into NaN
      for (int t = lane; t < VGICP_LINEARIZED_DOUBLES - 1; t += 32) o[t] = 0.0;
      if (lane == 0) o[VGICP_LINEARIZED_DOUBLES - 1] = 0.0, out_inl[f] = 0;
      return;
    }
    for (int t = lane; t < 36; t += 32) {
      const int i = t / 6, j = t % 6;
      // H_tt = [[Q, P], [Pᵀ, Ω]]
      const int qi[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
      double h;
      if (i < 3 && j < 3) h = tot[qi[i][j]];
      else if (i < 3) h = tot[6 + 3 * i + (j - 3)];
      else if (j < 3) h = tot[6 + 3 * j + (i - 3)];
      else h = tot[15 + qi[i - 3][j - 3]];
      H[t] = h;
      // Ad(T_ts) = [[R, 0], [[t]x R, R]]
      double ad = 0.0;
      if (i < 3 && j < 3) ad = T[3 * i + j];
      else if (i >= 3 && j >= 3) ad = T[3 * (i - 3) + (j - 3)];
      else if (i >= 3 && j < 3) {
        const int r = i - 3;
        const double tx = T[9], ty = T[10], tz = T[11];
        const double sk[3][3] = {{0.0, -tz, ty}, {tz, 0.0, -tx}, {-ty, tx, 0.0}};
        ad = dot3_rn(sk[r][0], sk[r][1], sk[r][2], T[j], T[3 + j], T[6 + j]);
      }
      Ad[t] = ad;
    }
    __syncwarp();
    for (int t = lane; t < 36; t += 32) {
      const int i = t / 6, j = t % 6;
      double sum = 0.0;
#pragma unroll
      for (int m = 0; m < 6; ++m) sum += H[6 * i + m] * Ad[6 * m + j];
      HA[t] = sum;  // H_tt · Ad
    }
    __syncwarp();
    for (int t = lane; t < 36; t += 32) {
      const int i = t / 6, j = t % 6;
      double sum = 0.0;
#pragma unroll
      for (int m = 0; m < 6; ++m) sum += Ad[6 * m + i] * HA[6 * m + j];
      Hss[t] = sum;  // Adᵀ · H_tt · Ad
    }
    __syncwarp();
    for (int t = lane; t < 36; t += 32) {
      const int i = t / 6, j = t % 6;
      o[t] = H[t];                                       // H_ii (exactly symmetric)
      o[36 + t] = -HA[t];                                // H_ij
      o[72 + t] = 0.5 * (Hss[6 * i + j] + Hss[6 * j + i]);  // H_jj, symmetrised (factors.cpp:141)
    }
    if (lane < 6) {
      o[108 + lane] = tot[21 + lane];  // b_i = b_t
      double sum = 0.0;
#pragma unroll
      for (int m = 0; m < 6; ++m) sum += Ad[6 * m + lane] * tot[21 + m];
      o[114 + lane] = -sum;  // b_j = -Adᵀ b_t
    }
    if (lane == 0) {
      o[120] = tot[27];
      out_inl[f] = tinl;
    }
  }
}

// Shared memory of one CTA. Every warp owns a private kStages-deep ring of source tiles that it
// fills itself with TMA bulk copies (cp.async.bulk, mbarrier completion), so warps never wait on
// each other inside the point loop; after the loop the rings are reused for the reduction.
constexpr int kStages = VG_STAGES;
using WarpTile = PointBlock;  // one Morton-ordered 64-point block of the source cloud
static_assert(kWarpTile == kPointBlock, "a warp tile is one point block");
// Per-warp FIFO of probe hits waiting for the math phase. The probe phase appends the hits of a
// tile; the math phase consumes them only in full batches of 32 (every lane busy), carrying the
// remainder over to the next tile. Entries are self-contained (the ring slot of their tile may be
// refilled before they are consumed). SoA float4 columns: conflict-free 128-bit stores / loads.
#ifndef VG_QUEUE
#define VG_QUEUE 128
#endif
constexpr int kQueue = VG_QUEUE;  // > 31 carried + kWarpTile new
static_assert(kQueue >= 31 + kWarpTile, "hit queue too small");
struct HitQueue {
  float4 a[kQueue];  // l.x l.y l.z q.x   (l = q - voxel corner, q = T_ts·mu)
  float4 b[kQueue];  // q.y q.z slot c_xx
  float4 c[kQueue];  // c_xy c_xz c_yy c_yz
  float d[kQueue];   // c_zz
  int e[kQueue];     // float64 source clouds only: the point's Morton position in the cloud
};
#ifndef VG_MAP_SMEM
#define VG_MAP_SMEM 1  // the linearize kernel reads the work item's map descriptor from shared memory
#endif
struct __align__(128) FactorSmem {
  union {
    WarpTile ring[kWarps][kStages];
  } u;
  HitQueue hq[kWarps];
  unsigned long long bar[kWarps][kStages];
  double T[12];
  float Rf[9];
#if VG_MAP_SMEM
  MapDev map;
#endif
};
static_assert(sizeof(WarpTile) * kStages >= sizeof(double) * 180, "epilogue scratch must fit in the warp's ring");

#ifndef VG_MINB
#define VG_MINB 2
#endif
// kRank: the target maps carry occupancy bitmaps with brick ranks and rank-ordered statistics
// (MapDev::sa / sb indexed by rank): a probe is ONE 16-B load of the brick record, spatially
// coherent across the Morton-ordered lanes, instead of two hash-bucket loads (one of them random).
// kF64: the launch's items belong to float64 source clouds (their float64 means are transformed
// instead of the float32 tile copies); such items follow the float32 ones and run in their own
// launch, so the float32 kernel keeps its register budget. item_base: first item of this launch.
template <bool kLinearize, bool kRank, bool kF64>
#ifdef VG_MAXNREG  // experiment switch: explicit register cap instead of the occupancy-derived one
#define VG_FACTOR_BOUNDS __maxnreg__(VG_MAXNREG)
#else
#define VG_FACTOR_BOUNDS __launch_bounds__(kFactorThreads, VG_MINB)
#endif
__global__ void VG_FACTOR_BOUNDS factor_kernel(
    const FactorDev* __restrict__ factors, const WorkItem* __restrict__ items, int item_base,
    const double* __restrict__ poses, double* __restrict__ partials, int* __restrict__ part_inl,
    unsigned* __restrict__ counters, double* __restrict__ out, int* __restrict__ out_inl) {
  constexpr int kAcc = kLinearize ? kLinAcc : 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  FactorSmem& sm = *reinterpret_cast<FactorSmem*>(smem_raw);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const WorkItem w = items[blockIdx.x];  // `items` starts at this launch's first item
  const FactorDev* __restrict__ fp = factors + w.factor;
  VG_CHECK(w.begin >= 0 && w.begin < w.end && w.end <= fp->n && w.begin % kPointBlock == 0);
  const PointBlock* __restrict__ gblk = fp->blk + w.begin / kPointBlock;
  // float64 means of the same blocks when the cloud is not float32-exact (submap clouds): the
  // transform reads them instead of the tile's float32 copies (warp-uniform branch)
  const PointBlock64* __restrict__ gblk64 = kF64 ? fp->blk64 + w.begin / kPointBlock : nullptr;
  // Warp `warp` processes the item's 64-point tiles warp, warp + kWarps, ... (balanced, no CTA
  // barrier in the loop); lane 0 streams them into the warp's ring with TMA bulk copies.
  const int ntiles_all = (w.end - w.begin + kWarpTile - 1) / kWarpTile;
  const int my_tiles = ntiles_all > warp ? (ntiles_all - warp + kWarps - 1) / kWarps : 0;
  unsigned long long* bars = sm.bar[warp];
  auto issue_tile = [&](int k) {  // k-th tile of this warp (one 64-point block) -> ring slot k % kStages
    const int stage = k % kStages;
    mbar_expect_tx(&bars[stage], static_cast<unsigned>(sizeof(PointBlock)));
    bulk_g2s(&sm.u.ring[warp][stage], gblk + warp + k * kWarps, static_cast<unsigned>(sizeof(PointBlock)),
             &bars[stage]);
  };
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < kStages; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < kStages && k < my_tiles; ++k) issue_tile(k);
  }
  if (tid < 12) sm.T[tid] = relative_pose_entry(poses + 12 * fp->tgt, poses + 12 * fp->src, tid);
#if VG_MAP_SMEM
  static_assert(sizeof(MapDev) % 4 == 0, "MapDev is copied as words");
  if (tid >= 32 && tid < 32 + static_cast<int>(sizeof(MapDev) / 4))
    reinterpret_cast<unsigned*>(&sm.map)[tid - 32] = reinterpret_cast<const unsigned*>(&fp->map)[tid - 32];
#endif
  __syncthreads();
  if (tid < 9) sm.Rf[tid] = (float)sm.T[tid];
  __syncthreads();

  // The linearize kernel reads the map descriptor (20 words) from shared memory instead of holding it
  // in registers: it then fits its 128 registers without spills or rematerialised reloads (C3
  // linearize 1.350 -> 1.317 ms); the error-only kernel has registers to spare and is faster with
  // the register copy (1.110 vs 1.172 ms).
  MapDev map_regs;
  if constexpr (!(kLinearize && VG_MAP_SMEM)) map_regs = fp->map;
  const MapDev& map = (kLinearize && VG_MAP_SMEM) ? sm.map : map_regs;
  const double* T = sm.T;  // T_ts stays in shared memory (broadcast reads)
  HitQueue& hq = sm.hq[warp];
  const unsigned lane_lt = (1u << lane) - 1u;

  float acc[kAcc];
#pragma unroll
  for (int k = 0; k < kAcc; ++k) acc[k] = 0.f;
  int inl = 0;
  unsigned head = 0, tail = 0;  // hit queue cursors (warp-uniform)

  // ---- math phase for one queued hit ----
  auto consume = [&](unsigned idx) {
    const float4 qa = hq.a[idx];
    const float4 qb = hq.b[idx];
    const float4 qc = hq.c[idx];
    const int sl = __float_as_int(qb.z);
    float4 v0, v1;  // (mx my mz cxx) (cxy cxz cyy cyz)
    ldg256(map.sa + sl, reinterpret_cast<unsigned&>(v0.x), reinterpret_cast<unsigned&>(v0.y),
           reinterpret_cast<unsigned&>(v0.z), reinterpret_cast<unsigned&>(v0.w), reinterpret_cast<unsigned&>(v1.x),
           reinterpret_cast<unsigned&>(v1.y), reinterpret_cast<unsigned&>(v1.z), reinterpret_cast<unsigned&>(v1.w));
    const float2 v2 = __ldg(reinterpret_cast<const float2*>(map.sb + sl));  // czz vid
    hit_math<kLinearize, kF64>(sm.Rf, T, map, qa, qb.x, qb.y, qb.w, qc, hq.d[idx], v0, v1, v2, acc, inl, fp,
                               kF64 ? hq.e[idx] : 0);
  };

  for (int k = 0; k < my_tiles; ++k) {
    const int stage = k % kStages;
    while (!mbar_try_wait(&bars[stage], (k / kStages) & 1)) {
    }
    const WarpTile& tb = sm.u.ring[warp][stage];
    const int tile_n = min(kWarpTile, w.end - (w.begin + (warp + k * kWarps) * kWarpTile));

    // ---- probe phase: kILP points per lane — fp64 transform (reference op order, T_ts in
    //      registers for this tile only), exact key, both bucket loads of all points issued before
    //      any compare ----
#ifndef VG_T_REGS
#define VG_T_REGS 1
#endif
#if VG_T_REGS
    double Tr[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) Tr[q] = T[q];
#else
    const double* Tr = T;  // broadcast shared-memory reads inside the transform
#endif
    unsigned hi[kILP], lo[kILP], b1[kILP], b2[kILP];
    float l0[kILP], l1[kILP], l2[kILP], q0[kILP], q1[kILP], q2[kILP], cxx[kILP];
    bool ok[kILP];
#pragma unroll
    for (int u = 0; u < kILP; ++u) {
      const int p = u * 32 + lane;
      const int lp = min(p, tile_n - 1);  // clamped: every lane computes, in-range lanes count
      const float4 A = tb.pa[lp];
      cxx[u] = A.w;  // error-only pass: kept in a register (the strided .w re-read at append time is
                     // a 4-way bank conflict); the linearize pass re-reads it (no registers to spare)
      double px = A.x, py = A.y, pz = A.z;
      if constexpr (kF64) {
        const PointBlock64* __restrict__ b64 = gblk64 + warp + k * kWarps;
        px = __ldg(&b64->x[lp]), py = __ldg(&b64->y[lp]), pz = __ldg(&b64->z[lp]);
      }
      double qd0, qd1, qd2;
      apply_pose_rn(Tr, px, py, pz, qd0, qd1, qd2);
      unsigned k0 = 0, k1 = 0, k2 = 0;
      double ld0, ld1, ld2;
      ok[u] = voxel_key(qd0, qd1, qd2, map.res, map.inv_res, k0, k1, k2, ld0, ld1, ld2) && (p < tile_n);
      l0[u] = (float)ld0, l1[u] = (float)ld1, l2[u] = (float)ld2;
      if constexpr (kRank) {  // biased voxel coordinates, located in the bitmap below
        b1[u] = k0, b2[u] = k1, hi[u] = k2;
      } else {
        pack_key32(k0, k1, k2, hi[u], lo[u]);
        b1[u] = bucket1(k0, k1, k2, map.shift);
        b2[u] = bucket2(k0, k1, k2, map.shift);
      }
      q0[u] = (float)qd0, q1[u] = (float)qd1, q2[u] = (float)qd2;
    }
    if constexpr (kRank) {
      // ---- rank lookups: brick record (bits, rank) of every point first, then the hit test ----
      unsigned word[kILP], bit[kILP];
      bool in_box[kILP];
#pragma unroll
      for (int u = 0; u < kILP; ++u) in_box[u] = ok[u] && occ_locate(map.occ, b1[u], b2[u], hi[u], word[u], bit[u]);
      uint4 rec[kILP];
#pragma unroll
      for (int u = 0; u < kILP; ++u)
        rec[u] = in_box[u] ? __ldg(reinterpret_cast<const uint4*>(map.occ.occ + word[u])) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int u = 0; u < kILP; ++u) {
        const unsigned long long bits = (static_cast<unsigned long long>(rec[u].y) << 32) | rec[u].x;
        const bool hit = (bits >> bit[u]) & 1ull;
        const int s = static_cast<int>(rec[u].z + static_cast<unsigned>(__popcll(bits & ((1ull << bit[u]) - 1ull))));
        const unsigned ball = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int p = u * 32 + lane;
#if VG_PREFETCH >= 1  // pull the hit's statistics into L1 now; the math phase gathers them soon after
          asm volatile("prefetch.global.L1 [%0];" ::"l"(map.sa + s));
#endif
#if VG_PREFETCH >= 2
          asm volatile("prefetch.global.L1 [%0];" ::"l"(map.sb + s));
#endif
          const unsigned idx = (tail + __popc(ball & lane_lt)) % static_cast<unsigned>(kQueue);
          const float4 B = tb.pb[p];
          hq.a[idx] = make_float4(l0[u], l1[u], l2[u], q0[u]);
          hq.b[idx] = make_float4(q1[u], q2[u], __int_as_float(s), kLinearize ? tb.pa[p].w : cxx[u]);
          hq.c[idx] = B;
          hq.d[idx] = tb.pc[p];
        if constexpr (kF64) hq.e[idx] = w.begin + (warp + k * kWarps) * kPointBlock + p;
        }
        tail += __popc(ball);
      }
    } else {
#if VG_B2_LAZY
    // bucket1 first; the alternative bucket is read only when bucket1 is full and misses (a key
    // lives in its bucket2 only if its bucket1 was full when it was placed, and slots never empty)
    int sl[kILP];
    {
      uint4 A[kILP];
#pragma unroll
      for (int u = 0; u < kILP; ++u) A[u] = __ldg(reinterpret_cast<const uint4*>(map.keys + kBucket * b1[u]));
      bool need2[kILP];
      bool any2 = false;
#pragma unroll
      for (int u = 0; u < kILP; ++u) {
        int s1 = -1;
        s1 = (A[u].x == lo[u] && A[u].y == hi[u]) ? static_cast<int>(kBucket * b1[u]) : s1;
        s1 = (A[u].z == lo[u] && A[u].w == hi[u]) ? static_cast<int>(kBucket * b1[u] + 1) : s1;
        sl[u] = s1;
        need2[u] = ok[u] && s1 < 0 && A[u].y != 0xFFFFFFFFu && A[u].w != 0xFFFFFFFFu;
        any2 |= need2[u];
      }
      if (__any_sync(0xffffffffu, any2)) {
#pragma unroll
        for (int u = 0; u < kILP; ++u) {
          if (need2[u]) {
            const uint4 B = ldg_bucket2(map.keys + kBucket * b2[u]);
            int s2 = -1;
            s2 = (B.x == lo[u] && B.y == hi[u]) ? static_cast<int>(kBucket * b2[u]) : s2;
            s2 = (B.z == lo[u] && B.w == hi[u]) ? static_cast<int>(kBucket * b2[u] + 1) : s2;
            sl[u] = s2;
          }
        }
      }
    }
#else
    BucketPair bp[kILP];
#pragma unroll
    for (int u = 0; u < kILP; ++u) bp[u] = load_buckets(map.keys, b1[u], b2[u]);  // always in-bounds
#endif
#pragma unroll
    for (int u = 0; u < kILP; ++u) {
#if VG_B2_LAZY
      const int s = sl[u];
#else
      const int s = match_buckets(bp[u], b1[u], b2[u], hi[u], lo[u]);
#endif
      const bool hit = ok[u] && s >= 0;
      const unsigned ball = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const int p = u * 32 + lane;
        const unsigned idx = (tail + __popc(ball & lane_lt)) % static_cast<unsigned>(kQueue);
        const float4 B = tb.pb[p];
        hq.a[idx] = make_float4(l0[u], l1[u], l2[u], q0[u]);
        hq.b[idx] = make_float4(q1[u], q2[u], __int_as_float(s), kLinearize ? tb.pa[p].w : cxx[u]);
        hq.c[idx] = B;
        hq.d[idx] = tb.pc[p];
        if constexpr (kF64) hq.e[idx] = w.begin + (warp + k * kWarps) * kPointBlock + p;
      }
      tail += __popc(ball);
    }
    }  // kRank
    __syncwarp();  // queue entries visible; the warp is done with this ring slot
    if (lane == 0 && k + kStages < my_tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async refill
      issue_tile(k + kStages);
    }

    // ---- math phase: full batches of 32 queued hits (all lanes busy) ----
    while (tail - head >= 32u) {
      consume((head + lane) % static_cast<unsigned>(kQueue));
      head += 32u;
      __syncwarp();
    }
  }
  if (head + lane < tail) consume((head + lane) % static_cast<unsigned>(kQueue));  // the last partial batch
  __syncwarp();  // this warp is done with its ring (no CTA-wide barrier after the prologue)

  finish_factor<kLinearize>(acc, inl, lane, (size_t)(item_base + blockIdx.x) * kWarps + warp, kWarps, w, fp, sm.T,
                            reinterpret_cast<double*>(&sm.u.ring[warp][0]), partials, part_inl, counters, out, out_inl);
}

// gicp_error (factors.cpp:75-88) in fp64, bit-identical to the oracle.
// in: src_mean(3) src_cov(9) tgt_mean(3) tgt_cov(9) T(12); out: error, residual(3), info(9), valid
__global__ void gicp_error_kernel(const double* __restrict__ in, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double* sm = in;
  const double* sc = in + 3;
  const double* tm = in + 12;
  const double* tc = in + 15;
  const double* T = in + 24;
  double q0, q1, q2;
  apply_pose_rn(T, sm[0], sm[1], sm[2], q0, q1, q2);
  const double d0 = __dsub_rn(tm[0], q0), d1 = __dsub_rn(tm[1], q1), d2 = __dsub_rn(tm[2], q2);
  out[1] = d0;
  out[2] = d1;
  out[3] = d2;
  double M[9], O[9];
  combined_cov_rn(T, sc, tc, M);
  if (!invert_covariance_rn(M, O)) {
    out[0] = 0.0;
    for (int k = 0; k < 9; ++k) out[4 + k] = 0.0;
    out[13] = 0.0;
    return;
  }
  for (int k = 0; k < 9; ++k) out[4 + k] = O[k];
  const double w0 = dot3_rn(O[0], O[1], O[2], d0, d1, d2);
  const double w1 = dot3_rn(O[3], O[4], O[5], d0, d1, d2);
  const double w2 = dot3_rn(O[6], O[7], O[8], d0, d1, d2);
  out[0] = dot3_rn(d0, d1, d2, w0, w1, w2);
  out[13] = 1.0;
}


// Device-side assemble_normal_equations (block_solver.cpp:14-62): one CTA per output block, one
// thread per entry (36 H entries + 6 rhs entries for diagonal outputs), contributions summed in
// factor order starting from zero — the reference's `block += H` sequence, so the assembled system
// is bit-identical to a host assembly of the same factor blocks.
__global__ void assemble_kernel(const int* __restrict__ out_ptr, const int* __restrict__ contrib, int num_slots,
                                int num_outputs, const ShardBlocks blocks, double* __restrict__ assembled) {
  const int o = blockIdx.x;
  const int t = threadIdx.x;
  if (t >= 42 || (t >= 36 && o >= num_slots)) return;
  double sum = 0.0;
  for (int c = out_ptr[o]; c < out_ptr[o + 1]; ++c) {
    const int code = contrib[c];
    const int f = code >> 2;
    int r = 0;  // the shard holding factor f (a peer device's memory for a sharded graph)
    while (r + 1 < blocks.n && f >= blocks.first[r + 1]) ++r;
    VG_CHECK(f >= blocks.first[r] && f < blocks.first[r + 1]);
    const double* B = blocks.out[r] + (size_t)(f - blocks.first[r]) * VGICP_LINEARIZED_DOUBLES;
    const int kind = code & 3;
    double v;
    if (t < 36) {
      v = kind == 0 ? B[t] : kind == 1 ? B[72 + t] : kind == 2 ? B[36 + t] : B[36 + (t % 6) * 6 + t / 6];
    } else {
      v = B[(kind == 0 ? 108 : 114) + (t - 36)];
    }
    sum = __dadd_rn(sum, v);
  }
  if (t < 36) assembled[(size_t)o * 36 + t] = sum;
  else assembled[(size_t)num_outputs * 36 + (size_t)o * 6 + (t - 36)] = sum;
}
}  // namespace

cudaError_t launch_assemble(const int* out_ptr, const int* contrib, int num_slots, int num_outputs,
                            const ShardBlocks& blocks, double* assembled, cudaStream_t s) {
  if (num_outputs <= 0) return cudaSuccess;
  assemble_kernel<<<num_outputs, 64, 0, s>>>(out_ptr, contrib, num_slots, num_outputs, blocks, assembled);
  return cudaGetLastError();
}

cudaError_t launch_factor(bool linearize, bool rank, const FactorDev* factors, const WorkItem* items, int num_items,
                          int f64_begin, const double* poses, double* partials, int* part_inl, unsigned* counters,
                          int num_factors, double* out, int* out_inl, cudaStream_t s) {
  if (num_items <= 0) return cudaSuccess;
  constexpr size_t kSmem = sizeof(FactorSmem);
  // the > 48 KB shared-memory opt-in is a per-device function attribute: set it once per device
  // (a context on another GPU of the same process needs its own), thread-safely
  static std::atomic<unsigned long long> configured{0ull};
  int dev = 0;
  if (const cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    for (const void* k : {reinterpret_cast<const void*>(factor_kernel<true, false, false>),
                          reinterpret_cast<const void*>(factor_kernel<false, false, false>),
                          reinterpret_cast<const void*>(factor_kernel<true, true, false>),
                          reinterpret_cast<const void*>(factor_kernel<false, true, false>),
                          reinterpret_cast<const void*>(factor_kernel<true, false, true>),
                          reinterpret_cast<const void*>(factor_kernel<false, false, true>),
                          reinterpret_cast<const void*>(factor_kernel<true, true, true>),
                          reinterpret_cast<const void*>(factor_kernel<false, true, true>)}) {
      const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
      if (e != cudaSuccess) return e;
    }
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  f64_begin = f64_begin < 0 ? num_items : (f64_begin > num_items ? num_items : f64_begin);
  auto go = [&](auto kernel, int base, int count) {
    if (count > 0)
      kernel<<<count, kFactorThreads, kSmem, s>>>(factors, items + base, base, poses, partials, part_inl, counters,
                                                  out, out_inl);
  };
  auto both = [&](auto k32, auto k64) {
    go(k32, 0, f64_begin);
    go(k64, f64_begin, num_items - f64_begin);
  };
  if (linearize) {
    if (rank) both(factor_kernel<true, true, false>, factor_kernel<true, true, true>);
    else both(factor_kernel<true, false, false>, factor_kernel<true, false, true>);
  } else {
    if (rank) both(factor_kernel<false, true, false>, factor_kernel<false, true, true>);
    else both(factor_kernel<false, false, false>, factor_kernel<false, false, true>);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && num_factors > 0)  // a launch that did not run must not leave arrivals behind
    cudaMemsetAsync(counters, 0, sizeof(unsigned) * num_factors, s);
  return e;
}

cudaError_t launch_gicp_error(const double* in, double* out, cudaStream_t s) {
  gicp_error_kernel<<<1, 32, 0, s>>>(in, out);
  return cudaGetLastError();
}

}  // namespace vgicp
