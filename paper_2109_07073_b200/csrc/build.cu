// Hand-written batched Gaussian voxel-map build for float32 clouds (GaussianVoxelMap ctor,
// voxelmap.cpp:65-104; VoxelAccumulator + KahanSum, voxelmap.cpp:23-41 / parallel.hpp:97-114), one
// launch per stage for all maps of a batch, no library sort:
//
//   fast_zero        clear every map's occupancy bitmap (the box is known on the host: floor(p/r) is
//                    monotone, so the voxel box of the cloud's finite bounding box is exact)
//   fast_mark        per point: fp64 key (exact floor(p/r), ±2^20 check), brick record / bit of the
//                    voxel in the map's box; warp-aggregated atomicOr of the bits (points in input
//                    order are spatially coherent); per-point code = word·64 + bit
//   fast_rank        per map (one CTA): exclusive prefix of the records' popcounts -> brick ranks,
//                    V = occupied voxels. A voxel's id is its RANK (brick order), the same number the
//                    factor kernels compute from the bitmap — no key sort anywhere.
//   fast_order       per map (one CTA): per-voxel point counts (shared-memory atomics), exclusive scan
//                    -> CSR offsets, then ONE warp walks the points in input order and scatters each
//                    to its voxel's next list position (__match_any_sync ranks equal voxels inside the
//                    32-point step), so every voxel's list is in input order: a stable counting sort
//   fast_accumulate  thread per voxel: Kahan fp64 sums over its list in input order — exactly the
//                    reference's per-shard order (voxelmap.cpp:87-94), hence bit-identical statistics
//                    — finalize, and write the rank-ordered fp32 voxel-local statistics (ra / rb,
//                    the factor kernels' gather targets) and the fp64 covariance (the near-singular
//                    fallback). Key-ordered arrays (keys, counts, fp64 means) are produced only on
//                    demand (export mode), by the same kernels.
//
// Algorithmic bytes: 36 B per input point + 48 B per voxel written.
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace vgicp {

namespace {

__device__ __forceinline__ void kahan_add(double& sum, double& comp, double value) {  // parallel.hpp:106-111
  const double y = __dsub_rn(value, comp);
  const double t = __dadd_rn(sum, y);
  comp = __dsub_rn(__dsub_rn(t, sum), y);
  sum = t;
}

__global__ void fast_zero_kernel(const FastBuildJob* __restrict__ jobs) {
  const FastBuildJob& j = jobs[blockIdx.y];
  const unsigned words = j.words;
  OccWord* occ = j.occ;
  for (unsigned w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x)
    occ[w] = OccWord{0ull, 0u, 0u};
}

__global__ void __launch_bounds__(256) fast_mark_kernel(const FastBuildJob* __restrict__ jobs,
                                                        unsigned* __restrict__ code, int* __restrict__ err) {
  const FastBuildJob& j = jobs[blockIdx.y];
  const unsigned n = j.n;
  const float4* __restrict__ pa = j.pa;
  const double res = j.res, inv_res = j.inv_res;
  const unsigned kx0 = j.kx0, ky0 = j.ky0, kz0 = j.kz0, ex = j.ex, ey = j.ey, ez = j.ez, nby = j.nby, nbz = j.nbz;
  OccWord* __restrict__ occ = j.occ;
  unsigned* __restrict__ out = code + j.pt_off;
  const unsigned lane = threadIdx.x & 31;
  bool bad = false;
  // whole warps iterate together (the base is block-uniform): the match below needs all 32 lanes
  for (unsigned base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const unsigned i = base + threadIdx.x;
    unsigned word = 0xFFFFFFFFu, bit = 0u;
    if (i < n) {
      const float4 a = __ldg(pa + i);
      unsigned k0, k1, k2;
      double l0, l1, l2;
      bool ok = voxel_key(a.x, a.y, a.z, res, inv_res, k0, k1, k2, l0, l1, l2);
      const unsigned rx = k0 - kx0, ry = k1 - ky0, rz = k2 - kz0;
      ok = ok && rx < ex && ry < ey && rz < ez;  // always inside for finite in-range points
      if (ok) {
        word = ((rx >> 2) * nby + (ry >> 2)) * nbz + (rz >> 2);
        bit = ((rx & 3u) << 4) | ((ry & 3u) << 2) | (rz & 3u);
        VG_CHECK(word < j.words);
      } else {
        bad = true;
      }
      out[i] = ok ? (word << 6) | bit : 0xFFFFFFFFu;
    }
    // one atomicOr per distinct brick record of the warp
    const unsigned peers = __match_any_sync(0xffffffffu, word);
    const unsigned long long m = word != 0xFFFFFFFFu ? (1ull << bit) : 0ull;
    const unsigned lo = __reduce_or_sync(peers, static_cast<unsigned>(m));
    const unsigned hi = __reduce_or_sync(peers, static_cast<unsigned>(m >> 32));
    if (word != 0xFFFFFFFFu && lane == static_cast<unsigned>(__ffs(peers) - 1))
      atomicOr(&occ[word].bits, (static_cast<unsigned long long>(hi) << 32) | lo);
  }
  if (bad) atomicOr(&err[blockIdx.y], 1);
}

// One CTA per map: brick ranks = exclusive prefix of the records' popcounts; V = the total.
__global__ void __launch_bounds__(1024) fast_rank_kernel(const FastBuildJob* __restrict__ jobs,
                                                         unsigned* __restrict__ vcount) {
  const FastBuildJob& j = jobs[blockIdx.x];
  OccWord* __restrict__ occ = j.occ;
  const unsigned words = j.words;
  __shared__ unsigned warp_sums[32];
  __shared__ unsigned carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (unsigned w0 = 0; w0 < words; w0 += 1024) {
    const unsigned w = w0 + threadIdx.x;
    const unsigned c = w < words ? static_cast<unsigned>(__popcll(occ[w].bits)) : 0u;
    unsigned x = c;  // inclusive warp scan
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= static_cast<unsigned>(off)) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      unsigned t = warp_sums[lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, t, off);
        if (lane >= static_cast<unsigned>(off)) t += y;
      }
      warp_sums[lane] = t;
    }
    __syncthreads();
    if (w < words) occ[w].rank = carry + (warp ? warp_sums[warp - 1] : 0u) + (x - c);
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) vcount[blockIdx.x] = carry;
}

// Maps whose bitmap fits in shared memory (C3's 1 m maps: ~8k records): zero, mark and rank in one
// CTA per map — the bit marking is shared-memory atomics (no L2 atomic traffic, no contention on the
// records of dense bricks), then the ranked records are written out once.
constexpr int kMarkThreads = 1024;
__global__ void __launch_bounds__(kMarkThreads) fast_markrank_smem_kernel(const FastBuildJob* __restrict__ jobs,
                                                                          unsigned* __restrict__ code,
                                                                          int* __restrict__ err,
                                                                          unsigned* __restrict__ vcount) {
  extern __shared__ unsigned sbits[];  // 2 words (lo, hi) per brick record
  __shared__ unsigned warp_sums[32];
  __shared__ unsigned carry;
  const int k = blockIdx.x;
  const FastBuildJob& j = jobs[k];
  const unsigned n = j.n, words = j.words;
  const float4* __restrict__ pa = j.pa;
  const double res = j.res, inv_res = j.inv_res;
  const unsigned kx0 = j.kx0, ky0 = j.ky0, kz0 = j.kz0, ex = j.ex, ey = j.ey, ez = j.ez, nby = j.nby, nbz = j.nbz;
  unsigned* __restrict__ out = code + j.pt_off;
  for (unsigned w = threadIdx.x; w < 2 * words; w += kMarkThreads) sbits[w] = 0u;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  bool bad = false;
  constexpr int kU = 2;  // points per thread in flight
  for (unsigned base = 0; base < n; base += kU * kMarkThreads) {
    float4 a[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned i = base + u * kMarkThreads + threadIdx.x;
      a[u] = i < n ? __ldg(pa + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned i = base + u * kMarkThreads + threadIdx.x;
      if (i >= n) continue;
      unsigned k0, k1, k2;
      double l0, l1, l2;
      bool ok = voxel_key(a[u].x, a[u].y, a[u].z, res, inv_res, k0, k1, k2, l0, l1, l2);
      const unsigned rx = k0 - kx0, ry = k1 - ky0, rz = k2 - kz0;
      ok = ok && rx < ex && ry < ey && rz < ez;
      unsigned c = 0xFFFFFFFFu;
      if (ok) {
        const unsigned word = ((rx >> 2) * nby + (ry >> 2)) * nbz + (rz >> 2);
        const unsigned bit = ((rx & 3u) << 4) | ((ry & 3u) << 2) | (rz & 3u);
        VG_CHECK(word < words);
        atomicOr(&sbits[2 * word + (bit >> 5)], 1u << (bit & 31u));
        c = (word << 6) | bit;
      } else {
        bad = true;
      }
      out[i] = c;
    }
  }
  if (bad) atomicOr(&err[k], 1);
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  OccWord* __restrict__ occ = j.occ;
  for (unsigned w0 = 0; w0 < words; w0 += kMarkThreads) {
    const unsigned w = w0 + threadIdx.x;
    const unsigned long long bits =
        w < words ? (static_cast<unsigned long long>(sbits[2 * w + 1]) << 32) | sbits[2 * w] : 0ull;
    const unsigned c = static_cast<unsigned>(__popcll(bits));
    unsigned x = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= static_cast<unsigned>(off)) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      unsigned t = warp_sums[lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, t, off);
        if (lane >= static_cast<unsigned>(off)) t += y;
      }
      warp_sums[lane] = t;
    }
    __syncthreads();
    if (w < words) occ[w] = OccWord{bits, carry + (warp ? warp_sums[warp - 1] : 0u) + (x - c), 0u};
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) vcount[k] = carry;
}

constexpr int kOrderThreads = 512;

// Block-wide exclusive scan of cnt[0, V) in place (each thread owns a contiguous run).
__device__ void block_exclusive_scan(volatile unsigned* cnt, unsigned V, unsigned* warp_sums) {
  const unsigned per = (V + kOrderThreads - 1) / kOrderThreads;
  const unsigned b = threadIdx.x * per, e = min(V, b + per);
  unsigned local = 0;
  for (unsigned v = b; v < e; ++v) local += cnt[v];
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= static_cast<unsigned>(off)) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned t = lane < kOrderThreads / 32 ? warp_sums[lane] : 0u;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, t, off);
      if (lane >= static_cast<unsigned>(off)) t += y;
    }
    if (lane < kOrderThreads / 32) warp_sums[lane] = t;
  }
  __syncthreads();
  unsigned run = (warp ? warp_sums[warp - 1] : 0u) + (x - local);
  for (unsigned v = b; v < e; ++v) {
    const unsigned c = cnt[v];
    cnt[v] = run;
    run += c;
  }
  __syncthreads();
}

template <bool kSmem>
__global__ void __launch_bounds__(kOrderThreads) fast_order_kernel(const FastBuildJob* __restrict__ jobs,
                                                                   const int* __restrict__ idx,
                                                                   const unsigned* __restrict__ code,
                                                                   unsigned* __restrict__ rank,
                                                                   unsigned* __restrict__ list,
                                                                   unsigned* __restrict__ offs,
                                                                   unsigned* __restrict__ gcnt) {
  extern __shared__ unsigned smem_cnt[];
  __shared__ unsigned warp_sums[32];
  const FastBuildJob& j = jobs[idx[blockIdx.x]];
  const unsigned n = j.n, V = j.V;
  volatile unsigned* cnt = kSmem ? smem_cnt : gcnt + j.vx_off;
  const unsigned* __restrict__ pcode = code + j.pt_off;
  unsigned* __restrict__ pc = rank + j.pt_off;  // per-point ranks (the codes stay: accumulate reads them)
  const OccWord* __restrict__ occ = j.occ;
  for (unsigned v = threadIdx.x; v < V; v += kOrderThreads) cnt[v] = 0u;
  __syncthreads();
  // per-point rank (brick rank + popcount of the lower bits) and per-voxel counts
  constexpr int kU = 4;  // points per thread in flight (code -> record -> rank is a dependent chain)
  for (unsigned base = 0; base < n; base += kU * kOrderThreads) {
    unsigned c[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned i = base + u * kOrderThreads + threadIdx.x;
      c[u] = i < n ? pcode[i] : 0u;
    }
    OccWord o[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) o[u] = occ[c[u] >> 6];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned i = base + u * kOrderThreads + threadIdx.x;
      if (i >= n) continue;
      const unsigned r = o[u].rank + static_cast<unsigned>(__popcll(o[u].bits & ((1ull << (c[u] & 63u)) - 1ull)));
      VG_CHECK(r < V);
      pc[i] = r;
      atomicAdd(const_cast<unsigned*>(cnt + r), 1u);
    }
  }
  __syncthreads();
  block_exclusive_scan(cnt, V, warp_sums);
  unsigned* __restrict__ off = offs + j.vx_off;
  for (unsigned v = threadIdx.x; v < V; v += kOrderThreads) off[v] = cnt[v];
  if (threadIdx.x == 0) off[V] = n;
  __syncthreads();  // every start offset is read before the scatter advances the cursors
  if (threadIdx.x >= 32) return;
  // stable scatter: one warp walks the points in input order; equal voxels inside a 32-point step
  // are ranked by lane (match_any), so every voxel's list keeps input order
  const unsigned lane = threadIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  unsigned* __restrict__ pl = list + j.pt_off;
  // the ranks of the next kDepth steps are loaded while the current kDepth steps run (each step is
  // only a match, a shared read and a shared write: the loads must be far ahead)
  constexpr int kDepth = 16;
  unsigned cur[kDepth];
#pragma unroll
  for (int q = 0; q < kDepth; ++q) {
    const unsigned i = q * 32 + lane;
    cur[q] = i < n ? __ldcg(pc + i) : 0xFFFFFFFFu;
  }
  for (unsigned base = 0; base < n; base += kDepth * 32) {
    unsigned nxt[kDepth];
#pragma unroll
    for (int q = 0; q < kDepth; ++q) {
      const unsigned i = base + (kDepth + q) * 32 + lane;
      nxt[q] = i < n ? __ldcg(pc + i) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int q = 0; q < kDepth; ++q) {
      const unsigned i = base + q * 32 + lane;
      const unsigned r = cur[q];
      const unsigned peers = __match_any_sync(0xffffffffu, r);
      unsigned pos = 0;
      if (i < n) pos = cnt[r] + static_cast<unsigned>(__popc(peers & lt));
      __syncwarp();
      if (i < n && (peers & lt) == 0u) cnt[r] += static_cast<unsigned>(__popc(peers));
      __syncwarp();
      VG_CHECK(i >= n || pos < n);
      if (i < n) pl[pos] = i;
    }
#pragma unroll
    for (int q = 0; q < kDepth; ++q) cur[q] = nxt[q];
  }
}

// Per-map stable counting sort as a hand-written LSD radix sort in shared memory (maps of <=
// kRadixMaxPoints points): keys (rank << 16 | point index) in input order, 4-bit digits of the rank,
// ceil(bits(V-1) / 4) passes. Each thread owns a contiguous run of k (odd: conflict-free) items and
// its own column of 16 digit counters, so a pass is: count the run, one block-wide exclusive scan over
// the 16 × 1024 counters (digit-major), scatter the run in order — stable without any warp-serial
// step. The sorted keys ARE the per-voxel lists in input order; run heads give the CSR offsets.
constexpr int kRadixThreads = 1024;
template <int kBits>
constexpr unsigned radix_counter_bytes() {
  return sizeof(unsigned short) * (1u << kBits) * kRadixThreads;  // 32 KB (4-bit digits) / 64 KB (5-bit)
}

template <int kBits>
__device__ void radix_block_scan(unsigned short* cnt, unsigned* warp_sums) {
  // exclusive scan over cnt[0, D·1024) in place; thread t owns entries [D·t, D·t + D), D = 2^kBits
  constexpr int kPer = 1 << kBits;
  constexpr int kWords = kPer / 2;  // u16 pairs
  uint4* my = reinterpret_cast<uint4*>(cnt + kPer * threadIdx.x);
  unsigned ws[kWords];
#pragma unroll
  for (int q = 0; q < kWords / 4; ++q) {
    const uint4 w = my[q];
    ws[4 * q] = w.x, ws[4 * q + 1] = w.y, ws[4 * q + 2] = w.z, ws[4 * q + 3] = w.w;
  }
  unsigned v[kPer];
#pragma unroll
  for (int q = 0; q < kWords; ++q) v[2 * q] = ws[q] & 0xFFFFu, v[2 * q + 1] = ws[q] >> 16;
  unsigned local = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) local += v[q];
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= static_cast<unsigned>(off)) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned t = warp_sums[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, t, off);
      if (lane >= static_cast<unsigned>(off)) t += y;
    }
    warp_sums[lane] = t;
  }
  __syncthreads();
  unsigned run = (warp ? warp_sums[warp - 1] : 0u) + (x - local);
  unsigned o[kWords];
#pragma unroll
  for (int q = 0; q < kWords; ++q) {
    const unsigned a = run;
    run += v[2 * q];
    const unsigned b = run;
    run += v[2 * q + 1];
    o[q] = a | (b << 16);
  }
#pragma unroll
  for (int q = 0; q < kWords / 4; ++q) my[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
}

template <int kBits>
__global__ void __launch_bounds__(kRadixThreads) fast_sort_kernel(const FastBuildJob* __restrict__ jobs,
                                                                  const int* __restrict__ idx,
                                                                  const unsigned* __restrict__ code,
                                                                  unsigned* __restrict__ list,
                                                                  unsigned* __restrict__ offs) {
  extern __shared__ __align__(16) unsigned char rsm[];
  __shared__ unsigned warp_sums[32];
  const FastBuildJob& j = jobs[idx[blockIdx.x]];
  const unsigned n = j.n, V = j.V;
  constexpr unsigned kDigits = 1u << kBits;
  unsigned short* cnt = reinterpret_cast<unsigned short*>(rsm);
  unsigned* src = reinterpret_cast<unsigned*>(rsm + radix_counter_bytes<kBits>());
  unsigned* dst = src + n;
  const unsigned* __restrict__ pc = code + j.pt_off;
  const OccWord* __restrict__ occ = j.occ;
  // keys in input order: rank (brick rank + popcount of the lower bits) << 16 | point index
  constexpr int kU = 4;
  for (unsigned base = 0; base < n; base += kU * kRadixThreads) {
    unsigned c[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned i = base + u * kRadixThreads + threadIdx.x;
      c[u] = i < n ? pc[i] : 0u;
    }
    OccWord o[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) o[u] = occ[c[u] >> 6];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned i = base + u * kRadixThreads + threadIdx.x;
      if (i < n) {
        VG_CHECK((c[u] >> 6) < j.words);
        const unsigned r = o[u].rank + static_cast<unsigned>(__popcll(o[u].bits & ((1ull << (c[u] & 63u)) - 1ull)));
        VG_CHECK(r < V && ((o[u].bits >> (c[u] & 63u)) & 1ull));
        src[i] = (r << 16) | i;
      }
    }
  }
  unsigned bits = 0;
  while (bits < 16 && ((V - 1u) >> bits) != 0u) bits += kBits;  // digits needed for the largest rank
  unsigned k = (n + kRadixThreads - 1) / kRadixThreads;
  k |= 1u;  // odd run length: the runs' first items fall in distinct banks
  const unsigned b0 = min(n, threadIdx.x * k), e0 = min(n, b0 + k);
  __syncthreads();
  for (unsigned shift = 16; shift < 16 + bits; shift += kBits) {
#pragma unroll
    for (unsigned d = 0; d < kDigits; ++d) cnt[d * kRadixThreads + threadIdx.x] = 0;
    for (unsigned i = b0; i < e0; ++i) ++cnt[((src[i] >> shift) & (kDigits - 1u)) * kRadixThreads + threadIdx.x];
    __syncthreads();
    radix_block_scan<kBits>(cnt, warp_sums);
    __syncthreads();
    for (unsigned i = b0; i < e0; ++i) {
      const unsigned key = src[i];
      unsigned short& slot = cnt[((key >> shift) & (kDigits - 1u)) * kRadixThreads + threadIdx.x];
      VG_CHECK(slot < n);
      dst[slot] = key;
      ++slot;
    }
    __syncthreads();
    unsigned* t = src;
    src = dst;
    dst = t;
  }
  // sorted by (rank, index): the per-voxel lists in input order; run heads are the CSR offsets
  unsigned* __restrict__ pl = list + j.pt_off;
  unsigned* __restrict__ off = offs + j.vx_off;
  for (unsigned q = threadIdx.x; q < n; q += kRadixThreads) {
    const unsigned key = src[q];
    pl[q] = key & 0xFFFFu;
    if (q == 0 || (src[q - 1] >> 16) != (key >> 16)) off[key >> 16] = q;
  }
  if (threadIdx.x == 0) off[V] = n;
}

// Accumulation, warp-cooperative: a warp owns 32 consecutive voxels, whose point lists are ONE
// contiguous CSR range (~45 points). The warp loads the range's list entries coalesced, gathers all of
// the range's point records at once (every lane a different point: the gathers are independent and in
// flight together) into shared memory, and then each lane folds its own voxel's points from there in
// input order. The voxel's key comes from its first point's code (brick record / bit), no fp64 redo.
constexpr int kAccThreads = 256;
constexpr int kAccWarps = kAccThreads / 32;
constexpr int kStage = 64;  // staged points per warp and round

template <bool kExport>
#ifndef VG_ACC_MINB
#define VG_ACC_MINB 3
#endif
__global__ void __launch_bounds__(kAccThreads, VG_ACC_MINB) fast_accumulate_kernel(const FastBuildJob* __restrict__ jobs,
                                                                         const unsigned* __restrict__ list,
                                                                         const unsigned* __restrict__ offs,
                                                                         const unsigned* __restrict__ code) {
  __shared__ float4 sA[kAccWarps][kStage];
  __shared__ float4 sB[kAccWarps][kStage];
  __shared__ float sZ[kAccWarps][kStage];
  constexpr int kCovW = kExport ? 9 : 6;  // row-major 3×3 for export, else the 6 unique entries
  __shared__ __align__(16) double stage[kAccWarps][32 * kCovW];  // the warp's fp64 covariances, written out coalesced
  const FastBuildJob& j = jobs[blockIdx.y];
  const unsigned V = j.V;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned v0 = blockIdx.x * kAccThreads + warp * 32;
  if (v0 >= V) return;  // (warp-uniform)
  const unsigned nv = min(32u, V - v0);
  const unsigned v = v0 + lane;
  const bool act = lane < nv;
  const float4* __restrict__ pa = j.pa;
  const float4* __restrict__ pb = j.pb;
  const float* __restrict__ pcz = j.pc;
  const unsigned* __restrict__ pl = list + j.pt_off;
  const unsigned* __restrict__ off = offs + j.vx_off;
  const unsigned b = off[v0 + min(lane, nv)];  // this lane's list begin (lanes >= nv: the range end)
  const unsigned re = off[v0 + nv];             // end of the warp's range (one broadcast load)
  const unsigned nb = __shfl_down_sync(0xffffffffu, b, 1);
  const unsigned e = lane + 1 < nv ? nb : re;
  const unsigned rb = __shfl_sync(0xffffffffu, b, 0);
  VG_CHECK(!act || (b < e && e <= j.n));  // every voxel holds >= 1 point
  // VoxelAccumulator::add (voxelmap.cpp:28-32) with KahanSum, component-wise; float32 clouds have
  // symmetric covariances, so the 6 unique second-moment sums equal the reference's 9 bit for bit
  double ms[3] = {0, 0, 0}, mc[3] = {0, 0, 0};
  double ss[6] = {0, 0, 0, 0, 0, 0}, sc[6] = {0, 0, 0, 0, 0, 0};  // xx xy xz yy yz zz
  for (unsigned c0 = rb; c0 < re; c0 += kStage) {
    const unsigned cn = min(static_cast<unsigned>(kStage), re - c0);
    unsigned p[kStage / 32];
#pragma unroll
    for (int u = 0; u < kStage / 32; ++u) p[u] = lane + 32 * u < cn ? pl[c0 + lane + 32 * u] : 0u;
#pragma unroll
    for (int u = 0; u < kStage / 32; ++u) VG_CHECK(p[u] < j.n);
#pragma unroll
    for (int u = 0; u < kStage / 32; ++u) {
      if (lane + 32 * u < cn) {
        sA[warp][lane + 32 * u] = __ldg(pa + p[u]);
        sB[warp][lane + 32 * u] = __ldg(pb + p[u]);
        sZ[warp][lane + 32 * u] = __ldg(pcz + p[u]);
      }
    }
    __syncwarp();
    if (act) {
      const unsigned q1 = min(e, c0 + cn);
      for (unsigned q = max(b, c0); q < q1; ++q) {  // this lane's points of the round, in input order
        const float4 A = sA[warp][q - c0];
        const float4 B = sB[warp][q - c0];
        const float Z = sZ[warp][q - c0];
        const double m0 = A.x, m1 = A.y, m2 = A.z;
        kahan_add(ms[0], mc[0], m0);
        kahan_add(ms[1], mc[1], m1);
        kahan_add(ms[2], mc[2], m2);
        kahan_add(ss[0], sc[0], __dadd_rn((double)A.w, __dmul_rn(m0, m0)));
        kahan_add(ss[1], sc[1], __dadd_rn((double)B.x, __dmul_rn(m0, m1)));
        kahan_add(ss[2], sc[2], __dadd_rn((double)B.y, __dmul_rn(m0, m2)));
        kahan_add(ss[3], sc[3], __dadd_rn((double)B.z, __dmul_rn(m1, m1)));
        kahan_add(ss[4], sc[4], __dadd_rn((double)B.w, __dmul_rn(m1, m2)));
        kahan_add(ss[5], sc[5], __dadd_rn((double)Z, __dmul_rn(m2, m2)));
      }
    }
    __syncwarp();
  }
  if (act) {
    // finalize (voxelmap.cpp:34-40); x / 1 == x exactly, so single-point voxels skip the divisions
    const unsigned count = e - b;
    const double cnt = static_cast<double>(count);
    double mean[3], cov[6];
    const int r6[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
    if (count == 1u) {
#pragma unroll
      for (int a = 0; a < 3; ++a) mean[a] = ms[a];
#pragma unroll
      for (int q = 0; q < 6; ++q) cov[q] = __dsub_rn(ss[q], __dmul_rn(mean[r6[q][0]], mean[r6[q][1]]));
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) mean[a] = __ddiv_rn(ms[a], cnt);
#pragma unroll
      for (int q = 0; q < 6; ++q) cov[q] = __dsub_rn(__ddiv_rn(ss[q], cnt), __dmul_rn(mean[r6[q][0]], mean[r6[q][1]]));
    }
    // the voxel's biased coordinates from its first point's code: record index -> brick, bit -> cell
    const unsigned c = code[j.pt_off + pl[b]];
    const unsigned word = c >> 6, bit = c & 63u;
    const unsigned bz = word % j.nbz, t = word / j.nbz, by = t % j.nby, bx = t / j.nby;
    const unsigned k0 = j.kx0 + 4 * bx + ((bit >> 4) & 3u);
    const unsigned k1 = j.ky0 + 4 * by + ((bit >> 2) & 3u);
    const unsigned k2 = j.kz0 + 4 * bz + (bit & 3u);
    const double corner0 = __dmul_rn(static_cast<double>(static_cast<int>(k0) - (1 << 20)), j.res);
    const double corner1 = __dmul_rn(static_cast<double>(static_cast<int>(k1) - (1 << 20)), j.res);
    const double corner2 = __dmul_rn(static_cast<double>(static_cast<int>(k2) - (1 << 20)), j.res);
    SlotStatsA a;
    a.mx = static_cast<float>(__dsub_rn(mean[0], corner0));
    a.my = static_cast<float>(__dsub_rn(mean[1], corner1));
    a.mz = static_cast<float>(__dsub_rn(mean[2], corner2));
    a.cxx = static_cast<float>(cov[0]);
    a.cxy = static_cast<float>(cov[1]);
    a.cxz = static_cast<float>(cov[2]);
    a.cyy = static_cast<float>(cov[3]);
    a.cyz = static_cast<float>(cov[4]);
    j.ra[v] = a;
    j.rb[v] = SlotStatsB{static_cast<float>(cov[5]), static_cast<int>(v)};
    if constexpr (kExport) {
      const int full[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};  // row-major 3×3 from the unique entries
#pragma unroll
      for (int q = 0; q < 9; ++q) stage[warp][9 * lane + q] = cov[full[q]];
    } else {
#pragma unroll
      for (int q = 0; q < 6; ++q) stage[warp][6 * lane + q] = cov[q];
    }
    if constexpr (kExport) {
      unsigned hi, lo;
      pack_key32(k0, k1, k2, hi, lo);
      j.keys[v] = key64(hi, lo);
      j.counts[v] = static_cast<int>(count);
      j.mean64[3 * static_cast<size_t>(v) + 0] = mean[0];
      j.mean64[3 * static_cast<size_t>(v) + 1] = mean[1];
      j.mean64[3 * static_cast<size_t>(v) + 2] = mean[2];
    }
  }
  __syncwarp();
  // the warp's covariances leave as one contiguous, coalesced run of kCovW·nv doubles, 16 B per store
  // (v0 is a multiple of 32, so the run starts 16-B aligned)
  double2* __restrict__ dst = reinterpret_cast<double2*>(j.cov9 + kCovW * static_cast<size_t>(v0));
  const double2* src2 = reinterpret_cast<const double2*>(stage[warp]);
  for (unsigned t = lane; t < (kCovW * nv) / 2; t += 32) dst[t] = src2[t];
  if ((kCovW * nv) % 2 && lane == 0)
    j.cov9[kCovW * static_cast<size_t>(v0) + kCovW * nv - 1] = stage[warp][kCovW * nv - 1];
}

// Hash table of a rank-numbered map (on demand): slot <- the statistics of its key's rank.
__global__ void place_rank_kernel(const InsertJob* __restrict__ job, unsigned V, const SlotStatsA* __restrict__ ra,
                                  const SlotStatsB* __restrict__ rb) {
  const InsertJob& j = *job;
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    const unsigned long long key = j.keys[v];
    unsigned k0, k1, k2;
    unpack_key(key, k0, k1, k2);
    const unsigned bb[2] = {bucket1(k0, k1, k2, j.shift), bucket2(k0, k1, k2, j.shift)};
    int slot = -1;
    for (int c = 0; c < 2; ++c)
      for (int q = 0; q < kBucket; ++q)
        if (j.tkeys[kBucket * bb[c] + q] == key) slot = kBucket * bb[c] + q;
    if (slot < 0) continue;  // cannot happen after a successful insert pass
    j.sa[slot] = ra[v];
    j.sb[slot] = rb[v];
  }
}

unsigned grid_for(unsigned n, unsigned threads, unsigned cap) {
  unsigned g = (n + threads - 1) / threads;
  if (g == 0) g = 1;
  return g < cap ? g : cap;
}

}  // namespace

cudaError_t launch_fast_mark(const FastBuildJob* jobs, int m, unsigned max_n, unsigned max_words, unsigned* code,
                             int* err, cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  for (int m0 = 0; m0 < m; m0 += 65535) {
    const unsigned mm = static_cast<unsigned>(std::min(65535, m - m0));
    fast_zero_kernel<<<dim3(grid_for(max_words, 256, 64), mm), 256, 0, s>>>(jobs + m0);
    fast_mark_kernel<<<dim3(grid_for(max_n, 256, 128), mm), 256, 0, s>>>(jobs + m0, code, err + m0);
  }
  return cudaGetLastError();
}

unsigned fast_markrank_smem_words(int device) {
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const int avail = optin - 1024;
  return avail > 0 ? static_cast<unsigned>(avail) / 8u : 0u;
}

cudaError_t launch_fast_markrank_smem(const FastBuildJob* jobs, int count, unsigned max_words, unsigned* code,
                                      int* err, unsigned* vcount, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const size_t bytes = 8 * static_cast<size_t>(std::max(1u, max_words));
  if (const cudaError_t e = cudaFuncSetAttribute(fast_markrank_smem_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
      e != cudaSuccess)
    return e;
  fast_markrank_smem_kernel<<<count, kMarkThreads, bytes, s>>>(jobs, code, err, vcount);
  return cudaGetLastError();
}

cudaError_t launch_fast_rank(const FastBuildJob* jobs, int m, unsigned* vcount, cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  fast_rank_kernel<<<m, 1024, 0, s>>>(jobs, vcount);
  return cudaGetLastError();
}

unsigned fast_order_smem_voxels(int device) {
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const int avail = optin - 1024;  // static shared memory of the kernel + slack
  return avail > 0 ? static_cast<unsigned>(avail) / sizeof(unsigned) - 1u : 0u;
}

cudaError_t launch_fast_order(const FastBuildJob* jobs, const int* idx, int count, unsigned smem_v, const unsigned* code,
                              unsigned* rank, unsigned* list, unsigned* offs, unsigned* gcnt, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (smem_v > 0) {
    const size_t bytes = sizeof(unsigned) * (static_cast<size_t>(smem_v) + 1);
    // per-function, per-device attribute: set for this launch's size
    if (const cudaError_t e = cudaFuncSetAttribute(fast_order_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(bytes));
        e != cudaSuccess)
      return e;
    fast_order_kernel<true><<<count, kOrderThreads, bytes, s>>>(jobs, idx, code, rank, list, offs, gcnt);
  } else {
    fast_order_kernel<false><<<count, kOrderThreads, 0, s>>>(jobs, idx, code, rank, list, offs, gcnt);
  }
  return cudaGetLastError();
}

static long sort_points_for(int device, unsigned counter_bytes) {
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const long avail = static_cast<long>(optin) - static_cast<long>(counter_bytes) - 512;
  return avail > 0 ? std::min<long>(avail / 8, 65535) : 0;  // two key buffers of u32
}

unsigned fast_sort_max_points(int device) {
  return static_cast<unsigned>(sort_points_for(device, radix_counter_bytes<4>()));
}

// 4-bit digits (16 counters per thread, 32 KB): measured faster than 5-bit digits (3 passes but a
// 64 KB counter scan per pass: C3 211 vs 171 us); VGICP_SORT_5BIT=1 selects the latter when it fits
cudaError_t launch_fast_sort(const FastBuildJob* jobs, const int* idx, int count, unsigned max_n, const unsigned* code,
                             unsigned* list, unsigned* offs, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  const bool wide = std::getenv("VGICP_SORT_5BIT") != nullptr &&
                    static_cast<long>(max_n) <= sort_points_for(dev, radix_counter_bytes<5>());
  const size_t bytes = (wide ? radix_counter_bytes<5>() : radix_counter_bytes<4>()) +
                       8 * static_cast<size_t>(std::max(1u, max_n));
  auto go = [&](auto kernel) {
    if (const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(bytes));
        e != cudaSuccess)
      return e;
    kernel<<<count, kRadixThreads, bytes, s>>>(jobs, idx, code, list, offs);
    return cudaGetLastError();
  };
  return wide ? go(fast_sort_kernel<5>) : go(fast_sort_kernel<4>);
}

cudaError_t launch_fast_accumulate(const FastBuildJob* jobs, int m, unsigned max_v, const unsigned* list,
                                   const unsigned* offs, const unsigned* code, bool export_mode, cudaStream_t s) {
  if (m <= 0 || max_v == 0) return cudaSuccess;
  for (int m0 = 0; m0 < m; m0 += 65535) {
    const unsigned mm = static_cast<unsigned>(std::min(65535, m - m0));
    const dim3 grid((max_v + kAccThreads - 1) / kAccThreads, mm);
    if (export_mode) fast_accumulate_kernel<true><<<grid, kAccThreads, 0, s>>>(jobs + m0, list, offs, code);
    else fast_accumulate_kernel<false><<<grid, kAccThreads, 0, s>>>(jobs + m0, list, offs, code);
  }
  return cudaGetLastError();
}

cudaError_t launch_place_rank(const InsertJob* job, unsigned V, const SlotStatsA* ra, const SlotStatsB* rb,
                              cudaStream_t s) {
  if (V == 0) return cudaSuccess;
  place_rank_kernel<<<grid_for(V, 128, 4096), 128, 0, s>>>(job, V, ra, rb);
  return cudaGetLastError();
}

}  // namespace vgicp
