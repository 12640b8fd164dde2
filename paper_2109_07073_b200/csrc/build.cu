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
//                    the factor kernels' gather targets) and the fp64 covariance (6 unique entries,
//                    the near-singular fallback). Key-ordered arrays (keys, counts, fp64 means) are
//                    produced only on demand (export mode), by the same kernels.
//
// Algorithmic bytes: 36 B per input point + 48 B per voxel written.
#include <algorithm>

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
                                                                   unsigned* __restrict__ code,
                                                                   unsigned* __restrict__ list,
                                                                   unsigned* __restrict__ offs,
                                                                   unsigned* __restrict__ gcnt) {
  extern __shared__ unsigned smem_cnt[];
  __shared__ unsigned warp_sums[32];
  const FastBuildJob& j = jobs[idx[blockIdx.x]];
  const unsigned n = j.n, V = j.V;
  volatile unsigned* cnt = kSmem ? smem_cnt : gcnt + j.vx_off;
  unsigned* __restrict__ pc = code + j.pt_off;
  const OccWord* __restrict__ occ = j.occ;
  for (unsigned v = threadIdx.x; v < V; v += kOrderThreads) cnt[v] = 0u;
  __syncthreads();
  // per-point rank (brick rank + popcount of the lower bits) and per-voxel counts
  for (unsigned i = threadIdx.x; i < n; i += kOrderThreads) {
    const unsigned c = pc[i];
    const OccWord o = occ[c >> 6];
    const unsigned r = o.rank + static_cast<unsigned>(__popcll(o.bits & ((1ull << (c & 63u)) - 1ull)));
    pc[i] = r;
    atomicAdd(const_cast<unsigned*>(cnt + r), 1u);
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
  unsigned r_next = lane < n ? pc[lane] : 0xFFFFFFFFu;
  for (unsigned base = 0; base < n; base += 32) {
    const unsigned i = base + lane;
    const unsigned r = r_next;
    r_next = i + 32 < n ? pc[i + 32] : 0xFFFFFFFFu;  // next step's ranks in flight
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    unsigned pos = 0;
    if (i < n) pos = cnt[r] + static_cast<unsigned>(__popc(peers & lt));
    __syncwarp();
    if (i < n && (peers & lt) == 0u) cnt[r] += static_cast<unsigned>(__popc(peers));
    __syncwarp();
    if (i < n) pl[pos] = i;
  }
}

constexpr int kGroup = 8;  // points per batch of independent loads

__global__ void __launch_bounds__(128) fast_accumulate_kernel(const FastBuildJob* __restrict__ jobs,
                                                              const unsigned* __restrict__ list,
                                                              const unsigned* __restrict__ offs, bool export_mode) {
  const FastBuildJob& j = jobs[blockIdx.y];
  const unsigned V = j.V;
  const float4* __restrict__ pa = j.pa;
  const float4* __restrict__ pb = j.pb;
  const float* __restrict__ pcz = j.pc;
  const unsigned* __restrict__ pl = list + j.pt_off;
  const unsigned* __restrict__ off = offs + j.vx_off;
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    const unsigned b = off[v], e = off[v + 1];
    // VoxelAccumulator::add (voxelmap.cpp:28-32) with KahanSum, component-wise; float32 clouds have
    // symmetric covariances, so the 6 unique second-moment sums equal the reference's 9 bit for bit
    double ms[3] = {0, 0, 0}, mc[3] = {0, 0, 0};
    double ss[6] = {0, 0, 0, 0, 0, 0}, sc[6] = {0, 0, 0, 0, 0, 0};  // xx xy xz yy yz zz
    float4 first = make_float4(0.f, 0.f, 0.f, 0.f);
    for (unsigned q0 = b; q0 < e; q0 += kGroup) {
      float4 A[kGroup], B[kGroup];
      float Z[kGroup];
#pragma unroll
      for (int q = 0; q < kGroup; ++q) {  // independent loads first
        const unsigned p = pl[min(q0 + q, e - 1)];
        A[q] = __ldg(pa + p);
        B[q] = __ldg(pb + p);
        Z[q] = __ldg(pcz + p);
      }
      if (q0 == b) first = A[0];
#pragma unroll
      for (int q = 0; q < kGroup; ++q) {  // then the in-order Kahan adds
        if (q0 + q >= e) break;
        const double m0 = A[q].x, m1 = A[q].y, m2 = A[q].z;
        kahan_add(ms[0], mc[0], m0);
        kahan_add(ms[1], mc[1], m1);
        kahan_add(ms[2], mc[2], m2);
        kahan_add(ss[0], sc[0], __dadd_rn((double)A[q].w, __dmul_rn(m0, m0)));
        kahan_add(ss[1], sc[1], __dadd_rn((double)B[q].x, __dmul_rn(m0, m1)));
        kahan_add(ss[2], sc[2], __dadd_rn((double)B[q].y, __dmul_rn(m0, m2)));
        kahan_add(ss[3], sc[3], __dadd_rn((double)B[q].z, __dmul_rn(m1, m1)));
        kahan_add(ss[4], sc[4], __dadd_rn((double)B[q].w, __dmul_rn(m1, m2)));
        kahan_add(ss[5], sc[5], __dadd_rn((double)Z[q], __dmul_rn(m2, m2)));
      }
    }
    // finalize (voxelmap.cpp:34-40)
    const double cnt = static_cast<double>(e - b);
    const double mean[3] = {__ddiv_rn(ms[0], cnt), __ddiv_rn(ms[1], cnt), __ddiv_rn(ms[2], cnt)};
    double cov[6];
    {
      const int r6[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
      for (int q = 0; q < 6; ++q) cov[q] = __dsub_rn(__ddiv_rn(ss[q], cnt), __dmul_rn(mean[r6[q][0]], mean[r6[q][1]]));
    }
    // the voxel's key from its first point (all of its points share it)
    unsigned k0 = 0, k1 = 0, k2 = 0;
    double l0, l1, l2;
    voxel_key(first.x, first.y, first.z, j.res, j.inv_res, k0, k1, k2, l0, l1, l2);
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
    double* c6 = j.cov6 + 6 * static_cast<size_t>(v);
#pragma unroll
    for (int q = 0; q < 6; ++q) c6[q] = cov[q];
    if (export_mode) {
      unsigned hi, lo;
      pack_key32(k0, k1, k2, hi, lo);
      j.keys[v] = key64(hi, lo);
      j.counts[v] = static_cast<int>(e - b);
      j.mean64[3 * static_cast<size_t>(v) + 0] = mean[0];
      j.mean64[3 * static_cast<size_t>(v) + 1] = mean[1];
      j.mean64[3 * static_cast<size_t>(v) + 2] = mean[2];
      double* c9 = j.cov9 + 9 * static_cast<size_t>(v);
      c9[0] = cov[0], c9[1] = cov[1], c9[2] = cov[2];
      c9[3] = cov[1], c9[4] = cov[3], c9[5] = cov[4];
      c9[6] = cov[2], c9[7] = cov[4], c9[8] = cov[5];
    }
  }
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

cudaError_t launch_fast_order(const FastBuildJob* jobs, const int* idx, int count, unsigned smem_v, unsigned* code,
                              unsigned* list, unsigned* offs, unsigned* gcnt, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (smem_v > 0) {
    const size_t bytes = sizeof(unsigned) * (static_cast<size_t>(smem_v) + 1);
    // per-function, per-device attribute: set for this launch's size
    if (const cudaError_t e = cudaFuncSetAttribute(fast_order_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(bytes));
        e != cudaSuccess)
      return e;
    fast_order_kernel<true><<<count, kOrderThreads, bytes, s>>>(jobs, idx, code, list, offs, gcnt);
  } else {
    fast_order_kernel<false><<<count, kOrderThreads, 0, s>>>(jobs, idx, code, list, offs, gcnt);
  }
  return cudaGetLastError();
}

cudaError_t launch_fast_accumulate(const FastBuildJob* jobs, int m, unsigned max_v, const unsigned* list,
                                   const unsigned* offs, bool export_mode, cudaStream_t s) {
  if (m <= 0 || max_v == 0) return cudaSuccess;
  for (int m0 = 0; m0 < m; m0 += 65535) {
    const unsigned mm = static_cast<unsigned>(std::min(65535, m - m0));
    fast_accumulate_kernel<<<dim3(grid_for(max_v, 128, 1024), mm), 128, 0, s>>>(jobs + m0, list, offs, export_mode);
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
