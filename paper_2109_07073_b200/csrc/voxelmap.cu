// Gaussian voxel map build, lookup and overlap kernels (sm_100a).
//
// Build (GaussianVoxelMap ctor, voxelmap.cpp:65-104), batched over m maps per call:
//   K1 build_keys       fp64 transform-free key per point (exact floor(p/r), ±2^20 check)
//   (CUB)               stable segmented radix sort of (key, point index) per map
//   K2 build_heads      run heads of equal keys
//   (CUB)               exclusive scan of heads -> compact voxel ids (ascending key order)
//   K3 build_counts     voxels per map
//   K4 build_accumulate one thread per voxel: Kahan fp64 sums over the voxel's points in input
//                       order (exactly the reference's per-shard order, voxelmap.cpp:87-94),
//                       finalize (voxelmap.cpp:34-40), atomicCAS insert into the open-addressing
//                       table and write the fp32 voxel-local hot record + fp64 cold statistics.
// Sorting instead of float atomics makes the statistics deterministic and bit-identical to the
// reference's Kahan merge; the hash table itself is built with 64-bit atomicCAS.
#include <algorithm>

#include "internal.h"

namespace vgicp {

__global__ void build_keys_kernel(const BuildSeg* __restrict__ segs, unsigned long long* __restrict__ keys,
                                  unsigned* __restrict__ vals, int* __restrict__ range_err) {
  const BuildSeg s = segs[blockIdx.y];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    double x, y, z;
    if (s.xyz64) {
      x = s.xyz64[3 * (size_t)i], y = s.xyz64[3 * (size_t)i + 1], z = s.xyz64[3 * (size_t)i + 2];
    } else {
      const float4 a = __ldg(s.pa + i);
      x = a.x, y = a.y, z = a.z;
    }
    unsigned k0, k1, k2, hi, lo;
    double l0, l1, l2;
    unsigned long long key = 0;
    if (voxel_key(x, y, z, s.res, s.inv_res, k0, k1, k2, l0, l1, l2)) {
      pack_key32(k0, k1, k2, hi, lo);
      key = key64(hi, lo);
    } else {
      atomicOr(&range_err[blockIdx.y], 1);
    }
    keys[s.offset + i] = key;
    vals[s.offset + i] = i;
  }
}

__global__ void build_heads_kernel(const BuildSeg* __restrict__ segs, const unsigned long long* __restrict__ keys,
                                   unsigned* __restrict__ heads) {
  const BuildSeg s = segs[blockIdx.y];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const unsigned long long o = s.offset + i;
    heads[o] = (i == 0 || keys[o] != keys[o - 1]) ? 1u : 0u;
  }
}

__global__ void build_counts_kernel(const BuildSeg* __restrict__ segs, int m, const unsigned* __restrict__ heads,
                                    const unsigned* __restrict__ vidx, unsigned* __restrict__ vcount,
                                    unsigned* __restrict__ vbase) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const BuildSeg s = segs[k];
  if (s.n == 0) {
    vcount[k] = 0;
    vbase[k] = 0;
    return;
  }
  const unsigned long long last = s.offset + s.n - 1;
  vbase[k] = vidx[s.offset];
  vcount[k] = vidx[last] + heads[last] - vidx[s.offset];
}

__device__ __forceinline__ void kahan_add(double& sum, double& comp, double value) {  // parallel.hpp:106-111
  const double y = __dsub_rn(value, comp);
  const double t = __dadd_rn(sum, y);
  comp = __dsub_rn(__dsub_rn(t, sum), y);
  sum = t;
}

constexpr int kGroup = 8;    // points per batch of independent loads (float32 path)
constexpr int kGroup64 = 4;  // (float64 path)

__global__ void build_accumulate_kernel(const BuildSeg* __restrict__ segs, const BuildOut* __restrict__ outs,
                                        const unsigned long long* __restrict__ keys,
                                        const unsigned* __restrict__ vals, const unsigned* __restrict__ heads,
                                        const unsigned* __restrict__ vidx, VoxelStats* __restrict__ hot) {
  const BuildSeg s = segs[blockIdx.y];
  const BuildOut o = outs[blockIdx.y];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const unsigned long long g = s.offset + i;
    if (!heads[g]) continue;
    const unsigned long long key = keys[g];
    const unsigned v = vidx[g] - o.vbase;
    // VoxelAccumulator::add (voxelmap.cpp:28-32) with KahanSum, component-wise.
    double ms[3] = {0, 0, 0}, mc[3] = {0, 0, 0};
    double cov[9];  // finalized covariance, row-major
    int count = 0;
    if (!s.xyz64) {
      // float32 cloud: symmetric inputs, so the 6 unique second-moment sums equal the 9 of the
      // reference bit for bit ((0,1) and (1,0) receive identical addends)
      double ss[6] = {0, 0, 0, 0, 0, 0}, sc[6] = {0, 0, 0, 0, 0, 0};  // xx xy xz yy yz zz
      // the run's points in groups of kGroup: independent loads first, then the in-order Kahan adds
      for (unsigned j = i, more = 1; more; j += kGroup) {
        bool val[kGroup];
        float4 A[kGroup], B[kGroup];
        float Z[kGroup];
#pragma unroll
        for (int q = 0; q < kGroup; ++q) {
          const unsigned jj = j + q;
          val[q] = jj < s.n && (jj == i || !heads[s.offset + jj]);
        }
#pragma unroll
        for (int q = 1; q < kGroup; ++q) val[q] = val[q] && val[q - 1];
#pragma unroll
        for (int q = 0; q < kGroup; ++q) {
          const unsigned p = val[q] ? vals[s.offset + j + q] : vals[s.offset + i];
          A[q] = __ldg(s.pa + p);
          B[q] = __ldg(s.pb + p);
          Z[q] = __ldg(s.pc + p);
        }
#pragma unroll
        for (int q = 0; q < kGroup; ++q) {
          if (!val[q]) break;
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
          ++count;
        }
        more = val[kGroup - 1];
      }
      const double cnt = static_cast<double>(count);
      const double mean[3] = {__ddiv_rn(ms[0], cnt), __ddiv_rn(ms[1], cnt), __ddiv_rn(ms[2], cnt)};
      const int r6[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
      for (int e = 0; e < 6; ++e) {
        const int r = r6[e][0], c = r6[e][1];
        cov[3 * r + c] = cov[3 * c + r] = __dsub_rn(__ddiv_rn(ss[e], cnt), __dmul_rn(mean[r], mean[c]));
      }
      ms[0] = mean[0], ms[1] = mean[1], ms[2] = mean[2];
    } else {
      // fp64 cloud with full (possibly 1-ulp asymmetric) covariances: all 9 sums, as the reference
      double ss[9], sc[9];
      for (int e = 0; e < 9; ++e) ss[e] = sc[e] = 0.0;
      for (unsigned j = i, more = 1; more; j += kGroup64) {
        bool val[kGroup64];
        size_t pp[kGroup64];
#pragma unroll
        for (int q = 0; q < kGroup64; ++q) {
          const unsigned jj = j + q;
          val[q] = jj < s.n && (jj == i || !heads[s.offset + jj]);
        }
#pragma unroll
        for (int q = 1; q < kGroup64; ++q) val[q] = val[q] && val[q - 1];
#pragma unroll
        for (int q = 0; q < kGroup64; ++q) pp[q] = val[q] ? vals[s.offset + j + q] : vals[s.offset + i];
        double M[kGroup64][3], Cq[kGroup64][9];
#pragma unroll
        for (int q = 0; q < kGroup64; ++q) {
#pragma unroll
          for (int a = 0; a < 3; ++a) M[q][a] = s.xyz64[3 * pp[q] + a];
#pragma unroll
          for (int e = 0; e < 9; ++e) Cq[q][e] = s.cov9[9 * pp[q] + e];
        }
#pragma unroll
        for (int q = 0; q < kGroup64; ++q) {
          if (!val[q]) break;
          const double* m = M[q];
          const double* C = Cq[q];
          kahan_add(ms[0], mc[0], m[0]);
          kahan_add(ms[1], mc[1], m[1]);
          kahan_add(ms[2], mc[2], m[2]);
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              kahan_add(ss[3 * r + c], sc[3 * r + c], __dadd_rn(C[3 * r + c], __dmul_rn(m[r], m[c])));
          ++count;
        }
        more = val[kGroup64 - 1];
      }
      const double cnt = static_cast<double>(count);
      const double mean[3] = {__ddiv_rn(ms[0], cnt), __ddiv_rn(ms[1], cnt), __ddiv_rn(ms[2], cnt)};
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) cov[3 * r + c] = __dsub_rn(__ddiv_rn(ss[3 * r + c], cnt), __dmul_rn(mean[r], mean[c]));
      ms[0] = mean[0], ms[1] = mean[1], ms[2] = mean[2];
    }
    const double mean[3] = {ms[0], ms[1], ms[2]};
    // occupied-region bounds (overlap culling)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int c = static_cast<int>(key_coord(key, a));
      atomicMin(&o.cbox[a], c);
      atomicMax(&o.cbox[3 + a], c);
    }
    // cold fp64 statistics (ascending key order)
    o.keys[v] = key;
    o.counts[v] = count;
    o.mean64[3 * v + 0] = mean[0];
    o.mean64[3 * v + 1] = mean[1];
    o.mean64[3 * v + 2] = mean[2];
    double* c9 = o.cov64 + 9 * v;
#pragma unroll
    for (int e = 0; e < 9; ++e) c9[e] = cov[e];
    // hot record (compact by global voxel id): statistics relative to the voxel's lower corner
    const double corner0 = __dmul_rn(key_coord(key, 0), s.res);
    const double corner1 = __dmul_rn(key_coord(key, 1), s.res);
    const double corner2 = __dmul_rn(key_coord(key, 2), s.res);
    VoxelStats r;
    r.mx = static_cast<float>(__dsub_rn(mean[0], corner0));
    r.my = static_cast<float>(__dsub_rn(mean[1], corner1));
    r.mz = static_cast<float>(__dsub_rn(mean[2], corner2));
    r.cxx = static_cast<float>(cov[0]);
    r.cxy = static_cast<float>(cov[1]);
    r.cxz = static_cast<float>(cov[2]);
    r.cyy = static_cast<float>(cov[4]);
    r.cyz = static_cast<float>(cov[5]);
    r.czz = static_cast<float>(cov[8]);
    r.vid = static_cast<int>(v);
    r.pad0 = r.pad1 = 0;
    hot[vidx[g]] = r;
  }
}

// Bucketized cuckoo insertion of the keys (2 choices × 4 slots): a thread claims an empty slot in
// either of its key's buckets with atomicCAS; when both are full it evicts a resident key with
// atomicExch and carries the victim to the victim's other bucket. Every key is always either in
// the table or carried by exactly one thread, so the table is complete when all threads finish;
// a walk longer than kMaxKicks flags the map for a rebuild with twice the buckets. Slot positions
// depend on scheduling; lookup results never do.
constexpr int kMaxKicks = 256;

__global__ void build_insert_kernel(const InsertJob* __restrict__ jobs, int* __restrict__ overflow) {
  const InsertJob j = jobs[blockIdx.y];
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < j.voxels; v += gridDim.x * blockDim.x) {
    unsigned long long cur = j.keys[v];
    unsigned from = 0xFFFFFFFFu;  // bucket the carried key was evicted from
    bool placed = false;
    for (int kick = 0; kick < kMaxKicks && !placed; ++kick) {
      unsigned k0, k1, k2;
      unpack_key(cur, k0, k1, k2);
      const unsigned bb[2] = {bucket1(k0, k1, k2, j.shift), bucket2(k0, k1, k2, j.shift)};
      for (int c = 0; c < 2 && !placed; ++c) {
        if (bb[c] == from) continue;
        for (int q = 0; q < kBucket && !placed; ++q)
          placed = atomicCAS(&j.tkeys[kBucket * bb[c] + q], kEmptyKey, cur) == kEmptyKey;
      }
      if (placed) break;
      // both candidate buckets full: evict from the bucket we did not just come from
      const unsigned b = (from == bb[0]) ? bb[1] : (from == bb[1]) ? bb[0] : bb[kick & 1];
      const unsigned victim_slot = kBucket * b + ((v + kick) & (kBucket - 1));
      cur = atomicExch(&j.tkeys[victim_slot], cur);
      from = b;
      if (cur == kEmptyKey) placed = true;  // the slot emptied meanwhile: nothing to carry
    }
    if (!placed) atomicOr(&overflow[blockIdx.y], 1);
  }
}

// After insertion: every voxel finds its slot and writes its fp32 statistics there.
__global__ void build_place_kernel(const InsertJob* __restrict__ jobs, const VoxelStats* __restrict__ hot) {
  const InsertJob j = jobs[blockIdx.y];
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < j.voxels; v += gridDim.x * blockDim.x) {
    const unsigned long long key = j.keys[v];
    unsigned k0, k1, k2;
    unpack_key(key, k0, k1, k2);
    const unsigned bb[2] = {bucket1(k0, k1, k2, j.shift), bucket2(k0, k1, k2, j.shift)};
    int slot = -1;
    for (int c = 0; c < 2; ++c)
      for (int q = 0; q < kBucket; ++q)
        if (j.tkeys[kBucket * bb[c] + q] == key) slot = kBucket * bb[c] + q;
    if (slot < 0) continue;  // cannot happen after a successful insert pass
    const VoxelStats h = hot[j.vbase + v];
    SlotStatsA a;
    a.mx = h.mx, a.my = h.my, a.mz = h.mz, a.cxx = h.cxx, a.cxy = h.cxy, a.cxz = h.cxz, a.cyy = h.cyy, a.cyz = h.cyz;
    j.sa[slot] = a;
    j.sb[slot] = SlotStatsB{h.czz, h.vid};
  }
}

__global__ void lookup_kernel(MapDev map, const double* __restrict__ pts, size_t n,
                              unsigned long long* __restrict__ keys_out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned k0, k1, k2, hi, lo;
    double l0, l1, l2;
    unsigned long long out = kEmptyKey;
    if (voxel_key(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], map.res, map.inv_res, k0, k1, k2, l0, l1, l2) &&
        find_slot(map, k0, k1, k2) >= 0) {
      pack_key32(k0, k1, k2, hi, lo);
      out = key64(hi, lo);
    }
    keys_out[i] = out;
  }
}

// Point i of a cloud's Morton-ordered blocks as float64: the exact float64 means of a float64 cloud,
// else the float32 means (exact by the cloud's contract).
__device__ __forceinline__ void load_point64(const PointBlock* __restrict__ blk, const PointBlock64* __restrict__ blk64,
                                             unsigned i, double& x, double& y, double& z) {
  if (blk64) {
    const PointBlock64& b = blk64[i / kPointBlock];
    x = __ldg(&b.x[i % kPointBlock]), y = __ldg(&b.y[i % kPointBlock]), z = __ldg(&b.z[i % kPointBlock]);
  } else {
    const float4 a = __ldg(&blk[i / kPointBlock].pa[i % kPointBlock]);
    x = a.x, y = a.y, z = a.z;
  }
}

// overlap_rate (voxelmap.cpp:119-135), batched: blockIdx.y walks (cloud, pose, map) items,
// hits are integer-exact (warp-aggregated 64-bit atomics), so the result is exactly hits / N.
// Each thread keeps kOverlapILP points' bucket pairs in flight (keys first, then all loads).
#ifndef VG_OV_ILP
#define VG_OV_ILP 4
#endif
#ifndef VG_OV_MINB
#define VG_OV_MINB 1
#endif
constexpr int kOverlapILP = VG_OV_ILP;

__global__ void __launch_bounds__(256, VG_OV_MINB) overlap_kernel(const OverlapItem* __restrict__ items, int m,
                                                      unsigned long long* __restrict__ hits) {
  for (int k = blockIdx.y; k < m; k += gridDim.y) {
    const OverlapItem& it = items[k];
    const unsigned n = it.n;
    const unsigned stride = gridDim.x * blockDim.x;
    const unsigned first = blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.x * blockDim.x >= n) continue;
    double T[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) T[q] = it.T[q];
    const MapDev map = it.map;
    const OccDev occ = it.occ;
    const PointBlock* __restrict__ blk = it.blk;
    const PointBlock64* __restrict__ blk64 = it.blk64;
    unsigned count = 0;
    if (occ.occ) {  // occupancy bitmap: one 8-byte word per probe, no key compare
      for (unsigned base = first; base < n; base += kOverlapILP * stride) {
        unsigned long long wv[kOverlapILP];
        unsigned bit[kOverlapILP];
#pragma unroll
        for (int u = 0; u < kOverlapILP; ++u) {
          const unsigned i = base + u * stride;
          const unsigned ic = min(i, n - 1);
          double px, py, pz, q0, q1, q2, l0, l1, l2;
          load_point64(blk, blk64, ic, px, py, pz);
          apply_pose_rn(T, px, py, pz, q0, q1, q2);
          unsigned k0 = 0, k1 = 0, k2 = 0, word = 0;
          const bool ok = voxel_key(q0, q1, q2, map.res, map.inv_res, k0, k1, k2, l0, l1, l2) && i < n &&
                          occ_locate(occ, k0, k1, k2, word, bit[u]);
          wv[u] = ok ? __ldg(&occ.occ[word].bits) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kOverlapILP; ++u) count += static_cast<unsigned>((wv[u] >> bit[u]) & 1ull);
      }
    } else
    for (unsigned base = first; base < n; base += kOverlapILP * stride) {
      unsigned hi[kOverlapILP], lo[kOverlapILP], b1[kOverlapILP], b2[kOverlapILP];
      bool ok[kOverlapILP];
#pragma unroll
      for (int u = 0; u < kOverlapILP; ++u) {
        const unsigned i = base + u * stride;
        const unsigned ic = min(i, n - 1);
        double px, py, pz, q0, q1, q2, l0, l1, l2;
        load_point64(blk, blk64, ic, px, py, pz);
        apply_pose_rn(T, px, py, pz, q0, q1, q2);
        unsigned k0 = 0, k1 = 0, k2 = 0;
        ok[u] = voxel_key(q0, q1, q2, map.res, map.inv_res, k0, k1, k2, l0, l1, l2) && i < n;
        pack_key32(k0, k1, k2, hi[u], lo[u]);
        b1[u] = bucket1(k0, k1, k2, map.shift);
        b2[u] = bucket2(k0, k1, k2, map.shift);
      }
      BucketPair bp[kOverlapILP];
#pragma unroll
      for (int u = 0; u < kOverlapILP; ++u) bp[u] = load_buckets(map.keys, b1[u], b2[u]);
#pragma unroll
      for (int u = 0; u < kOverlapILP; ++u)
        if (ok[u] && match_buckets(bp[u], b1[u], b2[u], hi[u], lo[u]) >= 0) ++count;
    }
    count = __reduce_add_sync(0xffffffffu, count);
    if ((threadIdx.x & 31) == 0 && count) atomicAdd(&hits[k], static_cast<unsigned long long>(count));
  }
}

namespace {
unsigned grid_for(unsigned n, unsigned threads, unsigned cap) {
  unsigned g = (n + threads - 1) / threads;
  if (g == 0) g = 1;
  return g < cap ? g : cap;
}
}  // namespace

cudaError_t launch_build_keys(const BuildSeg* segs, int m, unsigned max_n, unsigned long long* keys, unsigned* vals,
                              int* range_err, cudaStream_t s) {
  build_keys_kernel<<<dim3(grid_for(max_n, 256, 4096), m), 256, 0, s>>>(segs, keys, vals, range_err);
  return cudaGetLastError();
}

cudaError_t launch_build_heads(const BuildSeg* segs, int m, unsigned max_n, const unsigned long long* keys,
                               unsigned* heads, cudaStream_t s) {
  build_heads_kernel<<<dim3(grid_for(max_n, 256, 4096), m), 256, 0, s>>>(segs, keys, heads);
  return cudaGetLastError();
}

cudaError_t launch_build_counts(const BuildSeg* segs, int m, const unsigned* heads, const unsigned* vidx,
                                unsigned* vcount, unsigned* vbase, cudaStream_t s) {
  build_counts_kernel<<<(m + 127) / 128, 128, 0, s>>>(segs, m, heads, vidx, vcount, vbase);
  return cudaGetLastError();
}

cudaError_t launch_build_accumulate(const BuildSeg* segs, const BuildOut* outs, int m, unsigned max_n,
                                    const unsigned long long* keys, const unsigned* vals, const unsigned* heads,
                                    const unsigned* vidx, VoxelStats* hot, cudaStream_t s) {
  build_accumulate_kernel<<<dim3(grid_for(max_n, 128, 4096), m), 128, 0, s>>>(segs, outs, keys, vals, heads, vidx,
                                                                              hot);
  return cudaGetLastError();
}

cudaError_t launch_build_insert(const InsertJob* jobs, int m, unsigned max_v, int* overflow, cudaStream_t s) {
  build_insert_kernel<<<dim3(grid_for(max_v, 128, 4096), m), 128, 0, s>>>(jobs, overflow);
  return cudaGetLastError();
}

cudaError_t launch_build_place(const InsertJob* jobs, int m, unsigned max_v, const VoxelStats* hot, cudaStream_t s) {
  build_place_kernel<<<dim3(grid_for(max_v, 128, 4096), m), 128, 0, s>>>(jobs, hot);
  return cudaGetLastError();
}

cudaError_t launch_lookup(MapDev map, const double* pts, size_t n, unsigned long long* keys_out, cudaStream_t s) {
  lookup_kernel<<<grid_for(static_cast<unsigned>(n < (1u << 30) ? n : (1u << 30)), 256, 4096), 256, 0, s>>>(
      map, pts, n, keys_out);
  return cudaGetLastError();
}

// One cloud against many maps (C4, and every per-frame factor-selection sweep): each thread loads
// its points ONCE and probes a chunk of kOvMaps maps with them, two maps at a time; per-map hit
// counts are summed in shared memory (integer atomics, exact) and added to the global count once
// per CTA.
constexpr int kOvPoints = 2;   // points per thread
constexpr int kOvMaps = kOverlapMapsPerChunk;  // maps per CTA

__global__ void __launch_bounds__(256) overlap_multi_kernel(const OverlapItem* __restrict__ items,
                                                            const int2* __restrict__ chunks,
                                                            unsigned long long* __restrict__ hits) {
  __shared__ unsigned cnt[kOvMaps];
  const int2 ch = chunks[blockIdx.y];  // (first item, count <= kOvMaps), one cloud per chunk
  const OverlapItem& it0 = items[ch.x];
  const unsigned n = it0.n;
  if (blockIdx.x * blockDim.x * kOvPoints >= n) return;
  const PointBlock* __restrict__ blk = it0.blk;
  const int m0 = ch.x;
  const int mc = ch.y;
  if (threadIdx.x < kOvMaps) cnt[threadIdx.x] = 0;
  double px[kOvPoints], py[kOvPoints], pz[kOvPoints];
  bool in[kOvPoints];
#pragma unroll
  for (int u = 0; u < kOvPoints; ++u) {
    const unsigned i = (blockIdx.x * kOvPoints + u) * blockDim.x + threadIdx.x;
    const unsigned ic = min(i, n - 1);
    load_point64(blk, it0.blk64, ic, px[u], py[u], pz[u]);
    in[u] = i < n;
  }
  __syncthreads();
  for (int k = 0; k < mc; k += 2) {
    unsigned hi[2][kOvPoints], lo[2][kOvPoints], b1[2][kOvPoints], b2[2][kOvPoints];
    bool ok[2][kOvPoints];
    const MapDev* mp[2];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const int kk = min(k + w, mc - 1);
      const OverlapItem& it = items[m0 + kk];
      mp[w] = &it.map;
      const MapDev& map = it.map;
#pragma unroll
      for (int u = 0; u < kOvPoints; ++u) {
        double q0, q1, q2, l0, l1, l2;
        apply_pose_rn(it.T, px[u], py[u], pz[u], q0, q1, q2);
        unsigned k0 = 0, k1 = 0, k2 = 0;
        ok[w][u] = voxel_key(q0, q1, q2, map.res, map.inv_res, k0, k1, k2, l0, l1, l2) && in[u] && (k + w < mc);
        pack_key32(k0, k1, k2, hi[w][u], lo[w][u]);
        b1[w][u] = bucket1(k0, k1, k2, map.shift);
        b2[w][u] = bucket2(k0, k1, k2, map.shift);
      }
    }
    BucketPair bp[2][kOvPoints];
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
      for (int u = 0; u < kOvPoints; ++u) bp[w][u] = load_buckets(mp[w]->keys, b1[w][u], b2[w][u]);
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      unsigned c = 0;
#pragma unroll
      for (int u = 0; u < kOvPoints; ++u)
        if (ok[w][u] && match_buckets(bp[w][u], b1[w][u], b2[w][u], hi[w][u], lo[w][u]) >= 0) ++c;
      c = __reduce_add_sync(0xffffffffu, c);
      if ((threadIdx.x & 31) == 0 && c) atomicAdd(&cnt[k + w < mc ? k + w : 0], c);
    }
  }
  __syncthreads();
  if (threadIdx.x < mc && cnt[threadIdx.x])
    atomicAdd(&hits[m0 + threadIdx.x], static_cast<unsigned long long>(cnt[threadIdx.x]));
}

// Occupancy bitmaps of a batch of maps: zero every record, set one bit per voxel key, rank the
// bricks (exclusive prefix of their popcounts, one CTA per map), then scatter every voxel's fp32
// statistics to its rank (rank-ordered copies of the hash table's slot statistics).
__global__ void occ_zero_kernel(const OccJob* __restrict__ jobs) {
  const OccJob& j = jobs[blockIdx.y];
  for (unsigned w = blockIdx.x * blockDim.x + threadIdx.x; w < j.words; w += gridDim.x * blockDim.x)
    j.occ[w] = OccWord{0ull, 0u, 0u};
}
__device__ __forceinline__ void occ_coords(const OccJob& j, unsigned long long key, unsigned& word, unsigned& bit) {
  const unsigned k0 = static_cast<unsigned>(key >> 42) & 0x1FFFFFu;
  const unsigned k1 = static_cast<unsigned>(key >> 21) & 0x1FFFFFu;
  const unsigned k2 = static_cast<unsigned>(key) & 0x1FFFFFu;
  const unsigned rx = k0 - j.kx0, ry = k1 - j.ky0, rz = k2 - j.kz0;
  word = ((rx >> 2) * j.nby + (ry >> 2)) * j.nbz + (rz >> 2);
  bit = ((rx & 3u) << 4) | ((ry & 3u) << 2) | (rz & 3u);
}
__global__ void occ_set_kernel(const OccJob* __restrict__ jobs) {
  const OccJob& j = jobs[blockIdx.y];
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < j.V; v += gridDim.x * blockDim.x) {
    unsigned word, bit;
    occ_coords(j, j.keys[v], word, bit);
    atomicOr(&j.occ[word].bits, 1ull << bit);
  }
}
__global__ void __launch_bounds__(1024) occ_rank_kernel(const OccJob* __restrict__ jobs) {
  const OccJob& j = jobs[blockIdx.x];
  __shared__ unsigned warp_sums[32];
  __shared__ unsigned carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (unsigned w0 = 0; w0 < j.words; w0 += 1024) {
    const unsigned w = w0 + threadIdx.x;
    const unsigned c = w < j.words ? static_cast<unsigned>(__popcll(j.occ[w].bits)) : 0u;
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
      warp_sums[lane] = t;  // inclusive prefix over warps
    }
    __syncthreads();
    const unsigned before = carry + (warp ? warp_sums[warp - 1] : 0u) + (x - c);
    if (w < j.words) j.occ[w].rank = before;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
}
__global__ void occ_place_kernel(const OccJob* __restrict__ jobs, const VoxelStats* __restrict__ hot) {
  const OccJob& j = jobs[blockIdx.y];
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < j.V; v += gridDim.x * blockDim.x) {
    unsigned word, bit;
    occ_coords(j, j.keys[v], word, bit);
    const OccWord o = j.occ[word];
    const unsigned rank = o.rank + static_cast<unsigned>(__popcll(o.bits & ((1ull << bit) - 1ull)));
    const VoxelStats h = hot[j.vbase + v];
    SlotStatsA a;
    a.mx = h.mx, a.my = h.my, a.mz = h.mz, a.cxx = h.cxx, a.cxy = h.cxy, a.cxz = h.cxz, a.cyy = h.cyy, a.cyz = h.cyz;
    j.ra[rank] = a;
    j.rb[rank] = SlotStatsB{h.czz, h.vid};
  }
}

cudaError_t launch_occ_build(const OccJob* jobs, int m, unsigned max_words, unsigned max_v, const VoxelStats* hot,
                             cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  occ_zero_kernel<<<dim3(grid_for(max_words, 256, 1024), m), 256, 0, s>>>(jobs);
  occ_set_kernel<<<dim3(grid_for(max_v, 256, 1024), m), 256, 0, s>>>(jobs);
  occ_rank_kernel<<<m, 1024, 0, s>>>(jobs);
  occ_place_kernel<<<dim3(grid_for(max_v, 256, 1024), m), 256, 0, s>>>(jobs, hot);
  return cudaGetLastError();
}

// Overlap of one cloud against a chunk of <= kOvMaps maps that all carry occupancy bitmaps.
// Warp w of the CTA owns kOccPoints·32 consecutive Morton-ordered points. Per map (the host has
// already culled maps whose box the whole cloud misses; finer in-kernel culling measured slower):
//  * fp32 screen: q = fl32(R)·p + fl32(t), y = q·fl32(1/r); when frac(y) keeps a margin
//    δ = 5e-7·(|p|₁ + max|t|)/r + 1e-7 from both faces on every axis (|fl32 y - q/r| is at most
//    ~4.2e-7·(|p|₁ + |t|)/r: five fp32 roundings of the transform plus the 1/r and product
//    roundings; the reference's own fp64 rounding is far inside), floor(y) IS the reference's
//    floor(fl64(q64 / r)); otherwise (rare) the point takes the exact fp64 path;
//  * one 8-byte bitmap word per probe.
#ifndef VG_OCC_POINTS
#define VG_OCC_POINTS 4
#endif
constexpr int kOccPoints = VG_OCC_POINTS;  // points per lane (amortise the per-map loads)
// The reference's key of one point (fp64 transform + exact floor), out of line: the fp32 screen
// keeps the kernel's registers for the common path.
__device__ __noinline__ uint4 exact_probe_key(const double* T, double x, double y, double z, double res, double inv_res) {
  double e0, e1, e2, l0, l1, l2;
  apply_pose_rn(T, x, y, z, e0, e1, e2);
  unsigned k0 = 0, k1 = 0, k2 = 0;
  const bool ok = voxel_key(e0, e1, e2, res, inv_res, k0, k1, k2, l0, l1, l2);
  return make_uint4(k0, k1, k2, ok ? 1u : 0u);
}
__global__ void __launch_bounds__(256, 4) overlap_occ_kernel(const OverlapItem* __restrict__ items,
                                                             const int2* __restrict__ chunks,
                                                             unsigned long long* __restrict__ hits) {
  __shared__ unsigned cnt[kOvMaps];
  __shared__ OccScreen scr[kOvMaps];
  __shared__ unsigned live_n[kOvMaps];
  const int2 ch = chunks[blockIdx.y];
  unsigned n = 0;  // points of the chunk's cloud (items culled on the device carry n = 0)
  for (int q = 0; q < ch.y; ++q) n = max(n, items[ch.x + q].n);
  if (blockIdx.x * (256 * kOccPoints) >= n) return;
  for (int t = threadIdx.x; t < ch.y * 7; t += 256)  // stage the chunk's screens (7 × 16 B each)
    reinterpret_cast<uint4*>(&scr[t / 7])[t % 7] = __ldg(reinterpret_cast<const uint4*>(&items[ch.x + t / 7].scr) + t % 7);
  if (threadIdx.x < ch.y) live_n[threadIdx.x] = items[ch.x + threadIdx.x].n;
  if (threadIdx.x < kOvMaps) cnt[threadIdx.x] = 0;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned base = blockIdx.x * (256 * kOccPoints) + warp * (32 * kOccPoints);
  const PointBlock* __restrict__ blk = items[ch.x].blk;
  float px[kOccPoints], py[kOccPoints], pz[kOccPoints], p1[kOccPoints];
  unsigned in = 0;
#pragma unroll
  for (int u = 0; u < kOccPoints; ++u) {
    const unsigned i = base + u * 32 + lane;
    const unsigned ic = min(i, n - 1);
    const float4 a = __ldg(&blk[ic / kPointBlock].pa[ic % kPointBlock]);
    px[u] = a.x, py[u] = a.y, pz[u] = a.z;
    p1[u] = fabsf(a.x) + fabsf(a.y) + fabsf(a.z);
    in |= (i < n ? 1u : 0u) << u;
  }
  __syncthreads();
  for (int k = 0; k < ch.y; ++k) {
    if (live_n[k] == 0u) continue;  // culled on the device (map-set sweeps): exactly 0 hits
    const OccScreen& sc = scr[k];
    unsigned word[kOccPoints], bit[kOccPoints];
    unsigned ok = 0, need = 0;
#pragma unroll
    for (int u = 0; u < kOccPoints; ++u) {
      const float q0 = fmaf(sc.R[2], pz[u], fmaf(sc.R[1], py[u], sc.R[0] * px[u])) + sc.t[0];
      const float q1 = fmaf(sc.R[5], pz[u], fmaf(sc.R[4], py[u], sc.R[3] * px[u])) + sc.t[1];
      const float q2 = fmaf(sc.R[8], pz[u], fmaf(sc.R[7], py[u], sc.R[6] * px[u])) + sc.t[2];
      const float y0 = q0 * sc.inv_r, y1 = q1 * sc.inv_r, y2 = q2 * sc.inv_r;
      const float c0 = floorf(y0), c1 = floorf(y1), c2 = floorf(y2);
      const float h = 0.5f - fmaf(sc.A2, p1[u], sc.C);  // NaN / far points fail the test below
      const bool sure = fabsf((y0 - c0) - 0.5f) <= h && fabsf((y1 - c1) - 0.5f) <= h && fabsf((y2 - c2) - 0.5f) <= h;
      const unsigned rx = static_cast<unsigned>(__float2int_rz(c0) - sc.cx0);
      const unsigned ry = static_cast<unsigned>(__float2int_rz(c1) - sc.cy0);
      const unsigned rz = static_cast<unsigned>(__float2int_rz(c2) - sc.cz0);
      word[u] = ((rx >> 2) * sc.nby + (ry >> 2)) * sc.nbz + (rz >> 2);
      bit[u] = ((rx & 3u) << 4) | ((ry & 3u) << 2) | (rz & 3u);
      const bool inside = (rx < sc.ex) & (ry < sc.ey) & (rz < sc.ez);
      ok |= (sure && inside ? 1u : 0u) << u;
      need |= (sure ? 0u : 1u) << u;
    }
    ok &= in;
    need &= in;
    if (__any_sync(0xffffffffu, need != 0u)) {  // rare: within the margin of a face, or non-finite
      const OverlapItem& it = items[ch.x + k];
#pragma unroll
      for (int u = 0; u < kOccPoints; ++u) {
        if (!((need >> u) & 1u)) continue;
        double ex = px[u], ey = py[u], ez = pz[u];
        if (it.blk64) load_point64(blk, it.blk64, min(base + u * 32 + lane, n - 1), ex, ey, ez);  // exact means
        const uint4 e = exact_probe_key(it.T, ex, ey, ez, it.map.res, it.map.inv_res);
        const unsigned rx = e.x - (static_cast<unsigned>(sc.cx0) + (1u << 20));
        const unsigned ry = e.y - (static_cast<unsigned>(sc.cy0) + (1u << 20));
        const unsigned rz = e.z - (static_cast<unsigned>(sc.cz0) + (1u << 20));
        word[u] = ((rx >> 2) * sc.nby + (ry >> 2)) * sc.nbz + (rz >> 2);
        bit[u] = ((rx & 3u) << 4) | ((ry & 3u) << 2) | (rz & 3u);
        ok |= (e.w != 0u && (rx < sc.ex) & (ry < sc.ey) & (rz < sc.ez) ? 1u : 0u) << u;
      }
    }
    unsigned long long v[kOccPoints];
#pragma unroll
    for (int u = 0; u < kOccPoints; ++u) v[u] = ((ok >> u) & 1u) ? __ldg(&sc.occ[word[u]].bits) : 0ull;
    unsigned c = 0;
#pragma unroll
    for (int u = 0; u < kOccPoints; ++u) c += static_cast<unsigned>((v[u] >> (bit[u] & 63u)) & 1ull);
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0 && c) atomicAdd(&cnt[k], c);
  }
  __syncthreads();
  if (threadIdx.x < ch.y && cnt[threadIdx.x])
    atomicAdd(&hits[ch.x + threadIdx.x], static_cast<unsigned long long>(cnt[threadIdx.x]));
}

// Item k of a map-set sweep: the map's template + pose k; fp32 screen constants as the host path
// computes them (fl32 of the fp64 values, same margin formula); exact culling of the cloud box
// (8 corners in fp64) against the map's occupied box grown by one voxel -> n = 0 (no work).
__global__ void mapset_prepare_kernel(const OverlapItem* __restrict__ templates, int m,
                                      const double* __restrict__ poses12, const PointBlock* blk,
                                      const PointBlock64* blk64, unsigned n, const float* __restrict__ box,
                                      OverlapItem* __restrict__ items, int2* __restrict__ chunks) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  OverlapItem it = templates[k];
  const double* T = poses12 + 12 * k;
#pragma unroll
  for (int q = 0; q < 12; ++q) it.T[q] = T[q];
  it.blk = blk;
  it.blk64 = blk64;
  it.n = n;
  float tmax = 0.f;
#pragma unroll
  for (int q = 0; q < 9; ++q) it.scr.R[q] = __double2float_rn(T[q]);
#pragma unroll
  for (int q = 0; q < 3; ++q) it.scr.t[q] = __double2float_rn(T[9 + q]), tmax = fmaxf(tmax, fabsf(it.scr.t[q]));
  it.scr.inv_r = __double2float_rn(it.map.inv_res);
  it.scr.A2 = __fmul_rn(blk64 ? kScreenA64 : kScreenA, it.scr.inv_r);
  it.scr.C = __fadd_rn(__fmul_rn(it.scr.A2, tmax), 1e-7f);
  // culling (the host's overlap_disjoint): the cloud box has no finite point when lo > hi
  bool live = box[0] <= box[3];
  if (live) {
    double wlo[3] = {INFINITY, INFINITY, INFINITY}, whi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int c = 0; c < 8; ++c) {
      const double p0 = (c & 1) ? box[3] : box[0], p1 = (c & 2) ? box[4] : box[1], p2 = (c & 4) ? box[5] : box[2];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double q = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(T[3 * a], p0), __dmul_rn(T[3 * a + 1], p1)),
                                             __dmul_rn(T[3 * a + 2], p2)),
                                   T[9 + a]);
        wlo[a] = fmin(wlo[a], q);
        whi[a] = fmax(whi[a], q);
      }
    }
    const int cmin[3] = {it.scr.cx0, it.scr.cy0, it.scr.cz0};
    const unsigned ext[3] = {it.scr.ex, it.scr.ey, it.scr.ez};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double mlo = (cmin[a] - 1.0) * it.map.res, mhi = (cmin[a] + static_cast<int>(ext[a]) + 1.0) * it.map.res;
      live = live && (whi[a] >= mlo && wlo[a] <= mhi);
    }
  }
  if (!live) it.n = 0;  // culled: exactly 0 hits
  items[k] = it;
  if (k % kOvMaps == 0) chunks[k / kOvMaps] = make_int2(k, min(kOvMaps, m - k));
}

cudaError_t launch_mapset_prepare(const OverlapItem* templates, int m, const double* poses12, const PointBlock* blk,
                                  const PointBlock64* blk64, unsigned n, const float* cloud_box, OverlapItem* items,
                                  int2* chunks, cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  mapset_prepare_kernel<<<(m + 127) / 128, 128, 0, s>>>(templates, m, poses12, blk, blk64, n, cloud_box, items,
                                                        chunks);
  return cudaGetLastError();
}

cudaError_t launch_overlap_occ(const OverlapItem* items, const int2* chunks, int num_chunks, unsigned max_n,
                               unsigned long long* hits, cudaStream_t s) {
  if (num_chunks <= 0 || max_n == 0) return cudaSuccess;
  for (int c0 = 0; c0 < num_chunks; c0 += 65535) {
    const dim3 grid((max_n + 256 * kOccPoints - 1) / (256 * kOccPoints), std::min(65535, num_chunks - c0));
    overlap_occ_kernel<<<grid, 256, 0, s>>>(items, chunks + c0, hits);
  }
  return cudaGetLastError();
}

cudaError_t launch_overlap_multi(const OverlapItem* items, const int2* chunks, int num_chunks, unsigned max_n,
                                 unsigned long long* hits, cudaStream_t s) {
  if (num_chunks <= 0 || max_n == 0) return cudaSuccess;
  for (int c0 = 0; c0 < num_chunks; c0 += 65535) {  // grid.y limit
    const dim3 grid((max_n + 256 * kOvPoints - 1) / (256 * kOvPoints), std::min(65535, num_chunks - c0));
    overlap_multi_kernel<<<grid, 256, 0, s>>>(items, chunks + c0, hits);
  }
  return cudaGetLastError();
}

cudaError_t launch_overlap(const OverlapItem* items, int m, unsigned max_n, unsigned long long* hits, cudaStream_t s) {
  const unsigned gy = m < 65535 ? m : 65535;
  overlap_kernel<<<dim3(grid_for(max_n, 256 * kOverlapILP, 1024), gy), 256, 0, s>>>(items, m, hits);
  return cudaGetLastError();
}


// transform_cloud (point_cloud.cpp:26-42): q = T.apply(mu) and C' = (R·C)·Rᵀ in fp64 with the
// reference's per-entry op order ((a0·b0 + a1·b1) + a2·b2), all 9 entries (R·C·Rᵀ is not exactly
// symmetric in floating point, and the reference keeps the full matrix).
__device__ __forceinline__ void transform_point(const double* T, double x, double y, double z, const double C[9],
                                                double* q, double* Co) {
  apply_pose_rn(T, x, y, z, q[0], q[1], q[2]);
  double RC[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) RC[3 * r + c] = dot3_rn(T[3 * r], T[3 * r + 1], T[3 * r + 2], C[c], C[3 + c], C[6 + c]);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      Co[3 * r + c] = dot3_rn(RC[3 * r], RC[3 * r + 1], RC[3 * r + 2], T[3 * c], T[3 * c + 1], T[3 * c + 2]);
}

__global__ void transform_kernel(const TransformItem* __restrict__ items, double* __restrict__ out_xyz,
                                 double* __restrict__ out_cov9) {
  const TransformItem& it = items[blockIdx.y];
  double T[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) T[q] = it.T[q];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < it.n; i += gridDim.x * blockDim.x) {
    const size_t o = it.offset + i;
    if (it.xyz64) {  // float64 frame: its exact values
      double C[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) C[e] = it.cov9[9 * (size_t)i + e];
      transform_point(T, it.xyz64[3 * (size_t)i], it.xyz64[3 * (size_t)i + 1], it.xyz64[3 * (size_t)i + 2], C,
                      out_xyz + 3 * o, out_cov9 + 9 * o);
      continue;
    }
    const float4 a = __ldg(it.pa + i);
    const float4 b = __ldg(it.pb + i);
    const double czz = __ldg(it.pc + i);
    const double C[9] = {a.w, b.x, b.y, b.x, b.z, b.w, b.y, b.w, czz};
    transform_point(T, a.x, a.y, a.z, C, out_xyz + 3 * o, out_cov9 + 9 * o);
  }
}

__global__ void transform64_kernel(const double* __restrict__ xyz, const double* __restrict__ cov9, size_t n,
                                   const double* __restrict__ Tg, double* __restrict__ out_xyz,
                                   double* __restrict__ out_cov9) {
  double T[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) T[q] = Tg[q];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double C[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) C[e] = cov9 ? cov9[9 * i + e] : 0.0;
    double q[3], Co[9];
    transform_point(T, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], C, q, Co);
    out_xyz[3 * i] = q[0], out_xyz[3 * i + 1] = q[1], out_xyz[3 * i + 2] = q[2];
    if (out_cov9)
#pragma unroll
      for (int e = 0; e < 9; ++e) out_cov9[9 * i + e] = Co[e];
  }
}

cudaError_t launch_transform(const TransformItem* items, int m, unsigned max_n, double* out_xyz, double* out_cov9,
                             cudaStream_t s) {
  if (m <= 0 || max_n == 0) return cudaSuccess;
  transform_kernel<<<dim3(grid_for(max_n, 256, 1024), m), 256, 0, s>>>(items, out_xyz, out_cov9);
  return cudaGetLastError();
}

cudaError_t launch_transform64(const double* xyz, const double* cov9, size_t n, const double* T, double* out_xyz,
                               double* out_cov9, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  transform64_kernel<<<grid_for(static_cast<unsigned>(std::min<size_t>(n, 1u << 30)), 256, 4096), 256, 0, s>>>(
      xyz, cov9, n, T, out_xyz, out_cov9);
  return cudaGetLastError();
}

}  // namespace vgicp
