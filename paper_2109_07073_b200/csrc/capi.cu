// C ABI (include/vgicp_b200.h): contexts, handles, validation and launch orchestration (uploads,
// builds, overlap sweeps, factor graphs incl. sharded ones, assembly, solver plans, replication).
// Host code only; the kernels live in build.cu, voxelmap.cu, factor.cu, cloud.cu, covariance.cu,
// solver.cu (and the native LM in lm.cu).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <new>
#include <thread>
#include <tuple>
#include <type_traits>

#include "internal.h"

namespace vgicp {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int cuda_fail(cudaError_t err, const char* what) {
  g_error = std::string(what) + ": " + cudaGetErrorString(err);
  return err == cudaErrorMemoryAllocation ? VGICP_E_OUT_OF_MEMORY : VGICP_E_CUDA;
}

int api_exception() noexcept {
  try {
    throw;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return VGICP_E_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    try {
      g_error = std::string("internal error: ") + e.what();
    } catch (...) {
    }
    return VGICP_E_CUDA;
  } catch (...) {
    g_error = "internal error";
    return VGICP_E_CUDA;
  }
}

namespace {

constexpr double kKeyBiasD = 1048576.0;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

unsigned next_pow2(unsigned long long x) {
  unsigned p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync on the context
// stream, release threshold raised at context creation): no implicit device synchronisation and
// no page-mapping cost on the repeated graph / map / submap builds.
cudaError_t dmalloc(vgicp_ctx ctx, void** p, size_t bytes) { return cudaMallocAsync(p, bytes, ctx->stream); }
void dfree(vgicp_ctx ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

// inverse of the device-side monotone float -> uint map (cloud.cu / covariance.cu bounding boxes)
static float unordered_host(unsigned u) {
  const unsigned v = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
  float f;
  std::memcpy(&f, &v, sizeof(f));
  return f;
}

// RAII device buffer for temporaries of the fp64 / submap paths.
struct DevBuf {  // stream-ordered temporary: freed on the context stream after its last use
  vgicp_ctx ctx;
  void* p = nullptr;
  explicit DevBuf(vgicp_ctx c) : ctx(c) {}
  cudaError_t alloc(size_t bytes) { return dmalloc(ctx, &p, bytes); }
  ~DevBuf() { dfree(ctx, p); }
};


int ensure_scratch(vgicp_ctx ctx, size_t bytes) {
  if (ctx->scratch_bytes >= bytes) return VGICP_OK;
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  const size_t want = std::max(bytes, ctx->scratch_bytes * 2);
  if (ctx->scratch) dfree(ctx, ctx->scratch);
  ctx->scratch = nullptr;
  ctx->scratch_bytes = 0;
  VG_CUDA(dmalloc(ctx, &ctx->scratch, want));
  ctx->scratch_bytes = want;
  return VGICP_OK;
}

int ensure_pinned(vgicp_ctx ctx, size_t bytes) {
  if (ctx->pinned_bytes >= bytes) return VGICP_OK;
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  const size_t want = std::max<size_t>(std::max(bytes, ctx->pinned_bytes * 2), 1 << 20);
  if (ctx->pinned) VG_CUDA(cudaFreeHost(ctx->pinned));
  ctx->pinned = nullptr;
  ctx->pinned_bytes = 0;
  VG_CUDA(cudaMallocHost(&ctx->pinned, want));
  ctx->pinned_bytes = want;
  return VGICP_OK;
}

// Runs `f` when the scope ends unless dismissed: error paths (including VG_CUDA early returns)
// release what a partially completed call allocated.
template <typename F>
struct ScopeFail {
  F f;
  bool armed = true;
  ~ScopeFail() {
    if (armed) f();
  }
  void dismiss() { armed = false; }
};
template <typename F>
ScopeFail<F> on_failure(F f) {
  return ScopeFail<F>{f};
}

template <typename T>
T* relocate(T* p, const void* old_base, void* new_base) {
  if (!p) return nullptr;
  return reinterpret_cast<T*>(static_cast<char*>(new_base) +
                              (reinterpret_cast<const char*>(p) - static_cast<const char*>(old_base)));
}
cudaError_t copy_whole(vgicp_ctx dst, void** out, const void* src, int src_device, size_t bytes) {
  *out = nullptr;
  if (!src || !bytes) return cudaSuccess;
  if (const cudaError_t e = dmalloc(dst, out, bytes); e != cudaSuccess) return e;
  return cudaMemcpyPeerAsync(*out, dst->device, src, src_device, bytes, dst->stream);
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void release(vgicp_cloud c) {
  if (c && c->refs.fetch_sub(1) == 1) {
    DeviceGuard g(c->ctx->device);
    dfree(c->ctx, c->block);
    dfree(c->ctx, c->block64);
    delete c;
  }
}

void release(vgicp_map m) {
  if (m && m->refs.fetch_sub(1) == 1) {
    DeviceGuard g(m->ctx->device);
    dfree(m->ctx, m->cold);
    dfree(m->ctx, m->table);
    dfree(m->ctx, m->occ_mem);
    release(m->src);
    delete m;
  }
}

// (Re)allocate a map's hash table with `buckets` buckets (power of two), all slots empty.
int alloc_table(vgicp_map mp, unsigned buckets, cudaStream_t s) {
  if (mp->table) dfree(mp->ctx, mp->table);
  mp->table = nullptr;
  mp->num_buckets = buckets;
  unsigned lg = 0;
  while ((1u << lg) < buckets) ++lg;
  mp->shift = 32 - lg;
  const size_t cap = static_cast<size_t>(kBucket) * buckets;
  const size_t b_keys = align_up(sizeof(unsigned long long) * cap, 256);
  const size_t b_sa = align_up(sizeof(SlotStatsA) * cap, 256);
  mp->table_bytes = b_keys + b_sa + sizeof(SlotStatsB) * cap;
  VG_CUDA(dmalloc(mp->ctx, &mp->table, mp->table_bytes));
  mp->tkeys = static_cast<unsigned long long*>(mp->table);
  mp->sa = reinterpret_cast<SlotStatsA*>(static_cast<char*>(mp->table) + b_keys);
  mp->sb = reinterpret_cast<SlotStatsB*>(static_cast<char*>(mp->table) + b_keys + b_sa);
  VG_CUDA(cudaMemsetAsync(mp->tkeys, 0xFF, sizeof(unsigned long long) * cap, s));
  return VGICP_OK;
}

// voxel_coord + pack_key on the host (voxelmap.cpp:45-63); same division/floor semantics.
int host_voxel_key(double resolution, const double p[3], uint64_t* key) {
  uint64_t k = 0;
  for (int a = 0; a < 3; ++a) {
    const double c = std::floor(p[a] / resolution);
    if (!(c >= -kKeyBiasD && c < kKeyBiasD))
      return fail(VGICP_E_OUT_OF_RANGE, "point beyond the +-2^20 voxel-per-axis range limit");
    k = (k << 21) | static_cast<uint64_t>(static_cast<int64_t>(c) + (1 << 20));
  }
  *key = k;
  return VGICP_OK;
}

}  // namespace
}  // namespace vgicp

using namespace vgicp;

extern "C" {

const char* vgicp_last_error(void) { return g_error.c_str(); }

const char* vgicp_version(void) { return "vgicp_b200 0.1 (sm_100a)"; }

int vgicp_device_count(int* count) try {
  if (!count) return fail(VGICP_E_INVALID_ARGUMENT, "null output");
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *count = n;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_ctx_create(int device, void* stream, vgicp_ctx* out) try {
  if (!out) return fail(VGICP_E_INVALID_ARGUMENT, "null output");
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail(VGICP_E_NO_DEVICE, "no CUDA device visible (vgicp_b200 has no CPU fallback)");
  if (device < 0 || device >= n) return fail(VGICP_E_INVALID_ARGUMENT, "device index out of range");
  cudaDeviceProp prop;
  VG_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(VGICP_E_NO_DEVICE, std::string("vgicp_b200 is built for sm_100a; device is ") + prop.name);
  DeviceGuard g(device);
  auto ctx = std::make_unique<vgicp_ctx_s>();
  ctx->device = device;
  if (stream) {
    ctx->stream = static_cast<cudaStream_t>(stream);
  } else {
    VG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  // keep freed blocks in the device's default pool (no return to the OS between builds)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t threshold = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  *out = ctx.release();
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_ctx_destroy(vgicp_ctx ctx) try {
  if (!ctx) return VGICP_OK;
  DeviceGuard g(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->scratch) dfree(ctx, ctx->scratch);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_ctx_create_multi(const int* devices, int n, vgicp_ctx* out) try {
  if (!devices || !out || n <= 0) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  for (int k = 0; k < n; ++k) out[k] = nullptr;
  for (int k = 0; k < n; ++k)
    if (int rc = vgicp_ctx_create(devices[k], nullptr, &out[k])) {
      for (int q = 0; q < k; ++q) vgicp_ctx_destroy(out[q]), out[q] = nullptr;
      return rc;
    }
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_ctx_stream(vgicp_ctx ctx, void** stream) try {
  if (!ctx || !stream) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *stream = ctx->stream;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_ctx_synchronize(vgicp_ctx ctx) try {
  if (!ctx) return fail(VGICP_E_INVALID_ARGUMENT, "null context");
  DeviceGuard g(ctx->device);
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_ctx_launch_count(vgicp_ctx ctx, uint64_t* launches) try {
  if (!ctx || !launches) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *launches = ctx->launches;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// ------------------------------------------------------------------------------------ clouds
// Float32 cloud upload: points (+ the 6 unique covariance entries) are staged through the pinned
// buffer and the layout is built on the device (cloud.cu): input-order SoA for the builds and the
// Morton-ordered 64-point blocks (finite bounding box, 10-bit Z-order codes, stable radix sort).
static int cloud_upload_packed(vgicp_ctx ctx, const float* xyz, const float* cov6, size_t n, vgicp_cloud* out) {
  if (!ctx || !out) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (n > 0 && !xyz) return fail(VGICP_E_INVALID_ARGUMENT, "null point array");
  if (n >= (1ull << 31)) return fail(VGICP_E_INVALID_ARGUMENT, "cloud too large (>= 2^31 points)");
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  auto c = std::make_unique<vgicp_cloud_s>();
  c->ctx = ctx;
  c->n = n;
  c->has_cov = (cov6 != nullptr) && n > 0;
  const size_t na = align_up(n * sizeof(float4), 256);
  const size_t nc = align_up(n * sizeof(float), 256);
  const size_t half = na * 2 + nc;
  const size_t nblk = (n + kPointBlock - 1) / kPointBlock;
  c->block_bytes = std::max<size_t>(half + nblk * sizeof(PointBlock), 256);
  VG_CUDA(dmalloc(ctx, &c->block, c->block_bytes));
  char* base = static_cast<char*>(c->block);
  c->pa = reinterpret_cast<float4*>(base);
  c->pb = reinterpret_cast<float4*>(base + na);
  c->pc = reinterpret_cast<float*>(base + 2 * na);
  c->sblk = reinterpret_cast<PointBlock*>(base + half);
  if (n == 0) {
    *out = c.release();
    return VGICP_OK;
  }
  size_t sort_bytes = 0;
  VG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const unsigned*)nullptr, (unsigned*)nullptr,
                                          (const unsigned*)nullptr, (unsigned*)nullptr, static_cast<int>(n), 0, 30, s));
  const size_t b_xyz = align_up(sizeof(float) * 3 * n, 256);
  const size_t b_cov = c->has_cov ? align_up(sizeof(float) * 6 * n, 256) : 0;
  const size_t b_vec = align_up(sizeof(unsigned) * n, 256);
  DevBuf tmp(ctx);
  VG_CUDA(tmp.alloc(b_xyz + b_cov + 256 + 4 * b_vec + sort_bytes));
  char* t = static_cast<char*>(tmp.p);
  auto* d_xyz = reinterpret_cast<float*>(t);
  auto* d_cov = c->has_cov ? reinterpret_cast<float*>(t + b_xyz) : nullptr;
  auto* box = reinterpret_cast<unsigned*>(t + b_xyz + b_cov);
  auto* codes = reinterpret_cast<unsigned*>(t + b_xyz + b_cov + 256);
  auto* idx = codes + b_vec / sizeof(unsigned);
  auto* codes2 = idx + b_vec / sizeof(unsigned);
  auto* perm = codes2 + b_vec / sizeof(unsigned);
  void* temp = t + b_xyz + b_cov + 256 + 4 * b_vec;
  if (int rc = ensure_pinned(ctx, b_xyz + b_cov)) return rc;
  VG_CUDA(cudaStreamSynchronize(s));  // the pinned staging buffer is free
  char* h = static_cast<char*>(ctx->pinned);
  std::memcpy(h, xyz, sizeof(float) * 3 * n);
  if (c->has_cov) std::memcpy(h + b_xyz, cov6, sizeof(float) * 6 * n);
  VG_CUDA(cudaMemcpyAsync(d_xyz, h, b_xyz + b_cov, cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemsetAsync(box, 0xFF, 3 * sizeof(unsigned), s));
  VG_CUDA(cudaMemsetAsync(box + 3, 0, 3 * sizeof(unsigned), s));
  VG_CUDA(launch_cloud_bbox(d_xyz, n, box, s));
  VG_CUDA(launch_cloud_morton(d_xyz, n, box, codes, idx, s));
  VG_CUDA(cub::DeviceRadixSort::SortPairs(temp, sort_bytes, codes, codes2, idx, perm, static_cast<int>(n), 0, 30, s));
  VG_CUDA(launch_cloud_fill(d_xyz, d_cov, n, perm, c->pa, c->pb, c->pc, c->sblk, s));
  ctx->launches += 4;
  unsigned hbox[6];
  VG_CUDA(cudaMemcpyAsync(hbox, box, sizeof(hbox), cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  if (hbox[0] <= hbox[3])  // at least one finite point
    for (int a = 0; a < 3; ++a) c->lo[a] = unordered_host(hbox[a]), c->hi[a] = unordered_host(hbox[3 + a]);
  *out = c.release();
  return VGICP_OK;
}

int vgicp_cloud_upload(vgicp_ctx ctx, const float* xyz, const float* cov6, size_t n, vgicp_cloud* out) try {
  NvtxRange nvtx_("vgicp_cloud_upload");
  return cloud_upload_packed(ctx, xyz, cov6, n, out);
} catch (...) {
  return api_exception();
}

static void parallel_copies(const std::vector<std::tuple<void*, const void*, size_t>>& copies);

// m float32 clouds in one staged H2D and one launch per stage (bounding boxes + Morton codes, one
// segmented stable radix sort, fill) instead of ~8 launches per cloud. Same layout as m single
// uploads: the stable sort of the same codes is the same permutation.
int vgicp_cloud_upload_batch(vgicp_ctx ctx, const float* const* xyz, const float* const* cov6, const size_t* n, int m,
                             vgicp_cloud* out) try {
  NvtxRange nvtx_("vgicp_cloud_upload_batch");
  if (!ctx || (m > 0 && (!xyz || !n || !out))) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (m <= 0) return VGICP_OK;
  for (int k = 0; k < m; ++k) out[k] = nullptr;
  unsigned long long total = 0;
  unsigned max_n = 0;
  for (int k = 0; k < m; ++k) {
    if (n[k] > 0 && !xyz[k]) return fail(VGICP_E_INVALID_ARGUMENT, "null point array");
    total += n[k];
    max_n = std::max<unsigned>(max_n, static_cast<unsigned>(std::min<size_t>(n[k], UINT32_MAX)));
  }
  if (total >= (1ull << 31)) return fail(VGICP_E_INVALID_ARGUMENT, "batch too large (>= 2^31 points)");
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  std::vector<vgicp_cloud> clouds(m, nullptr);
  auto cleanup = [&]() {
    for (auto*& c : clouds) release(c), c = nullptr;
  };
  auto guard = on_failure(cleanup);
  std::vector<UploadSeg> segs(m);
  unsigned long long off = 0;
  for (int k = 0; k < m; ++k) {
    auto* c = new vgicp_cloud_s();
    clouds[k] = c;
    c->ctx = ctx;
    c->n = n[k];
    c->has_cov = cov6 && cov6[k] && n[k] > 0;
    const size_t na = align_up(n[k] * sizeof(float4), 256), nc = align_up(n[k] * sizeof(float), 256);
    const size_t half = 2 * na + nc, nblk = (n[k] + kPointBlock - 1) / kPointBlock;
    c->block_bytes = std::max<size_t>(half + nblk * sizeof(PointBlock), 256);
    if (const cudaError_t e = dmalloc(ctx, &c->block, c->block_bytes);
        e != cudaSuccess) {
      cleanup();
      return cuda_fail(e, "cudaMallocAsync(cloud)");
    }
    char* base = static_cast<char*>(c->block);
    c->pa = reinterpret_cast<float4*>(base);
    c->pb = reinterpret_cast<float4*>(base + na);
    c->pc = reinterpret_cast<float*>(base + 2 * na);
    c->sblk = reinterpret_cast<PointBlock*>(base + half);
    segs[k] = UploadSeg{nullptr, nullptr, static_cast<unsigned>(off), static_cast<unsigned>(n[k]), c->pa, c->pb, c->pc,
                        c->sblk};
    off += n[k];
  }
  if (total > 0) {
    const size_t b_xyz = align_up(sizeof(float) * 3 * total, 256), b_cov = align_up(sizeof(float) * 6 * total, 256);
    const size_t b_vec = align_up(sizeof(unsigned) * total, 256);
    size_t sort_bytes = 0;
    std::vector<int> seg_off(m + 1);
    for (int k = 0; k < m; ++k) seg_off[k] = static_cast<int>(segs[k].offset);
    seg_off[m] = static_cast<int>(total);
    VG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, sort_bytes, (const unsigned*)nullptr, (unsigned*)nullptr,
                                                     (const unsigned*)nullptr, (unsigned*)nullptr,
                                                     static_cast<int>(total), m, (const int*)nullptr,
                                                     (const int*)nullptr, 0, 30, s));
    const size_t b_segs = align_up(sizeof(UploadSeg) * m, 256), b_box = align_up(sizeof(unsigned) * 6 * m, 256);
    const size_t b_off = align_up(sizeof(int) * (m + 1), 256);
    DevBuf tmp(ctx);
    VG_CUDA(tmp.alloc(b_xyz + b_cov + 4 * b_vec + b_segs + b_box + b_off + sort_bytes));
    char* t = static_cast<char*>(tmp.p);
    auto* d_xyz = reinterpret_cast<float*>(t);
    auto* d_cov = reinterpret_cast<float*>(t + b_xyz);
    auto* codes = reinterpret_cast<unsigned*>(t + b_xyz + b_cov);
    auto* idx = codes + b_vec / sizeof(unsigned);
    auto* codes2 = idx + b_vec / sizeof(unsigned);
    auto* perm = codes2 + b_vec / sizeof(unsigned);
    auto* d_segs = reinterpret_cast<UploadSeg*>(t + b_xyz + b_cov + 4 * b_vec);
    auto* d_box = reinterpret_cast<unsigned*>(t + b_xyz + b_cov + 4 * b_vec + b_segs);
    auto* d_off = reinterpret_cast<int*>(t + b_xyz + b_cov + 4 * b_vec + b_segs + b_box);
    void* temp = t + b_xyz + b_cov + 4 * b_vec + b_segs + b_box + b_off;
    for (int k = 0; k < m; ++k) {
      segs[k].xyz = d_xyz + 3 * static_cast<size_t>(segs[k].offset);
      segs[k].cov6 = clouds[k]->has_cov ? d_cov + 6 * static_cast<size_t>(segs[k].offset) : nullptr;
    }
    if (int rc = ensure_pinned(ctx, b_xyz + b_cov)) {
      cleanup();
      return rc;
    }
    VG_CUDA(cudaStreamSynchronize(s));  // the pinned staging buffer is free
    char* h = static_cast<char*>(ctx->pinned);
    std::vector<std::tuple<void*, const void*, size_t>> cp;
    for (int k = 0; k < m; ++k) {
      if (n[k] == 0) continue;
      cp.emplace_back(h + sizeof(float) * 3 * segs[k].offset, xyz[k], sizeof(float) * 3 * n[k]);
      if (clouds[k]->has_cov) cp.emplace_back(h + b_xyz + sizeof(float) * 6 * segs[k].offset, cov6[k], sizeof(float) * 6 * n[k]);
    }
    parallel_copies(cp);
    std::vector<unsigned> hbox(6 * m);
    for (int k = 0; k < m; ++k)
      for (int a = 0; a < 3; ++a) hbox[6 * k + a] = ~0u, hbox[6 * k + 3 + a] = 0u;
    VG_CUDA(cudaMemcpyAsync(d_xyz, h, b_xyz + b_cov, cudaMemcpyHostToDevice, s));
    VG_CUDA(cudaMemcpyAsync(d_segs, segs.data(), sizeof(UploadSeg) * m, cudaMemcpyHostToDevice, s));
    VG_CUDA(cudaMemcpyAsync(d_box, hbox.data(), sizeof(unsigned) * 6 * m, cudaMemcpyHostToDevice, s));
    VG_CUDA(cudaMemcpyAsync(d_off, seg_off.data(), sizeof(int) * (m + 1), cudaMemcpyHostToDevice, s));
    VG_CUDA(launch_upload_batch_prepare(d_segs, m, max_n, d_box, codes, idx, s));
    VG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(temp, sort_bytes, codes, codes2, idx, perm, static_cast<int>(total),
                                                     m, d_off, d_off + 1, 0, 30, s));
    VG_CUDA(launch_upload_batch_fill(d_segs, m, max_n, perm, s));
    ctx->launches += 4;  // bbox, morton, segmented sort (counted once), fill
    VG_CUDA(cudaMemcpyAsync(hbox.data(), d_box, sizeof(unsigned) * 6 * m, cudaMemcpyDeviceToHost, s));
    VG_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < m; ++k)
      if (hbox[6 * k] <= hbox[6 * k + 3])  // at least one finite point
        for (int a = 0; a < 3; ++a)
          clouds[k]->lo[a] = unordered_host(hbox[6 * k + a]), clouds[k]->hi[a] = unordered_host(hbox[6 * k + 3 + a]);
  }
  guard.dismiss();
  for (int k = 0; k < m; ++k) out[k] = clouds[k];
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

static int cloud_from_device_f64(vgicp_ctx ctx, const double* d_xyz, const double* d_cov9, size_t n, bool keep64,
                                 vgicp_cloud* out);

// Reference layout (PointCloud, point_cloud.hpp:21-37: n×3 double means, n×9 double covariances).
// Float32-exact inputs with symmetric covariances (KITTI scans, io.cpp:50) take the float32 layout
// unchanged; anything else (submap clouds: transform_cloud + voxel_downsample output,
// pipeline.cpp:100-111) is kept in float64 as well, so keys / correspondences / overlap hits and map
// statistics built from it are those of the reference's double arithmetic.
int vgicp_cloud_upload_f64(vgicp_ctx ctx, const double* xyz, const double* cov9, size_t n, vgicp_cloud* out) try {
  NvtxRange nvtx_("vgicp_cloud_upload_f64");
  if (!ctx || !out) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (n > 0 && !xyz) return fail(VGICP_E_INVALID_ARGUMENT, "null point array");
  if (n >= (1ull << 31)) return fail(VGICP_E_INVALID_ARGUMENT, "cloud too large (>= 2^31 points)");
  auto f32_exact = [](double v) { return static_cast<double>(static_cast<float>(v)) == v; };
  bool exact = true;
  for (size_t i = 0; i < 3 * n && exact; ++i) exact = f32_exact(xyz[i]);
  for (size_t i = 0; cov9 && i < n && exact; ++i) {
    const double* m = cov9 + 9 * i;
    for (int k = 0; k < 9 && exact; ++k) exact = f32_exact(m[k]);
    exact = exact && m[1] == m[3] && m[2] == m[6] && m[5] == m[7];
  }
  if (exact || n == 0) {
    std::vector<float> p(3 * n), c(cov9 ? 6 * n : 0);
    for (size_t i = 0; i < 3 * n; ++i) p[i] = static_cast<float>(xyz[i]);
    if (cov9) {
      for (size_t i = 0; i < n; ++i) {
        const double* m = cov9 + 9 * i;
        const int idx[6] = {0, 1, 2, 4, 5, 8};
        for (int k = 0; k < 6; ++k) c[6 * i + k] = static_cast<float>(m[idx[k]]);
      }
    }
    return cloud_upload_packed(ctx, p.data(), cov9 ? c.data() : nullptr, n, out);
  }
  DeviceGuard g(ctx->device);
  DevBuf buf(ctx);
  VG_CUDA(buf.alloc(n * (cov9 ? 12 : 3) * sizeof(double)));
  double* d_xyz = static_cast<double*>(buf.p);
  double* d_cov = cov9 ? d_xyz + 3 * n : nullptr;
  VG_CUDA(cudaMemcpyAsync(d_xyz, xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  if (cov9) VG_CUDA(cudaMemcpyAsync(d_cov, cov9, n * 9 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  return cloud_from_device_f64(ctx, d_xyz, d_cov, n, true, out);  // synchronises before returning
} catch (...) {
  return api_exception();
}

int vgicp_cloud_is_f64(vgicp_cloud cloud, int* f64) try {
  if (!cloud || !f64) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *f64 = cloud->f64 ? 1 : 0;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_cloud_size(vgicp_cloud cloud, size_t* n) try {
  if (!cloud || !n) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *n = cloud->n;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_cloud_has_covariances(vgicp_cloud cloud, int* has) try {
  if (!cloud || !has) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *has = cloud->has_cov ? 1 : 0;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_cloud_destroy(vgicp_cloud cloud) try {
  release(cloud);
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// ------------------------------------------------------------------------------------ voxel maps
static int build_segments(vgicp_ctx ctx, std::vector<BuildSeg>& segs, vgicp_map* out);

// Occupancy bitmaps + rank-ordered statistics for freshly built maps: one 16-B record per 4×4×4
// brick of the occupied voxel box; maps whose box would need more than kOccMaxWords records keep
// hash probes only. `hot` / `vbase` are the build's per-voxel fp32 statistics.
constexpr size_t kOccMaxWords = size_t(1) << 21;  // 32 MB of records per map
static int build_occupancy(vgicp_ctx ctx, vgicp_map* maps, int m, const VoxelStats* hot,
                           const std::vector<unsigned>& vbase, cudaStream_t s) {
  if (std::getenv("VGICP_NO_OCCUPANCY")) return VGICP_OK;  // measurement switch (hash probes only)
  std::vector<OccJob> jobs;
  unsigned max_words = 0, max_v = 0;
  for (int k = 0; k < m; ++k) {
    vgicp_map mp = maps[k];
    if (mp->voxels == 0 || mp->cmin[0] > mp->cmax[0]) continue;
    unsigned e[3];
    size_t words = 1;
    for (int a = 0; a < 3; ++a) {
      e[a] = static_cast<unsigned>(mp->cmax[a] - mp->cmin[a] + 1);
      words *= (e[a] + 3) / 4;
    }
    if (words > kOccMaxWords) continue;
    const size_t V = mp->voxels;
    const size_t b_occ = align_up(sizeof(OccWord) * words, 256), b_ra = align_up(sizeof(SlotStatsA) * V, 256);
    mp->occ_bytes = b_occ + b_ra + sizeof(SlotStatsB) * V;
    VG_CUDA(dmalloc(ctx, &mp->occ_mem, mp->occ_bytes));
    char* base = static_cast<char*>(mp->occ_mem);
    OccDev& o = mp->occ;
    o.occ = reinterpret_cast<const OccWord*>(base);
    o.kx0 = static_cast<unsigned>(mp->cmin[0] + (1 << 20));
    o.ky0 = static_cast<unsigned>(mp->cmin[1] + (1 << 20));
    o.kz0 = static_cast<unsigned>(mp->cmin[2] + (1 << 20));
    o.ex = e[0], o.ey = e[1], o.ez = e[2];
    o.nby = (e[1] + 3) / 4, o.nbz = (e[2] + 3) / 4;
    mp->ra = reinterpret_cast<SlotStatsA*>(base + b_occ);
    mp->rb = reinterpret_cast<SlotStatsB*>(base + b_occ + b_ra);
    jobs.push_back(OccJob{mp->keys, reinterpret_cast<OccWord*>(base), mp->ra, mp->rb, static_cast<unsigned>(V),
                          static_cast<unsigned>(words), o.kx0, o.ky0, o.kz0, o.nby, o.nbz, vbase[k]});
    max_words = std::max(max_words, static_cast<unsigned>(words));
    max_v = std::max(max_v, static_cast<unsigned>(V));
  }
  if (jobs.empty()) return VGICP_OK;
  DevBuf d_jobs(ctx);
  VG_CUDA(d_jobs.alloc(sizeof(OccJob) * jobs.size()));
  VG_CUDA(cudaMemcpyAsync(d_jobs.p, jobs.data(), sizeof(OccJob) * jobs.size(), cudaMemcpyHostToDevice, s));
  VG_CUDA(launch_occ_build(static_cast<const OccJob*>(d_jobs.p), static_cast<int>(jobs.size()), max_words, max_v, hot,
                           s));
  ctx->launches += 4;
  VG_CUDA(cudaStreamSynchronize(s));  // the job array is freed on return
  return VGICP_OK;
}

// ---- hand-written build of float32 clouds (build.cu) ----------------------------------------
// Occupied voxel box of a float32 cloud at resolution r, exactly: floor(fl(x / r)) is monotone in x,
// so the box of the finite bounding box is the box of the voxels (what the build would find). false
// when the cloud has no finite point; out_of_range when a bound lies beyond ±2^20 voxels.
static bool fast_box(const vgicp_cloud_s* c, double r, int cmin[3], int cmax[3], bool* out_of_range) {
  *out_of_range = false;
  if (c->lo[0] > c->hi[0]) return false;
  for (int a = 0; a < 3; ++a) {
    const double l = std::floor(static_cast<double>(c->lo[a]) / r), h = std::floor(static_cast<double>(c->hi[a]) / r);
    if (!(l >= -kKeyBiasD && h < kKeyBiasD)) {
      *out_of_range = true;
      return false;
    }
    cmin[a] = static_cast<int>(l);
    cmax[a] = static_cast<int>(h);
  }
  return true;
}

static size_t fast_words(const int cmin[3], const int cmax[3]) {
  size_t words = 1;
  for (int a = 0; a < 3; ++a) words *= static_cast<size_t>((cmax[a] - cmin[a] + 1 + 3) / 4);
  return words;
}

// Export buffers of a single-map rebuild (rank order).
struct FastExport {
  unsigned long long* keys = nullptr;
  int* counts = nullptr;
  double* mean64 = nullptr;
  double* cov9 = nullptr;
  unsigned V = 0;
  void* mem = nullptr;
};

// Builds maps of float32 clouds clouds[k] at res[k] with the hand-written kernels: zero + mark,
// rank, (sync: V per map, range errors), order, accumulate. With `exp` (one map): export mode — the
// key-ordered statistics are written to device buffers in rank order (exp->mem, freed by the caller).
static int build_fast_ordered(vgicp_ctx ctx, const vgicp_cloud* clouds, const double* res, int m, int m_smem,
                              vgicp_map* out, FastExport* exp);

// Jobs are ordered so that the maps whose bitmap fits in shared memory come first (one fused
// zero + mark + rank launch for them, the global-atomic kernels for the rest).
static int build_fast(vgicp_ctx ctx, const vgicp_cloud* clouds, const double* res, int m, vgicp_map* out,
                      FastExport* exp) {
  const unsigned smem_words = fast_markrank_smem_words(ctx->device);
  std::vector<int> perm;
  for (int pass = 0; pass < 2; ++pass)
    for (int k = 0; k < m; ++k) {
      int cmin[3], cmax[3];
      bool oor = false;
      const bool fits = fast_box(clouds[k], res[k], cmin, cmax, &oor) && fast_words(cmin, cmax) <= smem_words;
      if (fits == (pass == 0)) perm.push_back(k);
    }
  int m_smem = 0;
  for (int k = 0; k < m; ++k) {
    int cmin[3], cmax[3];
    bool oor = false;
    m_smem += fast_box(clouds[k], res[k], cmin, cmax, &oor) && fast_words(cmin, cmax) <= smem_words ? 1 : 0;
  }
  std::vector<vgicp_cloud> pc(m);
  std::vector<double> pr(m);
  for (int q = 0; q < m; ++q) pc[q] = clouds[perm[q]], pr[q] = res[perm[q]];
  std::vector<vgicp_map> pm(m, nullptr);
  if (int rc = build_fast_ordered(ctx, pc.data(), pr.data(), m, m_smem, pm.data(), exp)) return rc;
  for (int q = 0; q < m; ++q) out[perm[q]] = pm[q];
  return VGICP_OK;
}

static int build_fast_ordered(vgicp_ctx ctx, const vgicp_cloud* clouds, const double* res, int m, int m_smem,
                              vgicp_map* out, FastExport* exp) {
  cudaStream_t s = ctx->stream;
  std::vector<FastBuildJob> jobs(m);
  std::vector<vgicp_map> maps(m, nullptr);
  auto cleanup = [&]() {
    for (auto*& mp : maps) release(mp), mp = nullptr;
  };
  auto guard = on_failure(cleanup);
  unsigned long long total = 0;
  unsigned max_n = 0, max_words = 0;
  for (int k = 0; k < m; ++k) {
    const vgicp_cloud c = clouds[k];
    int cmin[3], cmax[3];
    bool oor = false;
    if (!fast_box(c, res[k], cmin, cmax, &oor)) {
      cleanup();
      return fail(oor || c->n > 0 ? VGICP_E_OUT_OF_RANGE : VGICP_E_INVALID_ARGUMENT,
                  "point beyond the +-2^20 voxel-per-axis range limit");
    }
    auto* mp = new vgicp_map_s();
    maps[k] = mp;
    mp->ctx = ctx;
    mp->res = res[k];
    mp->inv_res = 1.0 / res[k];
    mp->total_points = c->n;
    mp->fast = true;
    c->refs.fetch_add(1);
    mp->src = c;
    for (int a = 0; a < 3; ++a) mp->cmin[a] = cmin[a], mp->cmax[a] = cmax[a];
    const size_t words = fast_words(cmin, cmax);
    mp->occ_bytes = sizeof(OccWord) * words;
    VG_CUDA(dmalloc(ctx, &mp->occ_mem, mp->occ_bytes));
    OccDev& o = mp->occ;
    o.occ = static_cast<const OccWord*>(mp->occ_mem);
    o.kx0 = static_cast<unsigned>(cmin[0] + (1 << 20));
    o.ky0 = static_cast<unsigned>(cmin[1] + (1 << 20));
    o.kz0 = static_cast<unsigned>(cmin[2] + (1 << 20));
    o.ex = static_cast<unsigned>(cmax[0] - cmin[0] + 1);
    o.ey = static_cast<unsigned>(cmax[1] - cmin[1] + 1);
    o.ez = static_cast<unsigned>(cmax[2] - cmin[2] + 1);
    o.nby = (o.ey + 3) / 4, o.nbz = (o.ez + 3) / 4;
    FastBuildJob& j = jobs[k];
    j = FastBuildJob{};
    j.pa = c->pa, j.pb = c->pb, j.pc = c->pc;
    j.n = static_cast<unsigned>(c->n);
    j.pt_off = static_cast<unsigned>(total);
    j.vx_off = static_cast<unsigned>(total + k);  // V + 1 <= n + 1 offsets per map
    j.res = mp->res, j.inv_res = mp->inv_res;
    j.kx0 = o.kx0, j.ky0 = o.ky0, j.kz0 = o.kz0, j.ex = o.ex, j.ey = o.ey, j.ez = o.ez, j.nby = o.nby, j.nbz = o.nbz;
    j.words = static_cast<unsigned>(words);
    j.occ = static_cast<OccWord*>(mp->occ_mem);
    total += c->n;
    max_n = std::max(max_n, j.n);
    max_words = std::max(max_words, j.words);
  }
  if (total + m >= (1ull << 32)) {
    cleanup();
    return fail(VGICP_E_INVALID_ARGUMENT, "batched build exceeds 2^32 points");
  }
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t o_jobs = carve(sizeof(FastBuildJob) * m);
  const size_t o_idx = carve(sizeof(int) * m);
  const size_t o_err = carve(sizeof(int) * m);
  const size_t o_vc = carve(sizeof(unsigned) * m);
  const size_t o_code = carve(sizeof(unsigned) * total);
  const size_t o_list = carve(sizeof(unsigned) * total);
  const size_t o_offs = carve(sizeof(unsigned) * (total + m));
  const size_t o_gcnt = carve(sizeof(unsigned) * 2 * (total + m));  // per-point ranks | global cursors
  if (int rc = ensure_scratch(ctx, off)) {
    cleanup();
    return rc;
  }
  char* sb = static_cast<char*>(ctx->scratch);
  auto* d_jobs = reinterpret_cast<FastBuildJob*>(sb + o_jobs);
  auto* d_idx = reinterpret_cast<int*>(sb + o_idx);
  auto* d_err = reinterpret_cast<int*>(sb + o_err);
  auto* d_vc = reinterpret_cast<unsigned*>(sb + o_vc);
  auto* d_code = reinterpret_cast<unsigned*>(sb + o_code);
  auto* d_list = reinterpret_cast<unsigned*>(sb + o_list);
  auto* d_offs = reinterpret_cast<unsigned*>(sb + o_offs);
  auto* d_gcnt = reinterpret_cast<unsigned*>(sb + o_gcnt);
  int rc = VGICP_OK;
  auto step = [&](cudaError_t e, const char* what) {
    if (rc == VGICP_OK && e != cudaSuccess) rc = cuda_fail(e, what);
  };
  step(cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(FastBuildJob) * m, cudaMemcpyHostToDevice, s), "build jobs");
  step(cudaMemsetAsync(d_err, 0, sizeof(int) * m, s), "build flags");
  unsigned max_words_smem = 0, max_words_glob = 0, max_n_glob = 0;
  for (int k = 0; k < m; ++k) {
    if (k < m_smem) {
      max_words_smem = std::max(max_words_smem, jobs[k].words);
    } else {
      max_words_glob = std::max(max_words_glob, jobs[k].words);
      max_n_glob = std::max(max_n_glob, jobs[k].n);
    }
  }
  (void)max_words;
  (void)max_n;
  if (rc == VGICP_OK && m_smem > 0)
    step(launch_fast_markrank_smem(d_jobs, m_smem, max_words_smem, d_code, d_err, d_vc, s), "build mark+rank");
  if (rc == VGICP_OK && m > m_smem) {
    step(launch_fast_mark(d_jobs + m_smem, m - m_smem, max_n_glob, max_words_glob, d_code, d_err + m_smem, s),
         "build mark");
    if (rc == VGICP_OK) step(launch_fast_rank(d_jobs + m_smem, m - m_smem, d_vc + m_smem, s), "build rank");
  }
  std::vector<int> herr(m);
  std::vector<unsigned> hv(m);
  step(cudaMemcpyAsync(herr.data(), d_err, sizeof(int) * m, cudaMemcpyDeviceToHost, s), "build flags");
  step(cudaMemcpyAsync(hv.data(), d_vc, sizeof(unsigned) * m, cudaMemcpyDeviceToHost, s), "build counts");
  step(cudaStreamSynchronize(s), "build rank");
  if (rc != VGICP_OK) {
    cleanup();
    return rc;
  }
  ctx->launches += (m_smem > 0 ? 1 : 0) + (m > m_smem ? 3 : 0);  // mark+rank | zero, mark, rank
  for (int k = 0; k < m; ++k)
    if (herr[k]) {
      cleanup();
      return fail(VGICP_E_OUT_OF_RANGE, "point beyond the +-2^20 voxel-per-axis range limit");
    }
  // per-map voxel arrays: ra | rb | cov64 (rank order; the 6 unique entries — float32 clouds have
  // symmetric covariances, so the sums are symmetric bit for bit — except in export mode, whose
  // rebuilt map hands its full 9-entry rows to the caller)
  unsigned max_v = 0, smem_v = fast_order_smem_voxels(ctx->device);
  const unsigned sort_n = std::getenv("VGICP_BUILD_SCATTER") ? 0u : fast_sort_max_points(ctx->device);
  std::vector<int> in_sort, in_smem, in_global;
  for (int k = 0; k < m; ++k) {
    vgicp_map mp = maps[k];
    const size_t V = hv[k];
    mp->voxels = V;
    const size_t b_ra = align_up(sizeof(SlotStatsA) * V, 256), b_rb = align_up(sizeof(SlotStatsB) * V, 256);
    mp->cov6 = exp == nullptr;
    mp->cold_bytes = std::max<size_t>(b_ra + b_rb + sizeof(double) * (mp->cov6 ? 6 : 9) * V, 256);
    if (const cudaError_t e = dmalloc(ctx, &mp->cold, mp->cold_bytes);
        e != cudaSuccess) {
      cleanup();
      return cuda_fail(e, "cudaMallocAsync(voxel map)");
    }
    char* b = static_cast<char*>(mp->cold);
    mp->ra = reinterpret_cast<SlotStatsA*>(b);
    mp->rb = reinterpret_cast<SlotStatsB*>(b + b_ra);
    mp->cov64 = reinterpret_cast<double*>(b + b_ra + b_rb);
    jobs[k].V = static_cast<unsigned>(V);
    jobs[k].ra = mp->ra, jobs[k].rb = mp->rb, jobs[k].cov9 = mp->cov64;
    max_v = std::max(max_v, jobs[k].V);
    (jobs[k].n <= sort_n ? in_sort : V <= smem_v ? in_smem : in_global).push_back(k);
  }
  if (exp) {  // single map: key-ordered statistics in rank order
    const size_t V = hv[0];
    exp->V = static_cast<unsigned>(V);
    VG_CUDA(dmalloc(ctx, &exp->mem, std::max<size_t>(V * (8 + 4 + 24) + 1024, 256)));
    char* b = static_cast<char*>(exp->mem);
    exp->keys = reinterpret_cast<unsigned long long*>(b);
    exp->counts = reinterpret_cast<int*>(b + align_up(8 * V, 256));
    exp->mean64 = reinterpret_cast<double*>(b + align_up(8 * V, 256) + align_up(4 * V, 256));
    exp->cov9 = maps[0]->cov64;  // the rebuilt map's own rank-ordered fp64 covariances
    jobs[0].keys = exp->keys, jobs[0].counts = exp->counts, jobs[0].mean64 = exp->mean64;
  }
  std::vector<int> order(in_sort);
  order.insert(order.end(), in_smem.begin(), in_smem.end());
  order.insert(order.end(), in_global.begin(), in_global.end());
  unsigned smem_max = 0, sort_max = 0;
  for (int k : in_smem) smem_max = std::max(smem_max, jobs[k].V);
  for (int k : in_sort) sort_max = std::max(sort_max, jobs[k].n);
  step(cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(FastBuildJob) * m, cudaMemcpyHostToDevice, s), "build jobs");
  step(cudaMemcpyAsync(d_idx, order.data(), sizeof(int) * m, cudaMemcpyHostToDevice, s), "build jobs");
  if (rc == VGICP_OK && !in_sort.empty())
    step(launch_fast_sort(d_jobs, d_idx, static_cast<int>(in_sort.size()), sort_max, d_code, d_list, d_offs, s),
         "build sort");
  if (rc == VGICP_OK && !in_smem.empty())
    step(launch_fast_order(d_jobs, d_idx + in_sort.size(), static_cast<int>(in_smem.size()), std::max(1u, smem_max),
                           d_code, d_gcnt, d_list, d_offs, d_gcnt + total + m, s),
         "build order");
  if (rc == VGICP_OK && !in_global.empty())
    step(launch_fast_order(d_jobs, d_idx + in_sort.size() + in_smem.size(), static_cast<int>(in_global.size()), 0u,
                           d_code, d_gcnt, d_list, d_offs, d_gcnt + total + m, s),
         "build order (global cursors)");
  if (rc == VGICP_OK) step(launch_fast_accumulate(d_jobs, m, max_v, d_list, d_offs, d_code, exp != nullptr, s), "build accumulate");
  step(cudaStreamSynchronize(s), "build");
  if (rc != VGICP_OK) {
    cleanup();
    return rc;
  }
  ctx->launches += (in_sort.empty() ? 0 : 1) + (in_smem.empty() ? 0 : 1) + (in_global.empty() ? 0 : 1) + 1;
  guard.dismiss();
  for (int k = 0; k < m; ++k) out[k] = maps[k];
  return VGICP_OK;
}

// The key-ordered statistics of a hand-built map (export, on-demand hash table): the same kernels
// rerun on the map's source cloud in export mode, then ordered by key on the host.
static int fast_export(vgicp_map map, std::vector<uint64_t>* keys, std::vector<int32_t>* counts,
                       std::vector<double>* means, std::vector<double>* covs, std::vector<unsigned>* rank_of_sorted) {
  vgicp_ctx ctx = map->ctx;
  vgicp_map tmp = nullptr;
  FastExport ex;
  const double r = map->res;
  if (int rc = build_fast(ctx, &map->src, &r, 1, &tmp, &ex)) {
    dfree(ctx, ex.mem);
    return rc;
  }
  const size_t V = ex.V;
  std::vector<uint64_t> k(V);
  std::vector<int32_t> c(V);
  std::vector<double> mu(3 * V), cv(9 * V);
  cudaStream_t s = ctx->stream;
  int rc = VGICP_OK;
  if (V > 0) {
    cudaError_t e = cudaMemcpyAsync(k.data(), ex.keys, 8 * V, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && counts) e = cudaMemcpyAsync(c.data(), ex.counts, 4 * V, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && means) e = cudaMemcpyAsync(mu.data(), ex.mean64, 24 * V, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && covs) e = cudaMemcpyAsync(cv.data(), ex.cov9, 72 * V, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "voxel map export");
  }
  dfree(ctx, ex.mem);
  release(tmp);
  if (rc != VGICP_OK) return rc;
  std::vector<unsigned> perm(V);
  for (size_t v = 0; v < V; ++v) perm[v] = static_cast<unsigned>(v);
  std::sort(perm.begin(), perm.end(), [&](unsigned a, unsigned b) { return k[a] < k[b]; });
  if (keys) {
    keys->resize(V);
    for (size_t q = 0; q < V; ++q) (*keys)[q] = k[perm[q]];
  }
  if (counts) {
    counts->resize(V);
    for (size_t q = 0; q < V; ++q) (*counts)[q] = c[perm[q]];
  }
  if (means) {
    means->resize(3 * V);
    for (size_t q = 0; q < V; ++q) std::memcpy(&(*means)[3 * q], &mu[3 * perm[q]], 24);
  }
  if (covs) {
    covs->resize(9 * V);
    for (size_t q = 0; q < V; ++q) std::memcpy(&(*covs)[9 * q], &cv[9 * perm[q]], 72);
  }
  if (rank_of_sorted) rank_of_sorted->swap(perm);
  return VGICP_OK;
}

// Hash table of a hand-built map, on demand (lookups, hash-probe measurement modes): keys in rank
// order, cuckoo insertion (rebuilt with twice the buckets on overflow), slot <- rank statistics.
static int ensure_table(vgicp_map mp) {
  if (mp->table || mp->voxels == 0 || !mp->fast) return VGICP_OK;
  std::vector<uint64_t> sorted;
  std::vector<unsigned> rank;
  if (int rc = fast_export(mp, &sorted, nullptr, nullptr, nullptr, &rank)) return rc;
  const size_t V = mp->voxels;
  std::vector<unsigned long long> by_rank(V);
  for (size_t q = 0; q < V; ++q) by_rank[rank[q]] = sorted[q];
  vgicp_ctx ctx = mp->ctx;
  cudaStream_t s = ctx->stream;
  DevBuf buf(ctx);
  VG_CUDA(buf.alloc(align_up(8 * V, 256) + 256 + sizeof(InsertJob)));
  auto* d_keys = static_cast<unsigned long long*>(buf.p);
  auto* d_ovf = reinterpret_cast<int*>(static_cast<char*>(buf.p) + align_up(8 * V, 256));
  auto* d_job = reinterpret_cast<InsertJob*>(static_cast<char*>(buf.p) + align_up(8 * V, 256) + 256);
  VG_CUDA(cudaMemcpyAsync(d_keys, by_rank.data(), 8 * V, cudaMemcpyHostToDevice, s));
  unsigned buckets = std::max(16u, next_pow2((2ull * V + kBucket - 1) / kBucket));  // load <= 0.5
  for (int attempt = 0;; ++attempt) {
    if (attempt > 8) return fail(VGICP_E_CUDA, "voxel hash table insertion did not converge");
    if (int rc = alloc_table(mp, buckets, s)) return rc;
    InsertJob job{mp->tkeys, mp->sa, mp->sb, d_keys, 0u, static_cast<unsigned>(V), mp->shift, 0u};
    int ovf = 0;
    VG_CUDA(cudaMemcpyAsync(d_job, &job, sizeof(job), cudaMemcpyHostToDevice, s));
    VG_CUDA(cudaMemsetAsync(d_ovf, 0, sizeof(int), s));
    VG_CUDA(launch_build_insert(d_job, 1, static_cast<unsigned>(V), d_ovf, s));
    VG_CUDA(cudaMemcpyAsync(&ovf, d_ovf, sizeof(int), cudaMemcpyDeviceToHost, s));
    VG_CUDA(cudaStreamSynchronize(s));
    ctx->launches += 1;
    if (!ovf) {
      VG_CUDA(launch_place_rank(d_job, static_cast<unsigned>(V), mp->ra, mp->rb, s));
      VG_CUDA(cudaStreamSynchronize(s));
      ctx->launches += 1;
      return VGICP_OK;
    }
    buckets *= 2;
  }
}

// GaussianVoxelMap ctor's resolution check (voxelmap.cpp:66-68: `resolution <= 0` -> invalid_argument).
// A NaN resolution passes it there and fails the first voxel_coord as out_of_range — the callers map
// it after their covariance check, in the reference's order. +inf, which the reference accepts (every
// point in voxel 0), is rejected: voxel corners c·r would be 0·inf here.
static int check_resolution(double r) {
  if (r <= 0.0) return fail(VGICP_E_INVALID_ARGUMENT, "voxel resolution must be positive");
  if (std::isinf(r)) return fail(VGICP_E_INVALID_ARGUMENT, "voxel resolution must be finite");
  return VGICP_OK;
}

int vgicp_voxelmap_build_batch(vgicp_ctx ctx, const vgicp_cloud* clouds, const double* resolutions, int m,
                               vgicp_map* out) try {
  NvtxRange nvtx_("vgicp_voxelmap_build_batch");
  if (!ctx || !out || (m > 0 && (!clouds || !resolutions))) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (m <= 0) return VGICP_OK;
  for (int k = 0; k < m; ++k) out[k] = nullptr;
  // GaussianVoxelMap ctor validation order (voxelmap.cpp:67-72)
  for (int k = 0; k < m; ++k) {
    if (int rc = check_resolution(resolutions[k])) return rc;
    if (!clouds[k] || clouds[k]->ctx != ctx) return fail(VGICP_E_INVALID_ARGUMENT, "cloud of another context");
    if (!clouds[k]->has_cov)
      return fail(VGICP_E_INVALID_ARGUMENT, "voxel map construction requires per-point covariances");
  }
  for (int k = 0; k < m; ++k)  // NaN: the reference's voxel_coord range check fails (voxelmap.cpp:48-51)
    if (std::isnan(resolutions[k])) return fail(VGICP_E_OUT_OF_RANGE, "point beyond the +-2^20 voxel-per-axis range limit");
  DeviceGuard g(ctx->device);
  // float32 clouds whose occupied box has a bitmap of <= kOccMaxWords records take the hand-written
  // build (build.cu); float64 clouds and sprawling boxes the sort-based one below
  // (VGICP_SORTED_BUILD=1 forces the latter: measurement / cross-check switch)
  const bool sorted_only = std::getenv("VGICP_SORTED_BUILD") != nullptr;
  std::vector<int> fast_idx, slow_idx;
  for (int k = 0; k < m; ++k) {
    const vgicp_cloud c = clouds[k];
    int cmin[3], cmax[3];
    bool oor = false;
    const bool boxed = fast_box(c, resolutions[k], cmin, cmax, &oor);
    if (oor) return fail(VGICP_E_OUT_OF_RANGE, "point beyond the +-2^20 voxel-per-axis range limit");
    const bool fast = !sorted_only && !c->f64 && boxed && fast_words(cmin, cmax) <= kOccMaxWords;
    (fast ? fast_idx : slow_idx).push_back(k);
  }
  if (!fast_idx.empty()) {
    std::vector<vgicp_cloud> fc;
    std::vector<double> fr;
    for (int k : fast_idx) fc.push_back(clouds[k]), fr.push_back(resolutions[k]);
    std::vector<vgicp_map> fm(fast_idx.size(), nullptr);
    if (int rc = build_fast(ctx, fc.data(), fr.data(), static_cast<int>(fc.size()), fm.data(), nullptr)) return rc;
    if (slow_idx.empty()) {
      for (size_t q = 0; q < fast_idx.size(); ++q) out[fast_idx[q]] = fm[q];
      return VGICP_OK;
    }
    std::vector<vgicp_cloud> sc;
    std::vector<double> sr;
    for (int k : slow_idx) sc.push_back(clouds[k]), sr.push_back(resolutions[k]);
    std::vector<vgicp_map> sm(slow_idx.size(), nullptr);
    if (int rc = vgicp_voxelmap_build_batch(ctx, sc.data(), sr.data(), static_cast<int>(sc.size()), sm.data())) {
      for (auto* mp : fm) release(mp);
      return rc;
    }
    for (size_t q = 0; q < fast_idx.size(); ++q) out[fast_idx[q]] = fm[q];
    for (size_t q = 0; q < slow_idx.size(); ++q) out[slow_idx[q]] = sm[q];
    return VGICP_OK;
  }
  std::vector<BuildSeg> segs(m);
  for (int k = 0; k < m; ++k) {
    const vgicp_cloud c = clouds[k];
    // float64 clouds accumulate their exact float64 means / covariances (all 9 entries, as
    // VoxelAccumulator does); float32-exact clouds their float32 layout (identical values)
    segs[k] = c->f64 ? BuildSeg{nullptr, nullptr, nullptr, c->m64, c->c64, 0ull, static_cast<unsigned>(c->n), 0u,
                                resolutions[k], 1.0 / resolutions[k]}
                     : BuildSeg{c->pa, c->pb, c->pc, nullptr, nullptr, 0ull, static_cast<unsigned>(c->n), 0u,
                                resolutions[k], 1.0 / resolutions[k]};
  }
  return build_segments(ctx, segs, out);
} catch (...) {
  return api_exception();
}

// Batched build core: segments are float32 device clouds or fp64 device arrays (BuildSeg).
static int build_segments(vgicp_ctx ctx, std::vector<BuildSeg>& segs, vgicp_map* out) {
  const int m = static_cast<int>(segs.size());
  unsigned long long total = 0;
  unsigned max_n = 0;
  for (int k = 0; k < m; ++k) {
    segs[k].offset = total;
    total += segs[k].n;
    max_n = std::max<unsigned>(max_n, segs[k].n);
  }
  if (total >= (1ull << 31)) return fail(VGICP_E_INVALID_ARGUMENT, "batched build exceeds 2^31 points");
  const int ntot = static_cast<int>(total);

  // scratch layout
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t o_segs = carve(sizeof(BuildSeg) * m);
  const size_t o_outs = carve(sizeof(BuildOut) * m);
  const size_t o_offs = carve(sizeof(int) * (m + 1));
  const size_t o_err = carve(sizeof(int) * m);
  const size_t o_vcnt = carve(sizeof(unsigned) * m);
  const size_t o_vbase = carve(sizeof(unsigned) * m);
  const size_t o_k0 = carve(sizeof(unsigned long long) * total);
  const size_t o_k1 = carve(sizeof(unsigned long long) * total);
  const size_t o_v0 = carve(sizeof(unsigned) * total);
  const size_t o_v1 = carve(sizeof(unsigned) * total);
  const size_t o_heads = carve(sizeof(unsigned) * total);
  const size_t o_vidx = carve(sizeof(unsigned) * total);
  const size_t o_hot = carve(sizeof(VoxelStats) * total);  // compact hot records (V <= N)
  const size_t o_jobs = carve(sizeof(InsertJob) * m);
  const size_t o_ovf = carve(sizeof(int) * m);
  const size_t o_cbox = carve(sizeof(int) * 6 * m);
  std::vector<int> offsets(m + 1);
  for (int k = 0; k < m; ++k) offsets[k] = static_cast<int>(segs[k].offset);
  offsets[m] = ntot;
  size_t sort_bytes = 0, scan_bytes = 0;
  VG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, sort_bytes, (const unsigned long long*)nullptr,
                                                   (unsigned long long*)nullptr, (const unsigned*)nullptr,
                                                   (unsigned*)nullptr, ntot, m, (const int*)nullptr,
                                                   (const int*)nullptr, 0, 63, ctx->stream));
  VG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const unsigned*)nullptr, (unsigned*)nullptr, ntot,
                                        ctx->stream));
  const size_t o_temp = carve(std::max(sort_bytes, scan_bytes));
  if (int rc = ensure_scratch(ctx, off)) return rc;
  char* sb = static_cast<char*>(ctx->scratch);
  auto* d_segs = reinterpret_cast<BuildSeg*>(sb + o_segs);
  auto* d_outs = reinterpret_cast<BuildOut*>(sb + o_outs);
  auto* d_offs = reinterpret_cast<int*>(sb + o_offs);
  auto* d_err = reinterpret_cast<int*>(sb + o_err);
  auto* d_vcnt = reinterpret_cast<unsigned*>(sb + o_vcnt);
  auto* d_vbase = reinterpret_cast<unsigned*>(sb + o_vbase);
  auto* d_k0 = reinterpret_cast<unsigned long long*>(sb + o_k0);
  auto* d_k1 = reinterpret_cast<unsigned long long*>(sb + o_k1);
  auto* d_v0 = reinterpret_cast<unsigned*>(sb + o_v0);
  auto* d_v1 = reinterpret_cast<unsigned*>(sb + o_v1);
  auto* d_heads = reinterpret_cast<unsigned*>(sb + o_heads);
  auto* d_vidx = reinterpret_cast<unsigned*>(sb + o_vidx);
  auto* d_hot = reinterpret_cast<VoxelStats*>(sb + o_hot);
  auto* d_jobs = reinterpret_cast<InsertJob*>(sb + o_jobs);
  auto* d_ovf = reinterpret_cast<int*>(sb + o_ovf);
  auto* d_cbox = reinterpret_cast<int*>(sb + o_cbox);
  void* d_temp = sb + o_temp;
  cudaStream_t s = ctx->stream;

  VG_CUDA(cudaMemcpyAsync(d_segs, segs.data(), sizeof(BuildSeg) * m, cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemcpyAsync(d_offs, offsets.data(), sizeof(int) * (m + 1), cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int) * m, s));
  VG_CUDA(launch_build_keys(d_segs, m, max_n, d_k0, d_v0, d_err, s));
  VG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(d_temp, sort_bytes, d_k0, d_k1, d_v0, d_v1, ntot, m, d_offs,
                                                   d_offs + 1, 0, 63, s));
  VG_CUDA(launch_build_heads(d_segs, m, max_n, d_k1, d_heads, s));
  VG_CUDA(cub::DeviceScan::ExclusiveSum(d_temp, scan_bytes, d_heads, d_vidx, ntot, s));
  VG_CUDA(launch_build_counts(d_segs, m, d_heads, d_vidx, d_vcnt, d_vbase, s));
  ctx->launches += 5;  // keys, heads, counts + CUB sort/scan (counted as one each)
  std::vector<int> herr(m);
  std::vector<unsigned> hv(m), hbase(m);
  VG_CUDA(cudaMemcpyAsync(herr.data(), d_err, sizeof(int) * m, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaMemcpyAsync(hv.data(), d_vcnt, sizeof(unsigned) * m, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaMemcpyAsync(hbase.data(), d_vbase, sizeof(unsigned) * m, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < m; ++k)
    if (herr[k]) return fail(VGICP_E_OUT_OF_RANGE, "point beyond the +-2^20 voxel-per-axis range limit");

  // allocate maps: cold fp64 arrays + a two-choice table with >= V/2 buckets (load <= 0.5)
  std::vector<vgicp_map> maps(m, nullptr);
  auto cleanup = [&]() {
    for (auto* mp : maps) release(mp);
  };
  std::vector<BuildOut> outs(m);
  unsigned max_v = 1;
  for (int k = 0; k < m; ++k) {
    auto* mp = new (std::nothrow) vgicp_map_s();
    if (!mp) {
      cleanup();
      return fail(VGICP_E_OUT_OF_MEMORY, "host allocation failed");
    }
    maps[k] = mp;
    mp->ctx = ctx;
    mp->res = segs[k].res;
    mp->inv_res = segs[k].inv_res;
    mp->voxels = hv[k];
    mp->total_points = segs[k].n;
    max_v = std::max(max_v, hv[k]);
    const size_t V = hv[k];
    const size_t b_keys = align_up(sizeof(unsigned long long) * V, 256);
    const size_t b_counts = align_up(sizeof(int) * V, 256);
    const size_t b_mean = align_up(sizeof(double) * 3 * V, 256);
    const size_t b_cov = align_up(sizeof(double) * 9 * V, 256);
    mp->cold_bytes = std::max<size_t>(b_keys + b_counts + b_mean + b_cov, 256);
    const cudaError_t e = dmalloc(ctx, &mp->cold, mp->cold_bytes);
    if (e != cudaSuccess) {
      cleanup();
      return cuda_fail(e, "cudaMallocAsync(voxel map)");
    }
    char* b = static_cast<char*>(mp->cold);
    mp->keys = reinterpret_cast<unsigned long long*>(b);
    mp->counts = reinterpret_cast<int*>(b + b_keys);
    mp->mean64 = reinterpret_cast<double*>(b + b_keys + b_counts);
    mp->cov64 = reinterpret_cast<double*>(b + b_keys + b_counts + b_mean);
    if (int rc = alloc_table(mp, std::max(16u, next_pow2((2ull * hv[k] + kBucket - 1) / kBucket)), s)) {  // load <= 0.5
      cleanup();
      return rc;
    }
    outs[k] = BuildOut{d_cbox + 6 * k, mp->keys, mp->counts, mp->mean64, mp->cov64, hbase[k], 0u};
  }
  std::vector<int> hbox(6 * m);
  for (int k = 0; k < m; ++k)
    for (int a = 0; a < 3; ++a) hbox[6 * k + a] = INT32_MAX, hbox[6 * k + 3 + a] = INT32_MIN;
  cudaError_t e = cudaMemcpyAsync(d_outs, outs.data(), sizeof(BuildOut) * m, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_cbox, hbox.data(), sizeof(int) * 6 * m, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = launch_build_accumulate(d_segs, d_outs, m, max_n, d_k1, d_v1, d_heads, d_vidx, d_hot, s);
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "voxel map accumulate");
  }
  ctx->launches += 1;
  // cuckoo-insert the keys; maps whose insertion overflowed are rebuilt with twice the buckets
  std::vector<int> todo(m);
  for (int k = 0; k < m; ++k) todo[k] = k;
  for (int attempt = 0; !todo.empty(); ++attempt) {
    if (attempt > 8) {
      cleanup();
      return fail(VGICP_E_CUDA, "voxel hash table insertion did not converge");
    }
    std::vector<InsertJob> jobs;
    for (int k : todo) {
      vgicp_map mp = maps[k];
      jobs.push_back(InsertJob{mp->tkeys, mp->sa, mp->sb, mp->keys, hbase[k], static_cast<unsigned>(mp->voxels),
                               mp->shift, 0u});
    }
    const int nj = static_cast<int>(jobs.size());
    std::vector<int> hovf(nj, 0);
    e = cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(InsertJob) * nj, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_ovf, 0, sizeof(int) * nj, s);
    if (e == cudaSuccess) e = launch_build_insert(d_jobs, nj, max_v, d_ovf, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hovf.data(), d_ovf, sizeof(int) * nj, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      cleanup();
      return cuda_fail(e, "voxel map insert");
    }
    ctx->launches += 1;
    std::vector<int> next;
    for (int q = 0; q < nj; ++q) {
      if (!hovf[q]) continue;
      const int k = todo[q];
      if (int rc = alloc_table(maps[k], maps[k]->num_buckets * 2, s)) {
        cleanup();
        return rc;
      }
      next.push_back(k);
    }
    if (std::getenv("VGICP_VERBOSE"))
      std::fprintf(stderr, "[vgicp] build insert pass %d: %d maps, %zu overflowed\n", attempt, nj, next.size());
    todo.swap(next);
  }
  {
    std::vector<InsertJob> jobs;
    for (int k = 0; k < m; ++k) {
      vgicp_map mp = maps[k];
      jobs.push_back(InsertJob{mp->tkeys, mp->sa, mp->sb, mp->keys, hbase[k], static_cast<unsigned>(mp->voxels),
                               mp->shift, 0u});
    }
    e = cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(InsertJob) * m, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = launch_build_place(d_jobs, m, max_v, d_hot, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      cleanup();
      return cuda_fail(e, "voxel map place");
    }
    ctx->launches += 1;
  }
  e = cudaMemcpy(hbox.data(), d_cbox, sizeof(int) * 6 * m, cudaMemcpyDeviceToHost);  // stream already idle
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "voxel map bounds");
  }
  for (int k = 0; k < m; ++k)
    for (int a = 0; a < 3; ++a) maps[k]->cmin[a] = hbox[6 * k + a], maps[k]->cmax[a] = hbox[6 * k + 3 + a];
  if (int rc = build_occupancy(ctx, maps.data(), m, d_hot, hbase, s)) {
    cleanup();
    return rc;
  }
  for (int k = 0; k < m; ++k) out[k] = maps[k];
  return VGICP_OK;
}

int vgicp_voxelmap_build(vgicp_ctx ctx, vgicp_cloud cloud, double resolution, vgicp_map* out) try {
  if (!out) return fail(VGICP_E_INVALID_ARGUMENT, "null output");
  return vgicp_voxelmap_build_batch(ctx, &cloud, &resolution, 1, out);
} catch (...) {
  return api_exception();
}

int vgicp_voxelmap_build_f64(vgicp_ctx ctx, const double* xyz, const double* cov9, size_t n, double resolution,
                             vgicp_map* out) try {
  if (!ctx || !out) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  // GaussianVoxelMap ctor validation order (voxelmap.cpp:67-72)
  if (int rc = check_resolution(resolution)) return rc;
  if (!cov9 || n == 0) return fail(VGICP_E_INVALID_ARGUMENT, "voxel map construction requires per-point covariances");
  if (std::isnan(resolution)) return fail(VGICP_E_OUT_OF_RANGE, "point beyond the +-2^20 voxel-per-axis range limit");
  if (!xyz) return fail(VGICP_E_INVALID_ARGUMENT, "null point array");
  if (n >= (1ull << 31)) return fail(VGICP_E_INVALID_ARGUMENT, "cloud too large (>= 2^31 points)");
  DeviceGuard g(ctx->device);
  DevBuf buf(ctx);
  VG_CUDA(buf.alloc(n * 12 * sizeof(double)));
  double* d_xyz = static_cast<double*>(buf.p);
  double* d_cov = d_xyz + 3 * n;
  VG_CUDA(cudaMemcpyAsync(d_xyz, xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  VG_CUDA(cudaMemcpyAsync(d_cov, cov9, n * 9 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  std::vector<BuildSeg> segs{BuildSeg{nullptr, nullptr, nullptr, d_xyz, d_cov, 0ull, static_cast<unsigned>(n), 0u,
                                      resolution, 1.0 / resolution}};
  const int rc = build_segments(ctx, segs, out);
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  return rc;
} catch (...) {
  return api_exception();
}

int vgicp_transform_cloud(vgicp_ctx ctx, const double* xyz, const double* cov9, size_t n, const double pose[12],
                          double* out_xyz, double* out_cov9) try {
  if (!ctx || !pose || (n > 0 && (!xyz || !out_xyz))) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (n == 0) return VGICP_OK;
  const bool cov = cov9 && out_cov9;
  DeviceGuard g(ctx->device);
  DevBuf buf(ctx);
  const size_t per = cov ? 24 : 6;  // doubles per point: in + out
  VG_CUDA(buf.alloc((n * per + 12) * sizeof(double)));
  double* d_in = static_cast<double*>(buf.p);
  double* d_cin = d_in + 3 * n;
  double* d_out = cov ? d_cin + 9 * n : d_in + 3 * n;
  double* d_cout = cov ? d_out + 3 * n : nullptr;
  double* d_T = d_out + (cov ? 12 * n : 3 * n);
  cudaStream_t s = ctx->stream;
  VG_CUDA(cudaMemcpyAsync(d_in, xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
  if (cov) VG_CUDA(cudaMemcpyAsync(d_cin, cov9, n * 9 * sizeof(double), cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemcpyAsync(d_T, pose, 12 * sizeof(double), cudaMemcpyHostToDevice, s));
  VG_CUDA(launch_transform64(d_in, cov ? d_cin : nullptr, n, d_T, d_out, d_cout, s));
  ctx->launches += 1;
  VG_CUDA(cudaMemcpyAsync(out_xyz, d_out, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (cov) VG_CUDA(cudaMemcpyAsync(out_cov9, d_cout, n * 9 * sizeof(double), cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// Device cloud (same layout as cloud_upload_packed) from float64 device arrays (d_cov9 may be null:
// a raw cloud). keep64: the cloud also keeps the float64 values (exact input-order copies for builds /
// transforms + Morton-ordered float64 means for the probe kernels), i.e. it is a float64 cloud.
static int cloud_from_device_f64(vgicp_ctx ctx, const double* d_xyz, const double* d_cov9, size_t n, bool keep64,
                                 vgicp_cloud* out) {
  *out = nullptr;
  if (n >= (1ull << 31)) return fail(VGICP_E_INVALID_ARGUMENT, "cloud too large (>= 2^31 points)");
  cudaStream_t s = ctx->stream;
  auto c = std::make_unique<vgicp_cloud_s>();
  c->ctx = ctx;
  c->n = n;
  c->has_cov = n > 0 && d_cov9 != nullptr;
  const size_t na = align_up(n * sizeof(float4), 256);
  const size_t nc = align_up(n * sizeof(float), 256);
  const size_t half = na * 2 + nc;
  const size_t nblk = (n + kPointBlock - 1) / kPointBlock;
  c->block_bytes = std::max<size_t>(half + nblk * sizeof(PointBlock), 256);
  VG_CUDA(dmalloc(ctx, &c->block, c->block_bytes));
  char* base = static_cast<char*>(c->block);
  c->pa = reinterpret_cast<float4*>(base);
  c->pb = reinterpret_cast<float4*>(base + na);
  c->pc = reinterpret_cast<float*>(base + 2 * na);
  c->sblk = reinterpret_cast<PointBlock*>(base + half);
  if (keep64 && n > 0) {
    const size_t bm = align_up(n * 3 * sizeof(double), 256);
    const size_t bc = c->has_cov ? align_up(n * 9 * sizeof(double), 256) : 0;
    c->block64_bytes = bm + bc + nblk * sizeof(PointBlock64);
    VG_CUDA(dmalloc(ctx, &c->block64, c->block64_bytes));
    char* b64 = static_cast<char*>(c->block64);
    c->f64 = true;
    c->m64 = reinterpret_cast<double*>(b64);
    c->c64 = c->has_cov ? reinterpret_cast<double*>(b64 + bm) : nullptr;
    c->blk64 = reinterpret_cast<PointBlock64*>(b64 + bm + bc);
    VG_CUDA(cudaMemcpyAsync(c->m64, d_xyz, n * 3 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (c->has_cov) VG_CUDA(cudaMemcpyAsync(c->c64, d_cov9, n * 9 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  if (n > 0) {
    size_t sort_bytes = 0;
    VG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const unsigned*)nullptr, (unsigned*)nullptr,
                                            (const unsigned*)nullptr, (unsigned*)nullptr, static_cast<int>(n), 0, 30,
                                            s));
    DevBuf tmp(ctx);
    const size_t b_vec = align_up(sizeof(unsigned) * n, 256);
    VG_CUDA(tmp.alloc(256 + 4 * b_vec + sort_bytes));
    char* t = static_cast<char*>(tmp.p);
    auto* box = reinterpret_cast<unsigned*>(t);
    auto* codes = reinterpret_cast<unsigned*>(t + 256);
    auto* idx = reinterpret_cast<unsigned*>(t + 256 + b_vec);
    auto* codes2 = reinterpret_cast<unsigned*>(t + 256 + 2 * b_vec);
    auto* perm = reinterpret_cast<unsigned*>(t + 256 + 3 * b_vec);
    void* temp = t + 256 + 4 * b_vec;
    VG_CUDA(cudaMemsetAsync(box, 0xFF, 3 * sizeof(unsigned), s));
    VG_CUDA(cudaMemsetAsync(box + 3, 0, 3 * sizeof(unsigned), s));
    VG_CUDA(launch_cloud_bbox(d_xyz, n, box, s));
    VG_CUDA(launch_cloud_morton(d_xyz, n, box, codes, idx, s));
    VG_CUDA(cub::DeviceRadixSort::SortPairs(temp, sort_bytes, codes, codes2, idx, perm, static_cast<int>(n), 0, 30, s));
    VG_CUDA(launch_cloud_fill(d_xyz, d_cov9, n, perm, c->pa, c->pb, c->pc, c->sblk, c->blk64, s));
    ctx->launches += 4;
    unsigned hbox[6];
    VG_CUDA(cudaMemcpyAsync(hbox, box, sizeof(hbox), cudaMemcpyDeviceToHost, s));
    VG_CUDA(cudaStreamSynchronize(s));
    if (hbox[0] <= hbox[3])  // at least one finite point
      for (int a = 0; a < 3; ++a) c->lo[a] = unordered_host(hbox[a]), c->hi[a] = unordered_host(hbox[3 + a]);
  }
  *out = c.release();
  return VGICP_OK;
}

int vgicp_submap_build(vgicp_ctx ctx, const vgicp_cloud* frames, const double* poses12, int m,
                       double downsample_resolution, double map_resolution, vgicp_map* out_downsampled,
                       vgicp_cloud* out_cloud, vgicp_map* out_map) try {
  NvtxRange nvtx_("vgicp_submap_build");
  if (!ctx || !out_map || (m > 0 && (!frames || !poses12))) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *out_map = nullptr;
  if (out_downsampled) *out_downsampled = nullptr;
  if (out_cloud) *out_cloud = nullptr;
  if (m <= 0) return fail(VGICP_E_INVALID_ARGUMENT, "submap requires at least one frame");
  if (int rc = check_resolution(map_resolution)) return rc;
  if (std::isinf(downsample_resolution)) return fail(VGICP_E_INVALID_ARGUMENT, "voxel resolution must be finite");
  size_t total = 0;
  unsigned max_n = 0;
  for (int k = 0; k < m; ++k) {
    if (!frames[k] || frames[k]->ctx != ctx) return fail(VGICP_E_INVALID_ARGUMENT, "cloud of another context");
    if (!frames[k]->has_cov)
      return fail(VGICP_E_INVALID_ARGUMENT, "voxel map construction requires per-point covariances");
    total += frames[k]->n;
    max_n = std::max<unsigned>(max_n, static_cast<unsigned>(frames[k]->n));
  }
  if (total == 0) return fail(VGICP_E_INVALID_ARGUMENT, "voxel map construction requires per-point covariances");
  if (std::isnan(downsample_resolution) || std::isnan(map_resolution))  // voxel_downsample / map voxel_coord
    return fail(VGICP_E_OUT_OF_RANGE, "point beyond the +-2^20 voxel-per-axis range limit");
  if (total >= (1ull << 31)) return fail(VGICP_E_INVALID_ARGUMENT, "submap too large (>= 2^31 points)");
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  const bool verbose = std::getenv("VGICP_VERBOSE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto stage = [&](const char* what) {
    if (!verbose) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[vgicp] submap %-12s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  // 1. transform_cloud of every frame into the submap frame, merged in frame order (pipeline.cpp:97-107)
  DevBuf merged(ctx), items(ctx);
  VG_CUDA(merged.alloc(total * 12 * sizeof(double)));
  VG_CUDA(items.alloc(m * sizeof(TransformItem)));
  double* d_xyz = static_cast<double*>(merged.p);
  double* d_cov = d_xyz + 3 * total;
  std::vector<TransformItem> hi(m);
  size_t off = 0;
  for (int k = 0; k < m; ++k) {
    TransformItem& it = hi[k];
    it.pa = frames[k]->pa;
    it.pb = frames[k]->pb;
    it.pc = frames[k]->pc;
    it.xyz64 = frames[k]->m64;  // float64 frames transform their exact values
    it.cov9 = frames[k]->c64;
    it.offset = off;
    it.n = static_cast<unsigned>(frames[k]->n);
    it.pad = 0;
    std::memcpy(it.T, poses12 + 12 * k, sizeof(it.T));
    off += frames[k]->n;
  }
  VG_CUDA(cudaMemcpyAsync(items.p, hi.data(), m * sizeof(TransformItem), cudaMemcpyHostToDevice, s));
  VG_CUDA(launch_transform(static_cast<const TransformItem*>(items.p), m, max_n, d_xyz, d_cov, s));
  ctx->launches += 1;
  stage("transform");
  // 2. voxel_downsample (voxelmap.cpp:137-169): the voxel means / covariances in ascending key
  //    order are exactly the cold arrays of the map built at the downsample resolution
  const double* src_xyz = d_xyz;
  const double* src_cov = d_cov;
  size_t src_n = total;
  vgicp_map ds = nullptr;
  if (downsample_resolution > 0.0) {
    std::vector<BuildSeg> segs{BuildSeg{nullptr, nullptr, nullptr, d_xyz, d_cov, 0ull, static_cast<unsigned>(total),
                                        0u, downsample_resolution, 1.0 / downsample_resolution}};
    if (int rc = build_segments(ctx, segs, &ds)) return rc;
    src_xyz = ds->mean64;
    src_cov = ds->cov64;
    src_n = ds->voxels;
    stage("downsample");
  }
  // 3. the submap's voxel map at the global resolution (pipeline.cpp:114)
  std::vector<BuildSeg> segs{BuildSeg{nullptr, nullptr, nullptr, src_xyz, src_cov, 0ull, static_cast<unsigned>(src_n),
                                      0u, map_resolution, 1.0 / map_resolution}};
  vgicp_map mp = nullptr;
  if (int rc = build_segments(ctx, segs, &mp)) {
    release(ds);
    return rc;
  }
  stage("map");
  // 4. the submap cloud as a float32 device cloud (source of submap-level factors), built on the
  //    device from the float64 arrays (no host round trip)
  if (out_cloud) {
    if (int rc = cloud_from_device_f64(ctx, src_xyz, src_cov, src_n, true, out_cloud)) {
      release(ds);
      release(mp);
      return rc;
    }
    stage("cloud");
  }
  VG_CUDA(cudaStreamSynchronize(s));
  if (out_downsampled) *out_downsampled = ds;
  else release(ds);
  *out_map = mp;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// ------------------------------------------------------------------------------- replication
// A handle's device state copied whole to another context's device (peer copy over NVLink, or
// through the host without peer access), internal pointers relocated: the replicated clouds / maps
// of a sharded graph (one transfer per map instead of a rebuild per device).

static int cloud_replicate(vgicp_cloud src, vgicp_ctx dst, vgicp_cloud* out) {
  *out = nullptr;
  VG_CUDA(cudaStreamSynchronize(src->ctx->stream));  // the source layout is complete
  DeviceGuard g(dst->device);
  auto c = std::make_unique<vgicp_cloud_s>();
  c->ctx = dst;
  c->n = src->n;
  c->has_cov = src->has_cov;
  c->f64 = src->f64;
  for (int a = 0; a < 3; ++a) c->lo[a] = src->lo[a], c->hi[a] = src->hi[a];
  auto guard = on_failure([&]() {
    dfree(dst, c->block);
    dfree(dst, c->block64);
  });
  VG_CUDA(copy_whole(dst, &c->block, src->block, src->ctx->device, src->block_bytes));
  VG_CUDA(copy_whole(dst, &c->block64, src->block64, src->ctx->device, src->block64_bytes));
  c->block_bytes = src->block_bytes, c->block64_bytes = src->block64_bytes;
  c->pa = relocate(src->pa, src->block, c->block);
  c->pb = relocate(src->pb, src->block, c->block);
  c->pc = relocate(src->pc, src->block, c->block);
  c->sblk = relocate(src->sblk, src->block, c->block);
  c->m64 = relocate(src->m64, src->block64, c->block64);
  c->c64 = relocate(src->c64, src->block64, c->block64);
  c->blk64 = relocate(src->blk64, src->block64, c->block64);
  guard.dismiss();
  *out = c.release();
  return VGICP_OK;
}

int vgicp_cloud_replicate(vgicp_cloud cloud, vgicp_ctx ctx, vgicp_cloud* out) try {
  if (!cloud || !ctx || !out) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  NvtxRange nvtx_("vgicp_cloud_replicate");
  return cloud_replicate(cloud, ctx, out);
} catch (...) {
  return api_exception();
}

int vgicp_voxelmap_replicate(vgicp_map map, vgicp_ctx ctx, vgicp_map* out) try {
  if (!map || !ctx || !out) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  NvtxRange nvtx_("vgicp_voxelmap_replicate");
  VG_CUDA(cudaStreamSynchronize(map->ctx->stream));
  DeviceGuard g(ctx->device);
  auto m = std::make_unique<vgicp_map_s>();
  m->ctx = ctx;
  m->res = map->res, m->inv_res = map->inv_res, m->voxels = map->voxels, m->total_points = map->total_points;
  for (int a = 0; a < 3; ++a) m->cmin[a] = map->cmin[a], m->cmax[a] = map->cmax[a];
  m->num_buckets = map->num_buckets, m->shift = map->shift, m->fast = map->fast, m->cov6 = map->cov6;
  auto guard = on_failure([&]() {
    dfree(ctx, m->cold);
    dfree(ctx, m->table);
    dfree(ctx, m->occ_mem);
    release(m->src);
  });
  const int sd = map->ctx->device;
  VG_CUDA(copy_whole(ctx, &m->cold, map->cold, sd, map->cold_bytes));
  VG_CUDA(copy_whole(ctx, &m->table, map->table, sd, map->table_bytes));
  VG_CUDA(copy_whole(ctx, &m->occ_mem, map->occ_mem, sd, map->occ_bytes));
  m->cold_bytes = map->cold_bytes, m->table_bytes = map->table_bytes, m->occ_bytes = map->occ_bytes;
  // every device pointer lies in one of the three allocations
  auto any = [&](auto* p) -> decltype(p) {
    using T = std::remove_pointer_t<decltype(p)>;
    if (!p) return nullptr;
    const char* c = reinterpret_cast<const char*>(p);
    auto in = [&](const void* base, size_t bytes) {
      return base && c >= static_cast<const char*>(base) && c < static_cast<const char*>(base) + bytes;
    };
    if (in(map->cold, map->cold_bytes)) return relocate(const_cast<std::remove_const_t<T>*>(p), map->cold, m->cold);
    if (in(map->table, map->table_bytes)) return relocate(const_cast<std::remove_const_t<T>*>(p), map->table, m->table);
    return relocate(const_cast<std::remove_const_t<T>*>(p), map->occ_mem, m->occ_mem);
  };
  m->keys = any(map->keys);
  m->counts = any(map->counts);
  m->mean64 = any(map->mean64);
  m->cov64 = any(map->cov64);
  m->tkeys = any(map->tkeys);
  m->sa = any(map->sa);
  m->sb = any(map->sb);
  m->ra = any(map->ra);
  m->rb = any(map->rb);
  m->occ = map->occ;
  m->occ.occ = any(map->occ.occ);
  if (map->src)
    if (int rc = cloud_replicate(map->src, ctx, &m->src)) return rc;
  guard.dismiss();
  *out = m.release();
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_voxelmap_destroy(vgicp_map map) try {
  release(map);
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_voxelmap_size(vgicp_map map, size_t* voxels) try {
  if (!map || !voxels) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *voxels = map->voxels;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_voxelmap_resolution(vgicp_map map, double* resolution) try {
  if (!map || !resolution) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *resolution = map->res;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_voxelmap_total_points(vgicp_map map, size_t* total) try {
  if (!map || !total) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *total = map->total_points;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_voxelmap_export(vgicp_map map, uint64_t* keys, int32_t* counts, double* means, double* covs) try {
  NvtxRange nvtx_("vgicp_voxelmap_export");
  if (!map) return fail(VGICP_E_INVALID_ARGUMENT, "null map");
  DeviceGuard g(map->ctx->device);
  cudaStream_t s = map->ctx->stream;
  const size_t V = map->voxels;
  if (V == 0) return VGICP_OK;
  if (map->fast) {  // rank-numbered map: recompute the key-ordered statistics with the same kernels
    std::vector<uint64_t> k;
    std::vector<int32_t> c;
    std::vector<double> mu, cv;
    if (int rc = fast_export(map, keys ? &k : nullptr, counts ? &c : nullptr, means ? &mu : nullptr,
                             covs ? &cv : nullptr, nullptr))
      return rc;
    if (keys) std::memcpy(keys, k.data(), sizeof(uint64_t) * V);
    if (counts) std::memcpy(counts, c.data(), sizeof(int32_t) * V);
    if (means) std::memcpy(means, mu.data(), sizeof(double) * 3 * V);
    if (covs) std::memcpy(covs, cv.data(), sizeof(double) * 9 * V);
    return VGICP_OK;
  }
  if (keys) VG_CUDA(cudaMemcpyAsync(keys, map->keys, sizeof(uint64_t) * V, cudaMemcpyDeviceToHost, s));
  if (counts) VG_CUDA(cudaMemcpyAsync(counts, map->counts, sizeof(int32_t) * V, cudaMemcpyDeviceToHost, s));
  if (means) VG_CUDA(cudaMemcpyAsync(means, map->mean64, sizeof(double) * 3 * V, cudaMemcpyDeviceToHost, s));
  if (covs) VG_CUDA(cudaMemcpyAsync(covs, map->cov64, sizeof(double) * 9 * V, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_voxelmap_lookup(vgicp_map map, const double* points, size_t n, uint64_t* keys_out) try {
  if (!map || (n > 0 && (!points || !keys_out))) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (n == 0) return VGICP_OK;
  vgicp_ctx ctx = map->ctx;
  DeviceGuard g(ctx->device);
  if (int rc = ensure_table(map)) return rc;
  const size_t bp = align_up(sizeof(double) * 3 * n, 256);
  if (int rc = ensure_scratch(ctx, bp + sizeof(uint64_t) * n)) return rc;
  char* sb = static_cast<char*>(ctx->scratch);
  double* d_pts = reinterpret_cast<double*>(sb);
  auto* d_keys = reinterpret_cast<unsigned long long*>(sb + bp);
  VG_CUDA(cudaMemcpyAsync(d_pts, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx->stream));
  VG_CUDA(launch_lookup(map->dev(), d_pts, n, d_keys, ctx->stream));
  ctx->launches += 1;
  VG_CUDA(cudaMemcpyAsync(keys_out, d_keys, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_voxel_key(double resolution, const double point[3], uint64_t* key) try {
  if (!point || !key) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  return host_voxel_key(resolution, point, key);
} catch (...) {
  return api_exception();
}

// ------------------------------------------------------------------------------------ overlap
// Conservative, exact culling of an overlap probe: when the axis-aligned box of the transformed
// cloud (its 8 box corners mapped by T, fp64) misses the map's occupied voxel region grown by one
// voxel on every side, no point can land in an occupied voxel and the hit count is exactly 0.
static bool overlap_disjoint(const vgicp_cloud_s* c, const double* T, const vgicp_map_s* m) {
  if (c->lo[0] > c->hi[0]) return true;  // no finite point: every lookup misses
  if (m->cmin[0] > m->cmax[0]) return true;
  double wlo[3] = {INFINITY, INFINITY, INFINITY}, whi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int corner = 0; corner < 8; ++corner) {
    const double p[3] = {(corner & 1) ? c->hi[0] : c->lo[0], (corner & 2) ? c->hi[1] : c->lo[1],
                         (corner & 4) ? c->hi[2] : c->lo[2]};
    for (int a = 0; a < 3; ++a) {
      const double q = T[3 * a] * p[0] + T[3 * a + 1] * p[1] + T[3 * a + 2] * p[2] + T[9 + a];
      wlo[a] = std::min(wlo[a], q);
      whi[a] = std::max(whi[a], q);
    }
  }
  for (int a = 0; a < 3; ++a) {
    const double mlo = (m->cmin[a] - 1.0) * m->res, mhi = (m->cmax[a] + 2.0) * m->res;
    if (!(whi[a] >= mlo && wlo[a] <= mhi)) return true;
  }
  return false;
}

// Overlap probe item k (cloud k's points through pose k against map k), written in place.
static void fill_overlap_item(OverlapItem& it, const vgicp_cloud_s* c, const double* T, const vgicp_map_s* mp) {
  it.blk = c->sblk;  // Morton order (hit counts are order-independent)
  it.blk64 = c->blk64;
  it.map = mp->dev();
  it.occ = mp->occ;
  std::memcpy(it.T, T, sizeof(double) * 12);
  it.n = static_cast<unsigned>(c->n);
  it.pad = 0;
  OccScreen& sc = it.scr;
  if (!it.occ.occ) {
    sc.occ = nullptr;
    return;
  }
  float tmax = 0.f;
  for (int q = 0; q < 9; ++q) sc.R[q] = static_cast<float>(T[q]);
  for (int q = 0; q < 3; ++q) sc.t[q] = static_cast<float>(T[9 + q]), tmax = std::max(tmax, std::fabs(sc.t[q]));
  sc.inv_r = static_cast<float>(mp->inv_res);
  sc.A2 = (c->f64 ? kScreenA64 : kScreenA) * sc.inv_r;
  sc.C = sc.A2 * tmax + 1e-7f;
  sc.cx0 = static_cast<int>(it.occ.kx0) - (1 << 20);
  sc.cy0 = static_cast<int>(it.occ.ky0) - (1 << 20);
  sc.cz0 = static_cast<int>(it.occ.kz0) - (1 << 20);
  sc.ex = it.occ.ex, sc.ey = it.occ.ey, sc.ez = it.occ.ez, sc.nby = it.occ.nby, sc.nbz = it.occ.nbz;
  sc.pad[0] = sc.pad[1] = 0u;
  sc.occ = it.occ.occ;
}

int vgicp_overlap_batch(vgicp_ctx ctx, const vgicp_cloud* clouds, const double* poses12, const vgicp_map* maps,
                        int m, uint64_t* hits) try {
  NvtxRange nvtx_("vgicp_overlap_batch");
  if (!ctx || (m > 0 && (!clouds || !poses12 || !maps || !hits)))
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (m <= 0) return VGICP_OK;
  const bool no_cull = std::getenv("VGICP_OVERLAP_NOCULL") != nullptr;  // measurement switch (un-culled)
  const bool per_item = std::getenv("VGICP_OVERLAP_PERITEM") != nullptr;  // measurement switch
  const bool verbose = std::getenv("VGICP_VERBOSE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto ms_since = [](std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  // pass 1: validation and exact culling (probes whose transformed cloud box misses the map's
  // occupied box: 0 hits, no launch work)
  std::vector<int> live;
  live.reserve(m);
  unsigned max_n = 0;
  for (int k = 0; k < m; ++k) {
    if (!clouds[k] || !maps[k]) return fail(VGICP_E_INVALID_ARGUMENT, "null cloud or map");
    if (clouds[k]->ctx != ctx || maps[k]->ctx != ctx) return fail(VGICP_E_INVALID_ARGUMENT, "handle of another context");
    if (clouds[k]->n == 0) return fail(VGICP_E_INVALID_ARGUMENT, "overlap_rate requires a nonempty cloud");
    hits[k] = 0;
    if (!no_cull && overlap_disjoint(clouds[k], poses12 + 12 * k, maps[k])) continue;
    max_n = std::max(max_n, static_cast<unsigned>(clouds[k]->n));
    live.push_back(k);
  }
  const int ml = static_cast<int>(live.size());
  if (ml == 0) return VGICP_OK;
  // Group the probes by cloud (stable), bitmap-carrying maps first within a cloud: every chunk of
  // <= 32 maps shares one cloud (its points are loaded once) and one kernel. Callers usually pass
  // probes grouped already (one frame against many maps), which skips the sort.
  auto before = [&](int a, int b) {
    const bool oa = maps[a]->occ.occ != nullptr, ob = maps[b]->occ.occ != nullptr;
    return clouds[a]->sblk != clouds[b]->sblk ? clouds[a]->sblk < clouds[b]->sblk : (oa && !ob);
  };
  std::vector<int> order = live;  // order[q] = probe index of sorted position q
  if (!std::is_sorted(order.begin(), order.end(), before)) std::stable_sort(order.begin(), order.end(), before);
  const double t_items = ms_since(t_start);
  DeviceGuard g(ctx->device);
  const size_t bi = align_up(sizeof(OverlapItem) * ml, 256);
  const size_t bc = align_up(sizeof(int2) * (ml + 1), 256);
  const size_t bh = sizeof(unsigned long long) * ml;
  if (int rc = ensure_scratch(ctx, bi + bc + bh)) return rc;
  if (int rc = ensure_pinned(ctx, bi + bc + bh)) return rc;
  char* hp = static_cast<char*>(ctx->pinned);  // page-locked staging: one fast H2D / D2H each
  auto* sorted = reinterpret_cast<OverlapItem*>(hp);
  auto* hchunks = reinterpret_cast<int2*>(hp + bi);
  auto* h = reinterpret_cast<unsigned long long*>(hp + bi + bc);
  int n_occ = 0;  // occupancy chunks first, then hash-probe chunks
  std::vector<int2> hash_chunks;
  for (int q = 0; q < ml; ++q) {
    const int k = order[q];
    fill_overlap_item(sorted[q], clouds[k], poses12 + 12 * k, maps[k]);
    const bool occ = sorted[q].occ.occ != nullptr;
    int2* last = occ ? (n_occ ? &hchunks[n_occ - 1] : nullptr) : (hash_chunks.empty() ? nullptr : &hash_chunks.back());
    if (!last || sorted[q].blk != sorted[last->x].blk || last->y == kOverlapMapsPerChunk) {
      if (occ) last = &(hchunks[n_occ++] = make_int2(q, 0));
      else last = &(hash_chunks.emplace_back(make_int2(q, 0)));
    }
    ++last->y;
  }
  const int n_hash = static_cast<int>(hash_chunks.size());
  for (int c = 0; c < n_hash; ++c) hchunks[n_occ + c] = hash_chunks[c];
  char* sb = static_cast<char*>(ctx->scratch);
  auto* d_items = reinterpret_cast<OverlapItem*>(sb);
  auto* d_chunks = reinterpret_cast<int2*>(sb + bi);
  auto* d_hits = reinterpret_cast<unsigned long long*>(sb + bi + bc);
  cudaStream_t s = ctx->stream;
  const double t_pack = ms_since(t_start);
  VG_CUDA(cudaMemcpyAsync(d_items, sorted, bi + sizeof(int2) * (n_occ + n_hash), cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemsetAsync(d_hits, 0, bh, s));
  if (per_item) {
    VG_CUDA(launch_overlap(d_items, ml, max_n, d_hits, s));
    ctx->launches += 1;
  } else {
    VG_CUDA(launch_overlap_occ(d_items, d_chunks, n_occ, max_n, d_hits, s));
    VG_CUDA(launch_overlap_multi(d_items, d_chunks + n_occ, n_hash, max_n, d_hits, s));
    ctx->launches += (n_occ > 0) + (n_hash > 0);
  }
  VG_CUDA(cudaMemcpyAsync(h, d_hits, bh, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  for (int q = 0; q < ml; ++q) hits[order[q]] = h[q];
  if (verbose)
    std::fprintf(stderr, "[vgicp] overlap batch: %d probes (%d live), cull+order %.3f ms, pack %.3f ms, gpu+sync %.3f ms\n",
                 m, ml, t_items, t_pack - t_items, ms_since(t_start) - t_pack);
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// ------------------------------------------------------------------------------- map sets
// Device block of a map set laid out for `cap` maps (templates | items | chunks | hits | poses + box);
// the first `keep` templates move over from the previous block.
static int mapset_reserve(vgicp_mapset set, int cap, int keep) {
  if (cap <= set->capacity) return VGICP_OK;
  vgicp_ctx ctx = set->ctx;
  const int nch = (cap + kOverlapMapsPerChunk - 1) / kOverlapMapsPerChunk;
  const size_t bt = align_up(sizeof(OverlapItem) * cap, 256), bc = align_up(sizeof(int2) * nch, 256);
  const size_t bh = align_up(sizeof(unsigned long long) * cap, 256), bp = align_up(sizeof(double) * 12 * cap + 64, 256);
  void* block = nullptr;
  if (const cudaError_t e = dmalloc(ctx, &block, 2 * bt + bc + bh + bp); e != cudaSuccess)
    return cuda_fail(e, ("mapset block of " + std::to_string(cap) + " maps, " + std::to_string(2 * bt + bc + bh + bp) +
                         " B").c_str());
  char* b = static_cast<char*>(block);
  auto* templates = reinterpret_cast<OverlapItem*>(b);
  if (keep > 0) {
    if (const cudaError_t e = cudaMemcpyAsync(templates, set->d_templates, sizeof(OverlapItem) * keep,
                                              cudaMemcpyDeviceToDevice, ctx->stream);
        e != cudaSuccess) {
      dfree(ctx, block);
      return cuda_fail(e, "cudaMemcpyAsync");
    }
  }
  if (set->block) {
    cudaStreamSynchronize(ctx->stream);  // the old block may still be read by a queued sweep / the copy
    dfree(ctx, set->block);
  }
  set->block = block;
  set->d_templates = templates;
  set->d_items = reinterpret_cast<OverlapItem*>(b + bt);
  set->d_chunks = reinterpret_cast<int2*>(b + 2 * bt);
  set->d_hits = reinterpret_cast<unsigned long long*>(b + 2 * bt + bc);
  set->d_poses = reinterpret_cast<double*>(b + 2 * bt + bc + bh);
  set->capacity = cap;
  return VGICP_OK;
}

// Appends maps[0..m) to the set: validation, then (device path) their templates after the existing
// ones — the block grows geometrically, so a keyframe database that gains one map per keyframe
// pays an amortised O(1) upload per map.
static int mapset_add(vgicp_mapset set, const vgicp_map* maps, int m) {
  vgicp_ctx ctx = set->ctx;
  bool occ = set->all_occ;
  for (int k = 0; k < m; ++k) {
    if (!maps[k]) return fail(VGICP_E_INVALID_ARGUMENT, "null map");
    if (maps[k]->ctx != ctx) return fail(VGICP_E_INVALID_ARGUMENT, "handle of another context");
    occ = occ && maps[k]->occ.occ != nullptr;
  }
  const int size = static_cast<int>(set->maps.size());
  if (occ && m > 0) {
    DeviceGuard g(ctx->device);
    if (size + m > set->capacity)
      if (int rc = mapset_reserve(set, std::max(size + m, 2 * set->capacity), size)) return rc;
    static const double kIdentity[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
    vgicp_cloud_s dummy;  // the template carries no cloud; fill_overlap_item needs one for blk / n
    std::vector<OverlapItem> templ(m);
    for (int k = 0; k < m; ++k) fill_overlap_item(templ[k], &dummy, kIdentity, maps[k]);
    VG_CUDA(cudaMemcpyAsync(set->d_templates + size, templ.data(), sizeof(OverlapItem) * m, cudaMemcpyHostToDevice,
                            ctx->stream));
    VG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  set->all_occ = occ;  // a map without a bitmap moves the whole set to the generic path
  for (int k = 0; k < m; ++k) {
    maps[k]->refs.fetch_add(1);
    set->maps.push_back(maps[k]);
  }
  return VGICP_OK;
}

int vgicp_mapset_create(vgicp_ctx ctx, const vgicp_map* maps, int m, vgicp_mapset* out) try {
  if (!ctx || !out || (m > 0 && !maps) || m < 0) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  auto set = std::make_unique<vgicp_mapset_s>();
  set->ctx = ctx;
  if (int rc = mapset_add(set.get(), maps, m)) {
    vgicp_mapset_destroy(set.release());
    return rc;
  }
  *out = set.release();
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_mapset_append(vgicp_mapset set, const vgicp_map* maps, int m) try {
  NvtxRange nvtx_("vgicp_mapset_append");
  if (!set || m < 0 || (m > 0 && !maps)) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  return mapset_add(set, maps, m);
} catch (...) {
  return api_exception();
}

int vgicp_mapset_size(vgicp_mapset set, int* size) try {
  if (!set || !size) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *size = static_cast<int>(set->maps.size());
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_mapset_destroy(vgicp_mapset set) try {
  if (!set) return VGICP_OK;
  {
    DeviceGuard g(set->ctx->device);
    cudaStreamSynchronize(set->ctx->stream);
    dfree(set->ctx, set->block);
  }
  for (auto mp : set->maps) release(mp);
  delete set;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_overlap_mapset(vgicp_ctx ctx, vgicp_cloud cloud, const double* rel12, vgicp_mapset set, uint64_t* hits) try {
  NvtxRange nvtx_("vgicp_overlap_mapset");
  if (!ctx || !cloud || !set || (!set->maps.empty() && (!rel12 || !hits)))
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (cloud->ctx != ctx || set->ctx != ctx) return fail(VGICP_E_INVALID_ARGUMENT, "handle of another context");
  if (cloud->n == 0) return fail(VGICP_E_INVALID_ARGUMENT, "overlap_rate requires a nonempty cloud");
  const int m = static_cast<int>(set->maps.size());
  if (m == 0) return VGICP_OK;
  if (!set->all_occ || std::getenv("VGICP_OVERLAP_PERITEM") || std::getenv("VGICP_OVERLAP_NOCULL")) {
    std::vector<vgicp_cloud> clouds(m, cloud);  // generic path (maps without bitmaps, measurement switches)
    return vgicp_overlap_batch(ctx, clouds.data(), rel12, set->maps.data(), m, hits);
  }
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  const size_t bp = sizeof(double) * 12 * m;
  if (int rc = ensure_pinned(ctx, align_up(bp + 6 * sizeof(float), 256) + sizeof(unsigned long long) * m)) return rc;
  char* hp = static_cast<char*>(ctx->pinned);
  std::memcpy(hp, rel12, bp);
  float* hbox = reinterpret_cast<float*>(hp + bp);
  for (int a = 0; a < 3; ++a) hbox[a] = cloud->lo[a], hbox[3 + a] = cloud->hi[a];
  auto* h = reinterpret_cast<unsigned long long*>(hp + align_up(bp + 6 * sizeof(float), 256));
  VG_CUDA(cudaMemcpyAsync(set->d_poses, hp, bp + 6 * sizeof(float), cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemsetAsync(set->d_hits, 0, sizeof(unsigned long long) * m, s));
  const float* d_box = reinterpret_cast<const float*>(reinterpret_cast<const char*>(set->d_poses) + bp);
  VG_CUDA(launch_mapset_prepare(set->d_templates, m, set->d_poses, cloud->sblk, cloud->blk64,
                                static_cast<unsigned>(cloud->n), d_box, set->d_items, set->d_chunks, s));
  const int nch = (m + kOverlapMapsPerChunk - 1) / kOverlapMapsPerChunk;
  VG_CUDA(launch_overlap_occ(set->d_items, set->d_chunks, nch, static_cast<unsigned>(cloud->n), set->d_hits, s));
  ctx->launches += 2;
  VG_CUDA(cudaMemcpyAsync(h, set->d_hits, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  std::memcpy(hits, h, sizeof(uint64_t) * m);
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_overlap_rate(vgicp_ctx ctx, vgicp_cloud cloud, const double pose_rel[12], vgicp_map map, double* rate) try {
  if (!rate || !cloud || !map || !pose_rel) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  uint64_t hits = 0;
  if (int rc = vgicp_overlap_batch(ctx, &cloud, pose_rel, &map, 1, &hits)) return rc;
  *rate = static_cast<double>(hits) / static_cast<double>(cloud->n);  // voxelmap.cpp:134
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// ------------------------------------------------------------------------------------ graphs
// kernels one factor pass launches: one for the float32-cloud items, one for the float64-cloud items
static int factor_launches(const vgicp_graph_s* g) {
  return (g->f64_begin > 0 ? 1 : 0) + (g->num_items > g->f64_begin ? 1 : 0);
}

// Work decomposition of a factor list (items in launch order: float32-cloud items first, then
// float64-cloud items; each factor's items contiguous). Items are one CTA each; a launch runs in
// ~equal waves of `slots` resident CTAs. With many factors, the last wave's factors are cut into
// quarter chunks so the tail wave is short; with fewer factors than slots, every factor is cut
// finer so that the launch still fills the GPU (C1 / C2). VGICP_NO_TAIL_SPLIT=1 keeps uniform
// chunks. A shard of a sharded graph uses the decomposition of the WHOLE list, so its per-factor
// blocks are bit-identical to a single-device graph's.
struct Decomp {
  std::vector<FactorDev> fd;
  std::vector<WorkItem> items;
  int f64_begin = 0;
  bool rank = false;
};

static int validate_factors(vgicp_ctx ctx, const vgicp_factor_desc* factors, int num_factors, int num_poses) {
  // MatchingCostFactor ctor validation (factors.cpp:57-66)
  for (int f = 0; f < num_factors; ++f) {
    const vgicp_factor_desc& d = factors[f];
    if (d.target_index == d.source_index)
      return fail(VGICP_E_INVALID_ARGUMENT, "matching cost factor requires distinct variables");
    if (!d.source || d.source->n == 0)
      return fail(VGICP_E_INVALID_ARGUMENT, "matching cost factor requires a nonempty source cloud");
    if (!d.source->has_cov) return fail(VGICP_E_INVALID_ARGUMENT, "matching cost factor requires source covariances");
    if (!d.target || d.target->voxels == 0)
      return fail(VGICP_E_INVALID_ARGUMENT, "matching cost factor requires a nonempty target voxel map");
    if (d.source->ctx != ctx || d.target->ctx != ctx)
      return fail(VGICP_E_INVALID_ARGUMENT, "factor handles belong to another context");
    if (d.target_index < 0 || d.target_index >= num_poses || d.source_index < 0 || d.source_index >= num_poses)
      return fail(VGICP_E_INVALID_ARGUMENT, "factor variable index out of range");
  }
  return VGICP_OK;
}

// Factor kernels probe the cuckoo tables (not the bitmaps) unless every target map has a bitmap
// (and VGICP_NO_RANK is unset): hand-built maps get their table, on demand, before descriptors
// capture their device pointers.
static bool use_rank_lookups(const vgicp_factor_desc* factors, int num_factors) {
  bool rank = std::getenv("VGICP_NO_RANK") == nullptr;
  for (int f = 0; f < num_factors && rank; ++f) rank = factors[f].target->occ.occ != nullptr;
  return rank;
}
static int ensure_tables_for_hash_mode(const vgicp_factor_desc* factors, int num_factors) {
  if (use_rank_lookups(factors, num_factors)) return VGICP_OK;
  for (int f = 0; f < num_factors; ++f)
    if (int rc = ensure_table(factors[f].target)) return rc;
  return VGICP_OK;
}

static void decompose(vgicp_ctx ctx, const vgicp_factor_desc* factors, int num_factors, int chunk, Decomp& g) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const int slots = 2 * sms;
  const bool split = std::getenv("VGICP_NO_TAIL_SPLIT") == nullptr;
  uint64_t total_points = 0;
  for (int f = 0; f < num_factors; ++f) total_points += factors[f].source->n;
  auto round_chunk = [](uint64_t c) {
    return static_cast<int>(std::max<uint64_t>(kFactorTile, (c + kFactorTile - 1) / kFactorTile * kFactorTile));
  };
  const int small_chunk = round_chunk(chunk / 4);
  const int few_chunk =
      std::min(chunk, round_chunk(total_points / std::max<uint64_t>(1, 2ull * static_cast<uint64_t>(slots))));
  g.fd.assign(num_factors, FactorDev{});
  g.items.clear();
  // rank lookups (occupancy bitmap + rank-ordered statistics) when every target map carries them;
  // VGICP_NO_RANK=1 keeps the cuckoo-hash probes (measurement switch)
  g.rank = use_rank_lookups(factors, num_factors);
  // items of float32-exact source clouds first, then those of float64 clouds (their own launch)
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) g.f64_begin = static_cast<int>(g.items.size());
    for (int f = 0; f < num_factors; ++f) {
      const vgicp_factor_desc& d = factors[f];
      if (d.source->f64 != (pass == 1)) continue;
      FactorDev& x = g.fd[f];
      const int fchunk =
          !split ? chunk : (num_factors < slots ? few_chunk : (f >= num_factors - slots ? small_chunk : chunk));
      x.blk = d.source->sblk;  // Morton order: neighbouring lanes probe neighbouring voxels
      x.blk64 = d.source->blk64;
      x.c64 = d.source->c64;
      x.map = g.rank ? d.target->dev_rank() : d.target->dev();
      x.n = static_cast<int>(d.source->n);
      x.tgt = d.target_index;
      x.src = d.source_index;
      x.item_begin = static_cast<int>(g.items.size());
      for (int b = 0; b < x.n; b += fchunk) g.items.push_back(WorkItem{f, b, std::min(x.n, b + fchunk), 0});
      x.item_count = static_cast<int>(g.items.size()) - x.item_begin;
      x.pad = 0;
    }
  }
}

// The graph of factors [first, first + count) of `factors` under the decomposition `g` of the whole
// list: local factor k is global factor first + k (its items keep their chunking; indices relabelled).
static int graph_from(vgicp_ctx ctx, const vgicp_factor_desc* factors, int num_poses, const Decomp& g, int first,
                      int count, vgicp_graph* out) {
  std::vector<FactorDev> fd(count);
  std::vector<WorkItem> items;
  int f64_begin = 0;
  uint64_t points = 0;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) f64_begin = static_cast<int>(items.size());
    const int i0 = pass == 0 ? 0 : g.f64_begin, i1 = pass == 0 ? g.f64_begin : static_cast<int>(g.items.size());
    for (int i = i0; i < i1; ++i) {
      const WorkItem& w = g.items[i];
      if (w.factor < first || w.factor >= first + count) continue;
      const int k = w.factor - first;
      if (i == g.fd[w.factor].item_begin) {
        fd[k] = g.fd[w.factor];
        fd[k].item_begin = static_cast<int>(items.size());
        points += static_cast<uint64_t>(fd[k].n);
      }
      items.push_back(WorkItem{k, w.begin, w.end, 0});
    }
  }
  auto gr = std::make_unique<vgicp_graph_s>();
  gr->ctx = ctx;
  gr->num_factors = count;
  gr->num_poses = num_poses;
  gr->num_items = static_cast<int>(items.size());
  gr->f64_begin = f64_begin;
  gr->num_points = points;
  gr->rank_lookup = g.rank;
  const size_t nf = std::max(count, 1), ni = std::max<size_t>(items.size(), 1);
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t o_f = carve(sizeof(FactorDev) * nf);
  const size_t o_i = carve(sizeof(WorkItem) * ni);
  const size_t o_p = carve(sizeof(double) * kPartialStride * kFactorWarps * ni);  // one partial per warp
  const size_t o_pi = carve(sizeof(int) * kFactorWarps * ni);
  const size_t o_c = carve(sizeof(unsigned) * nf);
  const size_t o_pose = carve(sizeof(double) * 12 * std::max(num_poses, 1));
  const size_t o_out = carve(sizeof(double) * VGICP_LINEARIZED_DOUBLES * nf);
  const size_t o_oi = carve(sizeof(int) * nf);
  const size_t o_err = carve(sizeof(double) * nf);
  VG_CUDA(dmalloc(ctx, &gr->block, off));
  char* b = static_cast<char*>(gr->block);
  gr->d_factors = reinterpret_cast<FactorDev*>(b + o_f);
  gr->d_items = reinterpret_cast<WorkItem*>(b + o_i);
  gr->d_partials = reinterpret_cast<double*>(b + o_p);
  gr->d_part_inl = reinterpret_cast<int*>(b + o_pi);
  gr->d_counters = reinterpret_cast<unsigned*>(b + o_c);
  gr->d_poses = reinterpret_cast<double*>(b + o_pose);
  gr->d_out = reinterpret_cast<double*>(b + o_out);
  gr->d_out_inl = reinterpret_cast<int*>(b + o_oi);
  gr->d_err = reinterpret_cast<double*>(b + o_err);
  cudaStream_t s = ctx->stream;
  int rc = VGICP_OK;
  auto step = [&](cudaError_t e, const char* what) {
    if (rc == VGICP_OK && e != cudaSuccess) rc = cuda_fail(e, what);
  };
  if (count > 0) {
    step(cudaMemcpyAsync(gr->d_factors, fd.data(), sizeof(FactorDev) * count, cudaMemcpyHostToDevice, s),
         "upload factors");
    if (!items.empty())
      step(cudaMemcpyAsync(gr->d_items, items.data(), sizeof(WorkItem) * items.size(), cudaMemcpyHostToDevice, s),
           "upload items");
  }
  step(cudaMemsetAsync(gr->d_counters, 0, sizeof(unsigned) * nf, s), "zero counters");
  step(cudaStreamSynchronize(s), "graph create");
  if (rc != VGICP_OK) {
    dfree(ctx, gr->block);
    return rc;
  }
  for (int k = 0; k < count; ++k) {
    const vgicp_factor_desc& d = factors[first + k];
    d.source->refs.fetch_add(1);
    d.target->refs.fetch_add(1);
    gr->clouds.push_back(d.source);
    gr->maps.push_back(d.target);
    gr->tgt_idx.push_back(d.target_index);
    gr->src_idx.push_back(d.source_index);
  }
  *out = gr.release();
  return VGICP_OK;
}

static int graph_create_range(vgicp_ctx ctx, const vgicp_factor_desc* factors, int num_factors, int num_poses,
                              int chunk, int first, int count, vgicp_graph* out) {
  if (!ctx || !out || (num_factors > 0 && !factors)) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (num_factors < 0 || num_poses < 0) return fail(VGICP_E_INVALID_ARGUMENT, "negative size");
  if (first < 0 || count < 0 || first + count > num_factors)
    return fail(VGICP_E_INVALID_ARGUMENT, "factor range outside the factor list");
  if (chunk <= 0) chunk = kDefaultChunk;
  chunk = std::max(kFactorTile, (chunk + kFactorTile - 1) / kFactorTile * kFactorTile);
  if (int rc = validate_factors(ctx, factors, num_factors, num_poses)) return rc;
  DeviceGuard g(ctx->device);
  if (int rc = ensure_tables_for_hash_mode(factors, num_factors)) return rc;
  Decomp d;
  decompose(ctx, factors, num_factors, chunk, d);
  return graph_from(ctx, factors, num_poses, d, first, count, out);
}

int vgicp_graph_create(vgicp_ctx ctx, const vgicp_factor_desc* factors, int num_factors, int num_poses, int chunk,
                       vgicp_graph* out) try {
  return graph_create_range(ctx, factors, num_factors, num_poses, chunk, 0, num_factors, out);
} catch (...) {
  return api_exception();
}

int vgicp_graph_create_range(vgicp_ctx ctx, const vgicp_factor_desc* factors, int num_factors, int num_poses,
                             int chunk, int first, int count, vgicp_graph* out) try {
  return graph_create_range(ctx, factors, num_factors, num_poses, chunk, first, count, out);
} catch (...) {
  return api_exception();
}

// Contiguous [begin, end) factor ranges, one per shard, balanced by Σ source points (the split of
// paper_2109_07073_b200/sharding.py: partition_factors).
static std::vector<int> partition_bounds(const vgicp_factor_desc* factors, int F, int n) {
  std::vector<double> cum(F);
  double run = 0.0;
  for (int f = 0; f < F; ++f) cum[f] = (run += static_cast<double>(factors[f].source->n));
  std::vector<int> bounds{0};
  for (int r = 1; r < n; ++r) {
    const double target = run * r / n;
    int b = static_cast<int>(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
    if (b < F && std::fabs(cum[b] - target) < std::fabs((b > 0 ? cum[b - 1] : 0.0) - target)) b = b + 1;
    bounds.push_back(std::min(std::max(b, bounds.back()), F));
  }
  bounds.push_back(F);
  return bounds;
}

int vgicp_graph_create_sharded(const vgicp_ctx* ctxs, int num_shards, const vgicp_factor_desc* const* factors,
                               int num_factors, int num_poses, int chunk, vgicp_graph* out) try {
  NvtxRange nvtx_("vgicp_graph_create_sharded");
  if (!ctxs || !out || !factors || num_shards <= 0) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (num_shards > kMaxShards) return fail(VGICP_E_INVALID_ARGUMENT, "at most 8 shards (one per device of a box)");
  if (num_factors < 0 || num_poses < 0) return fail(VGICP_E_INVALID_ARGUMENT, "negative size");
  for (int r = 0; r < num_shards; ++r) {
    if (!ctxs[r] || (num_factors > 0 && !factors[r])) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
    if (int rc = validate_factors(ctxs[r], factors[r], num_factors, num_poses)) return rc;
    for (int f = 0; f < num_factors; ++f)  // the lists must describe the same factors
      if (factors[r][f].target_index != factors[0][f].target_index ||
          factors[r][f].source_index != factors[0][f].source_index ||
          factors[r][f].source->n != factors[0][f].source->n)
        return fail(VGICP_E_INVALID_ARGUMENT, "shard factor lists differ");
  }
  if (chunk <= 0) chunk = kDefaultChunk;
  chunk = std::max(kFactorTile, (chunk + kFactorTile - 1) / kFactorTile * kFactorTile);
  vgicp_ctx root = ctxs[0];
  for (int r = 0; r < num_shards; ++r) {
    DeviceGuard gr(ctxs[r]->device);
    if (int rc = ensure_tables_for_hash_mode(factors[r], num_factors)) return rc;
  }
  DeviceGuard g(root->device);
  Decomp d;
  decompose(root, factors[0], num_factors, chunk, d);  // the whole list's decomposition, for every shard
  const std::vector<int> bounds = partition_bounds(factors[0], num_factors, num_shards);
  auto parent = std::make_unique<vgicp_graph_s>();
  auto cleanup = [&]() {
    for (auto* sh : parent->shards) vgicp_graph_destroy(sh);
    parent->shards.clear();
    for (auto ev : parent->shard_events) cudaEventDestroy(ev);
    parent->shard_events.clear();
    if (parent->root_event) cudaEventDestroy(parent->root_event);
    parent->root_event = nullptr;
  };
  for (int r = 0; r < num_shards; ++r) {
    Decomp dr;
    const Decomp* use = &d;
    if (r > 0) {  // the same chunking, with this shard's own device pointers
      dr = d;
      for (int f = 0; f < num_factors; ++f) {
        const vgicp_factor_desc& x = factors[r][f];
        dr.fd[f].blk = x.source->sblk;
        dr.fd[f].blk64 = x.source->blk64;
        dr.fd[f].c64 = x.source->c64;
        dr.fd[f].map = d.rank ? x.target->dev_rank() : x.target->dev();
      }
      use = &dr;
    }
    DeviceGuard gr(ctxs[r]->device);
    vgicp_graph sh = nullptr;
    if (int rc = graph_from(ctxs[r], factors[r], num_poses, *use, bounds[r], bounds[r + 1] - bounds[r], &sh)) {
      cleanup();
      return rc;
    }
    parent->shards.push_back(sh);
    parent->shard_first.push_back(bounds[r]);
    cudaEvent_t ev = nullptr;
    if (const cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming); e != cudaSuccess) {
      cleanup();
      return cuda_fail(e, "cudaEventCreate");
    }
    parent->shard_events.push_back(ev);
  }
  parent->shard_first.push_back(num_factors);
  // the root's assembly kernel reads the shards' blocks over peer memory (NVLink) when it can
  parent->peer_ok = true;
  for (int r = 1; r < num_shards; ++r) {
    const int dev = ctxs[r]->device;
    if (dev == root->device) continue;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, root->device, dev);
    if (!can) {
      parent->peer_ok = false;
      continue;
    }
    const cudaError_t e = cudaDeviceEnablePeerAccess(dev, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) parent->peer_ok = false;
    cudaGetLastError();
  }
  if (std::getenv("VGICP_SHARD_COPY")) parent->peer_ok = false;  // measurement switch: gather by peer copies
  if (const cudaError_t e = cudaEventCreateWithFlags(&parent->root_event, cudaEventDisableTiming); e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "cudaEventCreate");
  }
  parent->ctx = root;
  parent->num_factors = num_factors;
  parent->num_poses = num_poses;
  parent->rank_lookup = d.rank;
  for (auto* sh : parent->shards) parent->num_points += sh->num_points;
  const size_t nf = std::max(num_factors, 1);
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t o_pose = carve(sizeof(double) * 12 * std::max(num_poses, 1));
  const size_t o_out = carve(sizeof(double) * VGICP_LINEARIZED_DOUBLES * nf);
  const size_t o_oi = carve(sizeof(int) * nf);
  const size_t o_err = carve(sizeof(double) * nf);
  if (const cudaError_t e = dmalloc(root, &parent->block, off); e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "cudaMallocAsync(graph)");
  }
  char* b = static_cast<char*>(parent->block);
  parent->d_poses = reinterpret_cast<double*>(b + o_pose);
  parent->d_out = reinterpret_cast<double*>(b + o_out);
  parent->d_out_inl = reinterpret_cast<int*>(b + o_oi);
  parent->d_err = reinterpret_cast<double*>(b + o_err);
  for (int f = 0; f < num_factors; ++f) {
    parent->tgt_idx.push_back(factors[0][f].target_index);
    parent->src_idx.push_back(factors[0][f].source_index);
  }
  *out = parent.release();
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_graph_num_shards(vgicp_graph graph, int* num_shards) try {
  if (!graph || !num_shards) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *num_shards = graph->shards.empty() ? 1 : static_cast<int>(graph->shards.size());
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_graph_shard_range(vgicp_graph graph, int shard, int* first, int* count) try {
  if (!graph || !first || !count) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (graph->shards.empty()) {
    if (shard != 0) return fail(VGICP_E_INVALID_ARGUMENT, "shard index out of range");
    *first = 0;
    *count = graph->num_factors;
    return VGICP_OK;
  }
  if (shard < 0 || shard >= static_cast<int>(graph->shards.size()))
    return fail(VGICP_E_INVALID_ARGUMENT, "shard index out of range");
  *first = graph->shard_first[shard];
  *count = graph->shard_first[shard + 1] - graph->shard_first[shard];
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_graph_destroy(vgicp_graph graph) try {
  if (!graph) return VGICP_OK;
  for (auto* sh : graph->shards) vgicp_graph_destroy(sh);
  for (size_t r = 0; r < graph->shard_events.size(); ++r) cudaEventDestroy(graph->shard_events[r]);
  if (graph->root_event) cudaEventDestroy(graph->root_event);
  if (graph->ctx) {
    DeviceGuard g(graph->ctx->device);
    cudaStreamSynchronize(graph->ctx->stream);
    dfree(graph->ctx, graph->block);
    dfree(graph->ctx, graph->plan);
    dfree(graph->ctx, graph->band);
  }
  for (auto c : graph->clouds) release(c);
  for (auto m : graph->maps) release(m);
  delete graph;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_graph_num_factors(vgicp_graph graph, int* n) try {
  if (!graph || !n) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *n = graph->num_factors;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_graph_num_points(vgicp_graph graph, uint64_t* points) try {
  if (!graph || !points) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  *points = graph->num_points;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// One factor pass (linearize or evaluate) at device poses d_poses12 (root memory). A plain graph
// launches on its stream into d_res / d_inl. A sharded graph: the root stream marks the poses ready,
// every shard waits for that, pulls the poses to its device, launches its range into its own
// buffers and marks its event; the root stream waits for all shards. Then, when d_res != nullptr,
// the shards' results are gathered into d_res / d_inl (root memory, factor order) on the root
// stream; the assembly instead reads them in place over peer memory.
static int graph_pass(vgicp_graph g, bool linearize, const double* d_poses12, double* d_res, int32_t* d_inl) {
  if (g->shards.empty()) {
    DeviceGuard dg(g->ctx->device);
    if (g->num_items > 0) {
      VG_CUDA(launch_factor(linearize, g->rank_lookup, g->d_factors, g->d_items, g->num_items, g->f64_begin, d_poses12,
                            g->d_partials, g->d_part_inl, g->d_counters, g->num_factors, d_res, d_inl, g->ctx->stream));
      g->ctx->launches += factor_launches(g);
    } else if (g->num_factors > 0 && d_res) {  // zero-hit-free degenerate graph: all-zero blocks
      VG_CUDA(cudaMemsetAsync(d_res, 0, sizeof(double) * (linearize ? VGICP_LINEARIZED_DOUBLES : 1) * g->num_factors,
                              g->ctx->stream));
    }
    return VGICP_OK;
  }
  vgicp_ctx root = g->ctx;
  cudaStream_t s0 = root->stream;
  const size_t pose_bytes = sizeof(double) * 12 * g->num_poses;
  {
    DeviceGuard dg(root->device);
    VG_CUDA(cudaEventRecord(g->root_event, s0));
  }
  for (size_t r = 0; r < g->shards.size(); ++r) {
    vgicp_graph sh = g->shards[r];
    DeviceGuard dg(sh->ctx->device);
    cudaStream_t sr = sh->ctx->stream;
    VG_CUDA(cudaStreamWaitEvent(sr, g->root_event, 0));
    if (pose_bytes) VG_CUDA(cudaMemcpyAsync(sh->d_poses, d_poses12, pose_bytes, cudaMemcpyDefault, sr));
    if (int rc = graph_pass(sh, linearize, sh->d_poses, linearize ? sh->d_out : sh->d_err, sh->d_out_inl)) return rc;
    VG_CUDA(cudaEventRecord(g->shard_events[r], sr));
  }
  DeviceGuard dg(root->device);
  for (size_t r = 0; r < g->shards.size(); ++r) VG_CUDA(cudaStreamWaitEvent(s0, g->shard_events[r], 0));
  if (d_res) {
    const size_t per = linearize ? VGICP_LINEARIZED_DOUBLES : 1;
    for (size_t r = 0; r < g->shards.size(); ++r) {
      vgicp_graph sh = g->shards[r];
      if (sh->num_factors == 0) continue;
      const size_t f0 = static_cast<size_t>(g->shard_first[r]);
      VG_CUDA(cudaMemcpyAsync(d_res + f0 * per, linearize ? sh->d_out : sh->d_err, sizeof(double) * per * sh->num_factors,
                              cudaMemcpyDefault, s0));
      if (d_inl)
        VG_CUDA(cudaMemcpyAsync(d_inl + f0, sh->d_out_inl, sizeof(int32_t) * sh->num_factors, cudaMemcpyDefault, s0));
    }
  }
  return VGICP_OK;
}

int vgicp_graph_linearize_device(vgicp_graph graph, const double* d_poses12, double* d_out, int32_t* d_inliers) try {
  NvtxRange nvtx_("vgicp_graph_linearize_device");
  if (!graph || (graph->num_factors > 0 && (!d_poses12 || !d_out || !d_inliers)))
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  return graph_pass(graph, true, d_poses12, d_out, d_inliers);
} catch (...) {
  return api_exception();
}

int vgicp_graph_evaluate_device(vgicp_graph graph, const double* d_poses12, double* d_errors, int32_t* d_inliers) try {
  NvtxRange nvtx_("vgicp_graph_evaluate_device");
  if (!graph || (graph->num_factors > 0 && (!d_poses12 || !d_errors || !d_inliers)))
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  return graph_pass(graph, false, d_poses12, d_errors, d_inliers);
} catch (...) {
  return api_exception();
}

// Device-visible alias of `p` when it is page-locked host memory (cudaHostAlloc / cudaHostRegister /
// torch pin_memory; under UVA all of them are mapped), else null. Results can then be written by the
// kernel straight into the caller's buffer over PCIe, overlapping the D2H with the launch.
static void* mapped_alias(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

static int graph_run_host(vgicp_graph graph, bool linearize, const double* poses12, double* out, int32_t* inliers) {
  if (!graph || !poses12 || (graph->num_factors > 0 && (!out || !inliers)))
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  vgicp_ctx ctx = graph->ctx;
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  const int nf = graph->num_factors;
  if (nf == 0) return VGICP_OK;
  const size_t pose_bytes = sizeof(double) * 12 * graph->num_poses;
  const size_t per = linearize ? VGICP_LINEARIZED_DOUBLES : 1;
  const size_t res_bytes = sizeof(double) * per * nf;
  const size_t inl_bytes = sizeof(int32_t) * nf;
  // Page-locked caller buffers: the kernel's epilogue stores each factor's block directly into host
  // memory (zero-copy), so the result transfer overlaps the launch instead of following it.
  // VGICP_E2E_STAGED=1 keeps the copy-after-kernel path (for measurement).
  static const bool staged_only = [] {
    const char* e = std::getenv("VGICP_E2E_STAGED");
    return e && e[0] == '1';
  }();
  double* m_res = staged_only ? nullptr : static_cast<double*>(mapped_alias(out));
  auto* m_inl = staged_only ? nullptr : static_cast<int32_t*>(mapped_alias(inliers));
  const bool zero_copy = m_res && m_inl && graph->shards.empty();
  if (int rc = ensure_pinned(ctx, align_up(pose_bytes, 256) + (zero_copy ? 0 : align_up(res_bytes, 256) + inl_bytes)))
    return rc;
  char* h = static_cast<char*>(ctx->pinned);
  double* h_poses = reinterpret_cast<double*>(h);
  double* h_res = reinterpret_cast<double*>(h + align_up(pose_bytes, 256));
  auto* h_inl = reinterpret_cast<int32_t*>(h + align_up(pose_bytes, 256) + align_up(res_bytes, 256));
  const bool poses_pinned = mapped_alias(poses12) != nullptr;
  if (!poses_pinned) std::memcpy(h_poses, poses12, pose_bytes);
  VG_CUDA(cudaMemcpyAsync(graph->d_poses, poses_pinned ? poses12 : h_poses, pose_bytes, cudaMemcpyHostToDevice, s));
  if (!graph->shards.empty()) {
    // every shard's results go straight from its device to the host staging, on its own stream
    if (int rc = graph_pass(graph, linearize, graph->d_poses, nullptr, nullptr)) return rc;
    for (size_t r = 0; r < graph->shards.size(); ++r) {
      vgicp_graph sh = graph->shards[r];
      if (sh->num_factors == 0) continue;
      DeviceGuard dg(sh->ctx->device);
      const size_t f0 = static_cast<size_t>(graph->shard_first[r]);
      VG_CUDA(cudaMemcpyAsync(h_res + f0 * per, linearize ? sh->d_out : sh->d_err, sizeof(double) * per * sh->num_factors,
                              cudaMemcpyDeviceToHost, sh->ctx->stream));
      VG_CUDA(cudaMemcpyAsync(h_inl + f0, sh->d_out_inl, sizeof(int32_t) * sh->num_factors, cudaMemcpyDeviceToHost,
                              sh->ctx->stream));
    }
    for (auto* sh : graph->shards) {
      DeviceGuard dg(sh->ctx->device);
      VG_CUDA(cudaStreamSynchronize(sh->ctx->stream));
    }
    std::memcpy(out, h_res, res_bytes);
    std::memcpy(inliers, h_inl, inl_bytes);
    return VGICP_OK;
  }
  double* d_res = zero_copy ? m_res : (linearize ? graph->d_out : graph->d_err);
  int32_t* d_inl = zero_copy ? m_inl : graph->d_out_inl;
  if (int rc = graph_pass(graph, linearize, graph->d_poses, d_res, d_inl)) return rc;
  if (!zero_copy) {
    VG_CUDA(cudaMemcpyAsync(h_res, d_res, res_bytes, cudaMemcpyDeviceToHost, s));
    VG_CUDA(cudaMemcpyAsync(h_inl, d_inl, inl_bytes, cudaMemcpyDeviceToHost, s));
  }
  VG_CUDA(cudaStreamSynchronize(s));
  if (!zero_copy) {
    std::memcpy(out, h_res, res_bytes);
    std::memcpy(inliers, h_inl, inl_bytes);
  }
  return VGICP_OK;
}

int vgicp_graph_linearize(vgicp_graph graph, const double* poses12, double* out, int32_t* inliers) try {
  NvtxRange nvtx_("vgicp_graph_linearize");
  return graph_run_host(graph, true, poses12, out, inliers);
} catch (...) {
  return api_exception();
}

int vgicp_graph_evaluate(vgicp_graph graph, const double* poses12, double* errors, int32_t* inliers) try {
  NvtxRange nvtx_("vgicp_graph_evaluate");
  return graph_run_host(graph, false, poses12, errors, inliers);
} catch (...) {
  return api_exception();
}

// ------------------------------------------------------------------------------------ assembly
int vgicp_graph_assembly_plan(vgicp_graph graph, const uint8_t* fixed, int* num_slots, int* num_pairs,
                              int32_t* pairs) try {
  if (!graph || !num_slots || !num_pairs || (graph->num_poses > 0 && !fixed))
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  const int n = graph->num_poses;
  const int nf = graph->num_factors;
  // slot numbering: active variables in reverse insertion order (block_solver.cpp:26-34)
  std::vector<int> slot_of(n, -1);
  int active = 0;
  for (int v = 0; v < n; ++v) active += fixed[v] ? 0 : 1;
  for (int v = 0, rank = 0; v < n; ++v)
    if (!fixed[v]) slot_of[v] = active - 1 - rank++;
  // per-output contribution lists in factor order; pairs keyed by (col b, row a), a > b
  std::vector<std::vector<int>> diag(active);
  std::map<std::pair<int, int>, std::vector<int>> off;
  for (int f = 0; f < nf; ++f) {
    const int si = slot_of[graph->tgt_idx[f]], sj = slot_of[graph->src_idx[f]];
    if (si >= 0) diag[si].push_back(4 * f + 0);
    if (sj >= 0) diag[sj].push_back(4 * f + 1);
    if (si >= 0 && sj >= 0) {
      if (si >= sj) off[{sj, si}].push_back(4 * f + 2);
      else off[{si, sj}].push_back(4 * f + 3);
    }
  }
  const int P = static_cast<int>(off.size());
  const int O = active + P;
  std::vector<int> out_ptr(O + 1, 0), contrib;
  for (int o = 0; o < active; ++o) {
    contrib.insert(contrib.end(), diag[o].begin(), diag[o].end());
    out_ptr[o + 1] = static_cast<int>(contrib.size());
  }
  int o = active;
  for (const auto& [key, list] : off) {
    contrib.insert(contrib.end(), list.begin(), list.end());
    out_ptr[++o] = static_cast<int>(contrib.size());
    if (pairs) {
      pairs[2 * (o - 1 - active)] = key.second;  // row slot a
      pairs[2 * (o - 1 - active) + 1] = key.first;  // column slot b
    }
  }
  graph->pair_ab.clear();
  for (const auto& kv : off) {
    graph->pair_ab.push_back(kv.first.second);
    graph->pair_ab.push_back(kv.first.first);
  }
  DeviceGuard g(graph->ctx->device);
  if (graph->plan || graph->band) {
    VG_CUDA(cudaStreamSynchronize(graph->ctx->stream));
    dfree(graph->ctx, graph->plan);
    dfree(graph->ctx, graph->band);
    graph->plan = nullptr;
    graph->band = nullptr;
    graph->band_bw = -1;
    graph->band_cluster = 0;
  }
  const size_t b_ptr = align_up(sizeof(int) * (O + 1), 256);
  const size_t b_con = align_up(sizeof(int) * std::max<size_t>(contrib.size(), 1), 256);
  const size_t b_asm = sizeof(double) * (static_cast<size_t>(O) * 36 + static_cast<size_t>(active) * 6 + 1);
  VG_CUDA(dmalloc(graph->ctx, &graph->plan, b_ptr + b_con + b_asm));
  char* b = static_cast<char*>(graph->plan);
  graph->d_out_ptr = reinterpret_cast<int*>(b);
  graph->d_contrib = reinterpret_cast<int*>(b + b_ptr);
  graph->d_asm = reinterpret_cast<double*>(b + b_ptr + b_con);
  VG_CUDA(cudaMemcpyAsync(graph->d_out_ptr, out_ptr.data(), sizeof(int) * (O + 1), cudaMemcpyHostToDevice,
                          graph->ctx->stream));
  if (!contrib.empty())
    VG_CUDA(cudaMemcpyAsync(graph->d_contrib, contrib.data(), sizeof(int) * contrib.size(), cudaMemcpyHostToDevice,
                            graph->ctx->stream));
  VG_CUDA(cudaStreamSynchronize(graph->ctx->stream));
  graph->num_slots = active;
  graph->num_pairs = P;
  *num_slots = active;
  *num_pairs = P;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// Linearization pass + device assembly into d_asm (root memory), enqueued on the root stream. A
// sharded graph's assembly kernel reads the shards' blocks in place over peer memory (NVLink), or,
// without peer access, from the root copy that graph_pass gathers.
static int linearize_assemble(vgicp_graph graph, const double* d_poses12, double* d_asm) {
  const int S = graph->num_slots, O = S + graph->num_pairs;
  const bool gather = !graph->shards.empty() && !graph->peer_ok;
  if (int rc = graph_pass(graph, true, d_poses12, graph->shards.empty() || gather ? graph->d_out : nullptr,
                          graph->shards.empty() || gather ? graph->d_out_inl : nullptr))
    return rc;
  DeviceGuard g(graph->ctx->device);
  VG_CUDA(launch_assemble(graph->d_out_ptr, graph->d_contrib, S, O, graph->blocks(), d_asm, graph->ctx->stream));
  graph->ctx->launches += O > 0 ? 1 : 0;
  return VGICP_OK;
}

int vgicp_graph_linearize_assembled(vgicp_graph graph, const double* poses12, double* diag, double* offdiag,
                                    double* rhs) try {
  if (!graph || !poses12) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (!graph->plan) return fail(VGICP_E_INVALID_ARGUMENT, "no assembly plan (call vgicp_graph_assembly_plan)");
  const int S = graph->num_slots, P = graph->num_pairs, O = S + P;
  if ((S > 0 && (!diag || !rhs)) || (P > 0 && !offdiag)) return fail(VGICP_E_INVALID_ARGUMENT, "null output");
  vgicp_ctx ctx = graph->ctx;
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  const size_t pose_bytes = sizeof(double) * 12 * graph->num_poses;
  const size_t asm_bytes = sizeof(double) * (static_cast<size_t>(O) * 36 + static_cast<size_t>(S) * 6);
  if (int rc = ensure_pinned(ctx, align_up(pose_bytes, 256) + asm_bytes + 8)) return rc;
  char* h = static_cast<char*>(ctx->pinned);
  double* h_asm = reinterpret_cast<double*>(h + align_up(pose_bytes, 256));
  std::memcpy(h, poses12, pose_bytes);
  VG_CUDA(cudaMemcpyAsync(graph->d_poses, h, pose_bytes, cudaMemcpyHostToDevice, s));
  if (int rc = linearize_assemble(graph, graph->d_poses, graph->d_asm)) return rc;
  VG_CUDA(cudaMemcpyAsync(h_asm, graph->d_asm, asm_bytes, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  if (S > 0) std::memcpy(diag, h_asm, sizeof(double) * 36 * S);
  if (P > 0) std::memcpy(offdiag, h_asm + 36 * static_cast<size_t>(S), sizeof(double) * 36 * P);
  if (S > 0) std::memcpy(rhs, h_asm + 36 * static_cast<size_t>(O), sizeof(double) * 6 * S);
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_graph_linearize_assembled_device(vgicp_graph graph, const double* d_poses12, double* d_assembled) try {
  NvtxRange nvtx_("vgicp_graph_linearize_assembled_device");
  if (!graph || !d_poses12) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (!graph->plan) return fail(VGICP_E_INVALID_ARGUMENT, "no assembly plan (call vgicp_graph_assembly_plan)");
  const int S = graph->num_slots, O = S + graph->num_pairs;
  if (O > 0 && !d_assembled) return fail(VGICP_E_INVALID_ARGUMENT, "null output");
  return linearize_assemble(graph, d_poses12, d_assembled);
} catch (...) {
  return api_exception();
}

int vgicp_graph_assemble_device(vgicp_graph graph, const double* d_blocks, double* d_assembled) try {
  NvtxRange nvtx_("vgicp_graph_assemble_device");
  if (!graph) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (!graph->plan) return fail(VGICP_E_INVALID_ARGUMENT, "no assembly plan (call vgicp_graph_assembly_plan)");
  const int S = graph->num_slots, O = S + graph->num_pairs;
  if (O > 0 && (!d_assembled || (graph->num_factors > 0 && !d_blocks)))
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  ShardBlocks b{};
  b.n = 1;
  b.first[0] = 0;
  b.first[1] = graph->num_factors;
  b.out[0] = d_blocks;
  DeviceGuard g(graph->ctx->device);
  VG_CUDA(launch_assemble(graph->d_out_ptr, graph->d_contrib, S, O, b, d_assembled, graph->ctx->stream));
  graph->ctx->launches += O > 0 ? 1 : 0;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_graph_linearized_errors(vgicp_graph graph, double* errors, int32_t* inliers) try {
  NvtxRange nvtx_("vgicp_graph_linearized_errors");
  if (!graph || (graph->num_factors > 0 && (!errors || !inliers)))
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  const int nf = graph->num_factors;
  if (nf == 0) return VGICP_OK;
  vgicp_ctx ctx = graph->ctx;
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  const size_t err_bytes = sizeof(double) * nf;
  if (int rc = ensure_pinned(ctx, align_up(err_bytes, 256) + sizeof(int32_t) * nf)) return rc;
  auto* h_err = static_cast<double*>(ctx->pinned);
  auto* h_inl = reinterpret_cast<int32_t*>(static_cast<char*>(ctx->pinned) + align_up(err_bytes, 256));
  // strided gather of out[f·121 + 120] (the error member of each block): from the graph's blocks, or
  // from every shard's own blocks, each on its stream (after its last pass)
  const std::vector<vgicp_graph> parts = graph->shards.empty() ? std::vector<vgicp_graph>{graph} : graph->shards;
  for (size_t r = 0; r < parts.size(); ++r) {
    vgicp_graph sh = parts[r];
    if (sh->num_factors == 0) continue;
    const size_t f0 = graph->shards.empty() ? 0 : static_cast<size_t>(graph->shard_first[r]);
    DeviceGuard dg(sh->ctx->device);
    cudaStream_t sr = sh->ctx->stream;
    VG_CUDA(cudaMemcpy2DAsync(h_err + f0, sizeof(double), sh->d_out + (VGICP_LINEARIZED_DOUBLES - 1),
                              sizeof(double) * VGICP_LINEARIZED_DOUBLES, sizeof(double), sh->num_factors,
                              cudaMemcpyDeviceToHost, sr));
    VG_CUDA(cudaMemcpyAsync(h_inl + f0, sh->d_out_inl, sizeof(int32_t) * sh->num_factors, cudaMemcpyDeviceToHost, sr));
  }
  for (auto* sh : parts) {
    DeviceGuard dg(sh->ctx->device);
    VG_CUDA(cudaStreamSynchronize(sh->ctx->stream));
  }
  (void)s;
  std::memcpy(errors, h_err, err_bytes);
  std::memcpy(inliers, h_inl, sizeof(int32_t) * nf);
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// ------------------------------------------------------------------------------- band solver
int vgicp_graph_solver_plan(vgicp_graph graph, int* bandwidth, int* supported) try {
  if (!graph || !bandwidth || !supported) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (!graph->plan) return fail(VGICP_E_INVALID_ARGUMENT, "no assembly plan (call vgicp_graph_assembly_plan)");
  vgicp_ctx ctx = graph->ctx;
  DeviceGuard g(ctx->device);
  if (graph->band) {
    VG_CUDA(cudaStreamSynchronize(ctx->stream));
    dfree(ctx, graph->band);
    graph->band = nullptr;
  }
  const int S = graph->num_slots, P = graph->num_pairs;
  const BandPlanHost hp = make_band_plan(S, P, graph->pair_ab.data());
  graph->band_bw = hp.bw;
  graph->band_cluster = S > 0 && !std::getenv("VGICP_NO_BAND_SOLVER") ? band_cluster_size(hp.bw, S) : 0;
  cudaGetLastError();  // attribute / occupancy probes that failed are not launch errors
  *bandwidth = hp.bw;
  *supported = graph->band_cluster > 0 ? 1 : 0;
  if (!*supported) return VGICP_OK;
  const size_t b_perm = align_up(sizeof(int) * S, 256), b_reach = b_perm;
  const size_t b_ptr = align_up(sizeof(int) * (S + 1), 256);
  const size_t b_ent = align_up(sizeof(int2) * std::max<size_t>(hp.col_ent.size(), 1), 256);
  // two instances of the per-solve state (Lg, x, status, ready): a pair of damping values can be
  // solved concurrently by two clusters (vgicp_graph_solve_damped_pair)
  const size_t b_status = 512, b_x = align_up(sizeof(double) * 12 * S, 256), b_ready = align_up(sizeof(int) * 2 * S, 256);
  const size_t b_L = 2 * sizeof(double) * (36 * (static_cast<size_t>(hp.bw) + 1) + 16) * S;
  VG_CUDA(dmalloc(ctx, &graph->band, b_perm + b_reach + b_ptr + b_ent + b_status + b_x + b_ready + b_L));
  char* b = static_cast<char*>(graph->band);
  BandDev& d = graph->band_dev;
  d.S = S;
  d.bw = hp.bw;
  d.perm = reinterpret_cast<int*>(b);
  d.reach = reinterpret_cast<int*>(b + b_perm);
  d.col_ptr = reinterpret_cast<int*>(b + b_perm + b_reach);
  d.col_ent = reinterpret_cast<int2*>(b + b_perm + b_reach + b_ptr);
  d.status = reinterpret_cast<int*>(b + b_perm + b_reach + b_ptr + b_ent);
  d.x = reinterpret_cast<double*>(b + b_perm + b_reach + b_ptr + b_ent + b_status);
  d.ready = reinterpret_cast<int*>(b + b_perm + b_reach + b_ptr + b_ent + b_status + b_x);
  d.Lg = reinterpret_cast<double*>(b + b_perm + b_reach + b_ptr + b_ent + b_status + b_x + b_ready);
  graph->band_epoch = 0;
  VG_CUDA(cudaMemsetAsync(d.ready, 0, sizeof(int) * 2 * S, ctx->stream));
  cudaStream_t s = ctx->stream;
  VG_CUDA(cudaMemcpyAsync(const_cast<int*>(d.perm), hp.perm.data(), sizeof(int) * S, cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemcpyAsync(const_cast<int*>(d.reach), hp.reach.data(), sizeof(int) * S, cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemcpyAsync(const_cast<int*>(d.col_ptr), hp.col_ptr.data(), sizeof(int) * (S + 1),
                          cudaMemcpyHostToDevice, s));
  if (!hp.col_ent.empty())
    VG_CUDA(cudaMemcpyAsync(const_cast<int2*>(d.col_ent), hp.col_ent.data(), sizeof(int2) * hp.col_ent.size(),
                            cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaStreamSynchronize(s));
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// One launch solving the damped system for `count` (1 or 2) damping values, one cluster each.
static int solve_damped_n(vgicp_graph graph, const double* d_assembled, const double* lambdas, int count, double* x,
                          int* solved) {
  NvtxRange nvtx_(count > 1 ? "vgicp_graph_solve_damped_pair" : "vgicp_graph_solve_damped");
  if (!graph || !x || !solved || !lambdas || (graph->num_slots > 0 && !d_assembled))
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (!graph->band && graph->num_slots > 0)
    return fail(VGICP_E_INVALID_ARGUMENT, graph->band_bw >= 0
                                              ? "band solver unavailable for this bandwidth (use a dense solve)"
                                              : "no solver plan (call vgicp_graph_solver_plan)");
  const int S = graph->num_slots;
  for (int i = 0; i < count; ++i) solved[i] = 1;
  if (S == 0) return VGICP_OK;
  vgicp_ctx ctx = graph->ctx;
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  graph->band_epoch = graph->band_epoch == 0x7fffffff ? 1 : graph->band_epoch + 1;
  VG_CUDA(launch_band_solve(graph->band_dev, graph->band_cluster, d_assembled, graph->num_pairs, lambdas[0],
                            count > 1 ? lambdas[1] : lambdas[0], count, graph->band_epoch, s));
  ctx->launches += 1;
  const size_t b_x = sizeof(double) * 6 * S;
  if (int rc = ensure_pinned(ctx, align_up(count * b_x, 256) + 512)) return rc;
  auto* h_x = static_cast<double*>(ctx->pinned);
  auto* h_status = reinterpret_cast<int*>(static_cast<char*>(ctx->pinned) + align_up(count * b_x, 256));
  VG_CUDA(cudaMemcpyAsync(h_status, graph->band_dev.status, sizeof(int) * 64 * count, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaMemcpyAsync(h_x, graph->band_dev.x, count * b_x, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  if (std::getenv("VGICP_SOLVE_PROF")) {  // cycle profile of CTA 0 (diagnostic build)
    unsigned long long prof[8];
    VG_CUDA(cudaMemcpy(prof, reinterpret_cast<unsigned long long*>(graph->band_dev.status) + 8, sizeof(prof),
                       cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "band solve C=%d bw=%d S=%d cycles: wait %llu load %llu owner(publish) %llu update %llu sync %llu "
                 "back %llu owner-update %llu owner-factor %llu\n",
                 graph->band_cluster, graph->band_bw, S, prof[0], prof[1], prof[2], prof[3], prof[4], prof[5],
                 prof[6], prof[7]);
  }
  for (int i = 0; i < count; ++i) {
    solved[i] = h_status[64 * i] == 0 ? 1 : 0;  // else a pivot block was not positive definite
    if (solved[i]) std::memcpy(x + static_cast<size_t>(i) * 6 * S, h_x + static_cast<size_t>(i) * 6 * S, b_x);
  }
  return VGICP_OK;
}

int vgicp_graph_solve_damped(vgicp_graph graph, const double* d_assembled, double lambda, double* x, int* solved) try {
  return solve_damped_n(graph, d_assembled, &lambda, 1, x, solved);
} catch (...) {
  return api_exception();
}

int vgicp_graph_solve_damped_pair(vgicp_graph graph, const double* d_assembled, const double* lambdas, double* x,
                                  int* solved) try {
  return solve_damped_n(graph, d_assembled, lambdas, 2, x, solved);
} catch (...) {
  return api_exception();
}

// Single-factor entry points: a one-factor graph over poses {target, source}.
static int single_factor(vgicp_ctx ctx, const vgicp_factor_desc* factor, const double* T_target,
                         const double* T_source, bool linearize, double* out, int32_t* inliers) {
  if (!ctx || !factor || !T_target || !T_source || !out || !inliers)
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (factor->target_index == factor->source_index)
    return fail(VGICP_E_INVALID_ARGUMENT, "matching cost factor requires distinct variables");
  vgicp_factor_desc d = *factor;
  d.target_index = 0;
  d.source_index = 1;
  vgicp_graph gr = nullptr;
  if (int rc = vgicp_graph_create(ctx, &d, 1, 2, 0, &gr)) return rc;
  double poses[24];
  std::memcpy(poses, T_target, sizeof(double) * 12);
  std::memcpy(poses + 12, T_source, sizeof(double) * 12);
  const int rc = graph_run_host(gr, linearize, poses, out, inliers);
  vgicp_graph_destroy(gr);
  return rc;
}

int vgicp_linearize_matching_cost(vgicp_ctx ctx, const vgicp_factor_desc* factor, const double T_target[12],
                                  const double T_source[12], double out[VGICP_LINEARIZED_DOUBLES],
                                  int32_t* inliers) try {
  return single_factor(ctx, factor, T_target, T_source, true, out, inliers);
} catch (...) {
  return api_exception();
}

int vgicp_evaluate_matching_cost(vgicp_ctx ctx, const vgicp_factor_desc* factor, const double T_target[12],
                                 const double T_source[12], double* error, int32_t* inliers) try {
  return single_factor(ctx, factor, T_target, T_source, false, error, inliers);
} catch (...) {
  return api_exception();
}

int vgicp_gicp_error(vgicp_ctx ctx, const double source_mean[3], const double source_cov[9],
                     const double target_mean[3], const double target_cov[9], const double T[12], double* error,
                     double residual[3], double information[9], int* valid) try {
  if (!ctx || !source_mean || !source_cov || !target_mean || !target_cov || !T || !error || !residual ||
      !information || !valid)
    return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  DeviceGuard g(ctx->device);
  if (int rc = ensure_scratch(ctx, 64 * sizeof(double))) return rc;
  if (int rc = ensure_pinned(ctx, 64 * sizeof(double))) return rc;
  double* h = static_cast<double*>(ctx->pinned);
  std::memcpy(h, source_mean, 3 * sizeof(double));
  std::memcpy(h + 3, source_cov, 9 * sizeof(double));
  std::memcpy(h + 12, target_mean, 3 * sizeof(double));
  std::memcpy(h + 15, target_cov, 9 * sizeof(double));
  std::memcpy(h + 24, T, 12 * sizeof(double));
  double* d = static_cast<double*>(ctx->scratch);
  cudaStream_t s = ctx->stream;
  VG_CUDA(cudaMemcpyAsync(d, h, 36 * sizeof(double), cudaMemcpyHostToDevice, s));
  VG_CUDA(launch_gicp_error(d, d + 40, s));
  ctx->launches += 1;
  VG_CUDA(cudaMemcpyAsync(h + 40, d + 40, 14 * sizeof(double), cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  *error = h[40];
  std::memcpy(residual, h + 41, 3 * sizeof(double));
  std::memcpy(information, h + 44, 9 * sizeof(double));
  *valid = h[53] != 0.0 ? 1 : 0;
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

// ------------------------------------------------------------------------------------ preprocessing
// memcpy split over host threads (staging of large point / covariance batches)
static void parallel_copy(void* dst, const void* src, size_t bytes) {
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (bytes < (8u << 20) || hw == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t chunk = (bytes + hw - 1) / hw;
  for (unsigned t = 0; t < hw; ++t) {
    const size_t o = t * chunk;
    if (o >= bytes) break;
    th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(chunk, bytes - o)); });
  }
  for (auto& x : th) x.join();
}

// copies[k] = (dst, src, bytes), spread over host threads (fresh destination pages fault in parallel)
static void parallel_copies(const std::vector<std::tuple<void*, const void*, size_t>>& copies) {
  size_t total = 0;
  for (const auto& c : copies) total += std::get<2>(c);
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (total < (4u << 20) || hw == 1 || copies.size() == 1) {
    for (const auto& c : copies) parallel_copy(std::get<0>(c), std::get<1>(c), std::get<2>(c));
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> th;
  for (unsigned t = 0; t < hw; ++t)
    th.emplace_back([&] {
      for (size_t k; (k = next.fetch_add(1)) < copies.size();)
        std::memcpy(std::get<0>(copies[k]), std::get<1>(copies[k]), std::get<2>(copies[k]));
    });
  for (auto& x : th) x.join();
}


int vgicp_estimate_covariances_batch(vgicp_ctx ctx, const float* const* xyz, const size_t* n, int m, int k,
                                     double plane_epsilon, float* const* cov6) try {
  NvtxRange nvtx_("vgicp_estimate_covariances_batch");
  if (!ctx || (m > 0 && (!xyz || !n || !cov6))) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  if (m <= 0) return VGICP_OK;
  // estimate_covariances validation (point_cloud.cpp:47-53)
  if (k < 4) return fail(VGICP_E_INVALID_ARGUMENT, "covariance estimation requires k >= 4 neighbors");
  if (k > 32) return fail(VGICP_E_INVALID_ARGUMENT, "covariance estimation supports k <= 32 on the GPU");
  std::vector<CovSeg> segs(m);
  size_t total = 0;
  unsigned max_n = 0;
  for (int c = 0; c < m; ++c) {
    if (n[c] <= static_cast<size_t>(k))
      return fail(VGICP_E_INVALID_ARGUMENT, "covariance estimation requires more than k points");
    if (!xyz[c] || !cov6[c]) return fail(VGICP_E_INVALID_ARGUMENT, "null point or output array");
    segs[c] = CovSeg{};
    segs[c].offset = static_cast<unsigned>(total);
    segs[c].n = static_cast<unsigned>(n[c]);
    segs[c].eps = plane_epsilon;
    total += n[c];
    max_n = std::max(max_n, segs[c].n);
  }
  if (total >= (1ull << 31)) return fail(VGICP_E_INVALID_ARGUMENT, "batch too large");
  DeviceGuard gd(ctx->device);
  cudaStream_t s = ctx->stream;
  const bool verbose = std::getenv("VGICP_VERBOSE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto stage = [&](const char* what) {
    if (!verbose) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[vgicp] covariances %-10s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  // 1. points to the device (pinned staging), per-cloud bounding boxes on the device
  if (int rc = ensure_pinned(ctx, sizeof(float) * 6 * total)) return rc;
  DevBuf pts(ctx), meta(ctx);
  VG_CUDA(pts.alloc(align_up(sizeof(float) * 3 * total, 256) + sizeof(float) * 6 * total));
  VG_CUDA(meta.alloc(align_up(sizeof(CovSeg) * m, 256) + sizeof(unsigned) * 6 * m + sizeof(int) * m));
  auto* d_xyz = static_cast<float*>(pts.p);
  auto* d_cov = reinterpret_cast<float*>(static_cast<char*>(pts.p) + align_up(sizeof(float) * 3 * total, 256));
  auto* d_segs = static_cast<CovSeg*>(meta.p);
  auto* d_box = reinterpret_cast<unsigned*>(static_cast<char*>(meta.p) + align_up(sizeof(CovSeg) * m, 256));
  auto* d_bad = reinterpret_cast<int*>(d_box + 6 * m);
  VG_CUDA(cudaStreamSynchronize(s));
  float* h = static_cast<float*>(ctx->pinned);
  {
    std::vector<std::tuple<void*, const void*, size_t>> cp;
    for (int c = 0; c < m; ++c) cp.emplace_back(h + 3 * segs[c].offset, xyz[c], sizeof(float) * 3 * n[c]);
    parallel_copies(cp);
  }
  stage("stage-in");
  VG_CUDA(cudaMemcpyAsync(d_xyz, h, sizeof(float) * 3 * total, cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemcpyAsync(d_segs, segs.data(), sizeof(CovSeg) * m, cudaMemcpyHostToDevice, s));
  stage("h2d");
  for (int c = 0; c < m; ++c) {
    VG_CUDA(cudaMemsetAsync(d_box + 6 * c, 0xFF, 3 * sizeof(unsigned), s));
    VG_CUDA(cudaMemsetAsync(d_box + 6 * c + 3, 0, 3 * sizeof(unsigned), s));
  }
  VG_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int) * m, s));
  VG_CUDA(launch_cov_bbox(d_segs, m, max_n, d_xyz, d_box, d_bad, s));
  std::vector<unsigned> hbox(6 * m);
  std::vector<int> hbad(m);
  VG_CUDA(cudaMemcpyAsync(hbox.data(), d_box, sizeof(unsigned) * 6 * m, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaMemcpyAsync(hbad.data(), d_bad, sizeof(int) * m, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  stage("bbox");
  // 2. grid parameters per cloud (cell ~ (extent^2 k / n)^(1/2) in the dominant plane, <= 2^22 cells)
  unsigned long long cells = 0;
  for (int c = 0; c < m; ++c) {
    if (hbad[c]) return fail(VGICP_E_INVALID_ARGUMENT, "point cloud contains NaN/Inf coordinates");
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
      lo[a] = unordered_host(hbox[6 * c + a]);
      hi[a] = unordered_host(hbox[6 * c + 3 + a]);
    }
    const double ext = std::max({hi[0] - lo[0], hi[1] - lo[1], 1e-3});
    double cell = std::max(std::sqrt(ext * ext * k / static_cast<double>(n[c])), 1e-3);
    int g[3];
    for (;;) {
      unsigned long long gc = 1;
      for (int a = 0; a < 3; ++a) {
        g[a] = static_cast<int>(std::floor((hi[a] - lo[a]) / cell)) + 1;
        gc *= static_cast<unsigned long long>(g[a]);
      }
      if (gc <= (1ull << 22)) break;
      cell *= 1.5;
    }
    CovSeg& sg = segs[c];
    sg.cell_base = static_cast<unsigned>(cells);
    sg.gx = g[0], sg.gy = g[1], sg.gz = g[2];
    for (int a = 0; a < 3; ++a) sg.lo[a] = lo[a];
    sg.cell = cell;
    cells += static_cast<unsigned long long>(g[0]) * g[1] * g[2];
  }
  if (cells >= (1ull << 31)) return fail(VGICP_E_INVALID_ARGUMENT, "batch too large");
  // 3. counting sort into the cells, exact kNN, eigen regularisation
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t o_cell = carve(sizeof(unsigned) * total);
  const size_t o_sorted = carve(sizeof(float4) * total);
  const size_t o_cnt = carve(sizeof(unsigned) * (cells + 1));
  const size_t o_start = carve(sizeof(unsigned) * (cells + 1));
  const size_t o_cursor = carve(sizeof(unsigned) * cells);
  size_t scan_bytes = 0;
  VG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const unsigned*)nullptr, (unsigned*)nullptr,
                                        static_cast<int>(cells + 1), s));
  const size_t o_temp = carve(scan_bytes);
  if (int rc = ensure_scratch(ctx, off)) return rc;
  char* sb = static_cast<char*>(ctx->scratch);
  auto* d_cell = reinterpret_cast<unsigned*>(sb + o_cell);
  auto* d_sorted = reinterpret_cast<float4*>(sb + o_sorted);
  auto* d_cnt = reinterpret_cast<unsigned*>(sb + o_cnt);
  auto* d_start = reinterpret_cast<unsigned*>(sb + o_start);
  auto* d_cursor = reinterpret_cast<unsigned*>(sb + o_cursor);
  VG_CUDA(cudaMemcpyAsync(d_segs, segs.data(), sizeof(CovSeg) * m, cudaMemcpyHostToDevice, s));
  VG_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned) * (cells + 1), s));
  VG_CUDA(cudaMemsetAsync(d_cursor, 0, sizeof(unsigned) * cells, s));
  VG_CUDA(launch_cov_count(d_segs, m, max_n, d_xyz, d_cell, d_cnt, s));
  VG_CUDA(cub::DeviceScan::ExclusiveSum(sb + o_temp, scan_bytes, d_cnt, d_start, static_cast<int>(cells + 1), s));
  VG_CUDA(launch_cov_scatter(d_segs, m, max_n, d_xyz, d_cell, d_start, d_cursor, d_sorted, s));
  stage("grid");
  VG_CUDA(launch_cov_knn(d_segs, m, max_n, d_xyz, d_start, d_sorted, k, d_cov, s));
  ctx->launches += 5;
  stage("knn");
  VG_CUDA(cudaMemcpyAsync(h, d_cov, sizeof(float) * 6 * total, cudaMemcpyDeviceToHost, s));
  VG_CUDA(cudaStreamSynchronize(s));
  stage("d2h");
  {
    std::vector<std::tuple<void*, const void*, size_t>> cp;
    for (int c = 0; c < m; ++c) cp.emplace_back(cov6[c], h + 6 * segs[c].offset, sizeof(float) * 6 * n[c]);
    parallel_copies(cp);
  }
  stage("stage-out");
  return VGICP_OK;
} catch (...) {
  return api_exception();
}

int vgicp_estimate_covariances(vgicp_ctx ctx, const float* xyz, size_t n, int k, double plane_epsilon,
                               float* cov6) try {
  return vgicp_estimate_covariances_batch(ctx, &xyz, &n, 1, k, plane_epsilon, &cov6);
} catch (...) {
  return api_exception();
}

}  // extern "C"
