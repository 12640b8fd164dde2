// Device-side construction of a cloud's layout (every vgicp_cloud_upload, and the submap cloud of
// vgicp_submap_build from float64 device arrays): input-order SoA for the builds and the
// Morton-ordered 64-point blocks for the probe kernels (Z-order code of 10 bits per axis over the
// finite bounding box, stable radix sort: ties in input order).
#include <algorithm>
#include <type_traits>

#include "internal.h"

namespace vgicp {

namespace {

__device__ __forceinline__ unsigned ordered(float f) {  // monotone float -> uint map
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unordered(unsigned u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

template <typename T>
__global__ void bbox_kernel(const T* __restrict__ xyz, size_t n, unsigned* __restrict__ box) {
  unsigned lo[3] = {~0u, ~0u, ~0u}, hi[3] = {0u, 0u, 0u};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = static_cast<float>(xyz[3 * i + a]);
      if (isfinite(v)) {
        lo[a] = min(lo[a], ordered(v));
        hi[a] = max(hi[a], ordered(v));
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    atomicMin(&box[a], lo[a]);
    atomicMax(&box[3 + a], hi[a]);
  }
}

__device__ __forceinline__ unsigned spread10(unsigned x) {  // 10 bits -> every third bit
  x &= 0x3FFu;
  x = (x | (x << 16)) & 0x030000FFu;
  x = (x | (x << 8)) & 0x0300F00Fu;
  x = (x | (x << 4)) & 0x030C30C3u;
  x = (x | (x << 2)) & 0x09249249u;
  return x;
}

template <typename T>
__global__ void morton_kernel(const T* __restrict__ xyz, size_t n, const unsigned* __restrict__ box,
                              unsigned* __restrict__ codes, unsigned* __restrict__ idx) {
  float lo[3], ext[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = unordered(box[a]);
    ext[a] = unordered(box[3 + a]) - lo[a];
  }
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = static_cast<float>(xyz[3 * i + a]);
      const float u = (isfinite(v) && ext[a] > 0.f) ? (v - lo[a]) / ext[a] : 0.f;
      c[a] = static_cast<unsigned>(fminf(1023.f, fmaxf(0.f, u * 1024.f)));
    }
    codes[i] = spread10(c[0]) | (spread10(c[1]) << 1) | (spread10(c[2]) << 2);
    idx[i] = static_cast<unsigned>(i);
  }
}

// Source adaptors: float64 points + full 3×3 covariances (submap clouds) or float32 points + the
// 6 unique covariance entries (uploads; nullptr = raw cloud, zero covariances).
struct SrcF64 {
  const double* xyz;
  const double* cov9;  // nullptr: raw cloud
  __device__ void get(size_t j, float4& a, float4& b, float& z) const {
    const double* p = xyz + 3 * j;
    if (cov9) {
      const double* q = cov9 + 9 * j;
      a = make_float4((float)p[0], (float)p[1], (float)p[2], (float)q[0]);
      b = make_float4((float)q[1], (float)q[2], (float)q[4], (float)q[5]);
      z = (float)q[8];
    } else {
      a = make_float4((float)p[0], (float)p[1], (float)p[2], 0.f);
      b = make_float4(0.f, 0.f, 0.f, 0.f);
      z = 0.f;
    }
  }
  __device__ void get64(size_t j, double& x, double& y, double& w) const {
    x = xyz[3 * j], y = xyz[3 * j + 1], w = xyz[3 * j + 2];
  }
};
struct SrcF32 {
  const float* xyz;
  const float* cov6;
  __device__ void get(size_t j, float4& a, float4& b, float& z) const {
    const float* p = xyz + 3 * j;
    if (cov6) {
      const float* q = cov6 + 6 * j;
      a = make_float4(p[0], p[1], p[2], q[0]);
      b = make_float4(q[1], q[2], q[3], q[4]);
      z = q[5];
    } else {  // raw cloud
      a = make_float4(p[0], p[1], p[2], 0.f);
      b = make_float4(0.f, 0.f, 0.f, 0.f);
      z = 0.f;
    }
  }
};

template <typename Src>
__global__ void fill_cloud_kernel(Src src, size_t n, const unsigned* __restrict__ perm, float4* __restrict__ pa,
                                  float4* __restrict__ pb, float* __restrict__ pc, PointBlock* __restrict__ blk,
                                  PointBlock64* __restrict__ blk64, size_t padded) {
  for (size_t d = blockIdx.x * (size_t)blockDim.x + threadIdx.x; d < padded; d += (size_t)gridDim.x * blockDim.x) {
    const size_t dn = d < n ? d : n - 1;
#pragma unroll
    for (int copy = 0; copy < 2; ++copy) {
      const size_t j = copy == 0 ? dn : perm[dn];
      float4 a, b;
      float z;
      src.get(j, a, b, z);
      if (copy == 0) {
        if (d < n) pa[d] = a, pb[d] = b, pc[d] = z;
      } else {
        PointBlock& B = blk[d / kPointBlock];
        B.pa[d % kPointBlock] = a;
        B.pb[d % kPointBlock] = b;
        B.pc[d % kPointBlock] = z;
        if constexpr (std::is_same<Src, SrcF64>::value) {
          if (blk64) {  // the exact float64 means, same Morton position
            PointBlock64& B64 = blk64[d / kPointBlock];
            src.get64(j, B64.x[d % kPointBlock], B64.y[d % kPointBlock], B64.z[d % kPointBlock]);
            B64.idx[d % kPointBlock] = static_cast<unsigned>(j);
          }
        }
      }
    }
  }
}

unsigned grid_cloud(size_t n) {
  const size_t g = (n + 255) / 256;
  return static_cast<unsigned>(g == 0 ? 1 : (g < 4096 ? g : 4096));
}

// Batched float32 uploads (one launch per stage for all clouds; blockIdx.y = cloud).
__global__ void bbox_batch_kernel(const UploadSeg* __restrict__ segs, unsigned* __restrict__ boxes) {
  const UploadSeg& g = segs[blockIdx.y];
  const float* __restrict__ xyz = g.xyz;
  unsigned lo[3] = {~0u, ~0u, ~0u}, hi[3] = {0u, 0u, 0u};
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = xyz[3 * (size_t)i + a];
      if (isfinite(v)) {
        lo[a] = min(lo[a], ordered(v));
        hi[a] = max(hi[a], ordered(v));
      }
    }
  }
  unsigned* box = boxes + 6 * blockIdx.y;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    atomicMin(&box[a], lo[a]);
    atomicMax(&box[3 + a], hi[a]);
  }
}

__global__ void morton_batch_kernel(const UploadSeg* __restrict__ segs, const unsigned* __restrict__ boxes,
                                    unsigned* __restrict__ codes, unsigned* __restrict__ idx) {
  const UploadSeg& g = segs[blockIdx.y];
  const unsigned* box = boxes + 6 * blockIdx.y;
  float lo[3], ext[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = unordered(box[a]);
    ext[a] = unordered(box[3 + a]) - lo[a];
  }
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    unsigned c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = g.xyz[3 * (size_t)i + a];
      const float u = (isfinite(v) && ext[a] > 0.f) ? (v - lo[a]) / ext[a] : 0.f;
      c[a] = static_cast<unsigned>(fminf(1023.f, fmaxf(0.f, u * 1024.f)));
    }
    codes[g.offset + i] = spread10(c[0]) | (spread10(c[1]) << 1) | (spread10(c[2]) << 2);
    idx[g.offset + i] = i;
  }
}

__global__ void fill_batch_kernel(const UploadSeg* __restrict__ segs, const unsigned* __restrict__ perm) {
  const UploadSeg& g = segs[blockIdx.y];
  const unsigned n = g.n;
  const unsigned padded = (n + kPointBlock - 1) / kPointBlock * kPointBlock;
  const SrcF32 src{g.xyz, g.cov6};
  for (unsigned d = blockIdx.x * blockDim.x + threadIdx.x; d < padded; d += gridDim.x * blockDim.x) {
    const unsigned dn = d < n ? d : n - 1;
#pragma unroll
    for (int copy = 0; copy < 2; ++copy) {
      const unsigned j = copy == 0 ? dn : perm[g.offset + dn];
      float4 a, b;
      float z;
      src.get(j, a, b, z);
      if (copy == 0) {
        if (d < n) g.pa[d] = a, g.pb[d] = b, g.pc[d] = z;
      } else {
        PointBlock& B = g.blk[d / kPointBlock];
        B.pa[d % kPointBlock] = a;
        B.pb[d % kPointBlock] = b;
        B.pc[d % kPointBlock] = z;
      }
    }
  }
}

}  // namespace

cudaError_t launch_upload_batch_prepare(const UploadSeg* segs, int m, unsigned max_n, unsigned* boxes, unsigned* codes,
                                        unsigned* idx, cudaStream_t s) {
  if (m <= 0 || max_n == 0) return cudaSuccess;
  const unsigned gx = std::min<unsigned>((max_n + 255) / 256, 64);
  for (int m0 = 0; m0 < m; m0 += 65535) {
    const unsigned mm = static_cast<unsigned>(std::min(65535, m - m0));
    bbox_batch_kernel<<<dim3(gx, mm), 256, 0, s>>>(segs + m0, boxes + 6 * m0);
    morton_batch_kernel<<<dim3(gx, mm), 256, 0, s>>>(segs + m0, boxes + 6 * m0, codes, idx);
  }
  return cudaGetLastError();
}

cudaError_t launch_upload_batch_fill(const UploadSeg* segs, int m, unsigned max_n, const unsigned* perm, cudaStream_t s) {
  if (m <= 0 || max_n == 0) return cudaSuccess;
  const unsigned gx = std::min<unsigned>((max_n + kPointBlock + 255) / 256, 64);
  for (int m0 = 0; m0 < m; m0 += 65535) {
    const unsigned mm = static_cast<unsigned>(std::min(65535, m - m0));
    fill_batch_kernel<<<dim3(gx, mm), 256, 0, s>>>(segs + m0, perm);
  }
  return cudaGetLastError();
}

cudaError_t launch_cloud_bbox(const double* xyz, size_t n, unsigned* box, cudaStream_t s) {
  bbox_kernel<<<grid_cloud(n), 256, 0, s>>>(xyz, n, box);
  return cudaGetLastError();
}
cudaError_t launch_cloud_bbox(const float* xyz, size_t n, unsigned* box, cudaStream_t s) {
  bbox_kernel<<<grid_cloud(n), 256, 0, s>>>(xyz, n, box);
  return cudaGetLastError();
}

cudaError_t launch_cloud_morton(const double* xyz, size_t n, const unsigned* box, unsigned* codes, unsigned* idx,
                                cudaStream_t s) {
  morton_kernel<<<grid_cloud(n), 256, 0, s>>>(xyz, n, box, codes, idx);
  return cudaGetLastError();
}
cudaError_t launch_cloud_morton(const float* xyz, size_t n, const unsigned* box, unsigned* codes, unsigned* idx,
                                cudaStream_t s) {
  morton_kernel<<<grid_cloud(n), 256, 0, s>>>(xyz, n, box, codes, idx);
  return cudaGetLastError();
}

cudaError_t launch_cloud_fill(const double* xyz, const double* cov9, size_t n, const unsigned* perm, float4* pa,
                              float4* pb, float* pc, PointBlock* blk, PointBlock64* blk64, cudaStream_t s) {
  const size_t padded = (n + kPointBlock - 1) / kPointBlock * kPointBlock;
  fill_cloud_kernel<<<grid_cloud(padded), 256, 0, s>>>(SrcF64{xyz, cov9}, n, perm, pa, pb, pc, blk, blk64, padded);
  return cudaGetLastError();
}
cudaError_t launch_cloud_fill(const float* xyz, const float* cov6, size_t n, const unsigned* perm, float4* pa,
                              float4* pb, float* pc, PointBlock* blk, cudaStream_t s) {
  const size_t padded = (n + kPointBlock - 1) / kPointBlock * kPointBlock;
  fill_cloud_kernel<<<grid_cloud(padded), 256, 0, s>>>(SrcF32{xyz, cov6}, n, perm, pa, pb, pc, blk, nullptr, padded);
  return cudaGetLastError();
}

}  // namespace vgicp
