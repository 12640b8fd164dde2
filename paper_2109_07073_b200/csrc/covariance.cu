// Per-point covariance preprocessing on the GPU: estimate_covariances
// (proj/src/point_cloud.cpp:44-83) — the k nearest neighbours of every point (the point itself
// included; ties broken by lower index like oracles.hpp:24-35), their covariance (divided by k),
// eigenvectors kept and the spectrum clamped to (eps, 1, 1): C = I - (1 - eps)·v0·v0ᵀ with v0 the
// eigenvector of the smallest eigenvalue.
//
// Batched over clouds. Exact kNN on a uniform grid: points are counting-sorted into cells, each
// thread scans Chebyshev rings of cells around its point with a sorted top-k list in registers and
// stops once the k-th distance is below the distance to any unvisited cell.
#include <algorithm>

#include "internal.h"

namespace vgicp {

namespace {


__device__ __forceinline__ int cell_axis(double v, double lo, double cell, int g) {
  const int c = static_cast<int>(floor((v - lo) / cell));
  return c < 0 ? 0 : (c >= g ? g - 1 : c);
}

__device__ __forceinline__ unsigned cell_of_point(const CovSeg& s, const float* p) {
  const int cx = cell_axis(p[0], s.lo[0], s.cell, s.gx);
  const int cy = cell_axis(p[1], s.lo[1], s.cell, s.gy);
  const int cz = cell_axis(p[2], s.lo[2], s.cell, s.gz);
  return s.cell_base + static_cast<unsigned>((cx * s.gy + cy) * s.gz + cz);
}

__global__ void cov_count_kernel(const CovSeg* __restrict__ segs, const float* __restrict__ xyz,
                                 unsigned* __restrict__ cell_of, unsigned* __restrict__ cnt) {
  const CovSeg s = segs[blockIdx.y];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const unsigned g = s.offset + i;
    const unsigned c = cell_of_point(s, xyz + 3 * (size_t)g);
    cell_of[g] = c;
    atomicAdd(&cnt[c], 1u);
  }
}

// Cell-ordered copy of the points: (x, y, z, cloud-local index) so that a cell's candidates are one
// contiguous run of 16-B records (the kNN scan reads them sequentially instead of gathering).
__global__ void cov_scatter_kernel(const CovSeg* __restrict__ segs, const float* __restrict__ xyz,
                                   const unsigned* __restrict__ cell_of, const unsigned* __restrict__ start,
                                   unsigned* __restrict__ cursor, float4* __restrict__ sorted) {
  const CovSeg s = segs[blockIdx.y];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const unsigned g = s.offset + i;
    const unsigned c = cell_of[g];
    const float* p = xyz + 3 * (size_t)g;
    sorted[start[c] + atomicAdd(&cursor[c], 1u)] = make_float4(p[0], p[1], p[2], __uint_as_float(i));
  }
}

// Smallest-eigenvalue eigenvector of a symmetric 3×3 (cyclic Jacobi, double), same iteration as
// the host preprocessing (csrc/host/synthetic.cpp); rotations fully unrolled (register arrays).
__device__ __forceinline__ void jacobi_rotate(double (&A)[3][3], double (&V)[3][3], int p, int q) {
  if (A[p][q] == 0.0) return;
  const double theta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
  const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
  const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double akp = A[k][p], akq = A[k][q];
    A[k][p] = c * akp - s * akq;
    A[k][q] = s * akp + c * akq;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double apk = A[p][k], aqk = A[q][k];
    A[p][k] = c * apk - s * aqk;
    A[q][k] = s * apk + c * aqk;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double vkp = V[k][p], vkq = V[k][q];
    V[k][p] = c * vkp - s * vkq;
    V[k][q] = s * vkp + c * vkq;
  }
}

__device__ void smallest_eigenvector(double (&A)[3][3], double v[3]) {
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 50; ++sweep) {
    const double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    if (off < 1e-30 * (A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2]) + 1e-300) break;
    jacobi_rotate(A, V, 0, 1);
    jacobi_rotate(A, V, 0, 2);
    jacobi_rotate(A, V, 1, 2);
  }
  const int m = (A[1][1] < A[0][0]) ? ((A[2][2] < A[1][1]) ? 2 : 1) : ((A[2][2] < A[0][0]) ? 2 : 0);
  v[0] = m == 0 ? V[0][0] : (m == 1 ? V[0][1] : V[0][2]);
  v[1] = m == 0 ? V[1][0] : (m == 1 ? V[1][1] : V[1][2]);
  v[2] = m == 0 ? V[2][0] : (m == 1 ? V[2][1] : V[2][2]);
}

// (d, j) before (bd, bj): ascending distance, ties by lower index (oracles.hpp:24-35)
__device__ __forceinline__ bool knn_before(double d, unsigned j, double bd, unsigned bj) {
  return d < bd || (d == bd && j < bj);
}

// One thread per point; the exact top-K list lives in registers (K is a compile-time constant, the
// insertion is an unrolled shift network).
template <int K>
__global__ void __launch_bounds__(128) cov_knn_kernel(const CovSeg* __restrict__ segs, const float* __restrict__ xyz,
                                                      const unsigned* __restrict__ start,
                                                      const float4* __restrict__ sorted, float* __restrict__ cov6) {
  const CovSeg s = segs[blockIdx.y];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const unsigned g = s.offset + i;
    const double q0 = xyz[3 * (size_t)g], q1 = xyz[3 * (size_t)g + 1], q2 = xyz[3 * (size_t)g + 2];
    const int cx = cell_axis(q0, s.lo[0], s.cell, s.gx);
    const int cy = cell_axis(q1, s.lo[1], s.cell, s.gy);
    const int cz = cell_axis(q2, s.lo[2], s.cell, s.gz);
    double bd[K];
    unsigned bi[K];
#pragma unroll
    for (int a = 0; a < K; ++a) bd[a] = INFINITY, bi[a] = 0xFFFFFFFFu;
    const int rmax = max(s.gx, max(s.gy, s.gz));
    for (int r = 0; r <= rmax; ++r) {
      for (int dx = -r; dx <= r; ++dx) {
        const int x = cx + dx;
        if (x < 0 || x >= s.gx) continue;
        for (int dy = -r; dy <= r; ++dy) {
          const int y = cy + dy;
          if (y < 0 || y >= s.gy) continue;
          const bool edge_xy = (dx == -r || dx == r || dy == -r || dy == r);
          for (int dz = -r; dz <= r; dz += (edge_xy ? 1 : 2 * r > 0 ? 2 * r : 1)) {
            const int z = cz + dz;
            if (z < 0 || z >= s.gz) continue;
            const unsigned c = s.cell_base + static_cast<unsigned>((x * s.gy + y) * s.gz + z);
            const unsigned t1 = start[c + 1];
            for (unsigned t = start[c]; t < t1; ++t) {
              const float4 P = __ldg(sorted + t);
              const double d0 = P.x - q0, d1 = P.y - q1, d2 = P.z - q2;
              const double d = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
              const unsigned jl = __float_as_uint(P.w);
              if (!knn_before(d, jl, bd[K - 1], bi[K - 1])) continue;
#pragma unroll
              for (int a = K - 1; a > 0; --a) {
                const bool shift = knn_before(d, jl, bd[a - 1], bi[a - 1]);
                const bool here = !shift && knn_before(d, jl, bd[a], bi[a]);
                bd[a] = shift ? bd[a - 1] : (here ? d : bd[a]);
                bi[a] = shift ? bi[a - 1] : (here ? jl : bi[a]);
              }
              if (knn_before(d, jl, bd[0], bi[0])) bd[0] = d, bi[0] = jl;
            }
          }
        }
      }
      // every unvisited point lies at least r·cell away from q
      if (bd[K - 1] <= (r * s.cell) * (r * s.cell)) break;
    }
    // neighbourhood covariance (point_cloud.cpp:62-71) in neighbour order
    double P[K][3];
    double mean[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const size_t j = s.offset + bi[a];
      P[a][0] = xyz[3 * j], P[a][1] = xyz[3 * j + 1], P[a][2] = xyz[3 * j + 2];
      mean[0] += P[a][0];
      mean[1] += P[a][1];
      mean[2] += P[a][2];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) mean[a] /= static_cast<double>(K);
    double C[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const double d[3] = {P[a][0] - mean[0], P[a][1] - mean[1], P[a][2] - mean[2]};
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) C[r][c] += d[r] * d[c];
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) C[r][c] /= static_cast<double>(K);
    double v[3];
    smallest_eigenvector(C, v);
    const double w = 1.0 - s.eps;
    float* o = cov6 + 6 * (size_t)g;
    o[0] = static_cast<float>(1.0 - w * v[0] * v[0]);
    o[1] = static_cast<float>(-w * v[0] * v[1]);
    o[2] = static_cast<float>(-w * v[0] * v[2]);
    o[3] = static_cast<float>(1.0 - w * v[1] * v[1]);
    o[4] = static_cast<float>(-w * v[1] * v[2]);
    o[5] = static_cast<float>(1.0 - w * v[2] * v[2]);
  }
}

__device__ __forceinline__ unsigned ord_f(float f) {  // monotone float -> uint
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Per-cloud bounding box (ordered-uint atomics) and a non-finite flag, for the grid parameters.
__global__ void cov_bbox_kernel(const CovSeg* __restrict__ segs, const float* __restrict__ xyz,
                                unsigned* __restrict__ box, int* __restrict__ bad) {
  const CovSeg s = segs[blockIdx.y];
  unsigned lo[3] = {~0u, ~0u, ~0u}, hi[3] = {0u, 0u, 0u};
  int nonfinite = 0;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const float* p = xyz + 3 * (size_t)(s.offset + i);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = p[a];
      if (!isfinite(v)) nonfinite = 1;
      lo[a] = min(lo[a], ord_f(v));
      hi[a] = max(hi[a], ord_f(v));
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  }
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(&box[6 * blockIdx.y + a], lo[a]);
      atomicMax(&box[6 * blockIdx.y + 3 + a], hi[a]);
    }
    if (nonfinite) atomicOr(&bad[blockIdx.y], 1);
  }
}

unsigned grid_for_cov(unsigned n, unsigned threads) {
  unsigned g = (n + threads - 1) / threads;
  if (g == 0) g = 1;
  return g < 4096 ? g : 4096;
}

}  // namespace

cudaError_t launch_cov_bbox(const CovSeg* segs, int m, unsigned max_n, const float* xyz, unsigned* box, int* bad,
                            cudaStream_t s) {
  cov_bbox_kernel<<<dim3(std::min(grid_for_cov(max_n, 256), 64u), m), 256, 0, s>>>(segs, xyz, box, bad);
  return cudaGetLastError();
}

cudaError_t launch_cov_count(const CovSeg* segs, int m, unsigned max_n, const float* xyz, unsigned* cell_of,
                             unsigned* cnt, cudaStream_t s) {
  cov_count_kernel<<<dim3(grid_for_cov(max_n, 256), m), 256, 0, s>>>(segs, xyz, cell_of, cnt);
  return cudaGetLastError();
}

cudaError_t launch_cov_scatter(const CovSeg* segs, int m, unsigned max_n, const float* xyz, const unsigned* cell_of,
                               const unsigned* start, unsigned* cursor, float4* sorted, cudaStream_t s) {
  cov_scatter_kernel<<<dim3(grid_for_cov(max_n, 256), m), 256, 0, s>>>(segs, xyz, cell_of, start, cursor, sorted);
  return cudaGetLastError();
}

cudaError_t launch_cov_knn(const CovSeg* segs, int m, unsigned max_n, const float* xyz, const unsigned* start,
                           const float4* sorted, int k, float* cov6, cudaStream_t s) {
  const dim3 grid(grid_for_cov(max_n, 128), m);
  switch (k) {
#define VG_KNN_CASE(K) \
  case K:              \
    cov_knn_kernel<K><<<grid, 128, 0, s>>>(segs, xyz, start, sorted, cov6); \
    break;
    VG_KNN_CASE(4) VG_KNN_CASE(5) VG_KNN_CASE(6) VG_KNN_CASE(7) VG_KNN_CASE(8) VG_KNN_CASE(9) VG_KNN_CASE(10)
    VG_KNN_CASE(11) VG_KNN_CASE(12) VG_KNN_CASE(13) VG_KNN_CASE(14) VG_KNN_CASE(15) VG_KNN_CASE(16)
    VG_KNN_CASE(17) VG_KNN_CASE(18) VG_KNN_CASE(19) VG_KNN_CASE(20) VG_KNN_CASE(21) VG_KNN_CASE(22)
    VG_KNN_CASE(23) VG_KNN_CASE(24) VG_KNN_CASE(25) VG_KNN_CASE(26) VG_KNN_CASE(27) VG_KNN_CASE(28)
    VG_KNN_CASE(29) VG_KNN_CASE(30) VG_KNN_CASE(31) VG_KNN_CASE(32)
#undef VG_KNN_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace vgicp
