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

constexpr int kMaxK = 32;  // largest supported k (the reference's configs use 10)

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

__global__ void cov_scatter_kernel(const CovSeg* __restrict__ segs, const unsigned* __restrict__ cell_of,
                                   const unsigned* __restrict__ start, unsigned* __restrict__ cursor,
                                   unsigned* __restrict__ sorted) {
  const CovSeg s = segs[blockIdx.y];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const unsigned g = s.offset + i;
    const unsigned c = cell_of[g];
    sorted[start[c] + atomicAdd(&cursor[c], 1u)] = g;
  }
}

// Smallest-eigenvalue eigenvector of a symmetric 3×3 (cyclic Jacobi, double), same iteration as
// the host preprocessing (csrc/host/synthetic.cpp).
__device__ void smallest_eigenvector(double A[3][3], double v[3]) {
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 50; ++sweep) {
    const double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    if (off < 1e-30 * (A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2]) + 1e-300) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (A[p][q] == 0.0) continue;
        const double theta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - s * vkq;
          V[k][q] = s * vkp + c * vkq;
        }
      }
  }
  int m = 0;
  if (A[1][1] < A[m][m]) m = 1;
  if (A[2][2] < A[m][m]) m = 2;
  v[0] = V[0][m];
  v[1] = V[1][m];
  v[2] = V[2][m];
}

template <int KM>
__global__ void __launch_bounds__(128) cov_knn_kernel(const CovSeg* __restrict__ segs, const float* __restrict__ xyz,
                                                      const unsigned* __restrict__ start,
                                                      const unsigned* __restrict__ sorted, int k,
                                                      float* __restrict__ cov6) {
  const CovSeg s = segs[blockIdx.y];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const unsigned g = s.offset + i;
    const double q0 = xyz[3 * (size_t)g], q1 = xyz[3 * (size_t)g + 1], q2 = xyz[3 * (size_t)g + 2];
    const int cx = cell_axis(q0, s.lo[0], s.cell, s.gx);
    const int cy = cell_axis(q1, s.lo[1], s.cell, s.gy);
    const int cz = cell_axis(q2, s.lo[2], s.cell, s.gz);
    double bd[KM];
    unsigned bi[KM];
    int nb = 0;
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
            for (unsigned t = start[c]; t < start[c + 1]; ++t) {
              const unsigned j = sorted[t];
              const double d0 = xyz[3 * (size_t)j] - q0, d1 = xyz[3 * (size_t)j + 1] - q1,
                           d2 = xyz[3 * (size_t)j + 2] - q2;
              const double d = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
              const unsigned jl = j - s.offset;
              // insert (d, jl) into the sorted top-k list (lexicographic: distance, then index)
              if (nb == k && !(d < bd[k - 1] || (d == bd[k - 1] && jl < bi[k - 1]))) continue;
              int pos = nb < k ? nb : k - 1;
              while (pos > 0 && (d < bd[pos - 1] || (d == bd[pos - 1] && jl < bi[pos - 1]))) {
                bd[pos] = bd[pos - 1];
                bi[pos] = bi[pos - 1];
                --pos;
              }
              bd[pos] = d;
              bi[pos] = jl;
              if (nb < k) ++nb;
            }
          }
        }
      }
      // every unvisited point lies at least r·cell away from q
      if (nb == k && bd[k - 1] <= (r * s.cell) * (r * s.cell)) break;
    }
    // neighbourhood covariance (point_cloud.cpp:62-71) in neighbour-index order
    double mean[3] = {0, 0, 0};
    for (int a = 0; a < nb; ++a) {
      const size_t j = s.offset + bi[a];
      mean[0] += xyz[3 * j];
      mean[1] += xyz[3 * j + 1];
      mean[2] += xyz[3 * j + 2];
    }
    for (int a = 0; a < 3; ++a) mean[a] /= static_cast<double>(nb);
    double C[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int a = 0; a < nb; ++a) {
      const size_t j = s.offset + bi[a];
      const double d[3] = {xyz[3 * j] - mean[0], xyz[3 * j + 1] - mean[1], xyz[3 * j + 2] - mean[2]};
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) C[r][c] += d[r] * d[c];
    }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) C[r][c] /= static_cast<double>(nb);
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

cudaError_t launch_cov_scatter(const CovSeg* segs, int m, unsigned max_n, const unsigned* cell_of,
                               const unsigned* start, unsigned* cursor, unsigned* sorted, cudaStream_t s) {
  cov_scatter_kernel<<<dim3(grid_for_cov(max_n, 256), m), 256, 0, s>>>(segs, cell_of, start, cursor, sorted);
  return cudaGetLastError();
}

cudaError_t launch_cov_knn(const CovSeg* segs, int m, unsigned max_n, const float* xyz, const unsigned* start,
                           const unsigned* sorted, int k, float* cov6, cudaStream_t s) {
  const dim3 grid(grid_for_cov(max_n, 128), m);
  if (k <= 12)
    cov_knn_kernel<12><<<grid, 128, 0, s>>>(segs, xyz, start, sorted, k, cov6);
  else
    cov_knn_kernel<kMaxK><<<grid, 128, 0, s>>>(segs, xyz, start, sorted, k, cov6);
  return cudaGetLastError();
}

}  // namespace vgicp
