// fp64 routines that reproduce the oracle bit for bit: every operation uses an explicit
// round-to-nearest intrinsic, so nvcc cannot contract it into an FMA. Used by the rare
// near-singular path of the factor kernels and by gicp_error.
#pragma once

#include "vgicp_device.cuh"

namespace vgicp {

// Row-major 3×3 product (each entry a dot3 in the stated order).
__device__ __forceinline__ void mul33_rn(const double* A, const double* B, double* C) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) C[3 * i + j] = dot3_rn(A[3 * i], A[3 * i + 1], A[3 * i + 2], B[j], B[3 + j], B[6 + j]);
}

// M = C_t + (R·C_s)·Rᵀ  (factors.cpp:107, the nested product evaluated first).
__device__ __forceinline__ void combined_cov_rn(const double* R, const double* Cs, const double* Ct, double* M) {
  double RC[9];
  mul33_rn(R, Cs, RC);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      M[3 * i + j] = __dadd_rn(Ct[3 * i + j], dot3_rn(RC[3 * i], RC[3 * i + 1], RC[3 * i + 2], R[3 * j], R[3 * j + 1], R[3 * j + 2]));
}

__device__ __forceinline__ void dswap(double& a, double& b) {
  const double t = a;
  a = b;
  b = t;
}

// invert_covariance (factors.cpp:38-46): Eigen-style LDLT with diagonal pivoting on the lower
// triangle; rejects on failure or any pivot <= 0; Omega = solve(I), symmetrised.
// Same operation sequence as the CPU checker's LDLT restatement.
static __device__ __noinline__ bool invert_covariance_rn(const double* M, double* out) {
  double a[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) a[i][j] = M[3 * i + j];
  int tr[3];
  bool found_zero_pivot = false;
  bool ret = true;
  double temp[3];
  for (int k = 0; k < 3; ++k) {
    int biggest = k;
    double best = fabs(a[k][k]);
    for (int i = k + 1; i < 3; ++i) {
      if (fabs(a[i][i]) > best) {
        best = fabs(a[i][i]);
        biggest = i;
      }
    }
    tr[k] = biggest;
    if (k != biggest) {
      for (int j = 0; j < k; ++j) dswap(a[k][j], a[biggest][j]);
      for (int i = biggest + 1; i < 3; ++i) dswap(a[i][k], a[i][biggest]);
      dswap(a[k][k], a[biggest][biggest]);
      for (int i = k + 1; i < biggest; ++i) {
        const double tmp = a[i][k];
        a[i][k] = a[biggest][i];
        a[biggest][i] = tmp;
      }
    }
    const int rs = 2 - k;
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = __dmul_rn(a[j][j], a[k][j]);
      double s = __dmul_rn(a[k][0], temp[0]);
      if (k == 2) s = __dadd_rn(s, __dmul_rn(a[k][1], temp[1]));
      a[k][k] = __dsub_rn(a[k][k], s);
      for (int i = k + 1; i < 3; ++i) {
        double si = __dmul_rn(a[i][0], temp[0]);
        if (k == 2) si = __dadd_rn(si, __dmul_rn(a[i][1], temp[1]));
        a[i][k] = __dsub_rn(a[i][k], si);
      }
    }
    const double akk = a[k][k];
    const bool pivot_is_valid = fabs(akk) > 0.0;
    if (k == 0 && !pivot_is_valid) return false;  // zero pivot => D <= 0 => rejected
    if (rs > 0 && pivot_is_valid) {
      for (int i = k + 1; i < 3; ++i) a[i][k] = __ddiv_rn(a[i][k], akk);
    } else if (rs > 0) {
      for (int i = k + 1; i < 3; ++i) ret = ret && (a[i][k] == 0.0);
    }
    if (found_zero_pivot && pivot_is_valid) {
      ret = false;
    } else if (!pivot_is_valid) {
      found_zero_pivot = true;
    }
  }
  if (!ret) return false;
  if (a[0][0] <= 0.0 || a[1][1] <= 0.0 || a[2][2] <= 0.0) return false;  // (vectorD() <= 0).any()
  double X[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int k = 0; k < 3; ++k) {
    const int t = tr[k];
    if (t != k)
      for (int j = 0; j < 3; ++j) dswap(X[k][j], X[t][j]);
  }
  for (int j = 0; j < 3; ++j) {
    X[1][j] = __dsub_rn(X[1][j], __dmul_rn(a[1][0], X[0][j]));
    X[2][j] = __dsub_rn(X[2][j], __dadd_rn(__dmul_rn(a[2][0], X[0][j]), __dmul_rn(a[2][1], X[1][j])));
  }
  for (int i = 0; i < 3; ++i) {
    const double d = a[i][i];
    for (int j = 0; j < 3; ++j) X[i][j] = fabs(d) > 2.2250738585072014e-308 ? __ddiv_rn(X[i][j], d) : 0.0;
  }
  for (int j = 0; j < 3; ++j) {
    X[1][j] = __dsub_rn(X[1][j], __dmul_rn(a[2][1], X[2][j]));
    X[0][j] = __dsub_rn(X[0][j], __dadd_rn(__dmul_rn(a[1][0], X[1][j]), __dmul_rn(a[2][0], X[2][j])));
  }
  for (int k = 2; k >= 0; --k) {
    const int t = tr[k];
    if (t != k)
      for (int j = 0; j < 3; ++j) dswap(X[k][j], X[t][j]);
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) out[3 * i + j] = __dmul_rn(0.5, __dadd_rn(X[i][j], X[j][i]));
  return true;
}

}  // namespace vgicp
