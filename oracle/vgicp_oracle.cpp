// TEST INFRASTRUCTURE ONLY — CPU oracle for the VGICP matching-cost hot path.
//
// A plain-C++20 (Eigen-free) restatement of the reference's CPU implementation, used by tests/
// as the parity checker and by bench.py as the timed CPU baseline (cpu_baseline.kind = "port").
// It is never linked into, imported by, or called from the product path
// (paper_2109_07073_b200/), which fails loudly when its CUDA library is missing.
//
// Every function cites the reference file:line it restates (paths relative to
// /root/reference/proj). Build: oracle/Makefile, the reference's Release flags
// (-O3 -DNDEBUG -fopenmp -std=c++20, no -march, so no FMA contraction can occur on x86-64),
// plus -ffp-contract=off to make the no-FMA rule explicit.
//
// Arithmetic-order contract: every fixed-size 3-term inner product is
// evaluated as (a0*b0 + a1*b1) + a2*b2, one rounding per operation. Eigen's own order for
// 3-term reductions depends on its version and vectorisation flags and cannot be pinned here
// (Eigen is absent); the GPU path follows the same stated order, so voxel keys, hit sets and
// inlier counts are bit-identical between this oracle and the GPU by construction, and would
// differ from a given Eigen build only for points within one ulp of a voxel face.
//
// Parity pinning: no golden vectors exist in the reference; this restatement is pinned against
// every KAT / brute-force oracle of the reference's hot-path tests (tests/test_oracle_kats.py).

#include "vgicp_oracle.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <exception>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

thread_local std::string g_last_error;

// ------------------------------------------------------------------------------------------
// Small fixed-size linear algebra (replaces Eigen::Vector3d / Matrix3d / Matrix6d).
// ------------------------------------------------------------------------------------------
struct V3 {
  double v[3] = {0, 0, 0};
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};
struct M3 {
  double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  static M3 identity() {
    M3 r;
    r.m[0][0] = r.m[1][1] = r.m[2][2] = 1.0;
    return r;
  }
};
struct M6 {
  double m[6][6] = {};
};
struct V6 {
  double v[6] = {};
};

inline double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
  return (a0 * b0 + a1 * b1) + a2 * b2;
}
inline double dot(const V3& a, const V3& b) { return dot3(a[0], a[1], a[2], b[0], b[1], b[2]); }

inline V3 mul(const M3& A, const V3& x) {
  V3 r;
  for (int i = 0; i < 3; ++i) r[i] = dot3(A.m[i][0], A.m[i][1], A.m[i][2], x[0], x[1], x[2]);
  return r;
}
inline M3 mul(const M3& A, const M3& B) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = dot3(A.m[i][0], A.m[i][1], A.m[i][2], B.m[0][j], B.m[1][j], B.m[2][j]);
  return r;
}
inline M3 transpose(const M3& A) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = A.m[j][i];
  return r;
}
inline M3 add(const M3& A, const M3& B) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = A.m[i][j] + B.m[i][j];
  return r;
}
inline V3 add(const V3& a, const V3& b) { return V3{{a[0] + b[0], a[1] + b[1], a[2] + b[2]}}; }
inline V3 sub(const V3& a, const V3& b) { return V3{{a[0] - b[0], a[1] - b[1], a[2] - b[2]}}; }
inline M3 scale(double s, const M3& A) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = s * A.m[i][j];
  return r;
}

// se3.cpp:34-40
inline M3 skew(const V3& v) {
  M3 m;
  m.m[0][0] = 0.0;
  m.m[0][1] = -v[2];
  m.m[0][2] = v[1];
  m.m[1][0] = v[2];
  m.m[1][1] = 0.0;
  m.m[1][2] = -v[0];
  m.m[2][0] = -v[1];
  m.m[2][1] = v[0];
  m.m[2][2] = 0.0;
  return m;
}

// ------------------------------------------------------------------------------------------
// Pose (se3.hpp:33-56, se3.cpp:42-44)
// ------------------------------------------------------------------------------------------
struct Pose {
  M3 R = M3::identity();
  V3 t;
  int updates = 0;
  V3 apply(const V3& p) const { return add(mul(R, p), t); }  // se3.hpp:43
  Pose inverse() const {                                      // se3.hpp:45
    Pose r;
    r.R = transpose(R);
    const V3 rt = mul(r.R, t);
    r.t = V3{{-rt[0], -rt[1], -rt[2]}};
    return r;
  }
};
inline Pose compose(const Pose& a, const Pose& b) {  // se3.cpp:42-44
  Pose r;
  r.R = mul(a.R, b.R);
  r.t = add(mul(a.R, b.t), a.t);
  return r;
}
Pose pose_from(const double p[12]) {
  Pose r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.R.m[i][j] = p[3 * i + j];
  for (int i = 0; i < 3; ++i) r.t[i] = p[9 + i];
  return r;
}
void pose_to(const Pose& P, double p[12]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) p[3 * i + j] = P.R.m[i][j];
  for (int i = 0; i < 3; ++i) p[9 + i] = P.t[i];
}

constexpr double kSmallAngle = 1e-8;  // se3.cpp:10

inline double norm3(const V3& v) { return std::sqrt(dot(v, v)); }

// se3.cpp:14-24
M3 so3_left_jacobian(const V3& omega) {
  const double theta = norm3(omega);
  const M3 W = skew(omega);
  const M3 WW = mul(W, W);
  M3 r;
  if (theta < kSmallAngle) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = ((i == j ? 1.0 : 0.0) + 0.5 * W.m[i][j]) + WW.m[i][j] / 6.0;
    return r;
  }
  const double t2 = theta * theta;
  const double a = (1.0 - std::cos(theta)) / t2;
  const double b = (theta - std::sin(theta)) / (t2 * theta);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = ((i == j ? 1.0 : 0.0) + a * W.m[i][j]) + b * WW.m[i][j];
  return r;
}

// se3.cpp:46-55
M3 so3_exp(const V3& omega) {
  const double theta = norm3(omega);
  const M3 W = skew(omega);
  const M3 WW = mul(W, W);
  M3 r;
  if (theta < kSmallAngle) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = ((i == j ? 1.0 : 0.0) + W.m[i][j]) + 0.5 * WW.m[i][j];
    return r;
  }
  const double t2 = theta * theta;
  const double s = std::sin(theta) / theta;
  const double c = (1.0 - std::cos(theta)) / t2;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = ((i == j ? 1.0 : 0.0) + s * W.m[i][j]) + c * WW.m[i][j];
  return r;
}

// se3.cpp:74-78
Pose se3_exp(const V3& rot, const V3& trans) {
  Pose p;
  p.R = so3_exp(rot);
  p.t = mul(so3_left_jacobian(rot), trans);
  return p;
}

// se3.cpp:107-113
M6 adjoint(const Pose& T) {
  M6 ad;
  const M3 tR = mul(skew(T.t), T.R);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      ad.m[i][j] = T.R.m[i][j];
      ad.m[3 + i][3 + j] = T.R.m[i][j];
      ad.m[3 + i][j] = tR.m[i][j];
    }
  return ad;
}

// ------------------------------------------------------------------------------------------
// Execution contract (parallel.hpp:17-95)
// ------------------------------------------------------------------------------------------
struct ExecPolicy {
  int threads = 0;
  bool deterministic = false;
  int resolved_threads() const { return threads > 0 ? threads : omp_get_max_threads(); }
};

template <typename F>
void parallel_for(std::size_t n, const ExecPolicy& policy, F&& body) {  // parallel.hpp:24-40
  const int nt = policy.resolved_threads();
  std::exception_ptr failure;
#pragma omp parallel for schedule(static) num_threads(nt) shared(failure)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
    try {
      body(static_cast<std::size_t>(i));
    } catch (...) {
#pragma omp critical(oracle_parallel_for_failure)
      if (!failure) failure = std::current_exception();
    }
  }
  if (failure) std::rethrow_exception(failure);
}

template <typename Partial, typename MakeBlock, typename Combine>
Partial parallel_reduce(std::size_t n, const Partial& zero, const ExecPolicy& policy, MakeBlock&& make_block,
                        Combine&& combine) {  // parallel.hpp:48-95
  constexpr std::size_t kBlock = 1024;
  if (n == 0) return zero;
  if (!policy.deterministic) {
    const int nt = policy.resolved_threads();
    std::vector<Partial> per_thread(nt, zero);
#pragma omp parallel num_threads(nt)
    {
      const int tid = omp_get_thread_num();
      Partial local = zero;
#pragma omp for schedule(static) nowait
      for (std::int64_t b = 0; b < static_cast<std::int64_t>((n + kBlock - 1) / kBlock); ++b) {
        const std::size_t begin = static_cast<std::size_t>(b) * kBlock;
        const std::size_t end = begin + kBlock < n ? begin + kBlock : n;
        local = combine(local, make_block(begin, end));
      }
      per_thread[tid] = local;
    }
    Partial total = zero;
    for (const Partial& p : per_thread) total = combine(total, p);
    return total;
  }
  const std::size_t num_blocks = (n + kBlock - 1) / kBlock;
  std::vector<Partial> partials(num_blocks, zero);
  parallel_for(num_blocks, policy, [&](std::size_t b) {
    const std::size_t begin = b * kBlock;
    const std::size_t end = begin + kBlock < n ? begin + kBlock : n;
    partials[b] = make_block(begin, end);
  });
  for (std::size_t stride = 1; stride < num_blocks; stride *= 2) {
    const std::size_t pairs = (num_blocks + 2 * stride - 1) / (2 * stride);
    parallel_for(pairs, policy, [&](std::size_t p) {
      const std::size_t left = 2 * stride * p;
      const std::size_t right = left + stride;
      if (right < num_blocks) partials[left] = combine(partials[left], partials[right]);
    });
  }
  return partials[0];
}

// parallel.hpp:97-114, applied component-wise.
template <int N>
struct KahanSum {
  double sum[N] = {};
  double compensation[N] = {};
  void add(const double* value) {
    for (int i = 0; i < N; ++i) {
      const double y = value[i] - compensation[i];
      const double t = sum[i] + y;
      compensation[i] = (t - sum[i]) - y;
      sum[i] = t;
    }
  }
};

// ------------------------------------------------------------------------------------------
// Gaussian voxel map (voxelmap.cpp:12-135)
// ------------------------------------------------------------------------------------------
constexpr int kKeyBits = 21;                 // voxelmap.cpp:12
constexpr std::int64_t kKeyBias = 1 << 20;   // voxelmap.cpp:13
constexpr int kShards = 64;                  // voxelmap.cpp:14

std::uint64_t mix(std::uint64_t x) {  // voxelmap.cpp:16-21
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct Voxel {  // voxelmap.hpp:18-22
  V3 mean;
  M3 cov;
  int count = 0;
};

struct VoxelAccumulator {  // voxelmap.cpp:23-41
  KahanSum<3> mean_sum;
  KahanSum<9> second_moment_sum;
  int count = 0;
  void add(const V3& mean, const M3& cov) {
    mean_sum.add(mean.v);
    double sm[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) sm[3 * i + j] = cov.m[i][j] + mean[i] * mean[j];
    second_moment_sum.add(sm);
    ++count;
  }
  Voxel finalize() const {
    Voxel v;
    v.count = count;
    const double c = static_cast<double>(count);
    for (int i = 0; i < 3; ++i) v.mean[i] = mean_sum.sum[i] / c;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) v.cov.m[i][j] = second_moment_sum.sum[3 * i + j] / c - v.mean[i] * v.mean[j];
    return v;
  }
};

std::uint64_t pack_key(const int coord[3]) {  // voxelmap.cpp:57-63
  std::uint64_t key = 0;
  for (int a = 0; a < 3; ++a) key = (key << kKeyBits) | static_cast<std::uint64_t>(coord[a] + kKeyBias);
  return key;
}

void voxel_coord(double resolution, const V3& p, int coord[3]) {  // voxelmap.cpp:45-55
  for (int a = 0; a < 3; ++a) {
    const double c = std::floor(p[a] / resolution);
    if (!(c >= -static_cast<double>(kKeyBias) && c < static_cast<double>(kKeyBias))) {
      throw std::out_of_range("point beyond the +-2^20 voxel-per-axis range limit");
    }
    coord[a] = static_cast<int>(c);
  }
}

struct VoxelMap {
  double resolution = 1.0;
  std::size_t total_points = 0;
  std::unordered_map<std::uint64_t, Voxel> voxels;

  const Voxel* lookup(const V3& point) const {  // voxelmap.cpp:106-117
    int coord[3];
    for (int a = 0; a < 3; ++a) {
      const double c = std::floor(point[a] / resolution);
      if (!(c >= -static_cast<double>(kKeyBias) && c < static_cast<double>(kKeyBias))) return nullptr;
      coord[a] = static_cast<int>(c);
    }
    const auto it = voxels.find(pack_key(coord));
    return it == voxels.end() ? nullptr : &it->second;
  }
};

V3 v3_at(const double* a, std::size_t i) { return V3{{a[3 * i], a[3 * i + 1], a[3 * i + 2]}}; }
M3 m3_at(const double* a, std::size_t i) {
  M3 r;
  for (int k = 0; k < 9; ++k) r.m[k / 3][k % 3] = a[9 * i + k];
  return r;
}

// GaussianVoxelMap::GaussianVoxelMap (voxelmap.cpp:65-104)
void build_parallel(const double* means, const double* covs, std::size_t n, double resolution,
                    const ExecPolicy& policy, VoxelMap& map) {
  if (resolution <= 0.0) throw std::invalid_argument("voxel resolution must be positive");
  if (n == 0 || covs == nullptr) {
    throw std::invalid_argument("voxel map construction requires per-point covariances");
  }
  map.resolution = resolution;
  map.total_points = n;
  std::vector<std::uint64_t> keys(n);
  parallel_for(n, policy, [&](std::size_t i) {
    int c[3];
    voxel_coord(resolution, v3_at(means, i), c);
    keys[i] = pack_key(c);
  });
  std::array<std::vector<std::uint32_t>, kShards> shards;
  for (auto& s : shards) s.reserve(n / kShards + 1);
  for (std::size_t i = 0; i < n; ++i) shards[mix(keys[i]) & (kShards - 1)].push_back(static_cast<std::uint32_t>(i));
  std::array<std::unordered_map<std::uint64_t, VoxelAccumulator>, kShards> partials;
  parallel_for(kShards, policy, [&](std::size_t s) {
    auto& local = partials[s];
    local.reserve(shards[s].size());
    for (const std::uint32_t i : shards[s]) local[keys[i]].add(v3_at(means, i), m3_at(covs, i));
  });
  std::size_t total = 0;
  for (const auto& p : partials) total += p.size();
  map.voxels.reserve(total);
  for (const auto& p : partials)
    for (const auto& [key, acc] : p) map.voxels.emplace(key, acc.finalize());
}

// reference::build_voxelmap (reference.cpp:39-65)
void build_serial(const double* means, const double* covs, std::size_t n, double resolution, VoxelMap& map) {
  struct Accum {
    V3 mean_sum;
    M3 moment_sum;
    int count = 0;
  };
  std::unordered_map<std::uint64_t, Accum> accums;
  for (std::size_t i = 0; i < n; ++i) {
    const V3 p = v3_at(means, i);
    int coord[3];
    for (int a = 0; a < 3; ++a) coord[a] = static_cast<int>(std::floor(p[a] / resolution));
    Accum& acc = accums[pack_key(coord)];
    const M3 C = m3_at(covs, i);
    acc.mean_sum = add(acc.mean_sum, p);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) acc.moment_sum.m[r][c] = acc.moment_sum.m[r][c] + (C.m[r][c] + p[r] * p[c]);
    acc.count += 1;
  }
  map.resolution = resolution;
  map.total_points = n;
  map.voxels.reserve(accums.size());
  for (const auto& [key, acc] : accums) {
    Voxel v;
    v.count = acc.count;
    const double c = static_cast<double>(acc.count);
    for (int i = 0; i < 3; ++i) v.mean[i] = acc.mean_sum[i] / c;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) v.cov.m[i][j] = acc.moment_sum.m[i][j] / c - v.mean[i] * v.mean[j];
    map.voxels.emplace(key, v);
  }
}

// ------------------------------------------------------------------------------------------
// 3×3 LDLT with diagonal pivoting (Eigen::LDLT<Matrix3d>, lower storage), the decision and
// solve used by invert_covariance (factors.cpp:38-46).
// ------------------------------------------------------------------------------------------
struct Ldlt3 {
  double a[3][3];  // lower triangle holds L (unit diag implied) and D on the diagonal
  int transpositions[3];
  bool ok = true;
};

Ldlt3 ldlt_factor(const M3& M) {
  Ldlt3 f;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) f.a[i][j] = M.m[i][j];
  const int size = 3;
  bool found_zero_pivot = false;
  bool ret = true;
  double temp[3];
  for (int k = 0; k < size; ++k) {
    // largest |diagonal| in the trailing corner (first index on ties)
    int biggest = k;
    double best = std::abs(f.a[k][k]);
    for (int i = k + 1; i < size; ++i) {
      if (std::abs(f.a[i][i]) > best) {
        best = std::abs(f.a[i][i]);
        biggest = i;
      }
    }
    f.transpositions[k] = biggest;
    if (k != biggest) {
      // swap row k / row biggest in the leading k columns
      for (int j = 0; j < k; ++j) std::swap(f.a[k][j], f.a[biggest][j]);
      // swap column k / column biggest below row biggest
      for (int i = biggest + 1; i < size; ++i) std::swap(f.a[i][k], f.a[i][biggest]);
      std::swap(f.a[k][k], f.a[biggest][biggest]);
      for (int i = k + 1; i < biggest; ++i) {
        const double tmp = f.a[i][k];
        f.a[i][k] = f.a[biggest][i];
        f.a[biggest][i] = tmp;
      }
    }
    const int rs = size - k - 1;
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = f.a[j][j] * f.a[k][j];
      double s = 0.0;
      for (int j = 0; j < k; ++j) s = (j == 0) ? f.a[k][0] * temp[0] : s + f.a[k][j] * temp[j];
      f.a[k][k] -= s;
      for (int i = k + 1; i < size; ++i) {
        double si = 0.0;
        for (int j = 0; j < k; ++j) si = (j == 0) ? f.a[i][0] * temp[0] : si + f.a[i][j] * temp[j];
        f.a[i][k] -= si;
      }
    }
    const double realAkk = f.a[k][k];
    const bool pivot_is_valid = std::abs(realAkk) > 0.0;
    if (k == 0 && !pivot_is_valid) {
      for (int j = 0; j < size; ++j) {
        f.transpositions[j] = j;
        for (int i = j + 1; i < size; ++i) ret = ret && (f.a[i][j] == 0.0);
      }
      f.ok = ret;
      return f;
    }
    if (rs > 0 && pivot_is_valid) {
      for (int i = k + 1; i < size; ++i) f.a[i][k] /= realAkk;
    } else if (rs > 0) {
      for (int i = k + 1; i < size; ++i) ret = ret && (f.a[i][k] == 0.0);
    }
    if (found_zero_pivot && pivot_is_valid) {
      ret = false;
    } else if (!pivot_is_valid) {
      found_zero_pivot = true;
    }
  }
  f.ok = ret;
  return f;
}

// factors.cpp:38-46: LDLT, reject on failure or any D <= 0, solve(I), symmetrize.
bool invert_covariance(const M3& M, M3& out) {
  const Ldlt3 f = ldlt_factor(M);
  if (!f.ok) return false;
  for (int i = 0; i < 3; ++i)
    if (f.a[i][i] <= 0.0) return false;
  // X = P I
  double X[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int k = 0; k < 3; ++k) {
    const int t = f.transpositions[k];
    if (t != k)
      for (int j = 0; j < 3; ++j) std::swap(X[k][j], X[t][j]);
  }
  // L (unit lower) forward substitution, column by column
  for (int j = 0; j < 3; ++j) {
    X[1][j] -= f.a[1][0] * X[0][j];
    X[2][j] -= f.a[2][0] * X[0][j] + f.a[2][1] * X[1][j];
  }
  // D^-1 (zero rows for |d| <= DBL_MIN)
  for (int i = 0; i < 3; ++i) {
    const double d = f.a[i][i];
    for (int j = 0; j < 3; ++j) X[i][j] = std::abs(d) > std::numeric_limits<double>::min() ? X[i][j] / d : 0.0;
  }
  // L^T back substitution
  for (int j = 0; j < 3; ++j) {
    X[1][j] -= f.a[2][1] * X[2][j];
    X[0][j] -= f.a[1][0] * X[1][j] + f.a[2][0] * X[2][j];
  }
  // P^T (transpositions in reverse order)
  for (int k = 2; k >= 0; --k) {
    const int t = f.transpositions[k];
    if (t != k)
      for (int j = 0; j < 3; ++j) std::swap(X[k][j], X[t][j]);
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) out.m[i][j] = 0.5 * (X[i][j] + X[j][i]);
  return true;
}

// Matrix3d::inverse() (cofactor form), used by the serial reference (reference.cpp:90-91) and
// by frozen_cost (test_factors.cpp:80-82).
M3 inverse_cofactor(const M3& A) {
  auto cof = [&](int i, int j) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
    return A.m[i1][j1] * A.m[i2][j2] - A.m[i1][j2] * A.m[i2][j1];
  };
  const double c00 = cof(0, 0), c10 = cof(1, 0), c20 = cof(2, 0);
  const double det = dot3(c00, c10, c20, A.m[0][0], A.m[1][0], A.m[2][0]);
  const double invdet = 1.0 / det;
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = cof(j, i) * invdet;
  return r;
}

// R * C * R^T with the inner product evaluated first (Eigen evaluates the nested product).
M3 rotate_cov(const M3& R, const M3& C) { return mul(mul(R, C), transpose(R)); }

// ------------------------------------------------------------------------------------------
// Matching cost factor (factors.cpp:14-181)
// ------------------------------------------------------------------------------------------
struct FactorAccumulator {  // factors.cpp:14-34
  M6 H_tt, H_ts, H_ss;
  V6 b_t, b_s;
  double error = 0.0;
  int inliers = 0;
  FactorAccumulator combine(const FactorAccumulator& o) const {
    FactorAccumulator r;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) {
        r.H_tt.m[i][j] = H_tt.m[i][j] + o.H_tt.m[i][j];
        r.H_ts.m[i][j] = H_ts.m[i][j] + o.H_ts.m[i][j];
        r.H_ss.m[i][j] = H_ss.m[i][j] + o.H_ss.m[i][j];
      }
    for (int i = 0; i < 6; ++i) {
      r.b_t.v[i] = b_t.v[i] + o.b_t.v[i];
      r.b_s.v[i] = b_s.v[i] + o.b_s.v[i];
    }
    r.error = error + o.error;
    r.inliers = inliers + o.inliers;
    return r;
  }
};

// Jacobian blocks as 3×6 (factors.cpp:115-120)
struct J36 {
  double m[3][6];
};

// acc += Jl^T * (Omega * Jr)  (6×6 lazy product, 3-term inner dimension)
void accum_JtOJ(M6& acc, const J36& Jl, const J36& OJr) {
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j)
      acc.m[i][j] += dot3(Jl.m[0][i], Jl.m[1][i], Jl.m[2][i], OJr.m[0][j], OJr.m[1][j], OJr.m[2][j]);
}
J36 mul_OJ(const M3& O, const J36& J) {
  J36 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 6; ++j) r.m[i][j] = dot3(O.m[i][0], O.m[i][1], O.m[i][2], J.m[0][j], J.m[1][j], J.m[2][j]);
  return r;
}

struct SourceView {
  const double* means;
  const double* covs;
  std::size_t n;
};

// Per-point body shared by the parallel linearization (factors.cpp:101-131).
inline void linearize_point(const SourceView& src, std::size_t k, const VoxelMap& targets, const Pose& T_ts,
                            FactorAccumulator& acc) {
  const M3& R = T_ts.R;
  const V3 mu = v3_at(src.means, k);
  const V3 transformed = T_ts.apply(mu);
  const Voxel* voxel = targets.lookup(transformed);
  if (voxel == nullptr) return;
  const V3 e = sub(voxel->mean, transformed);
  M3 omega;
  if (!invert_covariance(add(voxel->cov, rotate_cov(R, m3_at(src.covs, k))), omega)) return;
  J36 A, B;
  const M3 sq = skew(transformed);
  const M3 Rs = mul(R, skew(mu));
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      A.m[i][j] = -sq.m[i][j];
      A.m[i][3 + j] = (i == j) ? 1.0 : 0.0;
      B.m[i][j] = Rs.m[i][j];
      B.m[i][3 + j] = -R.m[i][j];
    }
  const J36 omega_A = mul_OJ(omega, A);
  const J36 omega_B = mul_OJ(omega, B);
  accum_JtOJ(acc.H_tt, A, omega_A);
  accum_JtOJ(acc.H_ts, A, omega_B);
  accum_JtOJ(acc.H_ss, B, omega_B);
  const V3 oe = mul(omega, e);
  for (int i = 0; i < 6; ++i) {
    acc.b_t.v[i] -= dot3(A.m[0][i], A.m[1][i], A.m[2][i], oe[0], oe[1], oe[2]);
    acc.b_s.v[i] -= dot3(B.m[0][i], B.m[1][i], B.m[2][i], oe[0], oe[1], oe[2]);
  }
  acc.error += dot(e, oe);
  ++acc.inliers;
}

void pack_output(const FactorAccumulator& total, double* out, int32_t* inliers) {  // factors.cpp:134-147
  double* H_ii = out;
  double* H_ij = out + 36;
  double* H_jj = out + 72;
  double* b_i = out + 108;
  double* b_j = out + 114;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      H_ii[6 * i + j] = 0.5 * (total.H_tt.m[i][j] + total.H_tt.m[j][i]);
      H_ij[6 * i + j] = total.H_ts.m[i][j];
      H_jj[6 * i + j] = 0.5 * (total.H_ss.m[i][j] + total.H_ss.m[j][i]);
    }
  for (int i = 0; i < 6; ++i) {
    b_i[i] = total.b_t.v[i];
    b_j[i] = total.b_s.v[i];
  }
  out[120] = total.error;
  *inliers = total.inliers;
}

struct ErrPartial {
  double error = 0.0;
  int inliers = 0;
};

// evaluate_matching_cost per-point body (factors.cpp:165-176)
inline void evaluate_point(const SourceView& src, std::size_t k, const VoxelMap& targets, const Pose& T_ts,
                           ErrPartial& acc) {
  const V3 transformed = T_ts.apply(v3_at(src.means, k));
  const Voxel* voxel = targets.lookup(transformed);
  if (voxel == nullptr) return;
  const V3 e = sub(voxel->mean, transformed);
  M3 omega;
  if (!invert_covariance(add(voxel->cov, rotate_cov(T_ts.R, m3_at(src.covs, k))), omega)) return;
  acc.error += dot(e, mul(omega, e));
  ++acc.inliers;
}

}  // namespace

struct or_map_s {
  VoxelMap map;
};

struct or_rng_s {
  std::mt19937_64 engine;
  explicit or_rng_s(std::uint64_t seed) : engine(seed) {}
  // oracles.hpp:155-163
  double uniform(double lo, double hi) { return lo + (hi - lo) * (static_cast<double>(engine() >> 11) * 0x1.0p-53); }
  V3 vector(double s) {
    V3 r;
    r[0] = uniform(-s, s);
    r[1] = uniform(-s, s);
    r[2] = uniform(-s, s);
    return r;
  }
};

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 3;
  }
}

V3 normalized(const V3& v) {
  const double n = norm3(v);
  return V3{{v[0] / n, v[1] / n, v[2] / n}};
}
V3 cross(const V3& a, const V3& b) {
  return V3{{a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]}};
}
// Eigen's unitOrthogonal for 3-vectors
V3 unit_orthogonal(const V3& src) {
  const double prec = 1e-12;
  V3 perp;
  if (!(std::abs(src[0]) <= std::abs(src[2]) * prec) || !(std::abs(src[1]) <= std::abs(src[2]) * prec)) {
    const double invnm = 1.0 / std::sqrt(src[0] * src[0] + src[1] * src[1]);
    perp[0] = -src[1] * invnm;
    perp[1] = src[0] * invnm;
    perp[2] = 0.0;
  } else {
    const double invnm = 1.0 / std::sqrt(src[1] * src[1] + src[2] * src[2]);
    perp[0] = 0.0;
    perp[1] = -src[2] * invnm;
    perp[2] = src[1] * invnm;
  }
  return perp;
}
// V * diag(d) * V^T with V columns (c0, c1, c2)
M3 from_eigen(const V3& c0, const V3& c1, const V3& c2, double d0, double d1, double d2) {
  M3 V;
  for (int i = 0; i < 3; ++i) {
    V.m[i][0] = c0[i];
    V.m[i][1] = c1[i];
    V.m[i][2] = c2[i];
  }
  M3 VD = V;
  for (int i = 0; i < 3; ++i) {
    VD.m[i][0] *= d0;
    VD.m[i][1] *= d1;
    VD.m[i][2] *= d2;
  }
  return mul(VD, transpose(V));
}
Pose random_pose(or_rng_s& rng, double rot_scale, double trans_scale) {  // oracles.hpp:166-168
  const V3 rot = rng.vector(rot_scale);
  const V3 trans = rng.vector(trans_scale);
  return se3_exp(rot, trans);
}
M3 random_plane_covariance(or_rng_s& rng) {  // test_factors.cpp:23-32
  const V3 n = normalized(rng.vector(1.0));
  const V3 u = unit_orthogonal(n);
  const V3 v = cross(n, u);
  return from_eigen(n, u, v, 1e-3, 1.0, 1.0);
}
void put_m3(const M3& M, double* out) {
  for (int k = 0; k < 9; ++k) out[k] = M.m[k / 3][k % 3];
}

}  // namespace

extern "C" {

const char* or_last_error(void) { return g_last_error.c_str(); }

int or_voxelmap_build(const double* means, const double* covs, size_t n, double resolution, int threads,
                      int deterministic, or_map** out) {
  *out = nullptr;
  auto* m = new or_map_s();
  const int rc = guarded([&] {
    build_parallel(means, covs, n, resolution, ExecPolicy{threads, deterministic != 0}, m->map);
  });
  if (rc != 0) {
    delete m;
    return rc;
  }
  *out = m;
  return 0;
}

int or_voxelmap_build_serial(const double* means, const double* covs, size_t n, double resolution, or_map** out) {
  auto* m = new or_map_s();
  build_serial(means, covs, n, resolution, m->map);
  *out = m;
  return 0;
}

void or_voxelmap_destroy(or_map* map) { delete map; }
size_t or_voxelmap_size(const or_map* map) { return map->map.voxels.size(); }
size_t or_voxelmap_total_points(const or_map* map) { return map->map.total_points; }

void or_voxelmap_export(const or_map* map, uint64_t* keys, int32_t* counts, double* means, double* covs) {
  std::vector<std::uint64_t> sorted;
  sorted.reserve(map->map.voxels.size());
  for (const auto& kv : map->map.voxels) sorted.push_back(kv.first);
  std::sort(sorted.begin(), sorted.end());
  for (std::size_t i = 0; i < sorted.size(); ++i) {
    const Voxel& v = map->map.voxels.at(sorted[i]);
    if (keys) keys[i] = sorted[i];
    if (counts) counts[i] = v.count;
    if (means)
      for (int a = 0; a < 3; ++a) means[3 * i + a] = v.mean[a];
    if (covs) put_m3(v.cov, covs + 9 * i);
  }
}

void or_voxelmap_lookup(const or_map* map, const double* points, size_t n, uint64_t* keys_out) {
  for (size_t i = 0; i < n; ++i) {
    const V3 p = v3_at(points, i);
    const Voxel* v = map->map.lookup(p);
    if (v == nullptr) {
      keys_out[i] = UINT64_MAX;
      continue;
    }
    int c[3];
    voxel_coord(map->map.resolution, p, c);
    keys_out[i] = pack_key(c);
  }
}

int or_voxel_key(double resolution, const double p[3], uint64_t* key) {
  return guarded([&] {
    int c[3];
    voxel_coord(resolution, V3{{p[0], p[1], p[2]}}, c);
    *key = pack_key(c);
  });
}

int or_overlap_rate(const double* means, size_t n, const double pose[12], const or_map* map, int threads,
                    int deterministic, double* rate, uint64_t* hits_out) {
  return guarded([&] {
    if (n == 0) throw std::invalid_argument("overlap_rate requires a nonempty cloud");
    const Pose rel = pose_from(pose);
    const std::size_t hits = parallel_reduce(
        n, std::size_t{0}, ExecPolicy{threads, deterministic != 0},
        [&](std::size_t begin, std::size_t end) {
          std::size_t h = 0;
          for (std::size_t i = begin; i < end; ++i)
            if (map->map.lookup(rel.apply(v3_at(means, i))) != nullptr) ++h;
          return h;
        },
        [](std::size_t a, std::size_t b) { return a + b; });
    *rate = static_cast<double>(hits) / static_cast<double>(n);
    if (hits_out) *hits_out = hits;
  });
}

int or_overlap_rate_serial(const double* means, size_t n, const double pose[12], const or_map* map, double* rate) {
  return guarded([&] {
    if (n == 0) throw std::invalid_argument("overlap_rate requires a nonempty cloud");
    const Pose rel = pose_from(pose);
    std::size_t hits = 0;
    for (std::size_t i = 0; i < n; ++i)
      if (map->map.lookup(rel.apply(v3_at(means, i))) != nullptr) ++hits;
    *rate = static_cast<double>(hits) / static_cast<double>(n);
  });
}

int or_linearize(const double* src_means, const double* src_covs, size_t n, const or_map* target,
                 const double T_target[12], const double T_source[12], int threads, int deterministic, double* out,
                 int32_t* inliers) {
  return guarded([&] {
    const SourceView src{src_means, src_covs, n};
    const Pose T_ts = compose(pose_from(T_target).inverse(), pose_from(T_source));  // factors.cpp:94
    const FactorAccumulator total = parallel_reduce(
        n, FactorAccumulator{}, ExecPolicy{threads, deterministic != 0},
        [&](std::size_t begin, std::size_t end) {
          FactorAccumulator acc;
          for (std::size_t k = begin; k < end; ++k) linearize_point(src, k, target->map, T_ts, acc);
          return acc;
        },
        [](const FactorAccumulator& a, const FactorAccumulator& b) { return a.combine(b); });
    pack_output(total, out, inliers);
  });
}

// reference::linearize_matching_cost (reference.cpp:76-110)
int or_linearize_serial(const double* src_means, const double* src_covs, size_t n, const or_map* target,
                        const double T_target[12], const double T_source[12], double* out, int32_t* inliers) {
  return guarded([&] {
    const Pose T_ts = compose(pose_from(T_target).inverse(), pose_from(T_source));
    const M3& R = T_ts.R;
    M6 H_ii, H_ij, H_jj;
    V6 b_i, b_j;
    double error = 0.0;
    int count = 0;
    for (std::size_t k = 0; k < n; ++k) {
      const V3 mu = v3_at(src_means, k);
      const V3 transformed = T_ts.apply(mu);
      const Voxel* voxel = target->map.lookup(transformed);
      if (voxel == nullptr) continue;
      const M3 combined = add(voxel->cov, rotate_cov(R, m3_at(src_covs, k)));
      const M3 inv = inverse_cofactor(combined);
      M3 omega;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) omega.m[i][j] = 0.5 * (inv.m[i][j] + inv.m[j][i]);
      const V3 e = sub(voxel->mean, transformed);
      J36 A, B;
      const M3 sq = skew(transformed);
      const M3 Rs = mul(R, skew(mu));
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          A.m[i][j] = -sq.m[i][j];
          A.m[i][3 + j] = (i == j) ? 1.0 : 0.0;
          B.m[i][j] = Rs.m[i][j];
          B.m[i][3 + j] = -R.m[i][j];
        }
      accum_JtOJ(H_ii, A, mul_OJ(omega, A));
      accum_JtOJ(H_ij, A, mul_OJ(omega, B));
      accum_JtOJ(H_jj, B, mul_OJ(omega, B));
      const V3 oe = mul(omega, e);
      for (int i = 0; i < 6; ++i) {
        b_i.v[i] -= dot3(A.m[0][i], A.m[1][i], A.m[2][i], oe[0], oe[1], oe[2]);
        b_j.v[i] -= dot3(B.m[0][i], B.m[1][i], B.m[2][i], oe[0], oe[1], oe[2]);
      }
      error += dot(e, oe);
      ++count;
    }
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) {
        out[6 * i + j] = H_ii.m[i][j];
        out[36 + 6 * i + j] = H_ij.m[i][j];
        out[72 + 6 * i + j] = H_jj.m[i][j];
      }
    for (int i = 0; i < 6; ++i) {
      out[108 + i] = b_i.v[i];
      out[114 + i] = b_j.v[i];
    }
    out[120] = error;
    *inliers = count;
  });
}

int or_evaluate(const double* src_means, const double* src_covs, size_t n, const or_map* target,
                const double T_target[12], const double T_source[12], int threads, int deterministic, double* error,
                int32_t* inliers) {
  return guarded([&] {
    const SourceView src{src_means, src_covs, n};
    const Pose T_ts = compose(pose_from(T_target).inverse(), pose_from(T_source));
    const ErrPartial total = parallel_reduce(
        n, ErrPartial{}, ExecPolicy{threads, deterministic != 0},
        [&](std::size_t begin, std::size_t end) {
          ErrPartial acc;
          for (std::size_t k = begin; k < end; ++k) evaluate_point(src, k, target->map, T_ts, acc);
          return acc;
        },
        [](const ErrPartial& a, const ErrPartial& b) { return ErrPartial{a.error + b.error, a.inliers + b.inliers}; });
    *error = total.error;
    *inliers = total.inliers;
  });
}

void or_gicp_error(const double src_mean[3], const double src_cov[9], const double tgt_mean[3],
                   const double tgt_cov[9], const double T[12], double* error, double residual[3],
                   double information[9], int* valid) {
  const Pose P = pose_from(T);
  const V3 mu{{src_mean[0], src_mean[1], src_mean[2]}};
  const V3 tm{{tgt_mean[0], tgt_mean[1], tgt_mean[2]}};
  const V3 d = sub(tm, P.apply(mu));
  M3 Cs, Ct;
  for (int k = 0; k < 9; ++k) {
    Cs.m[k / 3][k % 3] = src_cov[k];
    Ct.m[k / 3][k % 3] = tgt_cov[k];
  }
  M3 omega;
  for (int a = 0; a < 3; ++a) residual[a] = d[a];
  if (!invert_covariance(add(Ct, rotate_cov(P.R, Cs)), omega)) {
    *valid = 0;
    *error = 0.0;
    for (int k = 0; k < 9; ++k) information[k] = 0.0;
    return;
  }
  *valid = 1;
  put_m3(omega, information);
  *error = dot(d, mul(omega, d));
}

int or_invert_covariance(const double M[9], double out[9]) {
  M3 A, O;
  for (int k = 0; k < 9; ++k) A.m[k / 3][k % 3] = M[k];
  if (!invert_covariance(A, O)) return 0;
  put_m3(O, out);
  return 1;
}

double or_frozen_cost(const double* src_means, const double* src_covs, size_t n, const or_map* target,
                      const double lin_target[12], const double lin_source[12], const double T_target[12],
                      const double T_source[12]) {
  const Pose T_lin = compose(pose_from(lin_target).inverse(), pose_from(lin_source));
  const Pose T_now = compose(pose_from(T_target).inverse(), pose_from(T_source));
  double cost = 0.0;
  for (std::size_t k = 0; k < n; ++k) {
    const V3 mu = v3_at(src_means, k);
    const Voxel* voxel = target->map.lookup(T_lin.apply(mu));
    if (voxel == nullptr) continue;
    const M3 omega = inverse_cofactor(add(voxel->cov, rotate_cov(T_lin.R, m3_at(src_covs, k))));
    const V3 e = sub(voxel->mean, T_now.apply(mu));
    cost += dot(e, mul(omega, e));
  }
  return cost;
}

void or_se3_exp(const double twist[6], double pose_out[12]) {
  pose_to(se3_exp(V3{{twist[0], twist[1], twist[2]}}, V3{{twist[3], twist[4], twist[5]}}), pose_out);
}
void or_compose(const double a[12], const double b[12], double out[12]) {
  pose_to(compose(pose_from(a), pose_from(b)), out);
}
void or_inverse(const double a[12], double out[12]) { pose_to(pose_from(a).inverse(), out); }
// Pose::retract without the every-50-updates re-orthonormalisation (se3.cpp:96-104); callers
// in the tests chain at most a handful of retractions.
void or_retract(const double a[12], const double twist[6], double out[12]) {
  pose_to(compose(pose_from(a), se3_exp(V3{{twist[0], twist[1], twist[2]}}, V3{{twist[3], twist[4], twist[5]}})),
          out);
}
void or_adjoint(const double a[12], double out[36]) {
  const M6 ad = adjoint(pose_from(a));
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) out[6 * i + j] = ad.m[i][j];
}

or_rng* or_rng_create(uint64_t seed) { return new or_rng_s(seed); }
void or_rng_destroy(or_rng* rng) { delete rng; }
double or_rng_uniform(or_rng* rng, double lo, double hi) { return rng->uniform(lo, hi); }
void or_rng_vector(or_rng* rng, double scale, double out[3]) {
  const V3 v = rng->vector(scale);
  for (int a = 0; a < 3; ++a) out[a] = v[a];
}
void or_random_pose(or_rng* rng, double rot_scale, double trans_scale, double pose_out[12]) {
  pose_to(random_pose(*rng, rot_scale, trans_scale), pose_out);
}
void or_random_plane_covariance(or_rng* rng, double cov_out[9]) { put_m3(random_plane_covariance(*rng), cov_out); }

void or_random_gaussian_cloud(or_rng* rng, int n, double scale, double* means, double* covs) {
  for (int i = 0; i < n; ++i) {
    const V3 m = rng->vector(scale);
    for (int a = 0; a < 3; ++a) means[3 * i + a] = m[a];
    const V3 axis = normalized(rng->vector(1.0));
    const V3 u = unit_orthogonal(axis);
    put_m3(from_eigen(axis, u, cross(axis, u), 1e-3, 1.0, 1.0), covs + 9 * i);
  }
}

void or_make_scene(or_rng* rng, int points, double resolution, double boundary_margin, double* T_target,
                   double* T_source, double* source_means, double* source_covs, double* target_means,
                   double* target_covs) {
  const Pose Tt = random_pose(*rng, 0.3, 2.0);
  const Pose Ts = random_pose(*rng, 0.3, 2.0);
  pose_to(Tt, T_target);
  pose_to(Ts, T_source);
  const Pose T_ts = compose(Tt.inverse(), Ts);
  for (int i = 0; i < points; ++i) {
    while (true) {
      const V3 p = rng->vector(8.0);
      const V3 q = T_ts.apply(p);
      bool clear = true;
      for (int a = 0; a < 3; ++a) {
        const double frac = q[a] / resolution - std::floor(q[a] / resolution);
        if (frac < boundary_margin || frac > 1.0 - boundary_margin) clear = false;
      }
      if (!clear) continue;
      for (int a = 0; a < 3; ++a) source_means[3 * i + a] = p[a];
      put_m3(random_plane_covariance(*rng), source_covs + 9 * i);
      const V3 jitter = rng->vector(1.0);
      V3 t{{q[0] + 0.05 * jitter[0], q[1] + 0.05 * jitter[1], q[2] + 0.05 * jitter[2]}};
      for (int a = 0; a < 3; ++a) {
        const double cell = std::floor(q[a] / resolution);
        t[a] = std::clamp(t[a], (cell + boundary_margin) * resolution, (cell + 1.0 - boundary_margin) * resolution);
      }
      for (int a = 0; a < 3; ++a) target_means[3 * i + a] = t[a];
      put_m3(random_plane_covariance(*rng), target_covs + 9 * i);
      break;
    }
  }
}

void or_rng_shuffle(or_rng* rng, uint64_t* perm, size_t n) { std::shuffle(perm, perm + n, rng->engine); }

// reference::estimate_covariances (reference.cpp:11-37) with the brute-force kNN of
// oracles.hpp:24-35 (full sort by (squared distance, index)) and a Jacobi eigen-solver in place of
// Eigen::SelfAdjointEigenSolver: V·diag(eps,1,1)·Vᵀ = I - (1-eps)·v0·v0ᵀ for the unit eigenvector
// v0 of the smallest eigenvalue. Means are n×3 doubles, output n×9 doubles.
int or_estimate_covariances(const double* means, size_t n, int k, double plane_epsilon, double* covs) {
  return guarded([&] {
    if (k < 4 || n <= static_cast<size_t>(k))
      throw std::invalid_argument("covariance estimation requires k >= 4 and more than k points");
    std::vector<std::pair<double, int>> all(n);
    for (size_t q = 0; q < n; ++q) {
      for (size_t i = 0; i < n; ++i) {
        double d2 = 0.0;
        for (int a = 0; a < 3; ++a) {
          const double d = means[3 * i + a] - means[3 * q + a];
          d2 += d * d;
        }
        all[i] = {d2, static_cast<int>(i)};
      }
      std::partial_sort(all.begin(), all.begin() + k, all.end());
      double mean[3] = {0, 0, 0};
      for (int j = 0; j < k; ++j)
        for (int a = 0; a < 3; ++a) mean[a] += means[3 * all[j].second + a];
      for (int a = 0; a < 3; ++a) mean[a] /= static_cast<double>(k);
      double A[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
      for (int j = 0; j < k; ++j) {
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = means[3 * all[j].second + a] - mean[a];
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) A[r][c] += d[r] * d[c];
      }
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) A[r][c] /= static_cast<double>(k);
      double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
      for (int sweep = 0; sweep < 100; ++sweep) {
        const double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
        if (off < 1e-32 * (A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2]) + 1e-300) break;
        for (int p = 0; p < 2; ++p)
          for (int r = p + 1; r < 3; ++r) {
            if (A[p][r] == 0.0) continue;
            const double theta = (A[r][r] - A[p][p]) / (2.0 * A[p][r]);
            const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
            const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
            for (int m = 0; m < 3; ++m) {
              const double amp = A[m][p], amr = A[m][r];
              A[m][p] = c * amp - sn * amr;
              A[m][r] = sn * amp + c * amr;
            }
            for (int m = 0; m < 3; ++m) {
              const double apm = A[p][m], arm = A[r][m];
              A[p][m] = c * apm - sn * arm;
              A[r][m] = sn * apm + c * arm;
            }
            for (int m = 0; m < 3; ++m) {
              const double vmp = V[m][p], vmr = V[m][r];
              V[m][p] = c * vmp - sn * vmr;
              V[m][r] = sn * vmp + c * vmr;
            }
          }
      }
      int mi = 0;
      if (A[1][1] < A[mi][mi]) mi = 1;
      if (A[2][2] < A[mi][mi]) mi = 2;
      const double v[3] = {V[0][mi], V[1][mi], V[2][mi]};
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) covs[9 * q + 3 * r + c] = (r == c ? 1.0 : 0.0) - (1.0 - plane_epsilon) * v[r] * v[c];
    }
  });
}

// transform_cloud (point_cloud.cpp:26-42): means -> T.apply(mean), covariances -> R·C·Rᵀ with
// Eigen's evaluation order ((R·C) first, then ·Rᵀ). covs / out_covs may be NULL.
void or_transform_cloud(const double* means, const double* covs, size_t n, const double pose[12], double* out_means,
                        double* out_covs) {
  const Pose T = pose_from(pose);
  for (size_t i = 0; i < n; ++i) {
    const V3 q = T.apply(v3_at(means, i));
    for (int a = 0; a < 3; ++a) out_means[3 * i + a] = q[a];
    if (covs && out_covs) {
      const M3 C = rotate_cov(T.R, m3_at(covs, i));
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) out_covs[9 * i + 3 * r + c] = C.m[r][c];
    }
  }
}

}  // extern "C"
