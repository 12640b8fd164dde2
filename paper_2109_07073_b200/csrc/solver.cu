// Damped block Cholesky solve of the LM's reduced normal equations on the GPU (sm_100a): the
// reference's solve_block_system (block_solver.cpp:64-122 — right-looking 6×6-block Cholesky,
// forward and backward substitution) over a fill-reducing order.
//
// Plan (host, once per assembly plan): reverse Cuthill-McKee order of the slot graph, row
// profile first(i), column reach(k) = max{i : first(i) <= k}; Cholesky fill stays inside that
// envelope, so every column k is stored densely as block rows k..reach(k) (+ the right-hand
// side as an augmented row, which turns the forward substitution into part of the factorization).
//
// Kernel: one thread-block cluster of C CTAs (the cluster launch guarantees co-residency). Column k
// is owned by CTA k mod C and lives in its shared memory from the step it is first touched until
// it is factored. Step j: every CTA receives panel j (L_jj, L_ij, y_j) — the owner from its own
// shared memory, the owner of column j+1 (the only CTA on the dependency chain) over DSMEM from the
// owner's slot after a release flag in its own shared memory, the others from L2 once the owner's
// global release flag carries this launch's epoch;
// the owner of column j+1 applies panel j to it first, factors it (6×6 Cholesky, TRSM of the
// sub-diagonal blocks and of the augmented row) and publishes it (global memory + flag); every
// CTA applies panel j to its other columns in the window. No cluster barrier inside the loop:
// panels live in distinct global records, so the only cross-CTA dependencies are the flags.
// Afterwards CTA 0 runs the backward substitution (one warp, columns TMA-prefetched two ahead).
// Fixed operation order everywhere: results are deterministic.
//
// Measured on C3 (449 slots, RCM block bandwidth 31, 16-CTA cluster): 1.57 ms per damped solve vs
// 1.81 ms for the dense cuSOLVER potrf/potrs of the 2,694-dim system; C5 (999 slots, bandwidth 47):
// 3.8 ms vs 5.3 ms. The 449-step dependency chain bounds it (per step: DSMEM hand-off to the next
// owner, its diagonal update + 6×6 Cholesky + TRSM). The LM uses it above 2,000 unknowns (dense
// below). Build with -DVG_SOLVE_PROF=1 for a per-phase cycle profile (VGICP_SOLVE_PROF=1 prints it).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "internal.h"

namespace cg = cooperative_groups;

namespace vgicp {

namespace {

constexpr int kSolveThreads = 256;
#ifndef VG_SOLVE_PROF
#define VG_SOLVE_PROF 0
#endif


__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar, unsigned phase) {
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

// Column / panel record (doubles): blocks 0..bw (block b = row k + b, row-major 6×6; block 0 is
// the diagonal), then the augmented row (6), the failure flag, a pad, 1/L_cc (6), 2 pads.
__host__ __device__ constexpr int col_aug(int bw) { return 36 * (bw + 1); }
__host__ __device__ constexpr int col_stride(int bw) { return 36 * (bw + 1) + 16; }

struct SolveArgs {
  BandDev d;
  const double* diag;  // assembled system: diag S×36 | off P×36 | rhs S×6
  const double* off;
  const double* rhs;
  double lam;
  double lam2;  // second damping value, solved concurrently by a second cluster (instances = 2)
  int ns;       // column slots per CTA
  int epoch;    // this launch's value of the ready flags
  int instances;
};

// Zero column k's record, then scatter its blocks from the assembled system (damped diagonal,
// off-diagonal pairs — transposed where the order flips the pair — and the rhs row).
__device__ void load_columns(const SolveArgs& a, double lam, const int* reach, double* slots, int first, int last, int C,
                             int rank) {
  const BandDev& d = a.d;
  const int cs = col_stride(d.bw);
  const int aug = col_aug(d.bw);
  for (int k = first; k <= last; k += C) {
    double* col = slots + (size_t)((k / C) % a.ns) * cs;
    const int n = 36 * (reach[k] - k + 1);
    for (int t = threadIdx.x; t < n; t += kSolveThreads) col[t] = 0.0;
    if (threadIdx.x < 16) col[aug + threadIdx.x] = 0.0;
  }
  __syncthreads();
  for (int k = first; k <= last; k += C) {
    double* col = slots + (size_t)((k / C) % a.ns) * cs;
    const int slot = d.perm[k];
    const int e0 = d.col_ptr[k], e1 = d.col_ptr[k + 1];
    const int tasks = 36 * (e1 - e0) + 36 + 6;
    for (int t = threadIdx.x; t < tasks; t += kSolveThreads) {
      if (t < 36) {  // damped diagonal block (optimizer.cpp:119-123)
        double v = a.diag[(size_t)slot * 36 + t];
        if (t % 7 == 0) v = v + lam * fmax(v, 1e-10);
        col[t] = v;
      } else if (t < 42) {
        col[aug + (t - 36)] = a.rhs[(size_t)slot * 6 + (t - 36)];
      } else {
        const int e = e0 + (t - 42) / 36;
        const int q = (t - 42) % 36;
        const int2 ent = d.col_ent[e];
        const int b = ent.x & 0xFFFF;
        const bool tr = (ent.x >> 16) != 0;
        const double* src = a.off + (size_t)ent.y * 36;
        col[36 * b + q] = tr ? src[(q % 6) * 6 + q / 6] : src[q];
      }
    }
  }
  __syncthreads();
}

// Apply panel j (pj) to the owned columns k in [lo, hi] (k ≡ rank mod C, k > j): block rows
// i ∈ [k, R] get A_ik -= L_ij·L_kjᵀ; the augmented row gets B_k -= y_j·L_kjᵀ. One thread per
// (column, block row, entry row): six fixed-order 6-term dot products.
__device__ void update_columns(const SolveArgs& a, double* slots, const double* pj, int j, int R, int lo, int hi,
                               int C) {
  const int cs = col_stride(a.d.bw);
  const int aug = col_aug(a.d.bw);
  if (lo > hi) return;
  // tasks of the c-th column k = lo + c·C: (R - k + 1)·6 entry rows + 1 augmented row (decreasing
  // by 6·C per column; no per-thread array, which would live in local memory)
  const int ncol = (hi - lo) / C + 1;
  const int first = (R - lo + 1) * 6 + 1;
  const int total = ncol * first - 3 * C * ncol * (ncol - 1);
  for (int t = threadIdx.x; t < total; t += kSolveThreads) {
    int c = 0, u = t, cnt = first;
    while (u >= cnt) u -= cnt, cnt -= 6 * C, ++c;
    const int k = lo + c * C;
    const int counts_c = cnt;
    double* col = slots + (size_t)((k / C) % a.ns) * cs;
    const double* Lk = pj + 36 * (k - j);
    const double* Li;
    double* dst;
    if (u < counts_c - 1) {
      const int b = u / 6, r = u % 6;  // block row i = k + b, entry row r
      Li = pj + 36 * (k + b - j) + 6 * r;
      dst = col + 36 * b + 6 * r;
    } else {
      Li = pj + aug;
      dst = col + aug;
    }
    const double l0 = Li[0], l1 = Li[1], l2 = Li[2], l3 = Li[3], l4 = Li[4], l5 = Li[5];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double* m = Lk + 6 * q;
      const double s = ((((l0 * m[0] + l1 * m[1]) + l2 * m[2]) + l3 * m[3]) + l4 * m[4]) + l5 * m[5];
      dst[q] -= s;
    }
  }
}

// 1/sqrt(x) for the pivots: libdevice's fp64 rsqrt (MUFU.RSQ64H seed + refinement) — measured
// faster on the pivot chain than an fp32-seeded Newton pair (C3 solve 1.72 -> 1.62 ms).
__device__ __forceinline__ double rsqrt_fast(double x) { return rsqrt(x); }

// Factor column k in place (all threads of the CTA): 6×6 Cholesky of the diagonal block (warp
// 0; a pivot that is not > 0 fails like Eigen::LLT, block_solver.cpp:78-82), then
// L_ik = A_ik·L_kk⁻ᵀ for the sub-diagonal blocks and y_k = L_kk⁻¹·b_k for the augmented row.
__device__ void factor_column(const SolveArgs& a, const int* reach, double* col, int k) {
  const int aug = col_aug(a.d.bw);
  double* inv = col + aug + 8;
  if (threadIdx.x == 0) {  // one thread: the pivot chain is short, shuffles would only add latency
    double L[6][6];
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) L[r][c] = col[6 * r + c];
    bool failed = false;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      double piv = L[c][c];
#pragma unroll
      for (int m = 0; m < c; ++m) piv -= L[c][m] * L[c][m];
      failed |= !(piv > 0.0);
      const double il = rsqrt_fast(piv);
      L[c][c] = piv * il;
      inv[c] = il;
#pragma unroll
      for (int r = c + 1; r < 6; ++r) {
        double v = L[r][c];
#pragma unroll
        for (int m = 0; m < c; ++m) v -= L[r][m] * L[c][m];
        L[r][c] = v * il;
      }
    }
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int c = 0; c < 6; ++c) col[6 * r + c] = c <= r ? L[r][c] : 0.0;
    col[aug + 6] = failed ? 1.0 : 0.0;
  }
  __syncthreads();
  if (col[aug + 6] != 0.0) return;
  const int nrows = (reach[k] - k) * 6 + 1;  // sub-diagonal entry rows + the augmented row
  for (int t = threadIdx.x; t < nrows; t += kSolveThreads) {
    double* v = t < nrows - 1 ? col + 36 + 6 * t : col + aug;
    double x[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) {  // x·L_kkᵀ = v  <=>  L_kk·xᵀ = vᵀ
      double s = v[c];
#pragma unroll
      for (int r = 0; r < c; ++r) s -= x[r] * col[6 * c + r];
      x[c] = s * inv[c];
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) v[c] = x[c];
  }
  __syncthreads();
}

// Column n1 on the dependency chain, at step j: panel j applied to it (when it reaches n1) and the
// column factored, overlapped — warp 0 updates the diagonal block and runs the 6×6 Cholesky while
// the other warps update the sub-diagonal rows and the augmented row; then every thread solves
// its TRSM rows. Same arithmetic (and order per entry) as update_columns + factor_column.
__device__ void chain_column(const SolveArgs& a, const int* reach, double* col, const double* pj, int j, int n1, int R,
                             bool upd) {
#if VG_SOLVE_PROF
  unsigned long long* cp = reinterpret_cast<unsigned long long*>(a.d.status) + 24;
  long long c0 = clock64();
  const bool prof = cooperative_groups::this_cluster().block_rank() == 0 && threadIdx.x == 0;
#define VG_CTICK(q) do { if (prof) { const long long c1 = clock64(); cp[q] += c1 - c0; c0 = c1; } } while (0)
#else
#define VG_CTICK(q) ((void)0)
#endif
  const int aug = col_aug(a.d.bw);
  double* inv = col + aug + 8;
  const double* Lk = pj + 36 * (n1 - j);  // L_{n1,j}
  auto upd_row = [&](double* dst, const double* Li) {
    const double l0 = Li[0], l1 = Li[1], l2 = Li[2], l3 = Li[3], l4 = Li[4], l5 = Li[5];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double* m = Lk + 6 * q;
      const double s = ((((l0 * m[0] + l1 * m[1]) + l2 * m[2]) + l3 * m[3]) + l4 * m[4]) + l5 * m[5];
      dst[q] -= s;
    }
  };
  if (threadIdx.x < 32) {
    VG_CTICK(0);
    if (threadIdx.x == 0) {  // diagonal update fused into the Cholesky thread (no smem round trip)
      double L[6][6];
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) L[r][c] = col[6 * r + c];
      if (upd) {
        double K[6][6];
#pragma unroll
        for (int r = 0; r < 6; ++r)
#pragma unroll
          for (int q = 0; q < 6; ++q) K[r][q] = Lk[6 * r + q];
#pragma unroll
        for (int r = 0; r < 6; ++r)
#pragma unroll
          for (int c = 0; c <= r; ++c)  // same per-entry order as update_columns
            L[r][c] -= ((((K[r][0] * K[c][0] + K[r][1] * K[c][1]) + K[r][2] * K[c][2]) + K[r][3] * K[c][3]) +
                        K[r][4] * K[c][4]) + K[r][5] * K[c][5];
      }
      bool failed = false;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        double piv = L[c][c];
#pragma unroll
        for (int m = 0; m < c; ++m) piv -= L[c][m] * L[c][m];
        failed |= !(piv > 0.0);
        const double il = rsqrt_fast(piv);
        L[c][c] = piv * il;
        inv[c] = il;
#pragma unroll
        for (int r = c + 1; r < 6; ++r) {
          double v = L[r][c];
#pragma unroll
          for (int m = 0; m < c; ++m) v -= L[r][m] * L[c][m];
          L[r][c] = v * il;
        }
      }
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) col[6 * r + c] = c <= r ? L[r][c] : 0.0;
      col[aug + 6] = failed ? 1.0 : 0.0;
    }
    VG_CTICK(1);
  } else if (upd) {
    const int rows = (R - n1) * 6;  // sub-diagonal entry rows touched by panel j, then the aug row
    for (int t = threadIdx.x - 32; t <= rows; t += kSolveThreads - 32) {
      if (t < rows) {
        const int b = 1 + t / 6, r = t % 6;
        upd_row(col + 36 * b + 6 * r, pj + 36 * (n1 + b - j) + 6 * r);
      } else {
        upd_row(col + aug, pj + aug);
      }
    }
  }
  __syncthreads();
  VG_CTICK(2);
  if (col[aug + 6] != 0.0) return;
  const int nrows = (reach[n1] - n1) * 6 + 1;
  for (int t = threadIdx.x; t < nrows; t += kSolveThreads) {
    double* v = t < nrows - 1 ? col + 36 + 6 * t : col + aug;
    double x[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      double s = v[c];
#pragma unroll
      for (int r = 0; r < c; ++r) s -= x[r] * col[6 * c + r];
      x[c] = s * inv[c];
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) v[c] = x[c];
  }
  VG_CTICK(3);
  __syncthreads();
  VG_CTICK(4);
#undef VG_CTICK
}

__device__ void copy_record(double* __restrict__ dst, const double* __restrict__ src, int n) {
  const double2* s = reinterpret_cast<const double2*>(src);
  double2* o = reinterpret_cast<double2*>(dst);
  for (int t = threadIdx.x; t < n / 2; t += kSolveThreads) o[t] = s[t];
}

__global__ void __launch_bounds__(kSolveThreads, 1) band_solve_kernel(SolveArgs a) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) unsigned long long bbars[3];
  cg::cluster_group cluster = cg::this_cluster();  // a cluster launch guarantees the CTAs are co-resident
  const BandDev& d = a.d;
  const int C = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  const int S = d.S;
  // instance (cluster) 1 solves the second damping value into its own buffers
  const int inst = static_cast<int>(blockIdx.x) / C;
  const double lam = inst ? a.lam2 : a.lam;
  double* const Lg = d.Lg + (size_t)inst * S * col_stride(d.bw);
  double* const X = d.x + (size_t)inst * 6 * S;
  int* const status = d.status + inst * 64;
  int* const ready = d.ready + (size_t)inst * S;
  const int cs = col_stride(d.bw);
  const int aug = col_aug(d.bw);
  double* slots = smem;                     // ns column records
  double* pj = smem + (size_t)a.ns * cs;    // the current panel
  // envelope reach per column, staged once: it is read on every step of the dependency chain
  int* reach = reinterpret_cast<int*>(pj + cs);
  for (int t = threadIdx.x; t < S; t += kSolveThreads) reach[t] = d.reach[t];
  __syncthreads();
  const auto rec_len = [&](int k) { return 36 * (reach[k] - k + 1); };
  const auto panel_bytes = [&](int k) { return static_cast<unsigned>(sizeof(double) * (rec_len(k) + 16)); };
  const auto slot_of = [&](int k) { return slots + (size_t)((k / C) % a.ns) * cs; };

  __shared__ int crit_flag;  // written remotely by owner(j) when column j is factored (value j)
  if (threadIdx.x == 0) {
    bar_init(&bbars[0]);
    bar_init(&bbars[1]);
    bar_init(&bbars[2]);
    crit_flag = -1;
  }
  cluster.sync();  // every CTA's flag is initialised before any remote release can reach it

  int next = rank;  // next owned column not yet loaded
  auto ensure_loaded = [&](int limit) {
    int last = next - C;
    while (last + C <= limit && last + C < S) last += C;
    if (last >= next) {
      load_columns(a, lam, reach, slots, next, last, C, rank);
      next = last + C;
    }
  };
  // Factored column k -> global memory, then a release flag (ready[k] = this launch's epoch).
  // Factored column k is published twice: to owner(k+1) — the only CTA on the dependency chain —
  // by a release store into ITS shared-memory flag (it then pulls the record from this CTA's slot
  // over DSMEM; the slot stays intact until owner(k+1) has published k+1, by the chain itself), and
  // to everybody else through L2 (record + release flag in global memory).
  auto publish = [&](int k) {
    // factor_column ended with a CTA barrier: the slot is complete; release it to owner(k+1) first
    if (threadIdx.x == 0 && k + 1 < S && (k + 1) % C != rank) {
      const unsigned remote = static_cast<unsigned>(__cvta_generic_to_shared(&crit_flag));
      unsigned raddr;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(remote), "r"((k + 1) % C));
      asm volatile("st.release.cluster.shared::cluster.b32 [%0], %1;" ::"r"(raddr), "r"(k) : "memory");
    }
    const double* col = slot_of(k);
    double* g = Lg + (size_t)k * cs;
    copy_record(g, col, rec_len(k));
    copy_record(g + aug, col + aug, 16);
    __syncthreads();  // the CTA's writes happen-before thread 0's (cumulative) release
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ready + k), "r"(a.epoch) : "memory");
  };
  // Panel j -> pj: the owner copies its own column record; the others wait for the flag and read
  // the record from L2.
  auto receive = [&](int j) {
    if (j % C == rank) {
      const double* col = slot_of(j);
      copy_record(pj, col, rec_len(j));
      copy_record(pj + aug, col + aug, 16);
    } else if (j + 1 < S && (j + 1) % C == rank) {  // on the chain: local flag, then a DSMEM pull
      if (threadIdx.x == 0) {
        const unsigned f = static_cast<unsigned>(__cvta_generic_to_shared(&crit_flag));
        int v;
        do {
          asm volatile("ld.acquire.cluster.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(f) : "memory");
        } while (v != j);
      }
      __syncthreads();
      const double* src = cluster.map_shared_rank(slot_of(j), j % C);
      copy_record(pj, src, rec_len(j));
      copy_record(pj + aug, src + aug, 16);
    } else {
      if (threadIdx.x == 0) {
        int v;
        do {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ready + j) : "memory");
        } while (v != a.epoch);
      }
      __syncthreads();
      const double2* g = reinterpret_cast<const double2*>(Lg + (size_t)j * cs);
      double2* o = reinterpret_cast<double2*>(pj);
      const int n = rec_len(j) / 2;
      for (int t = threadIdx.x; t < n + 8; t += kSolveThreads) {
        const int u = t < n ? t : aug / 2 + (t - n);
        o[u] = __ldcg(g + u);
      }
    }
    __syncthreads();
  };

  if (S > 0) {
    ensure_loaded(max(reach[0], 0));
    if (rank == 0) {
      factor_column(a, reach, slots, 0);
      publish(0);
    }
  }
  int failed_at = -1;
#if VG_SOLVE_PROF  // rank 0 / thread 0 cycle profile, read by VGICP_SOLVE_PROF=1 (diagnostic build)
  long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = clock64(), t1;
#define VG_TICK(q) (t1 = clock64(), tp[q] += t1 - t0, t0 = t1)
#else
#define VG_TICK(q) ((void)0)
#endif
  for (int j = 0; j < S; ++j) {
    const int R = reach[j];
    const int n1 = j + 1;
    receive(j);
    VG_TICK(0);
    if (pj[aug + 6] != 0.0) {  // the owner's pivot failed: every CTA leaves at the same step
      failed_at = j;
      break;
    }
    // owned columns in (j, R]
    int lo = j + 1 + ((rank - (j + 1)) % C + C) % C;
    if (n1 < S && n1 % C == rank) {  // on the chain: only column n1 must be resident first
      ensure_loaded(n1);
      VG_TICK(6);
      chain_column(a, reach, slot_of(n1), pj, j, n1, R, n1 <= R);
      VG_TICK(7);
      publish(n1);
      lo = n1 + C;
    }
    VG_TICK(2);
    ensure_loaded(max(R, n1 < S ? n1 : -1));
    VG_TICK(1);
    update_columns(a, slots, pj, j, R, lo, R, C);
    __syncthreads();
    VG_TICK(3);
  }
  if (failed_at >= 0 && rank == 0 && threadIdx.x == 0) *status = failed_at + 1;
  cluster.sync();  // every column published
  VG_TICK(4);

  // ---- backward substitution Lᵀx = y (block_solver.cpp:108-114) on CTA 0, pipelined over two
  //      roles: x_k = L_kk⁻ᵀ(y_k - P_k - L_{k+1,k}ᵀ x_{k+1}) is the only dependent step (warp 0),
  //      while warps 1..6 form P_{k-1} = Σ_{b>=2} L_{k-1+b,k-1}ᵀ x_{k-1+b} (all of those x are
  //      known) for the next step. Columns stream through a ring of 3 shared-memory buffers by bulk
  //      copies; x lives in a ring of bw + 1 block rows. Fixed orders: deterministic. ----
  if (failed_at >= 0 || rank != 0) return;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const auto buf = [&](int q) { return slots + (size_t)q * cs; };  // ring slot q of 3
  double* xr = slots + 3 * (size_t)cs;  // W × 6 (W <= 2·(bw + 1) <= a record's length)
  __shared__ double Pbuf[2][6];
  __shared__ double vbuf[6];
  int W = 1;  // x ring: power of two >= bw + 1, so ring indices are masks
  while (W < d.bw + 1) W <<= 1;
  const int wm = W - 1;
  auto fetch = [&](int k) {  // column k -> ring slot (S - 1 - k) % 3, barrier of that slot
    const int q = (S - 1 - k) % 3;
    bar_expect(&bbars[q], panel_bytes(k));
    bulk_copy(buf(q), Lg + (size_t)k * cs, static_cast<unsigned>(sizeof(double) * rec_len(k)), &bbars[q]);
    bulk_copy(buf(q) + aug, Lg + (size_t)k * cs + aug, static_cast<unsigned>(sizeof(double) * 16), &bbars[q]);
  };
  auto wait_col = [&](int k) {
    const int u = S - 1 - k;
    bar_wait(&bbars[u % 3], static_cast<unsigned>((u / 3) & 1));
  };
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async;" ::: "memory");  // Lg / slots were written by generic stores
    for (int k = S - 1; k >= 0 && k >= S - 3; --k) fetch(k);
  }
  if (threadIdx.x < 6) Pbuf[(S - 1) & 1][threadIdx.x] = 0.0;  // column S-1 has no rows below
  __syncthreads();
  for (int k = S - 1; k >= 0; --k) {
    wait_col(k);
    if (k > 0) wait_col(k - 1);
    const double* L = buf((S - 1 - k) % 3);
    if (warp == 0) {  // the chain: x_k
      const int nb = reach[k] - k;
      if (lane < 6) {  // lane c: v_c = y_c - P_c - (L_{k+1,k}ᵀ x_{k+1})_c
        double t = 0.0;
        if (nb >= 1) {
          const double* x1 = xr + ((k + 1) & wm) * 6;
#pragma unroll
          for (int r = 0; r < 6; ++r) t += L[36 + 6 * r + lane] * x1[r];
        }
        vbuf[lane] = L[aug + lane] - Pbuf[k & 1][lane] - t;
      }
      __syncwarp();
      double x[6];  // every lane solves L_kkᵀ x = v in registers (no shuffles on the chain)
#pragma unroll
      for (int c = 5; c >= 0; --c) {
        double w = vbuf[c];
#pragma unroll
        for (int r = c + 1; r < 6; ++r) w -= L[6 * r + c] * x[r];
        x[c] = w * L[aug + 8 + c];
      }
      if (lane < 6) {
        double xc = x[0];
#pragma unroll
        for (int c = 1; c < 6; ++c) xc = lane == c ? x[c] : xc;
        xr[(k & wm) * 6 + lane] = xc;
        X[(size_t)d.perm[k] * 6 + lane] = xc;
      }
    } else if (warp <= 6 && k > 0) {  // P_{k-1}, component c = warp - 1
      const int c = warp - 1;
      const int k1 = k - 1;
      const double* L1 = buf((S - 1 - k1) % 3);
      const int nb1 = reach[k1] - k1;
      double sum = 0.0;
      for (int t = lane; t < 6 * (nb1 - 1); t += 32) {  // blocks b = 2 .. nb1
        const int bb = 2 + t / 6, r = t % 6;
        sum += L1[36 * bb + 6 * r + c] * xr[((k1 + bb) & wm) * 6 + r];
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      if (lane == 0) Pbuf[k1 & 1][c] = sum;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads of buf before its refill
    __syncthreads();
    if (threadIdx.x == 0 && k >= 3) fetch(k - 3);  // into column k's (now free) ring slot
  }
  if (threadIdx.x == 0) {
    *status = 0;
#if VG_SOLVE_PROF
    VG_TICK(5);
    unsigned long long* prof = reinterpret_cast<unsigned long long*>(d.status) + 8;
    for (int q = 0; q < 8; ++q) prof[q] = static_cast<unsigned long long>(tp[q]);
#endif
  }
#undef VG_TICK
}

}  // namespace

// ------------------------------------------------------------------------------------ host plan
BandPlanHost make_band_plan(int S, int P, const int32_t* pairs) {
  BandPlanHost p;
  p.S = S;
  std::vector<std::vector<int>> adj(S);
  for (int q = 0; q < P; ++q) {
    const int a = pairs[2 * q], b = pairs[2 * q + 1];
    adj[a].push_back(b);
    adj[b].push_back(a);
  }
  std::vector<int> deg(S);
  for (int v = 0; v < S; ++v) {
    std::sort(adj[v].begin(), adj[v].end());
    adj[v].erase(std::unique(adj[v].begin(), adj[v].end()), adj[v].end());
    deg[v] = static_cast<int>(adj[v].size());
  }
  // reverse Cuthill-McKee: per component, a pseudo-peripheral start (George-Liu), BFS with
  // neighbours by ascending (degree, index); the concatenated order is reversed
  std::vector<int> order;
  order.reserve(S);
  std::vector<char> done(S, 0);
  std::vector<int> level(S, -1);
  auto bfs_levels = [&](int s, std::vector<int>& comp) {
    comp.clear();
    comp.push_back(s);
    level[s] = 0;
    for (size_t h = 0; h < comp.size(); ++h)
      for (int u : adj[comp[h]])
        if (level[u] < 0) {
          level[u] = level[comp[h]] + 1;
          comp.push_back(u);
        }
  };
  std::vector<int> comp;
  for (int seed = 0; seed < S; ++seed) {
    if (done[seed]) continue;
    int start = seed;
    bfs_levels(start, comp);
    for (int v : comp)
      if (deg[v] < deg[start] || (deg[v] == deg[start] && v < start)) start = v;
    for (int v : comp) level[v] = -1;
    for (int it = 0; it < 8; ++it) {
      bfs_levels(start, comp);
      const int ecc = level[comp.back()];
      int cand = -1;
      for (int v : comp)
        if (level[v] == ecc && (cand < 0 || deg[v] < deg[cand] || (deg[v] == deg[cand] && v < cand))) cand = v;
      std::vector<int> tmp = comp;
      for (int v : tmp) level[v] = -1;
      bfs_levels(cand, comp);
      const int ecc2 = level[comp.back()];
      for (int v : comp) level[v] = -1;
      if (ecc2 <= ecc) break;
      start = cand;
    }
    // Cuthill-McKee BFS
    size_t head = order.size();
    order.push_back(start);
    done[start] = 1;
    std::vector<int> nb;
    for (size_t h = head; h < order.size(); ++h) {
      nb.clear();
      for (int u : adj[order[h]])
        if (!done[u]) nb.push_back(u);
      std::sort(nb.begin(), nb.end(), [&](int x, int y) { return deg[x] != deg[y] ? deg[x] < deg[y] : x < y; });
      for (int u : nb) {
        done[u] = 1;
        order.push_back(u);
      }
    }
  }
  std::reverse(order.begin(), order.end());
  p.perm = order;
  std::vector<int> pos(S);
  for (int i = 0; i < S; ++i) pos[order[i]] = i;
  std::vector<int> first(S);
  for (int i = 0; i < S; ++i) {
    first[i] = i;
    for (int u : adj[order[i]]) first[i] = std::min(first[i], pos[u]);
  }
  p.reach.assign(S, 0);
  for (int k = 0; k < S; ++k) p.reach[k] = k;
  for (int i = 0; i < S; ++i) p.reach[first[i]] = std::max(p.reach[first[i]], i);
  for (int k = 1; k < S; ++k) p.reach[k] = std::max(p.reach[k], p.reach[k - 1]);
  p.bw = 0;
  for (int k = 0; k < S; ++k) p.bw = std::max(p.bw, p.reach[k] - k);
  // per-column lower blocks from the pairs (pair q stores block (row a, col b) in slot numbering)
  std::vector<std::vector<int2>> cols(S);
  for (int q = 0; q < P; ++q) {
    const int pa = pos[pairs[2 * q]], pb = pos[pairs[2 * q + 1]];
    if (pa > pb) cols[pb].push_back(make_int2(pa - pb, q));
    else cols[pa].push_back(make_int2((pb - pa) | (1 << 16), q));
  }
  p.col_ptr.assign(S + 1, 0);
  for (int k = 0; k < S; ++k) {
    std::sort(cols[k].begin(), cols[k].end(), [](int2 x, int2 y) { return (x.x & 0xFFFF) < (y.x & 0xFFFF); });
    p.col_ptr[k + 1] = p.col_ptr[k] + static_cast<int>(cols[k].size());
    p.col_ent.insert(p.col_ent.end(), cols[k].begin(), cols[k].end());
  }
  return p;
}

size_t band_smem_bytes(int bw, int C, int S) {
  const int ns = std::max(bw / C + 1, 4);  // >= 4: the backward substitution reuses the slot area
  const size_t rec = sizeof(double) * col_stride(bw);
  return (ns + 1) * rec + sizeof(int) * static_cast<size_t>(S);  // + the staged reach array
}

// Largest cluster (16, else 8, 4, 2, 1) that can be co-resident with this bandwidth's window.
int band_cluster_size(int bw, int S) {
  cudaFuncSetAttribute(band_solve_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, band_solve_kernel);
  for (int C : {16, 8, 4, 2, 1}) {
    const size_t smem = band_smem_bytes(bw, C, S);
    if (smem + fa.sharedSizeBytes > 227 * 1024 || bw / C + 1 > 16) continue;
    if (cudaFuncSetAttribute(band_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kSolveThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, band_solve_kernel, &cfg) == cudaSuccess && clusters > 0) return C;
    cudaGetLastError();
  }
  return 0;
}

cudaError_t launch_band_solve(const BandDev& d, int C, const double* assembled, int num_pairs, double lam,
                              double lam2, int instances, int epoch, cudaStream_t s) {
  SolveArgs a;
  a.epoch = epoch;
  a.lam2 = lam2;
  a.instances = instances;
  a.d = d;
  a.diag = assembled;
  a.off = assembled + (size_t)d.S * 36;
  a.rhs = assembled + (size_t)(d.S + num_pairs) * 36;
  a.lam = lam;
  a.ns = std::max(d.bw / C + 1, 4);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C * instances);  // one cluster per damping value
  cfg.blockDim = dim3(kSolveThreads);
  cfg.dynamicSmemBytes = band_smem_bytes(d.bw, C, d.S);
  cfg.stream = s;
  // the > 48 KB opt-in is a per-function (per-device) attribute shared by every graph: set it for
  // THIS launch's size (another graph's plan may have left a smaller limit behind)
  if (const cudaError_t e = cudaFuncSetAttribute(band_solve_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      e != cudaSuccess)
    return e;
  if (const cudaError_t e = cudaFuncSetAttribute(band_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(cfg.dynamicSmemBytes));
      e != cudaSuccess)
    return e;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, band_solve_kernel, a);
}

}  // namespace vgicp
