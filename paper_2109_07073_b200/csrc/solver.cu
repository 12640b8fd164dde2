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
// shared memory, the others from L2 once the owner's release flag carries this launch's epoch;
// the owner of column j+1 applies panel j to it first, factors it (6×6 Cholesky, TRSM of the
// sub-diagonal blocks and of the augmented row) and publishes it (global memory + flag); every
// CTA applies panel j to its other columns in the window. No cluster barrier inside the loop:
// panels live in distinct global records, so the only cross-CTA dependencies are the flags.
// Afterwards CTA 0 runs the backward substitution (one warp, columns TMA-prefetched two ahead).
// Fixed operation order everywhere: results are deterministic.
//
// Measured on C3 (449 slots, RCM block bandwidth 31, 16-CTA cluster): 2.4 ms per damped solve vs
// 1.8 ms for the dense cuSOLVER potrf/potrs of the 2,694-dim system — the 449-step dependency
// chain (panel hand-off through L2 + 6×6 pivots) costs ~5k cycles per step. The dense path stays
// the LM's default up to 6,000 unknowns; the band solver takes over beyond (memory O(S·bw) instead
// of O(S²), time O(S·bw²) instead of O(S³)).
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
  int ns;     // column slots per CTA
  int epoch;  // this launch's value of the ready flags
};

// Zero column k's record, then scatter its blocks from the assembled system (damped diagonal,
// off-diagonal pairs — transposed where the order flips the pair — and the rhs row).
__device__ void load_columns(const SolveArgs& a, double* slots, int first, int last, int C, int rank) {
  const BandDev& d = a.d;
  const int cs = col_stride(d.bw);
  const int aug = col_aug(d.bw);
  for (int k = first; k <= last; k += C) {
    double* col = slots + (size_t)((k / C) % a.ns) * cs;
    const int n = 36 * (d.reach[k] - k + 1);
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
        if (t % 7 == 0) v = v + a.lam * fmax(v, 1e-10);
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
  // tasks per column: (R - k + 1)·6 rows + 1 augmented row
  int counts[16];
  int ncol = 0, total = 0;
  for (int k = lo; k <= hi && ncol < 16; k += C) {
    counts[ncol++] = (R - k + 1) * 6 + 1;
    total += counts[ncol - 1];
  }
  for (int t = threadIdx.x; t < total; t += kSolveThreads) {
    int c = 0, u = t;
    while (u >= counts[c]) u -= counts[c++];
    const int k = lo + c * C;
    double* col = slots + (size_t)((k / C) % a.ns) * cs;
    const double* Lk = pj + 36 * (k - j);
    const double* Li;
    double* dst;
    if (u < counts[c] - 1) {
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

// 1/sqrt(x) for the pivots: MUFU fp32 estimate + two fp64 Newton steps (~1 ulp), IEEE fallback
// outside the fp32 range.
__device__ __forceinline__ double rsqrt_fast(double x) {
  if (!(x > 1e-30 && x < 1e30)) return 1.0 / sqrt(x);
  double y = static_cast<double>(rsqrtf(static_cast<float>(x)));
  const double hx = 0.5 * x;
  y = y * (1.5 - hx * y * y);
  y = y * (1.5 - hx * y * y);
  return y;
}

// Factor column k in place (all threads of the CTA): 6×6 Cholesky of the diagonal block (warp
// 0; a pivot that is not > 0 fails like Eigen::LLT, block_solver.cpp:78-82), then
// L_ik = A_ik·L_kk⁻ᵀ for the sub-diagonal blocks and y_k = L_kk⁻¹·b_k for the augmented row.
__device__ void factor_column(const SolveArgs& a, double* col, int k) {
  const int aug = col_aug(a.d.bw);
  double* inv = col + aug + 8;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double row[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) row[c] = lane < 6 ? col[6 * lane + c] : 0.0;
    bool failed = false;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      // lane c: pivot; lanes > c: column entries
      double s = row[c];
#pragma unroll
      for (int m = 0; m < c; ++m) s -= row[m] * __shfl_sync(0xffffffffu, row[m], c);
      const double piv = __shfl_sync(0xffffffffu, s, c);
      if (!(piv > 0.0)) failed = true;  // warp-uniform
      const double il = rsqrt_fast(piv);
      const double l = piv * il;
      if (lane == c) row[c] = l;
      if (lane > c && lane < 6) row[c] = s * il;
      if (lane == 0) inv[c] = il;
    }
    if (lane < 6) {
#pragma unroll
      for (int c = 0; c < 6; ++c) col[6 * lane + c] = c <= lane ? row[c] : 0.0;
    }
    if (lane == 0) col[aug + 6] = failed ? 1.0 : 0.0;
  }
  __syncthreads();
  if (col[aug + 6] != 0.0) return;
  const int nrows = (a.d.reach[k] - k) * 6 + 1;  // sub-diagonal entry rows + the augmented row
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

__device__ void copy_record(double* __restrict__ dst, const double* __restrict__ src, int n) {
  const double2* s = reinterpret_cast<const double2*>(src);
  double2* o = reinterpret_cast<double2*>(dst);
  for (int t = threadIdx.x; t < n / 2; t += kSolveThreads) o[t] = s[t];
}

__global__ void __launch_bounds__(kSolveThreads, 1) band_solve_kernel(SolveArgs a) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) unsigned long long bbars[2];
  cg::cluster_group cluster = cg::this_cluster();  // a cluster launch guarantees the CTAs are co-resident
  const BandDev& d = a.d;
  const int C = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  const int S = d.S;
  const int cs = col_stride(d.bw);
  const int aug = col_aug(d.bw);
  double* slots = smem;                     // ns column records
  double* pj = smem + (size_t)a.ns * cs;    // the current panel
  const auto rec_len = [&](int k) { return 36 * (d.reach[k] - k + 1); };
  const auto panel_bytes = [&](int k) { return static_cast<unsigned>(sizeof(double) * (rec_len(k) + 16)); };
  const auto slot_of = [&](int k) { return slots + (size_t)((k / C) % a.ns) * cs; };

  if (threadIdx.x == 0) {
    bar_init(&bbars[0]);
    bar_init(&bbars[1]);
  }

  int next = rank;  // next owned column not yet loaded
  auto ensure_loaded = [&](int limit) {
    int last = next - C;
    while (last + C <= limit && last + C < S) last += C;
    if (last >= next) {
      load_columns(a, slots, next, last, C, rank);
      next = last + C;
    }
  };
  // Factored column k -> global memory, then a release flag (ready[k] = this launch's epoch).
  auto publish = [&](int k) {
    const double* col = slot_of(k);
    double* g = d.Lg + (size_t)k * cs;
    copy_record(g, col, rec_len(k));
    copy_record(g + aug, col + aug, 16);
    __syncthreads();  // the CTA's writes happen-before thread 0's (cumulative) release
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(d.ready + k), "r"(a.epoch) : "memory");
  };
  // Panel j -> pj: the owner copies its own column record; the others wait for the flag and read
  // the record from L2.
  auto receive = [&](int j) {
    if (j % C == rank) {
      const double* col = slot_of(j);
      copy_record(pj, col, rec_len(j));
      copy_record(pj + aug, col + aug, 16);
    } else {
      if (threadIdx.x == 0) {
        int v;
        do {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(d.ready + j) : "memory");
        } while (v != a.epoch);
      }
      __syncthreads();
      const double2* g = reinterpret_cast<const double2*>(d.Lg + (size_t)j * cs);
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
    ensure_loaded(max(d.reach[0], 0));
    if (rank == 0) {
      factor_column(a, slots, 0);
      publish(0);
    }
  }
  int failed_at = -1;
  long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // rank 0 / thread 0 cycle profile (VGICP_SOLVE_PROF)
  long long t0 = clock64(), t1;
#define VG_TICK(q) (t1 = clock64(), tp[q] += t1 - t0, t0 = t1)
  for (int j = 0; j < S; ++j) {
    const int R = d.reach[j];
    const int n1 = j + 1;
    receive(j);
    VG_TICK(0);
    if (pj[aug + 6] != 0.0) {  // the owner's pivot failed: every CTA leaves at the same step
      failed_at = j;
      break;
    }
    ensure_loaded(max(R, n1 < S ? n1 : -1));
    VG_TICK(1);
    // owned columns in (j, R]
    int lo = j + 1 + ((rank - (j + 1)) % C + C) % C;
    if (n1 < S && n1 % C == rank) {
      if (n1 <= R) {
        update_columns(a, slots, pj, j, R, n1, n1, C);
        __syncthreads();
      }
      VG_TICK(6);
      factor_column(a, slot_of(n1), n1);
      VG_TICK(7);
      publish(n1);
      lo = n1 + C;
    }
    VG_TICK(2);
    update_columns(a, slots, pj, j, R, lo, R, C);
    __syncthreads();
    VG_TICK(3);
  }
  if (failed_at >= 0 && rank == 0 && threadIdx.x == 0) *d.status = failed_at + 1;
  cluster.sync();  // every column published
  VG_TICK(4);
  if (failed_at >= 0 || rank != 0 || threadIdx.x >= 32) return;

  // ---- backward substitution Lᵀx = y (block_solver.cpp:108-114) by warp 0 of CTA 0: columns from
  //      the last one, each prefetched two ahead into shared memory by bulk copies; x kept in a
  //      ring of bw + 1 block rows; partial sums in a fixed lane order + xor tree ----
  const int lane = threadIdx.x;
  double* buf[2] = {slots, slots + cs};
  double* xr = slots + 2 * (size_t)cs;  // (bw + 1) × 6
  const int W = d.bw + 1;
  auto fetch = [&](int k) {
    const int q = (S - 1 - k) & 1;
    bar_expect(&bbars[q], panel_bytes(k));
    bulk_copy(buf[q], d.Lg + (size_t)k * cs, static_cast<unsigned>(sizeof(double) * rec_len(k)), &bbars[q]);
    bulk_copy(buf[q] + aug, d.Lg + (size_t)k * cs + aug, static_cast<unsigned>(sizeof(double) * 16), &bbars[q]);
  };
  asm volatile("fence.proxy.async;" ::: "memory");  // Lg / slots were written by generic stores
  __syncwarp();
  if (lane == 0) {
    if (S > 0) fetch(S - 1);
    if (S > 1) fetch(S - 2);
  }
  for (int k = S - 1; k >= 0; --k) {
    const int q = (S - 1 - k) & 1;
    bar_wait(&bbars[q], static_cast<unsigned>(((S - 1 - k) >> 1) & 1));
    const double* L = buf[q];
    const int nb = d.reach[k] - k;
    double s[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int t = lane; t < 6 * nb; t += 32) {
      const int bb = 1 + t / 6, r = t % 6;
      const double xv = xr[((k + bb) % W) * 6 + r];
      const double* Lr = L + 36 * bb + 6 * r;  // row r of L_{k+bb,k}
#pragma unroll
      for (int c = 0; c < 6; ++c) s[c] += Lr[c] * xv;
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s[c] += __shfl_xor_sync(0xffffffffu, s[c], off);
    }
    double x[6];
#pragma unroll
    for (int c = 5; c >= 0; --c) {
      double v = L[aug + c] - s[c];
#pragma unroll
      for (int r = c + 1; r < 6; ++r) v -= L[6 * r + c] * x[r];
      x[c] = v * L[aug + 8 + c];
    }
    if (lane < 6) {
      double xc = x[0];
#pragma unroll
      for (int c = 1; c < 6; ++c) xc = lane == c ? x[c] : xc;
      xr[(k % W) * 6 + lane] = xc;
      d.x[(size_t)d.perm[k] * 6 + lane] = xc;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0 && k >= 2) fetch(k - 2);
  }
  if (lane == 0) {
    *d.status = 0;
    VG_TICK(5);
    unsigned long long* prof = reinterpret_cast<unsigned long long*>(d.status) + 8;
    for (int q = 0; q < 8; ++q) prof[q] = static_cast<unsigned long long>(tp[q]);
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

size_t band_smem_bytes(int bw, int C) {
  const int ns = std::max(bw / C + 1, 3);  // >= 3: the backward substitution reuses the slot area
  const size_t rec = sizeof(double) * col_stride(bw);
  return (ns + 1) * rec;
}

// Largest cluster (16, else 8, 4, 2, 1) that can be co-resident with this bandwidth's window.
int band_cluster_size(int bw) {
  cudaFuncSetAttribute(band_solve_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, band_solve_kernel);
  for (int C : {16, 8, 4, 2, 1}) {
    const size_t smem = band_smem_bytes(bw, C);
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
                              int epoch, cudaStream_t s) {
  SolveArgs a;
  a.epoch = epoch;
  a.d = d;
  a.diag = assembled;
  a.off = assembled + (size_t)d.S * 36;
  a.rhs = assembled + (size_t)(d.S + num_pairs) * 36;
  a.lam = lam;
  a.ns = std::max(d.bw / C + 1, 3);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kSolveThreads);
  cfg.dynamicSmemBytes = band_smem_bytes(d.bw, C);
  cfg.stream = s;
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
