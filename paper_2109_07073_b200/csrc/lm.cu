// Native Levenberg-Marquardt for graphs of matching-cost factors (optimizer.cpp:88-194), driving
// the device path: every candidate is linearized + assembled on the GPU (one launch + the assembly
// launch); its per-factor errors — bit-identical to evaluate_matching_cost — give total_error
// (summed in factor order, optimizer.cpp:66-75), so an accepted candidate's normal equations are
// already assembled for the next iteration; the damped system is solved on the GPU by the
// block-band Cholesky (solve_block_system, block_solver.cpp:64-122) when its envelope fits a
// cluster, else on the host. Retraction, damping schedule, acceptance and termination follow
// optimizer.cpp:113-186 and se3.cpp:46-105 exactly.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace vgicp {
namespace {

constexpr double kSmallAngle = 1e-8;    // se3.cpp:10
constexpr int kOrthonormalizeEvery = 50;  // se3.cpp:11

// T = (R row-major 9, t 3)
void se3_exp(const double* xi, double* T) {  // se3.cpp:46-78
  const double w0 = xi[0], w1 = xi[1], w2 = xi[2];
  const double th = std::sqrt(w0 * w0 + w1 * w1 + w2 * w2);
  const double W[9] = {0.0, -w2, w1, w2, 0.0, -w0, -w1, w0, 0.0};
  double WW[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) WW[3 * r + c] = W[3 * r] * W[c] + W[3 * r + 1] * W[3 + c] + W[3 * r + 2] * W[6 + c];
  double a, b, cc;
  if (th < kSmallAngle) {
    a = 1.0, b = 0.5, cc = 1.0 / 6.0;
  } else {
    a = std::sin(th) / th;
    b = (1.0 - std::cos(th)) / (th * th);
    cc = (th - std::sin(th)) / (th * th * th);
  }
  double J[9];
  for (int k = 0; k < 9; ++k) {
    const double I = (k % 4 == 0) ? 1.0 : 0.0;
    T[k] = I + a * W[k] + b * WW[k];
    J[k] = I + b * W[k] + cc * WW[k];
  }
  for (int r = 0; r < 3; ++r) T[9 + r] = J[3 * r] * xi[3] + J[3 * r + 1] * xi[4] + J[3 * r + 2] * xi[5];
}

void compose(const double* A, const double* B, double* out) {  // se3.cpp:42-44
  double R[9], t[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) R[3 * r + c] = A[3 * r] * B[c] + A[3 * r + 1] * B[3 + c] + A[3 * r + 2] * B[6 + c];
    t[r] = A[3 * r] * B[9] + A[3 * r + 1] * B[10] + A[3 * r + 2] * B[11] + A[9 + r];
  }
  std::memcpy(out, R, sizeof(R));
  std::memcpy(out + 9, t, sizeof(t));
}

// Orthogonal polar factor of the rotation block (se3.cpp:80-91 takes U·Vᵀ of the SVD): Newton's
// iteration X <- (X + X⁻ᵀ)/2 converges quadratically to it from a near-rotation.
void orthonormalize(double* T) {
  double X[9];
  std::memcpy(X, T, sizeof(X));
  for (int it = 0; it < 8; ++it) {
    const double c00 = X[4] * X[8] - X[5] * X[7], c01 = X[5] * X[6] - X[3] * X[8], c02 = X[3] * X[7] - X[4] * X[6];
    const double c10 = X[2] * X[7] - X[1] * X[8], c11 = X[0] * X[8] - X[2] * X[6], c12 = X[1] * X[6] - X[0] * X[7];
    const double c20 = X[1] * X[5] - X[2] * X[4], c21 = X[2] * X[3] - X[0] * X[5], c22 = X[0] * X[4] - X[1] * X[3];
    const double det = X[0] * c00 + X[1] * c01 + X[2] * c02;
    if (!(std::fabs(det) > 0.0)) return;
    const double id = 1.0 / det;  // X⁻ᵀ = cofactor matrix / det
    const double Y[9] = {c00 * id, c01 * id, c02 * id, c10 * id, c11 * id, c12 * id, c20 * id, c21 * id, c22 * id};
    double diff = 0.0;
    for (int k = 0; k < 9; ++k) {
      const double v = 0.5 * (X[k] + Y[k]);
      diff = std::max(diff, std::fabs(v - X[k]));
      X[k] = v;
    }
    if (diff < 1e-16) break;
  }
  std::memcpy(T, X, sizeof(X));
}

struct DeviceScope {  // selects the context's device for the call, restores the caller's
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceScope() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};
struct PoolBuffer {  // stream-ordered device temporary (the context's pool)
  cudaStream_t s;
  void* p = nullptr;
  explicit PoolBuffer(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes, s); }
  ~PoolBuffer() {
    if (p) cudaFreeAsync(p, s);
  }
};

// Banded Cholesky solve of the damped system on the host: lower band storage of half-bandwidth w
// (scalars), LAPACK dpbtrf/dpbtrs arithmetic without blocking, O(m·w²); false when not positive
// definite. pos[slot] = the slot's block position in the factored order: the identity (slot order)
// for narrow systems such as odometry chains, the reverse Cuthill-McKee order of the solver plan
// when the envelope is too wide for the device band kernel. x is returned in slot order.
bool host_band_solve(int S, int P, const std::vector<int32_t>& pairs, const double* asmb, double lam, int w,
                     const std::vector<int>& pos, std::vector<double>& x) {
  const int m = 6 * S;
  const int W = w + 1;
  std::vector<double> B(static_cast<size_t>(m) * W, 0.0), b(m);  // B[i*W + (i - j)] = A(i, j), i >= j
  auto at = [&](int i, int j) -> double& { return B[static_cast<size_t>(i) * W + (i - j)]; };
  const double* diag = asmb;
  const double* off = asmb + static_cast<size_t>(S) * 36;
  const double* rhs = asmb + static_cast<size_t>(S + P) * 36;
  for (int s = 0; s < S; ++s)
    for (int r = 0; r < 6; ++r) {
      const int p = pos[s];
      for (int c = 0; c <= r; ++c) at(6 * p + r, 6 * p + c) = diag[36 * s + 6 * r + c];
      b[6 * p + r] = rhs[6 * s + r];
    }
  for (int q = 0; q < P; ++q) {  // (row a, col b) block of the slot-order system
    const int pa = pos[pairs[2 * q]], pb = pos[pairs[2 * q + 1]];
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) {
        const double v = off[36 * q + 6 * r + c];
        if (pa > pb) at(6 * pa + r, 6 * pb + c) = v;
        else at(6 * pb + c, 6 * pa + r) = v;  // the transposed block below the diagonal
      }
  }
  for (int k = 0; k < m; ++k) {
    double& d = at(k, k);
    d = d + lam * std::max(d, 1e-10);
  }
  for (int j = 0; j < m; ++j) {
    double d = at(j, j);
    const int k0 = std::max(0, j - w);
    for (int k = k0; k < j; ++k) d -= at(j, k) * at(j, k);
    if (!(d > 0.0)) return false;
    const double l = std::sqrt(d);
    at(j, j) = l;
    const int i1 = std::min(m - 1, j + w);
    for (int i = j + 1; i <= i1; ++i) {
      double v = at(i, j);
      const int kk = std::max(k0, i - w);
      for (int k = kk; k < j; ++k) v -= at(i, k) * at(j, k);
      at(i, j) = v / l;
    }
  }
  x.assign(m, 0.0);
  for (int i = 0; i < m; ++i) {
    double v = b[i];
    for (int k = std::max(0, i - w); k < i; ++k) v -= at(i, k) * x[k];
    x[i] = v / at(i, i);
  }
  for (int i = m - 1; i >= 0; --i) {
    double v = x[i];
    for (int k = i + 1; k <= std::min(m - 1, i + w); ++k) v -= at(k, i) * x[k];
    x[i] = v / at(i, i);
  }
  std::vector<double> xs(m);
  for (int s = 0; s < S; ++s)
    for (int r = 0; r < 6; ++r) xs[6 * s + r] = x[6 * pos[s] + r];
  x.swap(xs);
  return true;
}

int find_root(std::vector<int>& parent, int x) {
  while (parent[x] != x) x = parent[x] = parent[parent[x]];
  return x;
}

}  // namespace
}  // namespace vgicp

using namespace vgicp;

extern "C" int vgicp_graph_optimize(vgicp_graph graph, double* poses12, const uint8_t* fixed_in, int32_t* updates,
                                    const vgicp_lm_settings* settings_in, vgicp_lm_report* report, double* trace,
                                    int max_trace, double* iteration_seconds) try {
  if (!graph || !report || (graph->num_poses > 0 && !poses12)) return fail(VGICP_E_INVALID_ARGUMENT, "null argument");
  const auto t_start = std::chrono::steady_clock::now();
  auto seconds = [&]() { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count(); };
  vgicp_lm_settings st{50, 1e-5, 10.0, 0.1, 1e10, 1e-6, 1e-8};  // optimizer.hpp:12-21
  if (settings_in) st = *settings_in;
  std::memset(report, 0, sizeof(*report));
  report->reason = VGICP_LM_MAX_ITERATIONS;
  const int n = graph->num_poses;
  const int nf = graph->num_factors;
  if (n == 0) {
    report->reason = VGICP_LM_CONVERGED_STEP_NORM;
    return VGICP_OK;
  }
  // effective fixed mask (optimizer.cpp:24-43): the first pose of every component without a fixed pose
  std::vector<int> parent(n);
  for (int v = 0; v < n; ++v) parent[v] = v;
  for (int f = 0; f < nf; ++f) parent[find_root(parent, graph->tgt_idx[f])] = find_root(parent, graph->src_idx[f]);
  std::vector<uint8_t> fixed(n, 0), has(n, 0);
  for (int v = 0; v < n; ++v) fixed[v] = fixed_in ? (fixed_in[v] ? 1 : 0) : 0;
  for (int v = 0; v < n; ++v)
    if (fixed[v]) has[find_root(parent, v)] = 1;
  for (int v = 0; v < n; ++v) {
    const int r = find_root(parent, v);
    if (!has[r]) fixed[v] = 1, has[r] = 1;
  }
  int S = 0, P = 0;
  if (int rc = vgicp_graph_assembly_plan(graph, fixed.data(), &S, &P, nullptr)) return rc;
  std::vector<int32_t> pairs(2 * static_cast<size_t>(P));
  if (P > 0 && (vgicp_graph_assembly_plan(graph, fixed.data(), &S, &P, pairs.data()) != VGICP_OK))
    return VGICP_E_CUDA;
  std::vector<int> var_of_slot(S);
  {
    int active = 0;
    for (int v = 0; v < n; ++v) active += fixed[v] ? 0 : 1;
    for (int v = 0, rank = 0; v < n; ++v)
      if (!fixed[v]) var_of_slot[active - 1 - rank++] = v;  // block_solver.cpp:26-34
  }
  int bw = 0, band = 0;
  if (S > 0)
    if (int rc = vgicp_graph_solver_plan(graph, &bw, &band)) return rc;
  // Narrow systems in slot order (odometry chains: a factor links nearby variables) are cheaper on
  // the host — one small D2H and an O(m·w²) band Cholesky — than a cluster launch whose dependency
  // chain runs over every slot.
  int slot_bw = 0;
  for (int q = 0; q < P; ++q) slot_bw = std::max(slot_bw, pairs[2 * q] - pairs[2 * q + 1]);
  int host_w = 6 * slot_bw + 5;
  const bool host_band = S > 0 && static_cast<double>(6 * S) * host_w * host_w <= 2.0e6 &&
                         !std::getenv("VGICP_LM_NO_HOST_BAND");  // (test switch: force the device solver)
  std::vector<int> host_pos(S);
  for (int sl = 0; sl < S; ++sl) host_pos[sl] = sl;  // slot order
  if (S > 0 && !band && !host_band) {
    // the envelope is too wide for one cluster: host band solve in the plan's reverse Cuthill-McKee
    // order (O(m·w²) time, O(m·w) memory), refused beyond ~4 GB of band storage
    const BandPlanHost hp = make_band_plan(S, P, pairs.data());
    for (int k = 0; k < S; ++k) host_pos[hp.perm[k]] = k;
    host_w = 6 * hp.bw + 5;
    if (static_cast<double>(6 * S) * (host_w + 1) > 5.0e8)
      return fail(VGICP_E_OUT_OF_MEMORY, "reduced system too wide for the host band fallback (" + std::to_string(S) +
                                             " slots, block bandwidth " + std::to_string(hp.bw) + ")");
  }

  vgicp_ctx ctx = graph->ctx;
  DeviceScope g(ctx->device);
  cudaStream_t s = ctx->stream;
  const size_t asm_doubles = static_cast<size_t>(S + P) * 36 + static_cast<size_t>(S) * 6;
  PoolBuffer d_buf(s);
  VG_CUDA(d_buf.alloc(sizeof(double) * (2 * std::max<size_t>(asm_doubles, 1) + 12 * static_cast<size_t>(n))));
  double* d_asm[2] = {static_cast<double*>(d_buf.p), static_cast<double*>(d_buf.p) + std::max<size_t>(asm_doubles, 1)};
  double* d_poses = static_cast<double*>(d_buf.p) + 2 * std::max<size_t>(asm_doubles, 1);
  std::vector<double> err(nf);
  std::vector<int32_t> inl(nf);
  std::vector<double> host_asm;
  int solves = 0, lins = 0;
  // The device solver runs the damping value the LM would try next (lam · lambda_increase, after a
  // failed factorization or a rejected step on the same system) in the same launch, on a second
  // cluster; that result is kept here until the system in its buffer is overwritten.
  std::vector<double> x_pair;
  struct {
    int which = -1;
    double lam = 0.0;
    int solved = 0;
  } next;
  // linearize + assemble `at` into d_asm[which]; returns the total error (factor order)
  // VGICP_LM_CUDA_GRAPH=1: a candidate's linearization — poses H2D, the factor pass, the device
  // assembly into d_asm[which], the per-factor errors and inliers D2H — becomes one CUDA graph per
  // assembly buffer (captured on the second use, replayed after): one graph launch and one
  // synchronisation per candidate. Measured (tools/lm_cuda_graph_ab.py, profiles/lm_cuda_graph_r02.log):
  // no change in ms per iteration on C2 / C3 / C5 — the loop is kernel-bound (linearize + band
  // solve), not launch-bound — and ~3 ms of capture + instantiation per run, so it is off by default.
  // Plain graphs only (a sharded graph's pass spans several devices' streams).
  const bool use_cuda_graph = graph->shards.empty() && nf > 0 && std::getenv("VGICP_LM_CUDA_GRAPH") != nullptr;
  struct PinnedHost {
    void* p = nullptr;
    ~PinnedHost() {
      if (p) cudaFreeHost(p);
    }
  } pin;
  double* h_poses = nullptr;
  double* h_err = nullptr;
  int32_t* h_inl = nullptr;
  cudaGraphExec_t cg_exec[2] = {nullptr, nullptr};
  uint64_t cg_launches[2] = {0, 0};
  int cg_uses[2] = {0, 0};
  struct GraphExecs {
    cudaGraphExec_t* e;
    ~GraphExecs() {
      for (int k = 0; k < 2; ++k)
        if (e[k]) cudaGraphExecDestroy(e[k]);
    }
  } cg_guard{cg_exec};
  if (use_cuda_graph) {
    const size_t bp = sizeof(double) * 12 * n, be = sizeof(double) * nf;
    VG_CUDA(cudaMallocHost(&pin.p, bp + be + sizeof(int32_t) * nf + 64));
    h_poses = static_cast<double*>(pin.p);
    h_err = reinterpret_cast<double*>(static_cast<char*>(pin.p) + bp);
    h_inl = reinterpret_cast<int32_t*>(static_cast<char*>(pin.p) + bp + be);
  }
  auto enqueue_linearization = [&](int which) -> int {
    VG_CUDA(cudaMemcpyAsync(d_poses, h_poses, sizeof(double) * 12 * n, cudaMemcpyHostToDevice, s));
    if (int rc = vgicp_graph_linearize_assembled_device(graph, d_poses, d_asm[which])) return rc;
    VG_CUDA(cudaMemcpy2DAsync(h_err, sizeof(double), graph->d_out + (VGICP_LINEARIZED_DOUBLES - 1),
                              sizeof(double) * VGICP_LINEARIZED_DOUBLES, sizeof(double), nf, cudaMemcpyDeviceToHost,
                              s));
    VG_CUDA(cudaMemcpyAsync(h_inl, graph->d_out_inl, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost, s));
    return VGICP_OK;
  };
  auto linearize = [&](const std::vector<double>& at, int which, double* total) -> int {
    if (next.which == which) next.which = -1;  // the pending pair result's system is overwritten
    if (use_cuda_graph) {
      std::memcpy(h_poses, at.data(), sizeof(double) * 12 * n);
      if (cg_exec[which]) {
        VG_CUDA(cudaGraphLaunch(cg_exec[which], s));
        ctx->launches += cg_launches[which];
      } else if (cg_uses[which]++ == 0) {  // first use: direct (configures the kernels' attributes)
        if (int rc = enqueue_linearization(which)) return rc;
      } else {
        const uint64_t l0 = ctx->launches;
        cudaGraph_t cg = nullptr;
        VG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const int rc = enqueue_linearization(which);
        const cudaError_t ce = cudaStreamEndCapture(s, &cg);
        if (rc) {
          if (cg) cudaGraphDestroy(cg);
          return rc;
        }
        VG_CUDA(ce);
        const cudaError_t ie = cudaGraphInstantiate(&cg_exec[which], cg, 0);
        cudaGraphDestroy(cg);
        VG_CUDA(ie);
        cg_launches[which] = ctx->launches - l0;
        VG_CUDA(cudaGraphLaunch(cg_exec[which], s));
      }
      VG_CUDA(cudaStreamSynchronize(s));
      std::copy(h_err, h_err + nf, err.begin());
      std::copy(h_inl, h_inl + nf, inl.begin());
    } else {
      VG_CUDA(cudaMemcpyAsync(d_poses, at.data(), sizeof(double) * 12 * n, cudaMemcpyHostToDevice, s));
      if (int rc = vgicp_graph_linearize_assembled_device(graph, d_poses, d_asm[which])) return rc;
      if (int rc = vgicp_graph_linearized_errors(graph, err.data(), inl.data())) return rc;
    }
    double e = 0.0;
    for (int f = 0; f < nf; ++f) e += err[f];
    *total = e;
    ++lins;
    return VGICP_OK;
  };
  std::vector<double> x;
  const bool pair_solve = !std::getenv("VGICP_LM_NO_PAIR_SOLVE");
  auto solve = [&](int which, double lam, bool* ok) -> int {
    ++solves;
    x.assign(6 * static_cast<size_t>(S), 0.0);
    if (S == 0) {
      *ok = true;
      return VGICP_OK;
    }
    if (band && !host_band) {
      if (next.which == which && next.lam == lam) {  // solved by the previous launch
        next.which = -1;
        *ok = next.solved != 0;
        if (*ok) std::copy(x_pair.begin() + 6 * static_cast<size_t>(S), x_pair.end(), x.begin());
        return VGICP_OK;
      }
      if (pair_solve) {
        const double lams[2] = {lam, lam * st.lambda_increase};
        int solved[2] = {0, 0};
        x_pair.assign(12 * static_cast<size_t>(S), 0.0);
        if (int rc = vgicp_graph_solve_damped_pair(graph, d_asm[which], lams, x_pair.data(), solved)) return rc;
        next.which = which, next.lam = lams[1], next.solved = solved[1];
        *ok = solved[0] != 0;
        if (*ok) std::copy(x_pair.begin(), x_pair.begin() + 6 * static_cast<size_t>(S), x.begin());
        return VGICP_OK;
      }
      int solved = 0;
      if (int rc = vgicp_graph_solve_damped(graph, d_asm[which], lam, x.data(), &solved)) return rc;
      *ok = solved != 0;
      return VGICP_OK;
    }
    host_asm.resize(asm_doubles);
    VG_CUDA(cudaMemcpyAsync(host_asm.data(), d_asm[which], sizeof(double) * asm_doubles, cudaMemcpyDeviceToHost, s));
    VG_CUDA(cudaStreamSynchronize(s));
    *ok = host_band_solve(S, P, pairs, host_asm.data(), lam, host_w, host_pos, x);
    return VGICP_OK;
  };

  std::vector<double> poses(poses12, poses12 + 12 * static_cast<size_t>(n));
  std::vector<int32_t> upd(n, 0);
  if (updates) std::copy(updates, updates + n, upd.begin());
  int buf = 0;
  double current = 0.0;
  if (int rc = linearize(poses, buf, &current)) return rc;
  report->initial_error = report->final_error = current;
  double lam = st.lambda_init;
  bool any_accepted = false;
  int ntrace = 0;
  auto record = [&](int it, double e, double l, double step, bool acc) {
    if (trace && ntrace < max_trace) {
      double* r = trace + 5 * static_cast<size_t>(ntrace);
      r[0] = it, r[1] = e, r[2] = l, r[3] = step, r[4] = acc ? 1.0 : 0.0;
    }
    ++ntrace;
  };
  std::vector<double> cand(poses.size());
  std::vector<int32_t> cand_upd(n);
  double t_prev = seconds();
  NvtxRange nvtx_run("vgicp_graph_optimize");
  for (int it = 0; it < st.max_iterations; ++it) {
    NvtxRange nvtx_it("LM iteration");
    bool accepted = false;
    while (true) {
      bool ok = false;
      if (int rc = solve(buf, lam, &ok)) return rc;
      if (!ok) {
        lam *= st.lambda_increase;
        if (lam > st.lambda_max) {
          if (!any_accepted) {
            report->aborted = 1;
            report->reason = VGICP_LM_SOLVER_ABORT;
          } else {
            report->reason = VGICP_LM_LAMBDA_LIMIT;
          }
          break;
        }
        continue;
      }
      double step_sq = 0.0;
      for (double v : x) step_sq += v * v;
      const double step_norm = std::sqrt(step_sq);
      if (step_norm < st.step_norm_tolerance) {
        record(it, current, lam, step_norm, false);
        report->reason = VGICP_LM_CONVERGED_STEP_NORM;
        break;
      }
      cand = poses;
      cand_upd = upd;
      for (int sl = 0; sl < S; ++sl) {  // Pose::retract (se3.cpp:93-105)
        const int v = var_of_slot[sl];
        double E[12];
        se3_exp(&x[6 * static_cast<size_t>(sl)], E);
        compose(&poses[12 * static_cast<size_t>(v)], E, &cand[12 * static_cast<size_t>(v)]);
        if (++cand_upd[v] >= kOrthonormalizeEvery) {
          orthonormalize(&cand[12 * static_cast<size_t>(v)]);
          cand_upd[v] = 0;
        }
      }
      double cand_error = 0.0;
      if (int rc = linearize(cand, 1 - buf, &cand_error)) return rc;
      if (cand_error < current) {
        const double decrease = (current - cand_error) / std::max(current, 1e-300);
        poses.swap(cand);
        upd.swap(cand_upd);
        buf = 1 - buf;  // the candidate's system is the next iteration's
        any_accepted = accepted = true;
        record(it, cand_error, lam, step_norm, true);
        current = cand_error;
        lam = std::max(lam * st.lambda_decrease, 1e-12);
        ++report->iterations;
        if (decrease < st.relative_error_decrease) report->reason = VGICP_LM_CONVERGED_RELATIVE_ERROR;
        break;
      }
      record(it, current, lam, step_norm, false);
      lam *= st.lambda_increase;
      if (lam > st.lambda_max) {
        report->reason = VGICP_LM_LAMBDA_LIMIT;
        break;
      }
    }
    const double t_now = seconds();
    if (iteration_seconds) iteration_seconds[it] = t_now - t_prev;
    t_prev = t_now;
    report->iteration_count_timed = it + 1;
    if (!accepted || report->reason == VGICP_LM_CONVERGED_RELATIVE_ERROR) break;
    report->reason = VGICP_LM_MAX_ITERATIONS;
  }
  if (!report->aborted) {
    std::copy(poses.begin(), poses.end(), poses12);
    if (updates) std::copy(upd.begin(), upd.end(), updates);
    report->final_error = current;
  }
  report->trace_length = ntrace;
  report->solves = solves;
  report->linearizations = lins;
  report->band_solver = band && !host_band;
  report->wall_time_seconds = seconds();
  return VGICP_OK;
} catch (...) {
  return api_exception();
}
