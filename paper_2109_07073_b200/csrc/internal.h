// Host-side handle structures and launch entry points shared by the translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/vgicp_b200.h"
#include "vgicp_device.cuh"

namespace vgicp {

// NVTX range around a C ABI operation (header-only NVTX3: a no-op unless a profiler is attached),
// so nsys / ncu timelines show builds, overlap sweeps, factor passes, solves and LM iterations.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t err, const char* what);
// Every extern "C" entry point is a function-try-block ending in `catch (...) { return
// api_exception(); }`: no C++ exception crosses the ABI (std::bad_alloc -> VGICP_E_OUT_OF_MEMORY,
// anything else -> VGICP_E_CUDA with the message in vgicp_last_error()).
int api_exception() noexcept;

#define VG_CUDA(call)                                  \
  do {                                                 \
    const cudaError_t _e = (call);                     \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

// Work decomposition of a batched factor launch: one CTA per (factor, point chunk).
struct WorkItem {
  int factor;
  int begin;
  int end;
  int pad;
};

// Source clouds are also stored Morton-ordered in blocks of 64 points (one TMA bulk copy per
// 64-point tile of the factor kernel): SoA inside the block.
constexpr int kPointBlock = 64;
struct PointBlock {
  float4 pa[kPointBlock];  // x y z c_xx
  float4 pb[kPointBlock];  // c_xy c_xz c_yy c_yz
  float pc[kPointBlock];   // c_zz
};
static_assert(sizeof(PointBlock) % 128 == 0, "blocks must stay 128-B aligned");
// Clouds whose means are not float32-exact (submap clouds: transform_cloud + voxel_downsample output,
// pipeline.cpp:100-111; any float64 upload) also keep their float64 means in the same Morton blocks,
// SoA per block: x[64] | y[64] | z[64] | idx[64] (1,792 B). The probe kernels transform THESE values, so keys,
// correspondences and overlap hits stay bit-exact against the reference's double arithmetic.
// idx: each point's input index (its float64 covariance is c64[9 * idx]; read only by the factor
// kernels' near-singular path, which must decide on the exact float64 source covariance).
struct PointBlock64 {
  double x[kPointBlock];
  double y[kPointBlock];
  double z[kPointBlock];
  unsigned idx[kPointBlock];
};
static_assert(sizeof(PointBlock64) % 128 == 0, "blocks must stay 128-B aligned");

struct FactorDev {
  const PointBlock* blk;
  const PointBlock64* blk64;  // float64 means of the same blocks, or nullptr (float32-exact cloud)
  const double* c64;          // float64 covariances (n×9, input order) of a float64 cloud, else nullptr
  MapDev map;
  int n;
  int tgt;
  int src;
  int item_begin;
  int item_count;
  int pad;
};

// Per-map constants of the occupancy overlap kernel's fp32 screen (host-computed, staged in
// shared memory per CTA): fl32(R), fl32(t), fl32(1/r), the margin δ = A2·|p|₁ + C (A2 = 5e-7/r,
// C = A2·max|t| + 1e-7: a bound on |fl32 y - q/r| with the reference's fp64 rounding inside it),
// the occupied box (unbiased voxel coordinates) and its bitmap.
struct alignas(16) OccScreen {
  float R[9];
  float t[3];
  float inv_r, A2, C;
  int cx0, cy0, cz0;
  unsigned ex, ey, ez, nby, nbz;
  unsigned pad[2];
  const OccWord* occ;
};
static_assert(sizeof(OccScreen) == 112, "OccScreen is staged as 7 uint4");
struct OverlapItem {
  const PointBlock* blk;
  const PointBlock64* blk64;  // float64 means (nullptr: the float32 means are exact)
  MapDev map;
  OccDev occ;  // occupancy bitmap (occ.occ == nullptr: hash probes)
  double T[12];
  unsigned n;
  unsigned pad;
  OccScreen scr;
};
static_assert(offsetof(OverlapItem, scr) % 16 == 0 && sizeof(OverlapItem) % 16 == 0, "OccScreen is read as uint4");
cudaError_t launch_overlap_occ(const OverlapItem* items, const int2* chunks, int num_chunks, unsigned max_n,
                               unsigned long long* hits, cudaStream_t s);
// Device-side item preparation for a map set swept by one cloud: item k = templates[k] + pose k
// (fp64 T, fp32 screen, exact culling against the cloud box -> n = 0 when culled); chunks of 32.
cudaError_t launch_mapset_prepare(const OverlapItem* templates, int m, const double* poses12, const PointBlock* blk,
                                  const PointBlock64* blk64, unsigned n, const float* cloud_box, OverlapItem* items,
                                  int2* chunks, cudaStream_t s);
// Screen margin coefficient of the occupancy overlap kernel: |fl32 y - q/r| <= ~4.2e-7·|p|₁/r for
// float32 means, + 6e-8·|p|₁/r when the float32 means are roundings of float64 ones.
constexpr float kScreenA = 5e-7f;
constexpr float kScreenA64 = 6e-7f;
// Occupancy bitmap build job for one map (cold keys -> bits -> brick ranks -> rank-ordered stats).
struct OccJob {
  const unsigned long long* keys;
  OccWord* occ;
  SlotStatsA* ra;
  SlotStatsB* rb;
  unsigned V;
  unsigned words;
  unsigned kx0, ky0, kz0, nby, nbz;
  unsigned vbase;  // first voxel of this map in the build's VoxelStats array
};
cudaError_t launch_occ_build(const OccJob* jobs, int m, unsigned max_words, unsigned max_v, const VoxelStats* hot,
                             cudaStream_t s);

struct InsertJob;
// Hand-written build of one float32 cloud's map (build.cu). The occupied voxel box is known before
// any device work (floor(p/r) is monotone, so the box of the cloud's finite bounding box IS the box
// of its voxels), so the map's occupancy bitmap exists from the start: voxels are numbered by rank
// (brick order), never sorted by key.
struct FastBuildJob {
  const float4* pa;  // float32 cloud, input order (x y z c_xx | c_xy c_xz c_yy c_yz | c_zz)
  const float4* pb;
  const float* pc;
  unsigned n;        // points
  unsigned V;        // voxels (known after the rank pass)
  unsigned pt_off;   // first point of this map in the batch's per-point scratch
  unsigned vx_off;   // first CSR offset of this map in the batch's per-voxel scratch (V + 1 entries)
  double res, inv_res;
  unsigned kx0, ky0, kz0;  // biased key coordinates of the box's lower corner
  unsigned ex, ey, ez;     // box extent in voxels
  unsigned nby, nbz, words;
  OccWord* occ;            // the map's bitmap (words records)
  SlotStatsA* ra;          // outputs by rank: voxel-local fp32 statistics ...
  SlotStatsB* rb;          //   ... (c_zz, rank)
  double* cov9;            //   ... and the fp64 covariance (the near-singular path: 6 unique entries; 9 row-major in export mode)
  unsigned long long* keys;  // export mode (else nullptr): packed key, count and fp64 mean by rank
  int* counts;
  double* mean64;
};
cudaError_t launch_fast_mark(const FastBuildJob* jobs, int m, unsigned max_n, unsigned max_words, unsigned* code,
                             int* err, cudaStream_t s);
cudaError_t launch_fast_rank(const FastBuildJob* jobs, int m, unsigned* vcount, cudaStream_t s);
// zero + mark + rank in one CTA per map for jobs[0, count), whose bitmaps (<= max_words records)
// fit in shared memory; err / vcount are indexed like jobs
cudaError_t launch_fast_markrank_smem(const FastBuildJob* jobs, int count, unsigned max_words, unsigned* code,
                                      int* err, unsigned* vcount, cudaStream_t s);
unsigned fast_markrank_smem_words(int device);
// count + scan + stable input-order scatter, one CTA per map; `idx` lists the jobs of this launch;
// smem_v > 0: per-voxel cursors in shared memory for maps with V <= smem_v, else in `gcnt`
cudaError_t launch_fast_order(const FastBuildJob* jobs, const int* idx, int count, unsigned smem_v, const unsigned* code,
                              unsigned* rank, unsigned* list, unsigned* offs, unsigned* gcnt, cudaStream_t s);
// the same result (list, offs) by a shared-memory LSD radix sort, one CTA per map, for maps of
// <= fast_sort_max_points() points (the serial-scatter order kernel covers larger ones)
cudaError_t launch_fast_sort(const FastBuildJob* jobs, const int* idx, int count, unsigned max_n, const unsigned* code,
                             unsigned* list, unsigned* offs, cudaStream_t s);
unsigned fast_sort_max_points(int device);
cudaError_t launch_fast_accumulate(const FastBuildJob* jobs, int m, unsigned max_v, const unsigned* list,
                                   const unsigned* offs, const unsigned* code, bool export_mode, cudaStream_t s);
unsigned fast_order_smem_voxels(int device);
// hash table of a rank-numbered map, built on demand (lookups, hash-probe measurement modes):
// cuckoo insert of keys[rank], then each slot receives ra / rb of its rank
cudaError_t launch_place_rank(const InsertJob* job, unsigned V, const SlotStatsA* ra, const SlotStatsB* rb,
                              cudaStream_t s);

struct BuildSeg {
  const float4* pa;           // float32 device cloud (input order) ...
  const float4* pb;
  const float* pc;
  const double* xyz64;        // ... or fp64 points (n×3) + full fp64 covariances (n×9) when non-null
  const double* cov9;         //     (transformed / downsampled submap clouds, point_cloud.cpp:26-42)
  unsigned long long offset;  // start of this map's points in the concatenated arrays
  unsigned n;
  unsigned pad;
  double res;
  double inv_res;
};

struct BuildOut {       // cold fp64 statistics of one map (ascending key order)
  int* cbox;               // occupied voxel-coordinate bounds (min xyz, max xyz), atomics
  unsigned long long* keys;
  int* counts;
  double* mean64;
  double* cov64;
  unsigned vbase;          // global voxel id of this map's first voxel
  unsigned pad;
};

struct InsertJob {       // hash-table insertion of one map's voxels
  unsigned long long* tkeys;
  SlotStatsA* sa;
  SlotStatsB* sb;
  const unsigned long long* keys;  // cold keys (ascending)
  unsigned vbase;
  unsigned voxels;
  unsigned shift;
  unsigned pad;
};

struct CovSeg {          // covariance preprocessing of one cloud
  unsigned offset;       // first point in the concatenated arrays
  unsigned n;
  unsigned cell_base;    // first cell of this cloud in the global cell arrays
  int gx, gy, gz;
  double lo[3];
  double cell;
  double eps;
};

#ifndef VG_THREADS
#define VG_THREADS 256
#endif
constexpr int kFactorThreads = VG_THREADS;
constexpr int kFactorWarps = kFactorThreads / 32;
constexpr int kFactorTile = 512;    // work-item granularity in points (a multiple of the 64-point block)
constexpr int kDefaultChunk = 20480;  // points per CTA work item (one item per typical 20k-point factor)
constexpr int kLinAcc = 28;     // Q(6) P(9) Omega(6) b(6) error(1)
constexpr int kPartialStride = 32;

// ---- kernel launchers (return cudaError_t of the launch) ----
cudaError_t launch_build_keys(const BuildSeg* segs, int m, unsigned max_n, unsigned long long* keys, unsigned* vals,
                              int* range_err, cudaStream_t s);
cudaError_t launch_build_heads(const BuildSeg* segs, int m, unsigned max_n, const unsigned long long* keys,
                               unsigned* heads, cudaStream_t s);
cudaError_t launch_build_counts(const BuildSeg* segs, int m, const unsigned* heads, const unsigned* vidx,
                                unsigned* vcount, unsigned* vbase, cudaStream_t s);
cudaError_t launch_build_accumulate(const BuildSeg* segs, const BuildOut* outs, int m, unsigned max_n,
                                    const unsigned long long* keys, const unsigned* vals, const unsigned* heads,
                                    const unsigned* vidx, VoxelStats* hot, cudaStream_t s);
cudaError_t launch_build_insert(const InsertJob* jobs, int m, unsigned max_v, int* overflow, cudaStream_t s);
cudaError_t launch_build_place(const InsertJob* jobs, int m, unsigned max_v, const VoxelStats* hot, cudaStream_t s);
cudaError_t launch_lookup(MapDev map, const double* pts, size_t n, unsigned long long* keys_out, cudaStream_t s);
cudaError_t launch_overlap(const OverlapItem* items, int m, unsigned max_n, unsigned long long* hits, cudaStream_t s);
// items [0, f64_begin) belong to float32-exact source clouds, [f64_begin, num_items) to float64 clouds
// (one launch each; the float64 launch transforms the exact float64 means)
cudaError_t launch_factor(bool linearize, bool rank, const FactorDev* factors, const WorkItem* items, int num_items,
                          int f64_begin, const double* poses, double* partials, int* part_inl, unsigned* counters,
                          int num_factors, double* out, int* out_inl, cudaStream_t s);
cudaError_t launch_gicp_error(const double* in, double* out, cudaStream_t s);
// overlap probes grouped by cloud: chunk = (first item, count <= kOverlapMapsPerChunk) of items that
// share one cloud; each thread loads its points once and probes the chunk's maps
constexpr int kOverlapMapsPerChunk = 32;
cudaError_t launch_overlap_multi(const OverlapItem* items, const int2* chunks, int num_chunks, unsigned max_n,
                                 unsigned long long* hits, cudaStream_t s);
// assemble_normal_equations (block_solver.cpp:14-62) from F×121 factor blocks: output o < S is
// slot o's diagonal block (+ rhs), o >= S the off-diagonal pair o - S; contrib codes f·4 + kind
// (0 H_ii/b_i, 1 H_jj/b_j, 2 H_ij, 3 H_ijᵀ) listed per output in factor order.
// The blocks of factors [first[r], first[r + 1]) live at out[r] (factor first[r] + k at row k): the
// shards of a sharded graph, read over peer memory; a plain graph is one shard.
constexpr int kMaxShards = 8;
struct ShardBlocks {
  int n;
  int first[kMaxShards + 1];
  const double* out[kMaxShards];
};
cudaError_t launch_assemble(const int* out_ptr, const int* contrib, int num_slots, int num_outputs,
                            const ShardBlocks& blocks, double* assembled, cudaStream_t s);
// Damped block Cholesky of the assembled reduced system (solver.cu; solve_block_system,
// block_solver.cpp:64-122) over a reverse Cuthill-McKee order: perm[pos] = slot, reach[k] = last
// block row of column k's envelope, per-column lower blocks (col_ent.x = row offset | transposed
// << 16, .y = pair index) in CSR form.
struct BandPlanHost {
  int S = 0, bw = 0;
  std::vector<int> perm, reach, col_ptr;
  std::vector<int2> col_ent;
};
struct BandDev {
  int S, bw;
  const int* perm;
  const int* reach;
  const int* col_ptr;
  const int2* col_ent;
  double* Lg;   // S factored columns (band records), per instance (2 concurrent damping values)
  double* x;    // S×6 solution, slot order, per instance
  int* status;  // 0 solved, k + 1: pivot of position k failed (instance i at status + 64·i)
  int* ready;   // S publication flags (launch epoch), per instance
};
BandPlanHost make_band_plan(int S, int P, const int32_t* pairs);
size_t band_smem_bytes(int bw, int C, int S);
int band_cluster_size(int bw, int S);
cudaError_t launch_band_solve(const BandDev& d, int C, const double* assembled, int num_pairs, double lam,
                              double lam2, int instances, int epoch, cudaStream_t s);
// transform_cloud (point_cloud.cpp:26-42) of float32 device clouds into fp64 arrays, batched:
// item k maps cloud k's points (input order) through poses12[k] into out_xyz / out_cov9 at `offset`.
struct TransformItem {
  const float4* pa;
  const float4* pb;
  const float* pc;
  const double* xyz64;  // float64 means (n×3) + covariances (n×9) of a float64 cloud, else nullptr
  const double* cov9;
  unsigned long long offset;
  unsigned n;
  unsigned pad;
  double T[12];
};
cudaError_t launch_transform(const TransformItem* items, int m, unsigned max_n, double* out_xyz, double* out_cov9,
                             cudaStream_t s);
// float32 cloud from float64 device arrays (cloud.cu)
cudaError_t launch_cloud_bbox(const double* xyz, size_t n, unsigned* box, cudaStream_t s);
cudaError_t launch_cloud_morton(const double* xyz, size_t n, const unsigned* box, unsigned* codes, unsigned* idx,
                                cudaStream_t s);
cudaError_t launch_cloud_fill(const double* xyz, const double* cov9, size_t n, const unsigned* perm, float4* pa,
                              float4* pb, float* pc, PointBlock* blk, PointBlock64* blk64, cudaStream_t s);
cudaError_t launch_cloud_bbox(const float* xyz, size_t n, unsigned* box, cudaStream_t s);
cudaError_t launch_cloud_morton(const float* xyz, size_t n, const unsigned* box, unsigned* codes, unsigned* idx,
                                cudaStream_t s);
cudaError_t launch_cloud_fill(const float* xyz, const float* cov6, size_t n, const unsigned* perm, float4* pa,
                              float4* pb, float* pc, PointBlock* blk, cudaStream_t s);
// Batched float32 upload (vgicp_cloud_upload_batch): per cloud, the staged device input and its
// destination layout. prepare = bounding boxes (boxes[6k], pre-set to empty) + Morton codes / local
// indices at `offset`; fill = input-order SoA + Morton blocks from the per-cloud sorted permutation.
struct UploadSeg {
  const float* xyz;   // staged n×3 (device)
  const float* cov6;  // staged n×6 (device) or nullptr (raw cloud)
  unsigned offset;    // first point of this cloud in the batch (codes / permutation arrays)
  unsigned n;
  float4* pa;
  float4* pb;
  float* pc;
  PointBlock* blk;
};
cudaError_t launch_upload_batch_prepare(const UploadSeg* segs, int m, unsigned max_n, unsigned* boxes, unsigned* codes,
                                        unsigned* idx, cudaStream_t s);
cudaError_t launch_upload_batch_fill(const UploadSeg* segs, int m, unsigned max_n, const unsigned* perm, cudaStream_t s);
// the same for fp64 host-provided input arrays (already on device)
cudaError_t launch_transform64(const double* xyz, const double* cov9, size_t n, const double* T, double* out_xyz,
                               double* out_cov9, cudaStream_t s);
cudaError_t launch_cov_bbox(const CovSeg* segs, int m, unsigned max_n, const float* xyz, unsigned* box, int* bad,
                            cudaStream_t s);
cudaError_t launch_cov_count(const CovSeg* segs, int m, unsigned max_n, const float* xyz, unsigned* cell_of,
                             unsigned* cnt, cudaStream_t s);
cudaError_t launch_cov_scatter(const CovSeg* segs, int m, unsigned max_n, const float* xyz, const unsigned* cell_of,
                               const unsigned* start, unsigned* cursor, float4* sorted, cudaStream_t s);
cudaError_t launch_cov_knn(const CovSeg* segs, int m, unsigned max_n, const float* xyz, const unsigned* start,
                           const float4* sorted, int k, float* cov6, cudaStream_t s);

}  // namespace vgicp

struct vgicp_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint64_t launches = 0;
  // growable device scratch and pinned host staging
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
};

struct vgicp_cloud_s {
  vgicp_ctx ctx = nullptr;
  size_t n = 0;
  bool has_cov = false;
  void* block = nullptr;  // single allocation: pa | pb | pc (input order) | Morton-ordered PointBlocks
  size_t block_bytes = 0, block64_bytes = 0;  // allocation sizes (replication copies them whole)
  float4* pa = nullptr;   // input order: voxel-map builds accumulate in this order (voxelmap.cpp:87-94)
  float4* pb = nullptr;
  float* pc = nullptr;
  vgicp::PointBlock* sblk = nullptr;  // Morton (Z-order) copy in 64-point blocks: streamed by the factor /
                               // overlap kernels so that consecutive points probe neighbouring voxels
  float lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};  // bounding box of the finite points (lo > hi: none)
  // float64 clouds (means not float32-exact): exact input-order arrays for builds / transforms and
  // the Morton-ordered float64 means for the probe kernels; all nullptr for float32-exact clouds
  bool f64 = false;
  void* block64 = nullptr;  // m64 | c64 | blk64
  double* m64 = nullptr;    // n×3 input order
  double* c64 = nullptr;    // n×9 input order (nullptr for a raw cloud)
  vgicp::PointBlock64* blk64 = nullptr;
  std::atomic<int> refs{1};
};

struct vgicp_map_s {
  vgicp_ctx ctx = nullptr;
  double res = 1.0;
  double inv_res = 1.0;
  size_t voxels = 0;
  int cmin[3] = {0, 0, 0}, cmax[3] = {-1, -1, -1};  // occupied voxel-coordinate bounds
  size_t total_points = 0;
  unsigned num_buckets = 0;
  unsigned shift = 0;
  void* cold = nullptr;   // keys | counts | mean64 | cov64
  void* table = nullptr;  // tkeys | stats
  size_t cold_bytes = 0, table_bytes = 0, occ_bytes = 0;  // allocation sizes (replication copies them whole)
  unsigned long long* keys = nullptr;
  int* counts = nullptr;
  double* mean64 = nullptr;
  double* cov64 = nullptr;
  unsigned long long* tkeys = nullptr;
  vgicp::SlotStatsA* sa = nullptr;
  vgicp::SlotStatsB* sb = nullptr;
  void* occ_mem = nullptr;  // occupancy bitmap + rank-ordered statistics; null when the box is too large
  vgicp::OccDev occ{};
  vgicp::SlotStatsA* ra = nullptr;  // statistics by rank (brick order), for rank lookups
  vgicp::SlotStatsB* rb = nullptr;
  std::atomic<int> refs{1};
  // Maps of float32 clouds built by the hand-written path (build.cu): voxels numbered by rank only
  // (ra / rb / cov64 by rank, `cold` holds them), no key-ordered arrays and no hash
  // table until one is needed (ensure_table); export recomputes the key-ordered statistics from `src`
  // with the same kernels.
  bool fast = false;
  bool cov6 = false;          // cov64 holds the 6 unique entries per voxel (hand-built: symmetric inputs)
  vgicp_cloud src = nullptr;  // the source cloud (kept alive: export / on-demand hash table)
  // device descriptors carry cov64 tagged in bit 0 when it is 6-wide (vgicp::cov_row decodes it)
  const double* cov_dev() const {
    return cov6 ? reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(cov64) | 1u) : cov64;
  }
  vgicp::MapDev dev() const { return vgicp::MapDev{tkeys, sa, sb, cov_dev(), res, inv_res, shift, 0u, occ}; }
  // rank lookups: slot statistics replaced by the rank-ordered copies (requires occ)
  vgicp::MapDev dev_rank() const { return vgicp::MapDev{tkeys, ra, rb, cov_dev(), res, inv_res, shift, 0u, occ}; }
};

struct vgicp_mapset_s {
  vgicp_ctx ctx = nullptr;
  std::vector<vgicp_map> maps;
  bool all_occ = true;            // every map carries an occupancy bitmap (device path)
  int capacity = 0;               // maps the device block is laid out for (vgicp_mapset_append grows it)
  void* block = nullptr;          // templates | items | chunks | hits | poses
  vgicp::OverlapItem* d_templates = nullptr;
  vgicp::OverlapItem* d_items = nullptr;
  int2* d_chunks = nullptr;
  unsigned long long* d_hits = nullptr;
  double* d_poses = nullptr;
};

struct vgicp_graph_s {
  vgicp_ctx ctx = nullptr;
  int num_factors = 0;
  int num_poses = 0;
  int num_items = 0;
  int f64_begin = 0;  // first work item of a float64 source cloud (items of float32 clouds come first)
  uint64_t num_points = 0;
  void* block = nullptr;  // factors | items | partials | part_inl | counters | poses | out | out_inl | err
  vgicp::FactorDev* d_factors = nullptr;
  vgicp::WorkItem* d_items = nullptr;
  double* d_partials = nullptr;
  int* d_part_inl = nullptr;
  unsigned* d_counters = nullptr;  // per-factor arrival counters (cleared by each factor's last warp)
  double* d_poses = nullptr;
  double* d_out = nullptr;
  int* d_out_inl = nullptr;
  double* d_err = nullptr;
  std::vector<vgicp_cloud> clouds;
  std::vector<vgicp_map> maps;
  std::vector<int32_t> tgt_idx, src_idx;  // factor variables (target i, source j)
  // device-side normal-equation assembly plan (vgicp_graph_assembly_plan)
  void* plan = nullptr;  // out_ptr[O+1] | contrib[C] | assembled[(S+P)·36 + S·6]
  int num_slots = 0, num_pairs = 0;
  int* d_out_ptr = nullptr;
  int* d_contrib = nullptr;
  double* d_asm = nullptr;
  std::vector<int32_t> pair_ab;  // (row slot a, column slot b) per off-diagonal pair
  // band Cholesky solver plan (vgicp_graph_solver_plan)
  void* band = nullptr;  // perm | reach | col_ptr | col_ent | status | x | Lg
  vgicp::BandDev band_dev{};
  int band_cluster = 0;
  int band_bw = -1;
  int band_epoch = 0;
  bool rank_lookup = false;  // factor kernels probe occupancy bitmaps (every target map has one)
  // sharded graph (vgicp_graph_create_sharded): the shards are plain graphs, each on its own
  // context, linearizing factors [shard_first[r], shard_first[r + 1]); this graph (on shard 0's
  // context, the root) plans, assembles (reading the shards' blocks over peer memory) and solves
  std::vector<vgicp_graph> shards;
  std::vector<int> shard_first;
  std::vector<cudaEvent_t> shard_events;  // on each shard's stream: its pass is done
  cudaEvent_t root_event = nullptr;       // on the root stream: the poses are in place
  bool peer_ok = true;                    // the root can read every shard's memory directly
  vgicp::ShardBlocks blocks() const {
    vgicp::ShardBlocks b{};
    if (shards.empty()) {
      b.n = 1;
      b.first[0] = 0;
      b.first[1] = num_factors;
      b.out[0] = d_out;
      return b;
    }
    b.n = static_cast<int>(shards.size());
    for (int r = 0; r <= b.n; ++r) b.first[r] = shard_first[r];
    for (int r = 0; r < b.n; ++r) b.out[r] = peer_ok ? shards[r]->d_out : d_out + (size_t)shard_first[r] * 121;
    return b;
  }
};
