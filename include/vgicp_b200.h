/*
 * vgicp_b200 — C ABI of the B200-native (sm_100a) VGICP matching-cost path.
 *
 * This is the drop-in boundary for the reference's hot path (/root/reference/proj):
 *   GaussianVoxelMap            include/vgicp/voxelmap.hpp:28-56, src/voxelmap.cpp:65-117
 *   overlap_rate                include/vgicp/voxelmap.hpp:60-61, src/voxelmap.cpp:119-135
 *   MatchingCostFactor          include/vgicp/factors.hpp:36-45, src/factors.cpp:50-67
 *   linearize_matching_cost     include/vgicp/factors.hpp:76-77, src/factors.cpp:90-148
 *   evaluate_matching_cost      include/vgicp/factors.hpp:80-81, src/factors.cpp:150-181
 *   gicp_error                  include/vgicp/factors.hpp:70,    src/factors.cpp:75-88
 * plus the batch entry points the paper's "issue all cost evaluations, sync, collect" needs
 * (SURVEY.md §8b): one launch linearizes / evaluates every matching-cost factor of a graph, the
 * integration point of linearize_all / total_error (src/optimizer.cpp:45-75).
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross this boundary, and no
 *    exception either: every call returns a vgicp_status and vgicp_last_error() (thread-local)
 *    holds the message. The reference's std::invalid_argument maps to
 *    VGICP_E_INVALID_ARGUMENT and std::out_of_range to VGICP_E_OUT_OF_RANGE.
 *  - A pose is 12 doubles: row-major rotation R (9) followed by the translation t (3), i.e.
 *    Pose{rotation, translation} of include/vgicp/se3.hpp:33-56.
 *  - Point means are float32 (KITTI .bin precision, src/io.cpp:50); covariances are the six
 *    unique float32 entries (xx, xy, xz, yy, yz, zz) of a symmetric 3×3. The _f64 upload
 *    variant accepts the reference's double layout and keeps float64 values when they are not
 *    float32-exact (float64 clouds).
 *  - A linearized factor is VGICP_LINEARIZED_DOUBLES doubles, the fields of LinearizedFactor
 *    (include/vgicp/factors.hpp:19-29) in order: H_ii(6×6) H_ij(6×6) H_jj(6×6) b_i(6) b_j(6)
 *    error(1), matrices row-major; inlier counts are returned separately as int32.
 *    Block i is the factor's target variable, j its source variable (src/factors.cpp:137-138).
 *  - Every device-side result is deterministic: reductions run in a fixed order, so repeated
 *    calls on identical inputs return bit-identical outputs.
 *  - One host thread drives a context (the optimizer is not reentrant either).
 *    Handles keep what they reference alive (reference counts), like the reference's
 *    shared_ptr<const ...> members.
 */
#ifndef VGICP_B200_H
#define VGICP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VGICP_LINEARIZED_DOUBLES 121
#define VGICP_KEY_MISS UINT64_MAX

typedef enum vgicp_status {
  VGICP_OK = 0,
  VGICP_E_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  VGICP_E_OUT_OF_RANGE = 2,     /* std::out_of_range (voxelmap.cpp:49-51) */
  VGICP_E_CUDA = 3,             /* CUDA runtime / launch failure */
  VGICP_E_NO_DEVICE = 4,        /* no usable sm_100 device */
  VGICP_E_OUT_OF_MEMORY = 5
} vgicp_status;

typedef struct vgicp_ctx_s* vgicp_ctx;
typedef struct vgicp_cloud_s* vgicp_cloud;
typedef struct vgicp_map_s* vgicp_map;
typedef struct vgicp_graph_s* vgicp_graph;
typedef struct vgicp_mapset_s* vgicp_mapset;

/* MatchingCostFactor (include/vgicp/factors.hpp:36-45): the older frame owns the map
 * (target), the newer frame supplies the points (source). */
typedef struct vgicp_factor_desc {
  int32_t target_index;
  int32_t source_index;
  vgicp_cloud source;
  vgicp_map target;
} vgicp_factor_desc;

/* ---------------------------------------------------------------- library / context */
const char* vgicp_last_error(void);
const char* vgicp_version(void);
int vgicp_device_count(int* count);

/* One context per device; it owns a CUDA stream (or adopts `stream` when non-NULL). */
int vgicp_ctx_create(int device, void* stream, vgicp_ctx* out);
int vgicp_ctx_destroy(vgicp_ctx ctx);
/* One context per device of devices[0, n) (each with its own stream): the contexts of a sharded
 * graph. All-or-nothing. */
int vgicp_ctx_create_multi(const int* devices, int n, vgicp_ctx* out);
int vgicp_ctx_stream(vgicp_ctx ctx, void** stream);
int vgicp_ctx_synchronize(vgicp_ctx ctx);
/* Kernels this context has launched so far (bench evidence for gpu_launches). */
int vgicp_ctx_launch_count(vgicp_ctx ctx, uint64_t* launches);

/* ---------------------------------------------------------------- point clouds (PointCloud,
 * include/vgicp/point_cloud.hpp:21-37). cov6 may be NULL for a raw cloud (overlap only). */
int vgicp_cloud_upload(vgicp_ctx ctx, const float* xyz, const float* cov6, size_t n, vgicp_cloud* out);
/* m clouds in one call (one staged copy, one launch per layout stage for the whole batch): out[k] equals
 * vgicp_cloud_upload(xyz[k], cov6[k] (cov6 or cov6[k] may be NULL), n[k]). All-or-nothing. */
int vgicp_cloud_upload_batch(vgicp_ctx ctx, const float* const* xyz, const float* const* cov6, const size_t* n, int m,
                             vgicp_cloud* out);
/* Reference layout: n×3 double means, n×9 double covariances (may be NULL). Float32-exact inputs
 * with symmetric covariances take the float32 layout; any other input (e.g. submap clouds, the output
 * of transform_cloud + voxel_downsample, pipeline.cpp:100-111) is a float64 cloud: its exact values
 * drive every key, correspondence, overlap hit and map statistic (bit-exact against the reference's
 * double arithmetic); only the per-hit H/b algebra reads float32 copies. */
int vgicp_cloud_upload_f64(vgicp_ctx ctx, const double* xyz, const double* cov9, size_t n, vgicp_cloud* out);
/* 1 when the cloud keeps float64 values (see vgicp_cloud_upload_f64), else 0. */
int vgicp_cloud_is_f64(vgicp_cloud cloud, int* f64);
int vgicp_cloud_size(vgicp_cloud cloud, size_t* n);
int vgicp_cloud_has_covariances(vgicp_cloud cloud, int* has);
int vgicp_cloud_destroy(vgicp_cloud cloud);
/* The cloud's device layout copied to ctx's device (peer copy over NVLink; through the host when the
 * devices cannot reach each other): the replicas of a sharded graph, identical in every bit. */
int vgicp_cloud_replicate(vgicp_cloud cloud, vgicp_ctx ctx, vgicp_cloud* out);

/* ---------------------------------------------------------------- Gaussian voxel maps */
/* GaussianVoxelMap(cloud, resolution) — voxelmap.cpp:65-104. Errors: resolution <= 0 or a
 * cloud without covariances -> INVALID_ARGUMENT; a coordinate beyond ±2^20 voxels, a NaN / Inf
 * point or a NaN resolution -> OUT_OF_RANGE (and no map), in the reference's check order. One
 * deviation: resolution = +inf (the reference maps every point to voxel 0) -> INVALID_ARGUMENT. */
int vgicp_voxelmap_build(vgicp_ctx ctx, vgicp_cloud cloud, double resolution, vgicp_map* out);
/* m maps in one batched build (all-or-nothing: on error no map is returned). */
int vgicp_voxelmap_build_batch(vgicp_ctx ctx, const vgicp_cloud* clouds, const double* resolutions, int m,
                               vgicp_map* out);
int vgicp_voxelmap_destroy(vgicp_map map);
/* The map (bitmap, statistics, tables) copied to ctx's device — one transfer per map instead of a
 * rebuild per device (maps are immutable); factor results are bit-identical. */
int vgicp_voxelmap_replicate(vgicp_map map, vgicp_ctx ctx, vgicp_map* out);
int vgicp_voxelmap_size(vgicp_map map, size_t* voxels);                 /* voxelmap.hpp:36 */
int vgicp_voxelmap_resolution(vgicp_map map, double* resolution);       /* voxelmap.hpp:35 */
int vgicp_voxelmap_total_points(vgicp_map map, size_t* total_points);   /* voxelmap.hpp:49 */
/* voxels() (voxelmap.hpp:47) in ascending key order: keys[V], counts[V], means[V×3],
 * covs[V×9] (row-major, float64 statistics). Any pointer may be NULL. */
int vgicp_voxelmap_export(vgicp_map map, uint64_t* keys, int32_t* counts, double* means, double* covs);
/* lookup() (voxelmap.cpp:106-117) for n points (n×3 double): the packed key of the
 * populated voxel containing each point, VGICP_KEY_MISS when absent or out of range. */
int vgicp_voxelmap_lookup(vgicp_map map, const double* points, size_t n, uint64_t* keys_out);
/* voxel_coord + pack_key (voxelmap.cpp:45-63) on the host; OUT_OF_RANGE beyond ±2^20. */
int vgicp_voxel_key(double resolution, const double point[3], uint64_t* key);
/* GaussianVoxelMap over a float64 cloud (the reference's PointCloud layout: n×3 means, n×9
 * covariances, all 9 entries accumulated) — voxelmap.cpp:65-104. With vgicp_voxelmap_export this
 * is voxel_downsample (voxelmap.cpp:137-169): one point per voxel, ascending packed-key order. */
int vgicp_voxelmap_build_f64(vgicp_ctx ctx, const double* xyz, const double* cov9, size_t n, double resolution,
                             vgicp_map* out);

/* ---------------------------------------------------------------- submap creation (§8f #2) */
/* transform_cloud (point_cloud.cpp:26-42) in float64 on the device: out = T.apply(mean),
 * out_cov = R·C·Rᵀ (full 9 entries). cov9 / out_cov9 may be NULL (means only). */
int vgicp_transform_cloud(vgicp_ctx ctx, const double* xyz, const double* cov9, size_t n, const double pose[12],
                          double* out_xyz, double* out_cov9);
/* The submap creation path of MappingPipeline::emit_submap (pipeline.cpp:92-114), on the device:
 * every frame k transformed by poses12[k] (frame -> submap) in float64 and merged in frame order,
 * voxel_downsample'd at downsample_resolution (skipped when <= 0), and the submap's voxel map built
 * at map_resolution from the float64 downsampled cloud. Optional outputs: out_downsampled (the
 * downsample map: export() = the submap cloud in float64, ascending key order) and out_cloud (that
 * cloud as a float64 device cloud, the source of submap-level factors and overlap probes). */
int vgicp_submap_build(vgicp_ctx ctx, const vgicp_cloud* frames, const double* poses12, int m,
                       double downsample_resolution, double map_resolution, vgicp_map* out_downsampled,
                       vgicp_cloud* out_cloud, vgicp_map* out_map);

/* ---------------------------------------------------------------- overlap (Eq. 7/8) */
/* overlap_rate(cloud, pose_rel, map) — voxelmap.cpp:119-135. Exact hits / N. */
int vgicp_overlap_rate(vgicp_ctx ctx, vgicp_cloud cloud, const double pose_rel[12], vgicp_map map, double* rate);
/* m independent (cloud, pose, map) probes in one launch; hits[k] is the exact hit count. */
int vgicp_overlap_batch(vgicp_ctx ctx, const vgicp_cloud* clouds, const double* poses12, const vgicp_map* maps,
                        int m, uint64_t* hits);
/* A fixed sequence of maps kept on the device (the keyframe database of pipeline.cpp:135-150):
 * vgicp_overlap_mapset sweeps ONE cloud against all of them — per-probe items are built and culled
 * on the device from the m poses (rel12: T_map⁻¹·T_cloud, m × 12), so a sweep costs one pose upload,
 * two launches and the hit download. Results equal vgicp_overlap_batch's. The set holds references
 * to its maps. */
int vgicp_mapset_create(vgicp_ctx ctx, const vgicp_map* maps, int m, vgicp_mapset* out);
/* Adds maps at the end of the set (a new keyframe's map): amortised O(1) device work per map (the
 * device block grows geometrically); earlier maps keep their positions in hits[]. */
int vgicp_mapset_append(vgicp_mapset set, const vgicp_map* maps, int m);
int vgicp_mapset_size(vgicp_mapset set, int* size);
int vgicp_mapset_destroy(vgicp_mapset set);
int vgicp_overlap_mapset(vgicp_ctx ctx, vgicp_cloud cloud, const double* rel12, vgicp_mapset set, uint64_t* hits);

/* ---------------------------------------------------------------- matching cost factors */
/* linearize_matching_cost (factors.cpp:90-148) for one factor. */
int vgicp_linearize_matching_cost(vgicp_ctx ctx, const vgicp_factor_desc* factor, const double T_target[12],
                                  const double T_source[12], double out[VGICP_LINEARIZED_DOUBLES],
                                  int32_t* inliers);
/* evaluate_matching_cost (factors.cpp:150-181) for one factor. */
int vgicp_evaluate_matching_cost(vgicp_ctx ctx, const vgicp_factor_desc* factor, const double T_target[12],
                                 const double T_source[12], double* error, int32_t* inliers);
/* gicp_error (factors.cpp:75-88): covariances as full row-major 3×3. */
int vgicp_gicp_error(vgicp_ctx ctx, const double source_mean[3], const double source_cov[9],
                     const double target_mean[3], const double target_cov[9], const double T[12], double* error,
                     double residual[3], double information[9], int* valid);

/* ---------------------------------------------------------------- batched factor graphs */
/* A fixed set of matching-cost factors over num_poses pose variables. Validation mirrors the
 * MatchingCostFactor constructor (factors.cpp:57-66): distinct variables, non-empty source with
 * covariances, non-empty target map; indices must lie in [0, num_poses). `chunk` is the number
 * of source points per CTA work item (0 = default 20480; rounded up to a multiple of 512). */
int vgicp_graph_create(vgicp_ctx ctx, const vgicp_factor_desc* factors, int num_factors, int num_poses, int chunk,
                       vgicp_graph* out);
int vgicp_graph_destroy(vgicp_graph graph);
/* The graph of factors [first, first + count) of the list, with the work decomposition of the WHOLE
 * list (so every per-factor block is bit-identical to vgicp_graph_create's): one rank's share of a
 * factor graph split across processes. Its blocks are indexed 0..count-1 (factor first + k at k);
 * plan / assemble / solve with a whole-list graph (vgicp_graph_assemble_device). */
int vgicp_graph_create_range(vgicp_ctx ctx, const vgicp_factor_desc* factors, int num_factors, int num_poses,
                             int chunk, int first, int count, vgicp_graph* out);
/* Multi-GPU split of ONE graph behind the C ABI (the loops of optimizer.cpp:53-56 /
 * :68-70 over factors): factors[r] is the factor list with context r's handles — the same factors,
 * their clouds / maps replicated on context r's device (contexts may share a device). Shard r
 * linearizes a contiguous, point-balanced factor range with the whole list's work decomposition;
 * context 0 is the root: it plans, assembles — its assembly kernel reads the shards' blocks in place
 * over peer memory (NVLink) — and solves, so assembled systems, errors and the native LM's trace are
 * bit-identical to a single-context graph. Every vgicp_graph_* call accepts the result (the
 * _device variants take and return root-device memory). At most 8 shards. */
int vgicp_graph_create_sharded(const vgicp_ctx* ctxs, int num_shards, const vgicp_factor_desc* const* factors,
                               int num_factors, int num_poses, int chunk, vgicp_graph* out);
int vgicp_graph_num_shards(vgicp_graph graph, int* num_shards);
int vgicp_graph_shard_range(vgicp_graph graph, int shard, int* first, int* count);
int vgicp_graph_num_factors(vgicp_graph graph, int* num_factors);
/* Σ source points over the graph's factors (the per-pass point-evaluation count). */
int vgicp_graph_num_points(vgicp_graph graph, uint64_t* points);
/* linearize_all for matching factors (optimizer.cpp:45-62): host poses in, host blocks out
 * (num_factors × VGICP_LINEARIZED_DOUBLES, factor order), synchronous. */
int vgicp_graph_linearize(vgicp_graph graph, const double* poses12, double* out, int32_t* inliers);
/* Per-factor errors / inliers for total_error (optimizer.cpp:66-75), synchronous. */
int vgicp_graph_evaluate(vgicp_graph graph, const double* poses12, double* errors, int32_t* inliers);
/* Device-side normal-equation assembly (§8f #3; assemble_normal_equations, block_solver.cpp:14-62).
 * vgicp_graph_assembly_plan fixes the variable mask (fixed[num_poses], non-zero = fixed): active
 * variables get slots in reverse insertion order (slot 0 = last active variable, :26-34); the
 * distinct off-diagonal blocks are the slot pairs (a > b) in ascending (b, a) order — written to
 * pairs[2·P] as (a, b) when pairs != NULL (call once with NULL to size it).
 * vgicp_graph_linearize_assembled runs one linearization pass and assembles on the device:
 * diag[S×36] = Σ H_ii / H_jj per slot, offdiag[P×36] = Σ H_ij (or H_ijᵀ) per pair, stored as the
 * (row a, col b) block, rhs[S×6] = Σ b_i / b_j — each summed in factor order from zero, i.e.
 * bit-identical to the reference's assembly of the same factor blocks. Only S·42 + P·36 doubles
 * cross PCIe instead of F·121. */
int vgicp_graph_assembly_plan(vgicp_graph graph, const uint8_t* fixed, int* num_slots, int* num_pairs, int32_t* pairs);
int vgicp_graph_linearize_assembled(vgicp_graph graph, const double* poses12, double* diag, double* offdiag,
                                    double* rhs);
/* Device-resident variant (enqueued on the context stream, no synchronisation): d_poses12 and
 * d_assembled are device memory; d_assembled receives [diag S×36 | offdiag P×36 | rhs S×6]. */
int vgicp_graph_linearize_assembled_device(vgicp_graph graph, const double* d_poses12, double* d_assembled);
/* Per-factor errors and inliers of the most recent vgicp_graph_linearize_assembled[_device] pass
 * (the `error` / `inliers` members of each LinearizedFactor, factors.hpp:27-28), synchronous.
 * They equal vgicp_graph_evaluate at the same poses bit for bit (same per-point arithmetic and
 * reduction order), so an LM can score a candidate with the linearization it needs anyway if the
 * candidate is accepted (total_error, optimizer.cpp:66-75 + linearize_all, :45-62). */
int vgicp_graph_linearized_errors(vgicp_graph graph, double* errors, int32_t* inliers);
/* Assembly (as vgicp_graph_linearize_assembled_device) of externally provided blocks: d_blocks holds
 * num_factors × VGICP_LINEARIZED_DOUBLES doubles in factor order on the context's device — e.g. the
 * blocks of every rank's vgicp_graph_create_range share, gathered over NCCL. */
int vgicp_graph_assemble_device(vgicp_graph graph, const double* d_blocks, double* d_assembled);
/* Damped solve of the assembled reduced system on the GPU (solve_block_system,
 * block_solver.cpp:64-122, with the Marquardt damping of optimizer.cpp:119-123: diagonal entries
 * d -> d + lambda·max(d, 1e-10)). vgicp_graph_solver_plan (after vgicp_graph_assembly_plan)
 * orders the slots by reverse Cuthill-McKee and reports the block bandwidth of the envelope;
 * supported = 0 when the envelope window does not fit one thread-block cluster's shared memory
 * (the caller then solves densely). vgicp_graph_solve_damped factors [diag | offdiag | rhs] as
 * written by vgicp_graph_linearize_assembled_device (device memory) with right-looking 6×6-block
 * Cholesky in one cluster launch and returns x[S×6] in slot order on the host; solved = 0 when a
 * pivot block is not positive definite (the reference's failed_slot, the LM then raises lambda). */
int vgicp_graph_solver_plan(vgicp_graph graph, int* bandwidth, int* supported);
int vgicp_graph_solve_damped(vgicp_graph graph, const double* d_assembled, double lambda, double* x, int* solved);
/* Two damping values in one launch (two clusters run concurrently): x receives 2 × S×6 doubles and
 * solved[2] the two outcomes — an LM that fails or rejects at lambdas[0] continues with lambdas[1]
 * without another solve. */
int vgicp_graph_solve_damped_pair(vgicp_graph graph, const double* d_assembled, const double* lambdas, double* x,
                                  int* solved);

/* ---------------------------------------------------------------- native Levenberg-Marquardt */
/* optimize (optimizer.cpp:88-194) for a graph whose factors are all matching-cost factors, in the
 * library: every candidate is linearized + assembled on the device and scored by its per-factor
 * errors (= total_error), the damped system is solved on the device (block-band Cholesky) or on the
 * host (a band Cholesky: in slot order for narrow systems such as odometry chains, in the reverse
 * Cuthill-McKee order when the envelope is too wide for the device kernel — the device kernel covers
 * envelopes up to ~80 blocks, e.g. C5's 1,000 poses need 47; systems whose host band storage would
 * exceed ~4 GB return VGICP_E_OUT_OF_MEMORY), Pose::retract (se3.cpp:93-105) on the host. Same damping schedule, acceptance rule,
 * termination reasons and gauge anchoring (effective_fixed_mask, optimizer.cpp:24-43) as the
 * reference. poses12 (num_poses × 12) is updated in place unless the solve aborts; fixed (may be
 * NULL) marks user-fixed poses; updates (may be NULL) carries each pose's
 * updates_since_orthonormalization in and out. trace (may be NULL) receives up to max_trace
 * IterationRecords as 5 doubles (iteration, error, lambda, step_norm, accepted);
 * iteration_seconds (may be NULL, >= max_iterations entries) the wall time of each outer iteration. */
typedef struct vgicp_lm_settings { /* LmSettings, optimizer.hpp:12-21 */
  int max_iterations;
  double lambda_init, lambda_increase, lambda_decrease, lambda_max;
  double relative_error_decrease, step_norm_tolerance;
} vgicp_lm_settings;
enum { /* TerminationReason, optimizer.hpp:23-29 (same order) */
  VGICP_LM_CONVERGED_RELATIVE_ERROR = 0,
  VGICP_LM_CONVERGED_STEP_NORM = 1,
  VGICP_LM_MAX_ITERATIONS = 2,
  VGICP_LM_LAMBDA_LIMIT = 3,
  VGICP_LM_SOLVER_ABORT = 4
};
typedef struct vgicp_lm_report { /* OptimizerReport, optimizer.hpp:41-50 (+ counters) */
  int iterations;               /* accepted re-linearizations */
  double initial_error, final_error;
  int reason;                   /* VGICP_LM_* */
  int aborted;
  double wall_time_seconds;
  int trace_length;             /* records produced (may exceed max_trace) */
  int iteration_count_timed;    /* entries written to iteration_seconds */
  int solves, linearizations, band_solver;
} vgicp_lm_report;
int vgicp_graph_optimize(vgicp_graph graph, double* poses12, const uint8_t* fixed, int32_t* updates,
                         const vgicp_lm_settings* settings, vgicp_lm_report* report, double* trace, int max_trace,
                         double* iteration_seconds);

/* Device-resident variants: every pointer is device memory of the context's device; the work
 * is enqueued on the context stream and the call returns without synchronising. */
int vgicp_graph_linearize_device(vgicp_graph graph, const double* d_poses12, double* d_out, int32_t* d_inliers);
int vgicp_graph_evaluate_device(vgicp_graph graph, const double* d_poses12, double* d_errors, int32_t* d_inliers);

/* ---------------------------------------------------------------- preprocessing */
/* estimate_covariances (point_cloud.cpp:44-83) on the GPU: exact k nearest neighbours (the point
 * itself included, ties by lower index), neighbourhood covariance, eigenvectors kept and the
 * spectrum clamped to (plane_epsilon, 1, 1). xyz: n×3 float32; cov6: n×6 float32 output
 * (xx xy xz yy yz zz). Errors: k < 4, n <= k, NaN/Inf -> INVALID_ARGUMENT; k > 32 unsupported. */
int vgicp_estimate_covariances(vgicp_ctx ctx, const float* xyz, size_t n, int k, double plane_epsilon, float* cov6);
int vgicp_estimate_covariances_batch(vgicp_ctx ctx, const float* const* xyz, const size_t* n, int m, int k,
                                     double plane_epsilon, float* const* cov6);

#ifdef __cplusplus
}
#endif

#endif /* VGICP_B200_H */
