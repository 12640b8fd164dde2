/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the VGICP hot path.
 *
 * This header is the C ABI of oracle/vgicp_oracle.cpp, a plain-C++20 restatement of the
 * reference's CPU implementation (/root/reference/proj, Eigen-free). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it,
 * and only as the checker or the timed CPU baseline — never as the product path.
 *
 * Parity pinning: the reference cannot be compiled here (Eigen3 and doctest are absent;
 * see DESIGN.md §Oracle), and it ships no golden vectors. The restatement is pinned against
 * every known-answer test and brute-force oracle the reference's own tests hold for this path
 * (tests/test_oracle_kats.py ports test_voxelmap.cpp, test_factors.cpp, test_reference.cpp and
 * oracles.hpp).
 *
 * Conventions: a pose is 12 doubles, row-major rotation R (9) then translation t (3).
 * Means are n×3 doubles, covariances n×9 doubles (row-major full 3×3).
 * Status codes: 0 ok, 1 invalid_argument, 2 out_of_range.
 */
#ifndef VGICP_ORACLE_H
#define VGICP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_map_s or_map;
typedef struct or_rng_s or_rng;

const char* or_last_error(void);

/* --- GaussianVoxelMap (voxelmap.cpp:65-104), parallel sharded Kahan build --- */
int or_voxelmap_build(const double* means, const double* covs, size_t n, double resolution, int threads,
                      int deterministic, or_map** out);
/* reference::build_voxelmap (reference.cpp:39-65): serial, plain sums, no range check */
int or_voxelmap_build_serial(const double* means, const double* covs, size_t n, double resolution, or_map** out);
void or_voxelmap_destroy(or_map* map);
size_t or_voxelmap_size(const or_map* map);
size_t or_voxelmap_total_points(const or_map* map);
/* Sorted by key. Any output pointer may be NULL. means: V×3, covs: V×9. */
void or_voxelmap_export(const or_map* map, uint64_t* keys, int32_t* counts, double* means, double* covs);
/* GaussianVoxelMap::lookup (voxelmap.cpp:106-117) for n points; key = UINT64_MAX on a miss. */
void or_voxelmap_lookup(const or_map* map, const double* points, size_t n, uint64_t* keys_out);
/* voxel_coord + pack_key (voxelmap.cpp:45-63); returns 2 when out of range */
int or_voxel_key(double resolution, const double p[3], uint64_t* key);

/* --- overlap_rate (voxelmap.cpp:119-135) and reference::overlap_rate (reference.cpp:67-74) --- */
int or_overlap_rate(const double* means, size_t n, const double pose[12], const or_map* map, int threads,
                    int deterministic, double* rate, uint64_t* hits);
int or_overlap_rate_serial(const double* means, size_t n, const double pose[12], const or_map* map, double* rate);

/* --- Matching cost factor (factors.cpp:90-181); out = 121 doubles:
 *     H_ii(36) H_ij(36) H_jj(36) b_i(6) b_j(6) error(1), all row-major. --- */
int or_linearize(const double* src_means, const double* src_covs, size_t n, const or_map* target,
                 const double T_target[12], const double T_source[12], int threads, int deterministic,
                 double* out, int32_t* inliers);
int or_linearize_serial(const double* src_means, const double* src_covs, size_t n, const or_map* target,
                        const double T_target[12], const double T_source[12], double* out, int32_t* inliers);
int or_evaluate(const double* src_means, const double* src_covs, size_t n, const or_map* target,
                const double T_target[12], const double T_source[12], int threads, int deterministic,
                double* error, int32_t* inliers);
/* gicp_error (factors.cpp:75-88). */
void or_gicp_error(const double src_mean[3], const double src_cov[9], const double tgt_mean[3],
                   const double tgt_cov[9], const double T[12], double* error, double residual[3],
                   double information[9], int* valid);
/* invert_covariance (factors.cpp:38-46): returns 1 when the LDLT accepts M. */
int or_invert_covariance(const double M[9], double out[9]);
/* frozen_cost (test_factors.cpp:72-88): association and Omega frozen at the linearization point. */
double or_frozen_cost(const double* src_means, const double* src_covs, size_t n, const or_map* target,
                      const double lin_target[12], const double lin_source[12], const double T_target[12],
                      const double T_source[12]);

/* --- SE3 subset (se3.cpp) --- */
void or_se3_exp(const double twist[6], double pose_out[12]);
void or_compose(const double a[12], const double b[12], double out[12]);
void or_inverse(const double a[12], double out[12]);
void or_retract(const double a[12], const double twist[6], double out[12]);
void or_adjoint(const double a[12], double out[36]);

/* --- Test RNG and scene builders (oracles.hpp:151-168, test_*.cpp scene helpers) --- */
or_rng* or_rng_create(uint64_t seed);
void or_rng_destroy(or_rng* rng);
double or_rng_uniform(or_rng* rng, double lo, double hi);
void or_rng_vector(or_rng* rng, double scale, double out[3]);
void or_random_pose(or_rng* rng, double rot_scale, double trans_scale, double pose_out[12]);
void or_random_plane_covariance(or_rng* rng, double cov_out[9]);
/* test_reference.cpp:15-30 */
void or_random_gaussian_cloud(or_rng* rng, int n, double scale, double* means, double* covs);
/* test_factors.cpp:33-68: target_means/covs and source_means/covs each points×3 / points×9 */
void or_make_scene(or_rng* rng, int points, double resolution, double boundary_margin, double* T_target,
                   double* T_source, double* source_means, double* source_covs, double* target_means,
                   double* target_covs);
/* reference::estimate_covariances (reference.cpp:11-37): brute-force kNN, eigen-regularised. */
int or_estimate_covariances(const double* means, size_t n, int k, double plane_epsilon, double* covs);
/* transform_cloud (point_cloud.cpp:26-42); covs / out_covs may be NULL. */
void or_transform_cloud(const double* means, const double* covs, size_t n, const double pose[12], double* out_means,
                        double* out_covs);
/* std::shuffle(perm, rng.engine) as in test_voxelmap.cpp:104 */
void or_rng_shuffle(or_rng* rng, uint64_t* perm, size_t n);

#ifdef __cplusplus
}
#endif

#endif
