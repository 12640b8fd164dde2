// vgicp_b200.hpp — header-only C++ façade over the C ABI (vgicp_b200.h) with the reference's
// operator API: same class / function names, argument meaning and exceptions as
//   proj/include/vgicp/voxelmap.hpp:28-61  (GaussianVoxelMap, overlap_rate)
//   proj/include/vgicp/factors.hpp:19-81   (LinearizedFactor, MatchingCostFactor,
//                                           gicp_error, linearize_/evaluate_matching_cost)
// plus the batch entry points (linearize_matching_costs / evaluate_matching_costs /
// overlap_rates) that optimizer.cpp:45-75 and pipeline.cpp:135-150 switch to.
//
// Eigen-free on purpose (the boundary carries plain arrays); INTEGRATION.md shows the few lines
// that adapt the reference's Eigen types to it. Errors: std::invalid_argument,
// std::out_of_range (as the reference) and vgicp::cuda_error for device failures.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "vgicp_b200.h"

namespace vgicp {

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == VGICP_OK) return;
  const std::string msg = vgicp_last_error();
  if (rc == VGICP_E_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == VGICP_E_OUT_OF_RANGE) throw std::out_of_range(msg);
  if (rc == VGICP_E_OUT_OF_MEMORY) throw std::bad_alloc();
  throw cuda_error(msg);
}

using Mat3 = std::array<double, 9>;   // row-major
using Vec3 = std::array<double, 3>;
using Mat6 = std::array<double, 36>;  // row-major
using Vec6 = std::array<double, 6>;

// Pose{rotation, translation} (se3.hpp:33-56) as 12 doubles: row-major R, then t.
struct Pose {
  std::array<double, 12> m{1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
  static Pose Identity() { return Pose{}; }
  static Pose from(const Mat3& R, const Vec3& t) {
    Pose p;
    for (int k = 0; k < 9; ++k) p.m[k] = R[k];
    for (int k = 0; k < 3; ++k) p.m[9 + k] = t[k];
    return p;
  }
  const double* data() const { return m.data(); }
};

class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) {
    vgicp_ctx c = nullptr;
    check(vgicp_ctx_create(device, stream, &c));
    h_.reset(c, [](vgicp_ctx x) { vgicp_ctx_destroy(x); });
  }
  vgicp_ctx get() const { return h_.get(); }
  void synchronize() const { check(vgicp_ctx_synchronize(get())); }
  std::uint64_t launch_count() const {
    std::uint64_t n = 0;
    check(vgicp_ctx_launch_count(get(), &n));
    return n;
  }

 private:
  std::shared_ptr<vgicp_ctx_s> h_;
};

// The reference's host PointCloud layout (point_cloud.hpp:21-37) for the float64 submap path.
struct HostCloud {
  std::vector<Vec3> means;
  std::vector<Mat3> covariances;  // empty or one per point (row-major)
  std::size_t size() const { return means.size(); }
  bool has_covariances() const { return !covariances.empty() && covariances.size() == means.size(); }
};

// Device-resident PointCloud (point_cloud.hpp:21-37). means: n×3, cov6: n×(xx xy xz yy yz zz).
class PointCloud {
 public:
  PointCloud(const Context& ctx, const std::vector<float>& xyz, const std::vector<float>& cov6 = {}) : ctx_(ctx) {
    if (xyz.size() % 3) throw std::invalid_argument("xyz must hold n*3 floats");
    const std::size_t n = xyz.size() / 3;
    if (!cov6.empty() && cov6.size() != 6 * n) throw std::invalid_argument("covariance count does not match point count");
    vgicp_cloud c = nullptr;
    check(vgicp_cloud_upload(ctx.get(), xyz.data(), cov6.empty() ? nullptr : cov6.data(), n, &c));
    h_.reset(c, [](vgicp_cloud x) { vgicp_cloud_destroy(x); });
  }
  // The reference's double layout: float32-exact clouds take the float32 layout, any other (submap
  // clouds) is kept in float64 too, so keys / correspondences / overlap hits stay bit-exact.
  PointCloud(const Context& ctx, const HostCloud& cloud) : ctx_(ctx) {
    vgicp_cloud c = nullptr;
    check(vgicp_cloud_upload_f64(ctx.get(), cloud.means.empty() ? nullptr : cloud.means[0].data(),
                                 cloud.has_covariances() ? cloud.covariances[0].data() : nullptr, cloud.size(), &c));
    h_.reset(c, [](vgicp_cloud x) { vgicp_cloud_destroy(x); });
  }
  bool is_f64() const {
    int v = 0;
    check(vgicp_cloud_is_f64(get(), &v));
    return v != 0;
  }
  std::size_t size() const {
    std::size_t n = 0;
    check(vgicp_cloud_size(get(), &n));
    return n;
  }
  bool empty() const { return size() == 0; }
  bool has_covariances() const {
    int has = 0;
    check(vgicp_cloud_has_covariances(get(), &has));
    return has != 0;
  }
  vgicp_cloud get() const { return h_.get(); }
  const Context& context() const { return ctx_; }
  // takes ownership of a handle returned by the C ABI (e.g. vgicp_submap_build)
  static PointCloud adopt(const Context& ctx, vgicp_cloud c) { return PointCloud(ctx, c); }
  // this cloud's device layout copied to another context's device (vgicp_cloud_replicate)
  PointCloud replicate(const Context& ctx) const {
    vgicp_cloud c = nullptr;
    check(vgicp_cloud_replicate(get(), ctx.get(), &c));
    return PointCloud(ctx, c);
  }

 private:
  PointCloud(const Context& ctx, vgicp_cloud c) : ctx_(ctx) { h_.reset(c, [](vgicp_cloud x) { vgicp_cloud_destroy(x); }); }
  Context ctx_;
  std::shared_ptr<vgicp_cloud_s> h_;
};

struct GaussianVoxel {  // voxelmap.hpp:18-22
  Vec3 mean{};
  Mat3 covariance{};
  int count = 0;
  bool operator==(const GaussianVoxel& o) const {
    return mean == o.mean && covariance == o.covariance && count == o.count;
  }
};

// GaussianVoxelMap (voxelmap.hpp:28-56): immutable after construction.
class GaussianVoxelMap {
 public:
  GaussianVoxelMap(const PointCloud& cloud, double resolution) : ctx_(cloud.context()) {
    vgicp_map m = nullptr;
    check(vgicp_voxelmap_build(ctx_.get(), cloud.get(), resolution, &m));
    h_.reset(m, [](vgicp_map x) { vgicp_voxelmap_destroy(x); });
  }
  // over a float64 host cloud (all 9 covariance entries accumulated, voxelmap.cpp:65-104)
  GaussianVoxelMap(const Context& ctx, const HostCloud& cloud, double resolution) : ctx_(ctx) {
    vgicp_map m = nullptr;
    check(vgicp_voxelmap_build_f64(ctx.get(), cloud.means.empty() ? nullptr : cloud.means[0].data(),
                                   cloud.has_covariances() ? cloud.covariances[0].data() : nullptr, cloud.size(),
                                   resolution, &m));
    h_.reset(m, [](vgicp_map x) { vgicp_voxelmap_destroy(x); });
  }
  static GaussianVoxelMap adopt(const Context& ctx, vgicp_map m) { return GaussianVoxelMap(ctx, m); }
  // the map copied to another context's device (vgicp_voxelmap_replicate): one transfer, no rebuild
  GaussianVoxelMap replicate(const Context& ctx) const {
    vgicp_map m = nullptr;
    check(vgicp_voxelmap_replicate(get(), ctx.get(), &m));
    return GaussianVoxelMap(ctx, m);
  }
  double resolution() const {
    double r = 0;
    check(vgicp_voxelmap_resolution(get(), &r));
    return r;
  }
  std::size_t size() const {
    std::size_t v = 0;
    check(vgicp_voxelmap_size(get(), &v));
    return v;
  }
  std::size_t total_points() const {
    std::size_t n = 0;
    check(vgicp_voxelmap_total_points(get(), &n));
    return n;
  }
  // voxels() in ascending key order
  std::vector<std::pair<std::uint64_t, GaussianVoxel>> voxels() const {
    const std::size_t v = size();
    std::vector<std::uint64_t> keys(v);
    std::vector<std::int32_t> counts(v);
    std::vector<double> means(3 * v), covs(9 * v);
    check(vgicp_voxelmap_export(get(), keys.data(), counts.data(), means.data(), covs.data()));
    std::vector<std::pair<std::uint64_t, GaussianVoxel>> out(v);
    for (std::size_t i = 0; i < v; ++i) {
      out[i].first = keys[i];
      for (int a = 0; a < 3; ++a) out[i].second.mean[a] = means[3 * i + a];
      for (int a = 0; a < 9; ++a) out[i].second.covariance[a] = covs[9 * i + a];
      out[i].second.count = counts[i];
    }
    return out;
  }
  // lookup (voxelmap.cpp:106-117): key of the populated voxel or VGICP_KEY_MISS
  std::vector<std::uint64_t> lookup(const std::vector<double>& points) const {
    std::vector<std::uint64_t> out(points.size() / 3);
    check(vgicp_voxelmap_lookup(get(), points.data(), out.size(), out.data()));
    return out;
  }
  // lookup (voxelmap.cpp:106-117) of one point: the populated voxel containing it, or nullptr
  const GaussianVoxel* lookup(const Vec3& point) const {
    const std::uint64_t key = lookup(std::vector<double>(point.begin(), point.end()))[0];
    if (key == VGICP_KEY_MISS) return nullptr;
    if (cache_.empty()) cache_ = voxels();  // immutable after construction (voxelmap.hpp:27)
    const auto it = std::lower_bound(cache_.begin(), cache_.end(), key,
                                     [](const auto& kv, std::uint64_t k) { return kv.first < k; });
    return it != cache_.end() && it->first == key ? &it->second : nullptr;
  }
  // voxel_coord (voxelmap.cpp:45-55); throws std::out_of_range beyond ±2^20 voxels
  std::array<int, 3> voxel_coord(const Vec3& point) const {
    const std::uint64_t k = pack_key(resolution(), point);
    return {static_cast<int>((k >> 42) & 0x1FFFFF) - (1 << 20), static_cast<int>((k >> 21) & 0x1FFFFF) - (1 << 20),
            static_cast<int>(k & 0x1FFFFF) - (1 << 20)};
  }
  static std::uint64_t pack_key(double resolution, const Vec3& point) {
    std::uint64_t k = 0;
    check(vgicp_voxel_key(resolution, point.data(), &k));
    return k;
  }
  vgicp_map get() const { return h_.get(); }
  const Context& context() const { return ctx_; }

 private:
  GaussianVoxelMap(const Context& ctx, vgicp_map m) : ctx_(ctx) { h_.reset(m, [](vgicp_map x) { vgicp_voxelmap_destroy(x); }); }
  Context ctx_;
  std::shared_ptr<vgicp_map_s> h_;
  mutable std::vector<std::pair<std::uint64_t, GaussianVoxel>> cache_;  // host copy for single lookups
};

// transform_cloud (point_cloud.cpp:26-42), float64 on the device.
inline HostCloud transform_cloud(const Context& ctx, const HostCloud& cloud, const Pose& T) {
  HostCloud out;
  out.means.resize(cloud.size());
  if (cloud.has_covariances()) out.covariances.resize(cloud.size());
  if (cloud.size() == 0) return out;
  check(vgicp_transform_cloud(ctx.get(), cloud.means[0].data(), cloud.has_covariances() ? cloud.covariances[0].data() : nullptr,
                              cloud.size(), T.data(), out.means[0].data(),
                              cloud.has_covariances() ? out.covariances[0].data() : nullptr));
  return out;
}

// voxel_downsample (voxelmap.cpp:137-169): one point per voxel, ascending packed-key order.
inline HostCloud voxel_downsample(const Context& ctx, const HostCloud& cloud, double resolution) {
  const GaussianVoxelMap map(ctx, cloud, resolution);
  HostCloud out;
  for (const auto& [key, v] : map.voxels()) {
    out.means.push_back(v.mean);
    out.covariances.push_back(v.covariance);
  }
  return out;
}

// MappingPipeline::emit_submap's data path (pipeline.cpp:92-114) on the device: frames transformed
// by frame_poses (frame -> submap), merged, voxel_downsample'd and mapped at map_resolution.
struct Submap {
  PointCloud cloud;         // float32 copy of the (downsampled) float64 submap cloud
  GaussianVoxelMap voxels;  // the submap's voxel map
};
inline Submap build_submap(const std::vector<const PointCloud*>& frames, const std::vector<Pose>& frame_poses,
                           double downsample_resolution, double map_resolution) {
  if (frames.empty()) throw std::invalid_argument("submap requires at least one frame");
  if (frames.size() != frame_poses.size()) throw std::invalid_argument("one pose per frame");
  const Context& ctx = frames[0]->context();
  std::vector<vgicp_cloud> fh(frames.size());
  std::vector<double> P(12 * frames.size());
  for (std::size_t k = 0; k < frames.size(); ++k) {
    fh[k] = frames[k]->get();
    for (int q = 0; q < 12; ++q) P[12 * k + q] = frame_poses[k].m[q];
  }
  vgicp_cloud c = nullptr;
  vgicp_map m = nullptr;
  check(vgicp_submap_build(ctx.get(), fh.data(), P.data(), static_cast<int>(frames.size()), downsample_resolution,
                           map_resolution, nullptr, &c, &m));
  return Submap{PointCloud::adopt(ctx, c), GaussianVoxelMap::adopt(ctx, m)};
}

inline double overlap_rate(const PointCloud& cloud, const Pose& pose_rel, const GaussianVoxelMap& map) {
  double r = 0.0;
  check(vgicp_overlap_rate(cloud.context().get(), cloud.get(), pose_rel.data(), map.get(), &r));
  return r;
}

// overlap_rates: one probe cloud against many maps in one launch (pipeline.cpp:135-150 loop).
inline std::vector<double> overlap_rates(const PointCloud& cloud, const std::vector<Pose>& poses,
                                         const std::vector<const GaussianVoxelMap*>& maps) {
  if (poses.size() != maps.size()) throw std::invalid_argument("poses and maps differ in length");
  const int m = static_cast<int>(maps.size());
  std::vector<vgicp_cloud> cl(m, cloud.get());
  std::vector<vgicp_map> mh(m);
  std::vector<double> P(12 * m);
  for (int k = 0; k < m; ++k) {
    mh[k] = maps[k]->get();
    for (int q = 0; q < 12; ++q) P[12 * k + q] = poses[k].m[q];
  }
  std::vector<std::uint64_t> hits(m);
  check(vgicp_overlap_batch(cloud.context().get(), cl.data(), P.data(), mh.data(), m, hits.data()));
  std::vector<double> out(m);
  for (int k = 0; k < m; ++k) out[k] = static_cast<double>(hits[k]) / static_cast<double>(cloud.size());
  return out;
}

// A keyframe database kept on the device (vgicp_mapset): sweeps of one new frame against all its
// maps build and cull their probe items on the GPU (pipeline.cpp:135-150 with the submap list fixed).
class KeyframeSet {
 public:
  KeyframeSet(const Context& ctx, const std::vector<const GaussianVoxelMap*>& maps) : ctx_(ctx) {
    std::vector<vgicp_map> mh;
    for (const auto* m : maps) mh.push_back(m->get());
    vgicp_mapset h = nullptr;
    check(vgicp_mapset_create(ctx.get(), mh.data(), static_cast<int>(mh.size()), &h));
    h_.reset(h, [](vgicp_mapset x) { vgicp_mapset_destroy(x); });
    size_ = maps.size();
  }
  // exact hits / N of `cloud` through poses[k] (T_map⁻¹·T_cloud) against map k
  std::vector<double> overlap_rates(const PointCloud& cloud, const std::vector<Pose>& poses) const {
    if (poses.size() != size_) throw std::invalid_argument("poses and maps differ in length");
    std::vector<double> P(12 * size_);
    for (std::size_t k = 0; k < size_; ++k)
      for (int q = 0; q < 12; ++q) P[12 * k + q] = poses[k].m[q];
    std::vector<std::uint64_t> hits(size_);
    check(vgicp_overlap_mapset(ctx_.get(), cloud.get(), P.data(), h_.get(), hits.data()));
    std::vector<double> out(size_);
    for (std::size_t k = 0; k < size_; ++k) out[k] = static_cast<double>(hits[k]) / static_cast<double>(cloud.size());
    return out;
  }
  // a new keyframe's map joins the set (amortised O(1) device work)
  void append(const GaussianVoxelMap& map) {
    vgicp_map mh = map.get();
    check(vgicp_mapset_append(h_.get(), &mh, 1));
    ++size_;
  }
  std::size_t size() const { return size_; }

 private:
  Context ctx_;
  std::shared_ptr<vgicp_mapset_s> h_;
  std::size_t size_ = 0;
};

struct LinearizedFactor {  // factors.hpp:19-29
  int i = -1;
  int j = -1;
  Mat6 H_ii{};
  Mat6 H_ij{};
  Mat6 H_jj{};
  Vec6 b_i{};
  Vec6 b_j{};
  double error = 0.0;
  int inliers = 0;

  static LinearizedFactor from(const double* raw, int i, int j, int inliers) {
    LinearizedFactor f;
    f.i = i;
    f.j = j;
    for (int k = 0; k < 36; ++k) {
      f.H_ii[k] = raw[k];
      f.H_ij[k] = raw[36 + k];
      f.H_jj[k] = raw[72 + k];
    }
    for (int k = 0; k < 6; ++k) {
      f.b_i[k] = raw[108 + k];
      f.b_j[k] = raw[114 + k];
    }
    f.error = raw[120];
    f.inliers = inliers;
    return f;
  }
};

struct MatchingCostFactor {  // factors.hpp:36-45, validation of factors.cpp:57-66
  int target_index = -1;
  int source_index = -1;
  std::shared_ptr<const PointCloud> source_points;
  std::shared_ptr<const GaussianVoxelMap> target_voxels;

  MatchingCostFactor(int target, int source, std::shared_ptr<const PointCloud> points,
                     std::shared_ptr<const GaussianVoxelMap> voxels)
      : target_index(target), source_index(source), source_points(std::move(points)), target_voxels(std::move(voxels)) {
    if (target_index == source_index) throw std::invalid_argument("matching cost factor requires distinct variables");
    if (!source_points || source_points->empty())
      throw std::invalid_argument("matching cost factor requires a nonempty source cloud");
    if (!source_points->has_covariances()) throw std::invalid_argument("matching cost factor requires source covariances");
    if (!target_voxels || target_voxels->size() == 0)
      throw std::invalid_argument("matching cost factor requires a nonempty target voxel map");
  }
  vgicp_factor_desc desc() const { return {target_index, source_index, source_points->get(), target_voxels->get()}; }
};

inline LinearizedFactor linearize_matching_cost(const MatchingCostFactor& f, const Pose& T_target, const Pose& T_source) {
  double raw[VGICP_LINEARIZED_DOUBLES];
  std::int32_t inl = 0;
  const vgicp_factor_desc d = f.desc();
  check(vgicp_linearize_matching_cost(f.source_points->context().get(), &d, T_target.data(), T_source.data(), raw, &inl));
  return LinearizedFactor::from(raw, f.target_index, f.source_index, inl);
}

inline std::pair<double, int> evaluate_matching_cost(const MatchingCostFactor& f, const Pose& T_target,
                                                     const Pose& T_source) {
  double err = 0.0;
  std::int32_t inl = 0;
  const vgicp_factor_desc d = f.desc();
  check(vgicp_evaluate_matching_cost(f.source_points->context().get(), &d, T_target.data(), T_source.data(), &err, &inl));
  return {err, inl};
}

struct GicpErrorResult {  // factors.hpp:62-67
  double error = 0.0;
  Vec3 residual{};
  Mat3 information{};
  bool valid = true;
};

inline GicpErrorResult gicp_error(const Context& ctx, const Vec3& source_mean, const Mat3& source_cov,
                                  const GaussianVoxel& target, const Pose& T) {
  GicpErrorResult r;
  int valid = 0;
  check(vgicp_gicp_error(ctx.get(), source_mean.data(), source_cov.data(), target.mean.data(), target.covariance.data(),
                         T.data(), &r.error, r.residual.data(), r.information.data(), &valid));
  r.valid = valid != 0;
  return r;
}

// Batched factors over a fixed graph: one launch linearizes / evaluates every factor.
// BlockSystem (block_solver.hpp): lower-triangle blocks per column slot, rhs per slot; slots are
// the active variables in reverse insertion order (block_solver.cpp:26-34).
struct BlockSystem {
  int num_slots = 0;
  std::vector<int> slot_of_var;  // -1 for fixed variables
  std::vector<int> var_of_slot;
  std::vector<std::map<int, Mat6>> columns;  // columns[b][a] = block (row a, col b), a >= b
  std::vector<Vec6> rhs;
};

class MatchingCostBatch {
 public:
  MatchingCostBatch(const Context& ctx, const std::vector<MatchingCostFactor>& factors, int num_poses, int chunk = 0)
      : ctx_(ctx), factors_(factors), num_poses_(num_poses) {
    std::vector<vgicp_factor_desc> d;
    d.reserve(factors.size());
    for (const auto& f : factors) d.push_back(f.desc());
    vgicp_graph g = nullptr;
    check(vgicp_graph_create(ctx.get(), d.data(), static_cast<int>(d.size()), num_poses, chunk, &g));
    h_.reset(g, [](vgicp_graph x) { vgicp_graph_destroy(x); });
  }
  // ONE batch split over several devices (vgicp_graph_create_sharded): per_device[r] holds the same
  // factors built on contexts[r] (clouds / maps replicated); every method below returns bit-identical
  // results to the single-device batch.
  MatchingCostBatch(const std::vector<Context>& contexts, const std::vector<std::vector<MatchingCostFactor>>& per_device,
                    int num_poses, int chunk = 0)
      : ctx_(contexts.at(0)), factors_(per_device.at(0)), num_poses_(num_poses), replicas_(per_device) {
    if (contexts.size() != per_device.size()) throw std::invalid_argument("one factor list per context");
    std::vector<std::vector<vgicp_factor_desc>> d(per_device.size());
    std::vector<const vgicp_factor_desc*> lists;
    std::vector<vgicp_ctx> cs;
    for (std::size_t r = 0; r < per_device.size(); ++r) {
      if (per_device[r].size() != factors_.size()) throw std::invalid_argument("factor lists differ in length");
      for (const auto& f : per_device[r]) d[r].push_back(f.desc());
      lists.push_back(d[r].data());
      cs.push_back(contexts[r].get());
    }
    vgicp_graph g = nullptr;
    check(vgicp_graph_create_sharded(cs.data(), static_cast<int>(cs.size()), lists.data(),
                                     static_cast<int>(factors_.size()), num_poses, chunk, &g));
    h_.reset(g, [](vgicp_graph x) { vgicp_graph_destroy(x); });
  }
  int num_shards() const {
    int n = 0;
    check(vgicp_graph_num_shards(h_.get(), &n));
    return n;
  }
  // linearize_all (optimizer.cpp:45-62), matching part, factor order
  std::vector<LinearizedFactor> linearize(const std::vector<Pose>& poses) const {
    const std::vector<double> P = flatten(poses);
    std::vector<double> raw(factors_.size() * VGICP_LINEARIZED_DOUBLES);
    std::vector<std::int32_t> inl(factors_.size());
    check(vgicp_graph_linearize(h_.get(), P.data(), raw.data(), inl.data()));
    std::vector<LinearizedFactor> out(factors_.size());
    for (std::size_t k = 0; k < factors_.size(); ++k)
      out[k] = LinearizedFactor::from(raw.data() + k * VGICP_LINEARIZED_DOUBLES, factors_[k].target_index,
                                      factors_[k].source_index, inl[k]);
    return out;
  }
  // per-factor (error, inliers) for total_error (optimizer.cpp:66-75)
  std::vector<std::pair<double, int>> evaluate(const std::vector<Pose>& poses) const {
    const std::vector<double> P = flatten(poses);
    std::vector<double> err(factors_.size());
    std::vector<std::int32_t> inl(factors_.size());
    check(vgicp_graph_evaluate(h_.get(), P.data(), err.data(), inl.data()));
    std::vector<std::pair<double, int>> out(factors_.size());
    for (std::size_t k = 0; k < out.size(); ++k) out[k] = {err[k], inl[k]};
    return out;
  }
  double total_error(const std::vector<Pose>& poses) const {
    double s = 0.0;
    for (const auto& e : evaluate(poses)) s += e.first;
    return s;
  }
  std::size_t size() const { return factors_.size(); }
  // optimize (optimizer.cpp:88-194) for this graph of matching factors, in the library
  // (vgicp_graph_optimize); `poses` updated in place unless the solve aborts (like graph.poses).
  struct IterationRecord {  // optimizer.hpp:33-39
    int iteration = 0;
    double error = 0.0, lambda = 0.0, step_norm = 0.0;
    bool accepted = false;
  };
  struct OptimizerReport {  // optimizer.hpp:41-50 (reason: VGICP_LM_*, TerminationReason order)
    int iterations = 0;
    double initial_error = 0.0, final_error = 0.0;
    std::vector<IterationRecord> trace;
    int reason = VGICP_LM_MAX_ITERATIONS;
    double wall_time_seconds = 0.0;
    bool aborted = false;
  };
  OptimizerReport optimize(std::vector<Pose>& poses, const std::vector<std::uint8_t>& fixed = {},
                           const vgicp_lm_settings* settings = nullptr) const {
    std::vector<double> P = flatten(poses);
    if (!fixed.empty() && static_cast<int>(fixed.size()) != num_poses_)
      throw std::invalid_argument("fixed mask size does not match");
    const int max_trace = 4 * (settings ? settings->max_iterations : 50) + 64;
    std::vector<double> trace(5 * static_cast<std::size_t>(max_trace));
    vgicp_lm_report rep{};
    check(vgicp_graph_optimize(h_.get(), P.data(), fixed.empty() ? nullptr : fixed.data(), nullptr, settings, &rep,
                               trace.data(), max_trace, nullptr));
    OptimizerReport out;
    out.iterations = rep.iterations;
    out.initial_error = rep.initial_error;
    out.final_error = rep.final_error;
    out.reason = rep.reason;
    out.wall_time_seconds = rep.wall_time_seconds;
    out.aborted = rep.aborted != 0;
    for (int k = 0; k < std::min(rep.trace_length, max_trace); ++k) {
      const double* r = trace.data() + 5 * k;
      out.trace.push_back({static_cast<int>(r[0]), r[1], r[2], r[3], r[4] != 0.0});
    }
    if (!out.aborted)
      for (std::size_t k = 0; k < poses.size(); ++k)
        for (int q = 0; q < 12; ++q) poses[k].m[q] = P[12 * k + q];
    return out;
  }
  // linearize_all + assemble_normal_equations (block_solver.cpp:14-62) with the assembly on the
  // device (matching factors only); bit-identical to assembling linearize()'s blocks on the host.
  BlockSystem linearize_assembled(const std::vector<Pose>& poses, const std::vector<std::uint8_t>& fixed) const {
    if (static_cast<int>(fixed.size()) != num_poses_) throw std::invalid_argument("fixed mask size does not match");
    int S = 0, P = 0;
    check(vgicp_graph_assembly_plan(h_.get(), fixed.data(), &S, &P, nullptr));
    std::vector<std::int32_t> pairs(2 * static_cast<std::size_t>(P));
    check(vgicp_graph_assembly_plan(h_.get(), fixed.data(), &S, &P, pairs.data()));
    const std::vector<double> Pz = flatten(poses);
    std::vector<double> diag(36 * static_cast<std::size_t>(S)), off(36 * static_cast<std::size_t>(P)),
        rhs(6 * static_cast<std::size_t>(S));
    check(vgicp_graph_linearize_assembled(h_.get(), Pz.data(), diag.data(), off.data(), rhs.data()));
    BlockSystem sys;
    sys.num_slots = S;
    sys.slot_of_var.assign(num_poses_, -1);
    sys.var_of_slot.assign(S, -1);
    for (int v = 0, rank = 0; v < num_poses_; ++v)
      if (!fixed[v]) {
        sys.slot_of_var[v] = S - 1 - rank++;
        sys.var_of_slot[sys.slot_of_var[v]] = v;
      }
    sys.columns.resize(S);
    sys.rhs.resize(S);
    for (int k = 0; k < S; ++k) {
      std::copy_n(diag.data() + 36 * k, 36, sys.columns[k][k].begin());
      std::copy_n(rhs.data() + 6 * k, 6, sys.rhs[k].begin());
    }
    for (int k = 0; k < P; ++k) std::copy_n(off.data() + 36 * k, 36, sys.columns[pairs[2 * k + 1]][pairs[2 * k]].begin());
    return sys;
  }

 private:
  std::vector<double> flatten(const std::vector<Pose>& poses) const {
    if (static_cast<int>(poses.size()) != num_poses_) throw std::invalid_argument("pose count does not match the batch");
    std::vector<double> P(12 * poses.size());
    for (std::size_t k = 0; k < poses.size(); ++k)
      for (int q = 0; q < 12; ++q) P[12 * k + q] = poses[k].m[q];
    return P;
  }
  Context ctx_;
  std::vector<MatchingCostFactor> factors_;
  int num_poses_;
  std::vector<std::vector<MatchingCostFactor>> replicas_;  // keeps the other devices' handles alive
  std::shared_ptr<vgicp_graph_s> h_;
};

inline std::vector<LinearizedFactor> linearize_matching_costs(const Context& ctx,
                                                              const std::vector<MatchingCostFactor>& factors,
                                                              const std::vector<Pose>& poses) {
  return MatchingCostBatch(ctx, factors, static_cast<int>(poses.size())).linearize(poses);
}

inline std::vector<std::pair<double, int>> evaluate_matching_costs(const Context& ctx,
                                                                   const std::vector<MatchingCostFactor>& factors,
                                                                   const std::vector<Pose>& poses) {
  return MatchingCostBatch(ctx, factors, static_cast<int>(poses.size())).evaluate(poses);
}

}  // namespace vgicp
