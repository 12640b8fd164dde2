// C++ façade smoke test (include/vgicp_b200.hpp): the reference-facing C++ API end to end on a
// GPU. Built by __graft_entry__.build(); run by tests/test_facade_cpp.py (-m gpu).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>

#include "vgicp_b200.hpp"

#define REQUIRE(c)                                                  \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                                 \
    }                                                               \
  } while (0)

int main() {
  using namespace vgicp;
  Context ctx(0);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<float> U(-10.f, 10.f);
  const int n = 5000;
  std::vector<float> xyz(3 * n), cov(6 * n);
  for (int i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) xyz[3 * i + a] = U(rng);
    // plane covariance with normal z: diag(1, 1, 1e-3)
    cov[6 * i + 0] = 1.f, cov[6 * i + 1] = 0.f, cov[6 * i + 2] = 0.f;
    cov[6 * i + 3] = 1.f, cov[6 * i + 4] = 0.f, cov[6 * i + 5] = 1e-3f;
  }
  auto cloud = std::make_shared<PointCloud>(ctx, xyz, cov);
  auto map = std::make_shared<GaussianVoxelMap>(*cloud, 1.0);
  REQUIRE(map->total_points() == static_cast<std::size_t>(n));
  REQUIRE(map->size() > 0 && map->size() <= static_cast<std::size_t>(n));
  std::size_t total = 0;
  for (const auto& kv : map->voxels()) total += kv.second.count;
  REQUIRE(total == static_cast<std::size_t>(n));

  // single-point lookup / voxel_coord (voxelmap.cpp:45-55, 106-117)
  {
    const Vec3 p0{xyz[0], xyz[1], xyz[2]};
    const GaussianVoxel* v = map->lookup(p0);
    REQUIRE(v != nullptr && v->count >= 1);
    REQUIRE(map->lookup(Vec3{1e7, 0, 0}) == nullptr);
    const auto c = map->voxel_coord(p0);
    REQUIRE(c[0] == static_cast<int>(std::floor(p0[0] / 1.0)) && c[2] == static_cast<int>(std::floor(p0[2] / 1.0)));
  }

  // overlap: self at identity = 1, far = 0 (test_voxelmap.cpp:138-149)
  REQUIRE(overlap_rate(*cloud, Pose::Identity(), *map) == 1.0);
  REQUIRE(overlap_rate(*cloud, Pose::from({1, 0, 0, 0, 1, 0, 0, 0, 1}, {500, 0, 0}), *map) == 0.0);
  const auto rates = overlap_rates(*cloud, {Pose::Identity(), Pose::from({1, 0, 0, 0, 1, 0, 0, 0, 1}, {0.5, 0, 0})},
                                   {map.get(), map.get()});
  REQUIRE(rates[0] == 1.0 && rates[1] > 0.0 && rates[1] < 1.0);

  // factor: identical clouds at equal poses -> every point hits its own voxel
  MatchingCostFactor factor(0, 1, cloud, map);
  const Pose T = Pose::from({1, 0, 0, 0, 1, 0, 0, 0, 1}, {0.3, -0.2, 0.1});
  const LinearizedFactor lin = linearize_matching_cost(factor, T, T);
  REQUIRE(lin.inliers == n);
  const auto ev = evaluate_matching_cost(factor, T, T);
  REQUIRE(ev.second == n);
  REQUIRE(std::abs(ev.first - lin.error) <= 1e-6 * std::max(1.0, lin.error));
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) REQUIRE(lin.H_ii[6 * r + c] == lin.H_ii[6 * c + r]);

  // batch == single
  MatchingCostBatch batch(ctx, {factor}, 2);
  const auto lins = batch.linearize({T, T});
  REQUIRE(lins.size() == 1 && lins[0].inliers == lin.inliers);
  for (int k = 0; k < 36; ++k) REQUIRE(lins[0].H_ij[k] == lin.H_ij[k]);
  REQUIRE(batch.total_error({T, T}) == ev.first);

  // exceptions mirror the reference
  bool threw = false;
  try {
    MatchingCostFactor bad(1, 1, cloud, map);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw);
  threw = false;
  try {
    PointCloud far(ctx, {2.0e6f, 0.f, 0.f}, {1, 0, 0, 1, 0, 1});
    GaussianVoxelMap m(far, 1.0);
  } catch (const std::out_of_range&) {
    threw = true;
  }
  REQUIRE(threw);
  threw = false;
  try {
    GaussianVoxelMap m(*cloud, -1.0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw);

  // gicp_error KAT (test_factors.cpp:107-111)
  GaussianVoxel v;
  v.mean = {2, 2, 3};
  v.covariance = {0.5, 0, 0, 0, 0.5, 0, 0, 0, 0.5};
  const auto g = gicp_error(ctx, {1, 2, 3}, {0.5, 0, 0, 0, 0.5, 0, 0, 0, 0.5}, v, Pose::Identity());
  REQUIRE(g.valid && std::abs(g.error - 1.0) < 1e-12);

  // device-side assembly (§8f #3) equals the host assembly of the same factor blocks
  {
    MatchingCostBatch b3(ctx, {MatchingCostFactor(0, 1, cloud, map), MatchingCostFactor(1, 2, cloud, map),
                               MatchingCostFactor(2, 0, cloud, map)}, 3);
    const std::vector<Pose> poses = {T, Pose::Identity(), Pose::from({1, 0, 0, 0, 1, 0, 0, 0, 1}, {0.1, 0.1, 0})};
    const BlockSystem sys = b3.linearize_assembled(poses, {1, 0, 0});
    REQUIRE(sys.num_slots == 2 && sys.var_of_slot[0] == 2 && sys.var_of_slot[1] == 1);
    const auto lins = b3.linearize(poses);
    for (int v = 1; v < 3; ++v) {
      Mat6 d{};
      Vec6 r{};
      for (const auto& lf : lins) {
        if (lf.i == v) for (int e = 0; e < 36; ++e) d[e] += lf.H_ii[e];
        if (lf.i == v) for (int e = 0; e < 6; ++e) r[e] += lf.b_i[e];
        if (lf.j == v) for (int e = 0; e < 36; ++e) d[e] += lf.H_jj[e];
        if (lf.j == v) for (int e = 0; e < 6; ++e) r[e] += lf.b_j[e];
      }
      const int sl = sys.slot_of_var[v];
      REQUIRE(sys.columns[sl].at(sl) == d && sys.rhs[sl] == r);
    }
  }

  // keyframe set sweep == per-map overlap_rate
  {
    KeyframeSet set(ctx, {map.get(), map.get()});
    const auto r = set.overlap_rates(*cloud, {Pose::Identity(), T});
    REQUIRE(r.size() == 2 && r[0] == overlap_rate(*cloud, Pose::Identity(), *map) &&
            r[1] == overlap_rate(*cloud, T, *map));
    set.append(*map);  // a new keyframe joins the set
    const auto r3 = set.overlap_rates(*cloud, {Pose::Identity(), T, T});
    REQUIRE(set.size() == 3 && r3[0] == r[0] && r3[1] == r[1] && r3[2] == r[1]);
  }

  // native LM (optimizer.cpp:88-194): the error never increases along the trace, the fixed pose
  // stays put, accepted records carry the new error
  {
    MatchingCostBatch b3(ctx, {MatchingCostFactor(0, 1, cloud, map), MatchingCostFactor(1, 2, cloud, map),
                               MatchingCostFactor(2, 0, cloud, map)}, 3);
    std::vector<Pose> poses = {Pose::Identity(), Pose::from({1, 0, 0, 0, 1, 0, 0, 0, 1}, {0.2, -0.1, 0.05}),
                               Pose::from({1, 0, 0, 0, 1, 0, 0, 0, 1}, {-0.1, 0.15, 0})};
    const Pose p0 = poses[0];
    const auto rep = b3.optimize(poses, {1, 0, 0});
    REQUIRE(!rep.aborted && rep.iterations >= 1 && rep.final_error <= rep.initial_error);
    double last = rep.initial_error;
    for (const auto& r : rep.trace)
      if (r.accepted) {
        REQUIRE(r.error < last);
        last = r.error;
      }
    REQUIRE(last == rep.final_error && std::abs(b3.total_error(poses) - rep.final_error) <= 1e-9 * rep.final_error);
    for (int q = 0; q < 12; ++q) REQUIRE(poses[0].m[q] == p0.m[q]);
  }

  // submap path (§8f #2): transform_cloud, voxel_downsample, build_submap
  {
    HostCloud hc;
    for (int i = 0; i < 200; ++i) {
      hc.means.push_back({0.05 * i, 0.1 * (i % 7), 0.02 * (i % 13)});
      hc.covariances.push_back({1, 0, 0, 0, 1, 0, 0, 0, 1e-3});
    }
    const HostCloud moved = transform_cloud(ctx, hc, Pose::from({1, 0, 0, 0, 1, 0, 0, 0, 1}, {1, 2, 3}));
    REQUIRE(moved.size() == 200 && std::abs(moved.means[10][0] - (hc.means[10][0] + 1)) < 1e-12);
    const HostCloud down = voxel_downsample(ctx, hc, 1.0);
    REQUIRE(down.size() == GaussianVoxelMap(ctx, hc, 1.0).size());
    const Submap sub = build_submap({cloud.get(), cloud.get()}, {Pose::Identity(), Pose::Identity()}, 0.5, 1.0);
    REQUIRE(sub.cloud.has_covariances() && sub.voxels.size() > 0 && sub.voxels.total_points() == sub.cloud.size());
  }

  // float64 host clouds keep their double values (not float32-exact -> a float64 device cloud)
  {
    HostCloud hc;
    for (int i = 0; i < 500; ++i) {
      hc.means.push_back({0.1 * i + 1e-9, 0.3 * (i % 11), 0.01 * (i % 17)});
      hc.covariances.push_back({1, 0, 0, 0, 1, 0, 0, 0, 1e-3});
    }
    PointCloud c64(ctx, hc);
    REQUIRE(c64.is_f64() && c64.size() == 500 && c64.has_covariances());
    HostCloud h32;
    for (int i = 0; i < 100; ++i) {
      h32.means.push_back({static_cast<double>(xyz[3 * i]), static_cast<double>(xyz[3 * i + 1]), static_cast<double>(xyz[3 * i + 2])});
      h32.covariances.push_back({1, 0, 0, 0, 1, 0, 0, 0, 1.0 / 1024});  // float32-exact (1e-3 is not)
    }
    REQUIRE(!PointCloud(ctx, h32).is_f64());
  }

  // ONE batch split over two contexts (two "devices"; here both on device 0): bit-identical blocks,
  // errors and LM result (vgicp_graph_create_sharded)
  {
    Context ctx2(0);
    auto cloud2 = std::make_shared<PointCloud>(cloud->replicate(ctx2));  // replicas: one copy each
    auto map2 = std::make_shared<GaussianVoxelMap>(map->replicate(ctx2));
    REQUIRE(map2->size() == map->size() && map2->voxels() == map->voxels());
    auto mk = [&](const std::shared_ptr<PointCloud>& c, const std::shared_ptr<GaussianVoxelMap>& m) {
      return std::vector<MatchingCostFactor>{MatchingCostFactor(0, 1, c, m), MatchingCostFactor(1, 2, c, m),
                                             MatchingCostFactor(2, 0, c, m), MatchingCostFactor(0, 2, c, m)};
    };
    MatchingCostBatch single(ctx, mk(cloud, map), 3);
    MatchingCostBatch sharded({ctx, ctx2}, {mk(cloud, map), mk(cloud2, map2)}, 3);
    REQUIRE(sharded.num_shards() == 2);
    const std::vector<Pose> poses = {Pose::Identity(), Pose::from({1, 0, 0, 0, 1, 0, 0, 0, 1}, {0.2, -0.1, 0.05}),
                                     Pose::from({1, 0, 0, 0, 1, 0, 0, 0, 1}, {-0.1, 0.15, 0})};
    const auto a = single.linearize(poses), b = sharded.linearize(poses);
    for (std::size_t k = 0; k < a.size(); ++k) {
      REQUIRE(a[k].inliers == b[k].inliers && a[k].error == b[k].error);
      for (int e = 0; e < 36; ++e) REQUIRE(a[k].H_ij[e] == b[k].H_ij[e] && a[k].H_jj[e] == b[k].H_jj[e]);
    }
    REQUIRE(single.total_error(poses) == sharded.total_error(poses));
    std::vector<Pose> p1 = poses, p2 = poses;
    const auto r1 = single.optimize(p1, {1, 0, 0}), r2 = sharded.optimize(p2, {1, 0, 0});
    REQUIRE(r1.final_error == r2.final_error && r1.iterations == r2.iterations);
    for (int k = 0; k < 3; ++k)
      for (int q = 0; q < 12; ++q) REQUIRE(p1[k].m[q] == p2[k].m[q]);
  }

  std::printf("facade ok: voxels=%zu inliers=%d error=%.6f launches=%llu\n", map->size(), lin.inliers, lin.error,
              static_cast<unsigned long long>(ctx.launch_count()));
  return 0;
}
