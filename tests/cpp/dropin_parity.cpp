// Drop-in parity suite (GPU): the reference's own types, fixtures and training loops, with
// the five hot-path operators bound to libgsct_b200.so through
// paper_2604_01844_b200/adapter/gsct_b200_dropin.hpp. The reference CPU operators stay
// available in-process as *_cpu and serve as the oracle. Tolerances follow the north_star
// (fp32 per-pair arithmetic): images/volumes 1e-4 of peak, gradients 1e-4 of the per-class
// maximum; integer counters exact; bitwise properties that survive fp32 (exact doubling,
// power-of-two homogeneity, fixed-order stability, duplicate-splat gradients) bitwise.
//
// Built by oracle/Makefile (needs /root/reference headers at build time) into
// oracle/_ref/dropin_parity; run by tests/test_dropin.py on the GPU box.
#include "gsct_b200_dropin.hpp"

#include <catch2/catch_amalgamated.hpp>
#include <cmath>

#include "gsct/bench.hpp"
#include "gsct/optim.hpp"
#include "gsct/synthetic.hpp"
#include "oracles.hpp"

using namespace gsct;

namespace {

ScanGeometry parallel_geometry(int n, double spacing, std::vector<double> angles) {
  ScanGeometry geom;
  geom.mode = BeamMode::parallel;
  geom.n_u = geom.n_v = n;
  geom.s_u = geom.s_v = spacing;
  geom.angles = std::move(angles);
  return geom;
}

ScanGeometry cone_geometry(int n, double spacing, std::vector<double> angles) {
  ScanGeometry geom = parallel_geometry(n, spacing, std::move(angles));
  geom.mode = BeamMode::cone;
  geom.source_to_origin = 50.0;
  geom.origin_to_detector = 25.0;
  return geom;
}

RasterSettings oracle_settings() {
  RasterSettings rs;
  rs.tau_cut = 1e-12;
  rs.sigma_cap = 6.0;
  rs.dilate = false;
  return rs;
}

template <class V>
double class_error(const std::vector<V>& a, const std::vector<V>& b) {
  double peak = 0.0, worst = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i)
    for (int k = 0; k < static_cast<int>(V::SizeAtCompileTime); ++k) {
      peak = std::max(peak, std::abs(b[i][k]));
      worst = std::max(worst, std::abs(a[i][k] - b[i][k]));
    }
  return peak > 0 ? worst / peak : worst;
}

double class_error(const std::vector<double>& a, const std::vector<double>& b) {
  return oracles::max_error_relative_to_peak(a, b);
}

void check_grads(const ParamGradients& g, const ParamGradients& r, double tol) {
  CHECK(class_error(g.positions, r.positions) <= tol);
  CHECK(class_error(g.log_scales, r.log_scales) <= tol);
  CHECK(class_error(g.rotations, r.rotations) <= tol);
  CHECK(class_error(g.raw_densities, r.raw_densities) <= tol);
  CHECK(class_error(g.pos_grad_norm, r.pos_grad_norm) <= tol);
  CHECK(g.visible == r.visible);
}

}  // namespace

TEST_CASE("drop-in rasterize_view matches the CPU reference (stats exact)") {
  const GaussianCloud cloud = oracles::random_cloud(35, 60);
  for (const bool cone : {false, true}) {
    for (const bool oracle : {false, true}) {
      const ScanGeometry geom = cone ? cone_geometry(48, 0.7, {0.9, 2.5}) : parallel_geometry(52, 0.55, {0.3, 2.4});
      const RasterSettings rs = oracle ? oracle_settings() : RasterSettings{};
      for (std::size_t v = 0; v < 2; ++v) {
        RenderStats sg, sc;
        const Image img = rasterize_view(cloud, geom, v, rs, &sg);
        const Image ref = rasterize_view_cpu(cloud, geom, v, rs, &sc);
        INFO("cone " << cone << " oracle " << oracle << " view " << v);
        CHECK(oracles::max_error_relative_to_peak(img.values, ref.values) <= 1e-4);
        CHECK(sg.culled == sc.culled);
        CHECK(sg.degenerate == sc.degenerate);
        CHECK(sg.tile_pairs == sc.tile_pairs);
        CHECK(sg.pixel_pairs == sc.pixel_pairs);
      }
    }
  }
}

TEST_CASE("drop-in rasterize_backward matches the CPU reference") {
  for (const bool cone : {false, true}) {
    const GaussianCloud cloud = oracles::random_cloud(cone ? 42 : 41, 12);
    const ScanGeometry geom = cone ? cone_geometry(36, 0.7, {0.9}) : parallel_geometry(36, 0.7, {0.9});
    Image grad = Image::zeros(geom.n_u, geom.n_v);
    Rng rng(99);
    for (double& x : grad.values) x = static_cast<float>(rng.uniform(-1, 1));
    for (const bool oracle : {false, true}) {
      const RasterSettings rs = oracle ? oracle_settings() : RasterSettings{};
      INFO("cone " << cone << " oracle " << oracle);
      check_grads(rasterize_backward(cloud, geom, 0, grad, rs), rasterize_backward_cpu(cloud, geom, 0, grad, rs),
                  1e-4);
    }
  }
}

TEST_CASE("drop-in voxelize / voxelize_full / voxelize_backward match the CPU reference") {
  const GaussianCloud cloud = oracles::random_cloud(54, 20, 4.0);
  const GridSpec grid = GridSpec::centered({20, 22, 18}, 0.8);
  for (const bool wide : {false, true}) {
    VoxelSettings vs;
    if (wide) {
      vs.tau_cut = 1e-12;
      vs.sigma_cap = 8.0;
    }
    RenderStats sg, sc;
    const Volume vol = voxelize_full(cloud, grid, vs, &sg);
    const Volume ref = voxelize_full_cpu(cloud, grid, vs, &sc);
    CHECK(oracles::max_error_relative_to_peak(vol.values, ref.values) <= 1e-4);
    CHECK(sg.culled == sc.culled);
    CHECK(sg.pixel_pairs == sc.pixel_pairs);
    const GridRegion region = GridRegion::of_parent(grid, {3, 2, 5}, {9, 11, 7});
    const Volume win = voxelize(cloud, region, vs);
    CHECK(oracles::max_error_relative_to_peak(win.values, voxelize_cpu(cloud, region, vs).values) <= 1e-4);
    Volume gv = Volume::zeros(grid.dims, grid.spacing, grid.origin);
    Rng rng(7);
    for (double& x : gv.values) x = static_cast<float>(rng.uniform(-1, 1));
    check_grads(voxelize_backward(cloud, GridRegion::covering(grid), gv, vs),
                voxelize_backward_cpu(cloud, GridRegion::covering(grid), gv, vs), 1e-4);
  }
}

TEST_CASE("drop-in bitwise properties (test_projector.cpp:177-268, 366-379)") {
  const ScanGeometry geom = parallel_geometry(33, 1.0, {0.0});
  SECTION("two identical splats render exactly twice one") {
    GaussianCloud one;
    one.push_back(Vec3(0.5, -1, 2), Vec3::Constant(std::log(3.0)), Vec4(1, 0, 0, 0), 0.9);
    GaussianCloud two = one;
    two.push_back(one.positions[0], one.log_scales[0], one.rotations[0], one.raw_densities[0]);
    const Image a = rasterize_view(one, geom, 0);
    const Image b = rasterize_view(two, geom, 0);
    for (std::size_t i = 0; i < a.values.size(); ++i) CHECK(b.values[i] == 2.0 * a.values[i]);
  }
  SECTION("power-of-two density factors scale exactly; fixed order is bit-stable") {
    const GaussianCloud cloud = oracles::random_cloud(33, 6);
    const ScanGeometry g2 = parallel_geometry(40, 0.6, {0.2});
    RasterSettings rs;
    rs.tau_cut = 1e-12;
    const Image base = rasterize_view(cloud, g2, 0, rs);
    for (const double c : {0.0, 0.5, 2.0, 4.0}) {
      GaussianCloud scaled = cloud;
      for (double& d : scaled.raw_densities) d *= c;
      const Image img = rasterize_view(scaled, g2, 0, rs);
      for (std::size_t i = 0; i < img.values.size(); ++i) CHECK(img.values[i] == c * base.values[i]);
    }
    const Image again = rasterize_view(cloud, g2, 0, rs);
    for (std::size_t i = 0; i < base.values.size(); ++i) CHECK(again.values[i] == base.values[i]);
  }
  SECTION("duplicated splats receive identical gradients") {
    GaussianCloud cloud = oracles::random_cloud(43, 3);
    cloud.push_back(cloud.positions[1], cloud.log_scales[1], cloud.rotations[1], cloud.raw_densities[1]);
    const ScanGeometry g3 = parallel_geometry(32, 0.7, {0.4});
    Image grad = Image::zeros(32, 32);
    Rng rng(5);
    for (double& x : grad.values) x = rng.uniform(-1, 1);
    const ParamGradients g = rasterize_backward(cloud, g3, 0, grad);
    CHECK(g.positions[1] == g.positions[3]);
    CHECK(g.log_scales[1] == g.log_scales[3]);
    CHECK(g.rotations[1] == g.rotations[3]);
    CHECK(g.raw_densities[1] == g.raw_densities[3]);
  }
}

TEST_CASE("drop-in contract errors are gsct::contract_error") {
  GaussianCloud cloud = oracles::random_cloud(1, 4);
  cloud.positions[2][1] = std::nan("");
  const ScanGeometry geom = parallel_geometry(16, 1.0, {0.0});
  try {
    rasterize_view(cloud, geom, 0);
    FAIL("expected contract_error");
  } catch (const contract_error& e) {
    CHECK(std::string(e.what()).find("splat 2") != std::string::npos);
  }
  CHECK_THROWS_AS(rasterize_view(oracles::random_cloud(1, 4), parallel_geometry(0, 1.0, {0.0}), 0), contract_error);
  CHECK_THROWS_AS(rasterize_backward(oracles::random_cloud(1, 4), geom, 0, Image::zeros(8, 16)), contract_error);
  CHECK_THROWS_AS(rasterize_view(oracles::random_cloud(1, 4), geom, 3), contract_error);
  GaussianCloud lockstep = oracles::random_cloud(1, 4);
  lockstep.raw_densities.push_back(1.0);
  CHECK_THROWS_AS(voxelize_full(lockstep, GridSpec::centered({8, 8, 8}, 1.0)), contract_error);
}

TEST_CASE("unchanged train_reconstruction converges on the B200 operators (test_optim.cpp:226-273)") {
  const int n_views = 12;
  GaussianCloud truth;
  Rng rng(77);
  for (int i = 0; i < 20; ++i) {
    truth.push_back(Vec3(rng.uniform(-6, 6), rng.uniform(-6, 6), rng.uniform(-6, 6)),
                    Vec3::Constant(std::log(rng.uniform(1.2, 2.5))), Vec4(1, 0, 0, 0), rng.uniform(0.4, 1.0));
  }
  ScanGeometry geom;
  geom.mode = BeamMode::parallel;
  geom.n_u = geom.n_v = 48;
  geom.s_u = geom.s_v = 0.55;
  geom.angles = default_angles(n_views, BeamMode::parallel);
  ProjectionSet projections;
  projections.geometry = geom;
  for (int view = 0; view < n_views; ++view) projections.images.push_back(rasterize_view(truth, geom, view));
  GaussianCloud start = truth;
  for (std::size_t i = 0; i < start.size(); ++i) {
    start.positions[i] += Vec3(rng.uniform(-0.4, 0.4), rng.uniform(-0.4, 0.4), rng.uniform(-0.4, 0.4));
    start.log_scales[i] += Vec3::Constant(rng.uniform(-0.15, 0.15));
    start.raw_densities[i] *= rng.uniform(0.7, 1.3);
  }
  TrainConfig config;
  config.densify_start = 1 << 20;  // adaptive control off (test_optim.cpp:106-110)
  config.iterations = 200;
  config.weights.alpha_tv = 0.0;
  config.weights.alpha_ssim = 0.25;
  config.seed = 5;
  config.lr_scale = 1e-3;
  config.lr_density = 2e-3;
  config.lr_rotation = 2e-4;
  TrainOptions options;
  options.deterministic = true;
  const TrainResult result = train_reconstruction(start, projections, config, options);
  REQUIRE_FALSE(result.diverged);
  REQUIRE(result.log.size() == 200);
  INFO("final L1 " << result.log.back().l1);
  CHECK(result.log.back().l1 < 1e-3);
  // determinism of the whole loop on the GPU operators
  const TrainResult again = train_reconstruction(start, projections, config, options);
  CHECK(again.log.back().l1 == result.log.back().l1);
}

TEST_CASE("unchanged train_volume_fit is stable at an exact fixed point (test_optim.cpp:307-333)") {
  GaussianCloud cloud;
  cloud.push_back(Vec3::Zero(), Vec3::Constant(std::log(1.2)), Vec4(1, 0, 0, 0), 1.0);
  cloud.push_back(Vec3(6, 6, 6), Vec3::Constant(std::log(0.9)), Vec4(1, 0, 0, 0), 0.5);
  cloud.push_back(Vec3(-6, 5, -4), Vec3::Constant(std::log(0.8)), Vec4(1, 0, 0, 0), 0.4);
  const GridSpec grid = GridSpec::centered({17, 17, 17}, 1.0);
  const Volume target = voxelize_full(cloud, grid);
  REQUIRE(target.max_value() == 1.0);
  TrainConfig config;
  config.densify_start = 1 << 20;  // adaptive control off (test_optim.cpp:106-110)
  config.iterations = 50;
  config.weights.alpha_ssim = 0.0;
  config.eval_interval = 1 << 20;
  const TrainResult result = train_volume_fit(cloud, target, config);
  CHECK(result.log.back().total == 0.0);
}

TEST_CASE("unchanged bench sweep runs on the B200 operators (test_bench.cpp:435-461)") {
  SweepConfig config;
  config.target = SweepTarget::rasterize;
  config.sides = {32, 64};
  config.counts = {200};
  config.repeats = 1;
  config.seed = 3;
  const std::vector<BenchRow> rows = sweep(config);
  REQUIRE(rows.size() == 2);
  CHECK(rows[0].work_pairs > 0);
  config.target = SweepTarget::voxelize;
  config.sides = {24};
  const std::vector<BenchRow> a = sweep(config);
  const std::vector<BenchRow> b = sweep(config);
  CHECK(a[0].work_pairs == b[0].work_pairs);
}
