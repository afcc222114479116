// One epoch of the UNCHANGED reference training loop train_reconstruction (optim.hpp:397-538)
// at a benchmark configuration, timed end to end. Built twice by oracle/Makefile:
//   dropin_train_b200: with gsct_b200_dropin.hpp, so the loop's rasterize_view /
//                      rasterize_backward / voxelize / voxelize_backward calls run on the
//                      B200 operators through the C++ adapter (libgsct_b200.so);
//   dropin_train_cpu:  the plain reference (the CPU baseline of the same loop).
// Everything else in the loop (view shuffling, sample_subvolume, total_loss_recon with
// L1 + SSIM2D + TV3D, accumulate_control_stats, lr_schedule, adam_step) is the reference's
// CPU code in both builds. Prints one JSON line.
//
//   dropin_train_{b200,cpu} <gaussians> <side> <views> <det> [epochs]
//
// Inputs: the benchmark's Shepp-Logan phantom cloud (bench.py make_workload, drawn with the
// reference Rng exactly as oracle/ref_capi.cpp ref_shepp_logan_cloud), default_geometry
// (synthetic.hpp:246-271); the targets are the projections of that cloud, the training
// starts from a second draw (seed 1). Harness only -- TEST / BENCH INFRASTRUCTURE.
#ifdef GSCT_DROPIN
#include "gsct_b200_dropin.hpp"
#endif

#include <sys/resource.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "gsct/optim.hpp"
#include "gsct/synthetic.hpp"

using namespace gsct;

namespace {

GaussianCloud shepp_logan_cloud(std::int64_t count, double side, double sp, std::uint64_t seed) {
  Rng rng(seed);
  const double half = 0.5 * side * sp;
  const double ax = 0.69 * half, ay = 0.92 * half, az = 0.81 * half;
  const double vfg = 4.0 / 3.0 * M_PI * ax * ay * az;
  const double s0 = 0.554 * std::cbrt(vfg / static_cast<double>(count > 0 ? count : 1));
  GaussianCloud c;
  for (std::int64_t i = 0; i < count; ++i) {
    double x, y, z;
    do {
      x = rng.uniform(-1.0, 1.0);
      y = rng.uniform(-1.0, 1.0);
      z = rng.uniform(-1.0, 1.0);
    } while (x * x + y * y + z * z > 1.0);
    double ls[3];
    for (double& l : ls) l = std::log(s0) + rng.uniform(-0.3, 0.3);
    double qq[4] = {rng.normal(), rng.normal(), rng.normal(), rng.normal()};
    double zz = qq[0] * qq[0];
    zz += qq[1] * qq[1];
    zz += qq[2] * qq[2];
    zz += qq[3] * qq[3];
    if (std::sqrt(zz) == 0.0) {
      qq[0] = 1;
      qq[1] = qq[2] = qq[3] = 0;
      zz = 1.0;
    }
    const double nrm = std::sqrt(zz);
    c.positions.push_back(Vec3(x * ax, y * ay, z * az));
    c.log_scales.push_back(Vec3(ls[0], ls[1], ls[2]));
    c.rotations.push_back(Vec4(qq[0] / nrm, qq[1] / nrm, qq[2] / nrm, qq[3] / nrm));
    c.raw_densities.push_back(0.15 * rng.uniform(0.2, 1.0));
  }
  return c;
}

}  // namespace

int main(int argc, char** argv) {
  const std::int64_t n = argc > 1 ? std::atoll(argv[1]) : 200000;
  const int side = argc > 2 ? std::atoi(argv[2]) : 256;
  const int views = argc > 3 ? std::atoi(argv[3]) : 75;
  const int det = argc > 4 ? std::atoi(argv[4]) : 512;
  const int epochs = argc > 5 ? std::atoi(argv[5]) : 1;

  const Volume vol = Volume::zeros({side, side, side}, 1.0, Vec3::Zero());
  ProjectionSet proj;
  proj.geometry = default_geometry(vol, static_cast<std::size_t>(views), BeamMode::cone, det, det);
  const GaussianCloud truth = shepp_logan_cloud(n, side, 1.0, 0);
  const auto t_targets = std::chrono::steady_clock::now();
  for (int v = 0; v < views; ++v) proj.images.push_back(rasterize_view(truth, proj.geometry, v));
  const double targets_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_targets).count();
  const GaussianCloud init = shepp_logan_cloud(n, side, 1.0, 1);

  TrainConfig cfg;
  cfg.iterations = epochs;
  cfg.max_gaussians = static_cast<std::size_t>(2 * n);
  TrainOptions opt;
  opt.deterministic = true;
#ifdef GSCT_DROPIN
  // warm-up: one view-step's operators (context creation, workspace growth, module load)
  {
    const Image r = rasterize_view(init, proj.geometry, 0);
    (void)rasterize_backward(init, proj.geometry, 0, r);
  }
  b200::op_times() = b200::OpTimes{};
#endif
  const auto t0 = std::chrono::steady_clock::now();
  const TrainResult res = train_reconstruction(init, proj, cfg, opt);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  double op_s = 0.0;
  long long op_calls = 0;
#ifdef GSCT_DROPIN
  op_s = b200::op_times().seconds;
  std::fprintf(stderr, "operator seconds inside the C ABI: %.3f\n", b200::op_times().api_seconds);
  for (int k = 0; k < 5; ++k)
    std::fprintf(stderr, "  kind %d: total %.3f api %.3f pre %.3f post %.3f\n", k, b200::op_times().kind_seconds[k],
                 b200::op_times().api_kind_seconds[k], b200::op_times().pre_seconds[k],
                 b200::op_times().post_seconds[k]);
  std::fprintf(stderr, "operator seconds by kind: fwd %.3f bwd %.3f vox %.3f voxbwd %.3f loss %.3f\n",
               b200::op_times().kind_seconds[0], b200::op_times().kind_seconds[1], b200::op_times().kind_seconds[2],
               b200::op_times().kind_seconds[3], b200::op_times().kind_seconds[4]);
  op_calls = static_cast<long long>(b200::op_times().calls);
  const char* impl = "b200_dropin";
#else
  const char* impl = "reference_cpu";
#endif
  const double steps = static_cast<double>(views) * epochs;

  // per-call wall times of one view-step's pieces (same call pattern as the loop body)
  auto ms_of = [](auto&& f) {
    f();
    const int reps = 5;
    const auto a = std::chrono::steady_clock::now();
    for (int k = 0; k < reps; ++k) f();
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count() / reps;
  };
  GaussianCloud cl = res.cloud;
  Rng rng(7);
  const GridSpec grid = GridSpec::of(Volume::zeros({side, side, side}, 1.0, Vec3::Zero()));
  const GridRegion region = sample_subvolume(grid, cfg.tv_subvolume, rng);
  const Image rendered = rasterize_view(cl, proj.geometry, 1);
  const Volume sub = voxelize(cl, region);
  const ReconLoss loss = total_loss_recon(rendered, proj.images[1], sub, cfg.weights);
  ParamGradients grads = rasterize_backward(cl, proj.geometry, 1, loss.grad_image);
  OptimState st;
  st.init(cl.size(), 0);
  LearningRates lrs;
  const double t_fwd = ms_of([&] { (void)rasterize_view(cl, proj.geometry, 1); });
  const double t_vox = ms_of([&] { (void)voxelize(cl, region); });
  const double t_loss = ms_of([&] { (void)total_loss_recon(rendered, proj.images[1], sub, cfg.weights); });
  const double t_bwd = ms_of([&] { (void)rasterize_backward(cl, proj.geometry, 1, loss.grad_image); });
  const double t_vbwd = ms_of([&] { (void)voxelize_backward(cl, region, loss.grad_subvolume); });
  const double t_adam = ms_of([&] { adam_step(cl, st, grads, lrs); });
  // the loop body of train_reconstruction (optim.hpp:456-492) restated with a timer per
  // piece, over 20 view-steps: where a view-step's wall time goes
  double piece[8] = {}, faults[8] = {};
  const char* piece_name[8] = {"sample_subvolume", "rasterize_view", "voxelize", "total_loss_recon",
                               "rasterize_backward", "accumulate_control_stats", "voxelize_backward+add",
                               "adam_step"};
  {
    OptimState s2;
    s2.init(cl.size(), 0);
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto minflt = [] {
      rusage u{};
      getrusage(RUSAGE_SELF, &u);
      return static_cast<long long>(u.ru_minflt);
    };
    long long flt_mark = minflt();
    auto tick = [&](int k, std::chrono::steady_clock::time_point& t) {
      const auto t2 = now();
      piece[k] += std::chrono::duration<double, std::milli>(t2 - t).count();
      const long long f = minflt();
      faults[k] += static_cast<double>(f - flt_mark);
      flt_mark = f;
      t = t2;
    };
    const int n_steps = 20;
    for (int s = 0; s < n_steps; ++s) {
      const std::size_t view = static_cast<std::size_t>(s % views);
      auto t = now();
      const GridRegion reg = sample_subvolume(grid, cfg.tv_subvolume, s2.rng);
      tick(0, t);
      const Image r = rasterize_view(cl, proj.geometry, view);
      tick(1, t);
      const Volume sv = voxelize(cl, reg);
      tick(2, t);
      const ReconLoss lo = total_loss_recon(r, proj.images[view], sv, cfg.weights);
      tick(3, t);
      ParamGradients g = rasterize_backward(cl, proj.geometry, view, lo.grad_image);
      tick(4, t);
      detail::accumulate_control_stats(s2, g);
      tick(5, t);
      const ParamGradients tg = voxelize_backward(cl, reg, lo.grad_subvolume);
      g.add(tg);
      tick(6, t);
      adam_step(cl, s2, g, lrs);
      tick(7, t);
    }
    for (double& p : piece) p /= n_steps;
    // minor page faults per piece (first touches of fresh heap / mmap pages)
    std::fprintf(stderr, "minor faults per view-step piece:");
    for (int k = 0; k < 8; ++k) std::fprintf(stderr, " %s %.0f", piece_name[k], faults[k] / n_steps);
    std::fprintf(stderr, "\n");
  }
  std::printf(
      "{\"impl\": \"%s\", \"gaussians\": %lld, \"views\": %d, \"detector\": %d, \"epochs\": %d, "
      "\"wall_s\": %.4f, \"view_steps_per_s\": %.4f, \"operator_s\": %.4f, \"operator_calls\": %lld, "
      "\"targets_s\": %.4f, \"loss_first\": %.6g, \"diverged\": %s, \"threads\": %d, "
      "\"call_ms\": {\"rasterize_view\": %.3f, \"voxelize_32\": %.3f, \"total_loss_recon\": %.3f, "
      "\"rasterize_backward\": %.3f, \"voxelize_backward_32\": %.3f, \"adam_step\": %.3f}, "
      "\"loop_piece_ms\": {\"%s\": %.3f, \"%s\": %.3f, \"%s\": %.3f, \"%s\": %.3f, \"%s\": %.3f, \"%s\": %.3f, "
      "\"%s\": %.3f, \"%s\": %.3f}}\n",
      impl, static_cast<long long>(n), views, det, epochs, wall, steps / wall, op_s, op_calls, targets_s,
      res.log.empty() ? 0.0 : res.log.front().total, res.diverged ? "true" : "false", thread_count(), t_fwd, t_vox,
      t_loss, t_bwd, t_vbwd, t_adam, piece_name[0], piece[0], piece_name[1], piece[1], piece_name[2], piece[2],
      piece_name[3], piece[3], piece_name[4], piece[4], piece_name[5], piece[5], piece_name[6], piece[6],
      piece_name[7], piece[7]);
  return 0;
}
