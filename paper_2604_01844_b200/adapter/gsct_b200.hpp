// gsct_b200.hpp — the reference's C++ operator API (namespace gsct) implemented on the
// B200 C ABI (include/gsct_cuda.h, libgsct_b200.so).
//
// Include AFTER the reference's "gsct/projector.hpp" and "gsct/voxelizer.hpp" (this header
// uses their types: GaussianCloud, ScanGeometry, Image, Volume, GridRegion, GridSpec,
// RasterSettings, VoxelSettings, RenderStats, ParamGradients, contract_error). It defines,
// in namespace gsct::b200, functions with exactly the reference signatures:
//
//   Image          rasterize_view    (cloud, geometry, angle_index, settings, stats)  projector.hpp:308-310
//   ParamGradients rasterize_backward(cloud, geometry, angle_index, grad_image, ...) projector.hpp:371-375
//   Volume         voxelize          (cloud, region, settings, stats)                 voxelizer.hpp:162-163
//   Volume         voxelize_full     (cloud, grid, settings, stats)                   voxelizer.hpp:203-206
//   ParamGradients voxelize_backward (cloud, region, grad_volume, settings, stats)    voxelizer.hpp:214-217
//
// plus batched forms (rasterize_views / rasterize_backward_views: many views per call,
// gradients summed in view order as ParamGradients::add). Semantics: inputs are validated
// like the reference (contract_error with the reference's messages), outputs are fresh
// by-value containers, RenderStats accumulate with +=, calls are synchronous. Images and
// volumes come back from fp32 device buffers widened to double; gradients are fp64.
//
// For a drop-in of the unchanged reference loops (optim.hpp, bench.hpp, CLI) include
// gsct_b200_dropin.hpp first instead (it renames the CPU operators to *_cpu and exposes
// these under the original names).
#pragma once

#include <malloc.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/gsct_cuda.h"

namespace gsct {
namespace b200 {

// The reference API returns fresh multi-MB containers from every call (ParamGradients:
// 96 B/splat, 19 MB at 200k splats, twice per view-step of train_reconstruction). glibc
// serves blocks that large with fresh mmaps by default, so every call pays first-touch page
// faults (measured: ~4 ms per 19 MB result, more than the GPU work of a one-view call). The
// first use of the adapter keeps such blocks in the heap instead (reused, already mapped);
// GSCT_B200_NO_MALLOC_TUNE=1 leaves the process's allocator settings alone.
inline void tune_host_allocator() {
  static const bool done = [] {
    const char* e = std::getenv("GSCT_B200_NO_MALLOC_TUNE");
    if (!(e && e[0] == '1')) {
      mallopt(M_MMAP_THRESHOLD, 32 << 20);    // glibc's upper limit on 64-bit
      mallopt(M_TRIM_THRESHOLD, 1024 << 20);  // keep freed heap for the next call's result
    }
    return true;
  }();
  (void)done;
}

// One context per thread and device (the C ABI context is single-threaded).
class Device {
 public:
  static gsct_ctx ctx(int device = -1) {
    tune_host_allocator();
    thread_local Device d;
    if (device >= 0 && device != d.device_) d.reset(device);
    if (!d.ctx_) d.reset(d.device_ < 0 ? 0 : d.device_);
    return d.ctx_;
  }
  ~Device() {
    if (ctx_) gsct_ctx_destroy(ctx_);
  }

 private:
  void reset(int device) {
    if (ctx_) gsct_ctx_destroy(ctx_);
    ctx_ = nullptr;
    device_ = device;
    if (gsct_ctx_create(device, &ctx_) != GSCT_OK)
      throw error("gsct::b200: no usable CUDA device " + std::to_string(device) + " (no CPU fallback)");
  }
  gsct_ctx ctx_ = nullptr;
  int device_ = -1;
};

// Wall time spent inside the B200 operators of this thread (drop-in accounting: the
// reference loop's own CPU work = its wall time minus this).
struct OpTimes {
  double seconds = 0.0;
  std::int64_t calls = 0;
  double kind_seconds[5] = {0, 0, 0, 0, 0};  // rasterize fwd, rasterize bwd, voxelize, voxelize bwd, loss
  double api_seconds = 0.0;                   // of which inside the C ABI calls (the rest: host-side conversions)
  double pre_seconds[5] = {0, 0, 0, 0, 0};    // per kind: operator entry -> first C ABI call
  double post_seconds[5] = {0, 0, 0, 0, 0};   // per kind: last C ABI call -> operator return
  double api_kind_seconds[5] = {0, 0, 0, 0, 0};
};
inline OpTimes& op_times() {
  static thread_local OpTimes t;
  return t;
}

namespace detail {

struct OpTimer;
inline OpTimer*& active_timer() {
  static thread_local OpTimer* t = nullptr;
  return t;
}

struct OpTimer {
  int kind;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  std::chrono::steady_clock::time_point first_api{}, last_api{};
  OpTimer* outer;
  explicit OpTimer(int k) : kind(k), outer(active_timer()) { active_timer() = this; }
  ~OpTimer() {
    using sec = std::chrono::duration<double>;
    const auto t1 = std::chrono::steady_clock::now();
    const double s = sec(t1 - t0).count();
    op_times().seconds += s;
    op_times().kind_seconds[kind] += s;
    op_times().calls += 1;
    if (first_api != std::chrono::steady_clock::time_point{}) {
      op_times().pre_seconds[kind] += sec(first_api - t0).count();
      op_times().post_seconds[kind] += sec(t1 - last_api).count();
    }
    active_timer() = outer;
  }
};

inline void check_status(gsct_ctx c, int status) {
  if (status == GSCT_OK) return;
  const std::string msg = gsct_ctx_last_error(c);
  if (status == GSCT_ERR_CONTRACT) throw contract_error(msg);
  throw error("gsct::b200: " + msg);
}

// C ABI call timed into op_times().api_seconds
template <class F>
inline void call_api(gsct_ctx c, F&& f) {
  const auto t0 = std::chrono::steady_clock::now();
  const int status = f();
  const auto t1 = std::chrono::steady_clock::now();
  const double s = std::chrono::duration<double>(t1 - t0).count();
  op_times().api_seconds += s;
  if (OpTimer* t = active_timer()) {
    op_times().api_kind_seconds[t->kind] += s;
    if (t->first_api == std::chrono::steady_clock::time_point{}) t->first_api = t0;
    t->last_api = t1;
  }
  check_status(c, status);
}

// GaussianCloud stores std::vector<Vec3/Vec4>: fixed-size Eigen vectors are dense doubles
// (24 / 32 bytes), so the vectors are used in place as AoS double arrays (no copy).
inline gsct_cloud c_cloud(const GaussianCloud& cloud) {
  cloud.validate();
  static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be 3 dense doubles");
  static_assert(sizeof(Vec4) == 4 * sizeof(double), "Vec4 must be 4 dense doubles");
  gsct_cloud c;
  c.n = static_cast<int64_t>(cloud.size());
  c.pos = reinterpret_cast<const double*>(cloud.positions.data());
  c.log_scale = reinterpret_cast<const double*>(cloud.log_scales.data());
  c.quat = reinterpret_cast<const double*>(cloud.rotations.data());
  c.raw_density = cloud.raw_densities.data();
  c.location = GSCT_HOST;
  return c;
}

inline gsct_geometry c_geometry(const ScanGeometry& g) {
  gsct_geometry c;
  c.cone = g.mode == BeamMode::cone ? 1 : 0;
  c.n_u = g.n_u;
  c.n_v = g.n_v;
  c.s_u = g.s_u;
  c.s_v = g.s_v;
  c.source_to_origin = g.source_to_origin;
  c.origin_to_detector = g.origin_to_detector;
  return c;
}

inline gsct_raster_settings c_raster(const RasterSettings& s) {
  gsct_raster_settings c;
  c.tau_cut = s.tau_cut;
  c.sigma_cap = s.sigma_cap;
  c.dilation_px2 = s.dilation_px2;
  c.tile_size = s.tile_size;
  c.dilate = s.dilate ? 1 : 0;
  c.bounding = s.bounding == BoundingMode::square_circumscribed ? 1 : 0;
  return c;
}

inline gsct_voxel_settings c_voxel(const VoxelSettings& s) { return gsct_voxel_settings{s.tau_cut, s.sigma_cap}; }

inline gsct_grid c_grid(const std::array<int, 3>& dims, double spacing, const Vec3& origin) {
  gsct_grid g;
  for (int a = 0; a < 3; ++a) {
    g.dims[a] = dims[a];
    g.origin[a] = origin[a];
  }
  g.spacing = spacing;
  return g;
}

inline void take_stats(const gsct_stats& s, RenderStats* stats) {
  if (!stats) return;
  stats->culled = s.culled;
  stats->degenerate = s.degenerate;
  stats->tile_pairs = s.tile_pairs;
  stats->pixel_pairs = s.pixel_pairs;
  stats->forward_ms = s.forward_ms;
  stats->backward_ms = s.backward_ms;
}

inline gsct_stats put_stats(const RenderStats* stats) {
  gsct_stats s{};
  if (stats) {
    s.culled = stats->culled;
    s.degenerate = stats->degenerate;
    s.tile_pairs = stats->tile_pairs;
    s.pixel_pairs = stats->pixel_pairs;
    s.forward_ms = stats->forward_ms;
    s.backward_ms = stats->backward_ms;
  }
  return s;
}

// zero = false: every element is overwritten by the call, so default-insert (no
// ParamGradients::resize zero pass; Eigen's fixed-size vectors are left uninitialised);
// zero = true: zero-filled, for calls that write only the rows they touch (GSCT_HOST_ZEROED)
inline void build_grads(ParamGradients& g, std::size_t n, bool zero) {
  if (zero) {
    g.resize(n);
    return;
  }
  g.positions.resize(n);
  g.log_scales.resize(n);
  g.rotations.resize(n);
  g.raw_densities.resize(n);
  g.pos_grad_norm.resize(n);
  g.visible.resize(n);
}

// The reference API returns a fresh ParamGradients (19 MB at 200k splats) from every backward
// call; constructing its six vectors is single-threaded host work on the call's critical path
// (measured in the unchanged train_reconstruction: 1.4-1.9 ms per call, two calls per
// view-step). A per-thread worker builds the NEXT result's containers while the caller works
// with the current one, so a call finds them ready (same size) and only moves them out.
// GSCT_B200_NO_PREBUILD=1 builds them inline.
class GradPrebuild {
 public:
  static GradPrebuild& get() {
    static thread_local GradPrebuild p;
    return p;
  }
  // zero: the caller needs zero-filled containers (the prebuilt ones always are)
  ParamGradients take(std::size_t n, bool zero) {
    ParamGradients g;
    if (!enabled_) {
      build_grads(g, n, zero);
      return g;
    }
    std::unique_lock<std::mutex> lk(mu_);
    if (!worker_.joinable()) worker_ = std::thread([this] { loop(); });
    done_cv_.wait(lk, [&] { return !want_; });
    if (ready_ && n_ == n) {
      g = std::move(next_);
    } else {
      lk.unlock();
      build_grads(g, n, zero);
      lk.lock();
    }
    ready_ = false;
    n_ = n;
    want_ = true;  // build the next one
    cv_.notify_one();
    return g;
  }
  ~GradPrebuild() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_one();
    if (worker_.joinable()) worker_.join();
  }

 private:
  GradPrebuild() {
    const char* e = std::getenv("GSCT_B200_NO_PREBUILD");
    enabled_ = !(e && e[0] == '1');
  }
  void loop() {
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return stop_ || want_; });
      if (stop_) return;
      const std::size_t n = n_;
      lk.unlock();
      ParamGradients g;
      bool ok = true;
      try {
        build_grads(g, n, true);  // off the critical path: zero-filled, usable by every call
      } catch (...) {  // e.g. bad_alloc: the next take() builds inline and reports it there
        ok = false;
      }
      lk.lock();
      if (ok) next_ = std::move(g);
      ready_ = ok;
      want_ = false;
      done_cv_.notify_all();
    }
  }
  bool enabled_ = true, want_ = false, ready_ = false, stop_ = false;
  std::size_t n_ = 0;
  ParamGradients next_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::thread worker_;
};

struct GradBuffers {
  ParamGradients g;
  gsct_grads c;
  // sparse = true: zero-filled containers, so a sparse call (voxelize_backward of a sub-region)
  // brings down and writes only the rows of the splats it touched
  explicit GradBuffers(std::size_t n, bool sparse = false) : g(GradPrebuild::get().take(n, sparse)) {
    c.pos = reinterpret_cast<double*>(g.positions.data());
    c.log_scale = reinterpret_cast<double*>(g.log_scales.data());
    c.quat = reinterpret_cast<double*>(g.rotations.data());
    c.raw_density = g.raw_densities.data();
    c.pos_grad_norm = g.pos_grad_norm.data();
    c.visible = g.visible.data();
    c.location = sparse ? GSCT_HOST_ZEROED : GSCT_HOST;
  }
};

}  // namespace detail

// Batched forward: images of angle_indices (all views when empty).
inline std::vector<Image> rasterize_views(const GaussianCloud& cloud, const ScanGeometry& geometry,
                                          const std::vector<std::size_t>& angle_indices,
                                          const RasterSettings& settings = {}, RenderStats* stats = nullptr) {
  geometry.validate();
  detail::OpTimer timer_(0);
  std::vector<double> angles;
  for (std::size_t v : angle_indices) {
    check(v < geometry.angles.size(), "view_frame: angle index out of range");
    angles.push_back(geometry.angles[v]);
  }
  gsct_ctx c = Device::ctx();
  const gsct_cloud cc = detail::c_cloud(cloud);
  const gsct_geometry cg = detail::c_geometry(geometry);
  const gsct_raster_settings rs = detail::c_raster(settings);
  const std::size_t npx = static_cast<std::size_t>(geometry.n_u) * geometry.n_v;
  std::vector<float> buf(npx * angles.size());
  gsct_stats st = detail::put_stats(stats);
  detail::call_api(c, [&] { return gsct_rasterize_fwd(c, &cc, &cg, angles.data(), static_cast<int>(angles.size()), &rs,
                                              buf.data(), GSCT_HOST, stats ? &st : nullptr); });
  detail::take_stats(st, stats);
  std::vector<Image> out(angles.size());
  for (std::size_t v = 0; v < angles.size(); ++v) {
    out[v] = Image::zeros(geometry.n_u, geometry.n_v);
    gsct_host_f32_to_f64(buf.data() + v * npx, out[v].values.data(), static_cast<int64_t>(npx), 1.0);
  }
  return out;
}

// gsct::rasterize_view (projector.hpp:308-360)
inline Image rasterize_view(const GaussianCloud& cloud, const ScanGeometry& geometry, std::size_t angle_index,
                            const RasterSettings& settings = {}, RenderStats* stats = nullptr) {
  return rasterize_views(cloud, geometry, {angle_index}, settings, stats)[0];
}

// Batched backward: sum over the views (ascending) of rasterize_backward.
inline ParamGradients rasterize_backward_views(const GaussianCloud& cloud, const ScanGeometry& geometry,
                                               const std::vector<std::size_t>& angle_indices,
                                               const std::vector<const Image*>& grad_images,
                                               const RasterSettings& settings = {}, RenderStats* stats = nullptr) {
  check(grad_images.size() == angle_indices.size(), "rasterize_backward: one grad image per view");
  detail::OpTimer timer_(1);
  std::vector<double> angles;
  const std::size_t npx = static_cast<std::size_t>(geometry.n_u) * geometry.n_v;
  std::vector<float> gi(npx * angle_indices.size());
  for (std::size_t k = 0; k < angle_indices.size(); ++k) {
    check(grad_images[k]->n_u == geometry.n_u && grad_images[k]->n_v == geometry.n_v,
          "rasterize_backward: grad image dims must match detector");
    check(angle_indices[k] < geometry.angles.size(), "view_frame: angle index out of range");
    angles.push_back(geometry.angles[angle_indices[k]]);
    gsct_host_f64_to_f32(grad_images[k]->values.data(), gi.data() + k * npx, static_cast<int64_t>(npx));
  }
  gsct_ctx c = Device::ctx();
  const gsct_cloud cc = detail::c_cloud(cloud);
  const gsct_geometry cg = detail::c_geometry(geometry);
  const gsct_raster_settings rs = detail::c_raster(settings);
  detail::GradBuffers gb(cloud.size());
  gsct_stats st = detail::put_stats(stats);
  detail::call_api(c, [&] { return gsct_rasterize_bwd(c, &cc, &cg, angles.data(), static_cast<int>(angles.size()), &rs,
                                              gi.data(), GSCT_HOST, &gb.c, stats ? &st : nullptr); });
  detail::take_stats(st, stats);
  return std::move(gb.g);  // a member: no implicit move, so move explicitly (19 MB at 200k)
}

// gsct::rasterize_backward (projector.hpp:371-482)
inline ParamGradients rasterize_backward(const GaussianCloud& cloud, const ScanGeometry& geometry,
                                         std::size_t angle_index, const Image& grad_image,
                                         const RasterSettings& settings = {}, RenderStats* stats = nullptr) {
  check(grad_image.n_u == geometry.n_u && grad_image.n_v == geometry.n_v,
        "rasterize_backward: grad image dims must match detector");
  return rasterize_backward_views(cloud, geometry, {angle_index}, {&grad_image}, settings, stats);
}

// gsct::voxelize (voxelizer.hpp:162-199)
inline Volume voxelize(const GaussianCloud& cloud, const GridRegion& region, const VoxelSettings& settings = {},
                       RenderStats* stats = nullptr) {
  detail::OpTimer timer_(2);
  gsct_ctx c = Device::ctx();
  const gsct_cloud cc = detail::c_cloud(cloud);
  const gsct_grid g = detail::c_grid(region.dims, region.spacing, region.origin);
  const gsct_voxel_settings vs = detail::c_voxel(settings);
  Volume out = Volume::zeros(region.dims, region.spacing, region.origin);
  std::vector<float> buf(out.values.size());
  gsct_stats st = detail::put_stats(stats);
  detail::call_api(c, [&] { return gsct_voxelize_fwd(c, &cc, &g, nullptr, &vs, buf.data(), GSCT_HOST, stats ? &st : nullptr); });
  detail::take_stats(st, stats);
  gsct_host_f32_to_f64(buf.data(), out.values.data(), static_cast<int64_t>(buf.size()), 1.0);
  return out;
}

// gsct::voxelize_full (voxelizer.hpp:203-206)
inline Volume voxelize_full(const GaussianCloud& cloud, const GridSpec& grid, const VoxelSettings& settings = {},
                            RenderStats* stats = nullptr) {
  return voxelize(cloud, GridRegion::covering(grid), settings, stats);
}

// gsct::voxelize_backward (voxelizer.hpp:214-263)
inline ParamGradients voxelize_backward(const GaussianCloud& cloud, const GridRegion& region,
                                        const Volume& grad_volume, const VoxelSettings& settings = {},
                                        RenderStats* stats = nullptr) {
  check(grad_volume.dims == region.dims, "voxelize_backward: grad dims must match region");
  detail::OpTimer timer_(3);
  gsct_ctx c = Device::ctx();
  const gsct_cloud cc = detail::c_cloud(cloud);
  const gsct_grid g = detail::c_grid(region.dims, region.spacing, region.origin);
  const gsct_voxel_settings vs = detail::c_voxel(settings);
  std::vector<float> gv(grad_volume.values.size());
  gsct_host_f64_to_f32(grad_volume.values.data(), gv.data(), static_cast<int64_t>(gv.size()));
  detail::GradBuffers gb(cloud.size(), /*sparse=*/true);
  gsct_stats st = detail::put_stats(stats);
  detail::call_api(c, [&] { return gsct_voxelize_bwd(c, &cc, &g, nullptr, &vs, gv.data(), GSCT_HOST, &gb.c,
                                             stats ? &st : nullptr); });
  detail::take_stats(st, stats);
  return std::move(gb.g);  // a member: no implicit move, so move explicitly (19 MB at 200k)
}

}  // namespace b200
}  // namespace gsct
