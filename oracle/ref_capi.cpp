// TEST INFRASTRUCTURE ONLY. A thin extern "C" wrapper that calls the UNCHANGED reference
// implementation (/root/reference/proj/include/gsct/*.hpp, compiled here with the
// Eigen-subset shim) so Python tests and bench.py's reference arm can call it through
// ctypes. Built by oracle/Makefile into oracle/_ref/libgsct_ref.so (git-ignored, travels
// to the GPU box prebuilt). Array layouts match oracle/gsct_oracle.h.
#include <cstdint>
#include <sstream>
#include <cstring>
#include <exception>
#include <string>

#include "gsct/bench.hpp"
#include "gsct/core.hpp"
#include "gsct/io.hpp"
#include "gsct/losses.hpp"
#include "gsct/optim.hpp"
#include "gsct/parallel.hpp"
#include "gsct/projector.hpp"
#include "gsct/synthetic.hpp"
#include "gsct/voxelizer.hpp"
#include "oracles.hpp"

using namespace gsct;

namespace {
std::string g_err;

struct Geo {
  int cone, n_u, n_v;
  double s_u, s_v, source_to_origin, origin_to_detector;
};
struct RS {
  double tau_cut, sigma_cap, dilation_px2;
  int tile_size, dilate, bounding;
};
struct VS {
  double tau_cut, sigma_cap;
};
struct Region {
  int dims[3];
  double spacing;
  double origin[3];
};
struct Stats {
  int64_t culled, degenerate, tile_pairs, pixel_pairs;
};

ScanGeometry to_geom(const Geo* g, const double* angles, int n_angles) {
  ScanGeometry geom;
  geom.mode = g->cone ? BeamMode::cone : BeamMode::parallel;
  geom.n_u = g->n_u;
  geom.n_v = g->n_v;
  geom.s_u = g->s_u;
  geom.s_v = g->s_v;
  geom.source_to_origin = g->source_to_origin;
  geom.origin_to_detector = g->origin_to_detector;
  geom.angles.assign(angles, angles + n_angles);
  return geom;
}
RasterSettings to_rs(const RS* r) {
  RasterSettings s;
  s.tau_cut = r->tau_cut;
  s.sigma_cap = r->sigma_cap;
  s.dilation_px2 = r->dilation_px2;
  s.tile_size = r->tile_size;
  s.dilate = r->dilate != 0;
  s.bounding = r->bounding ? BoundingMode::square_circumscribed : BoundingMode::rect_density_aware;
  return s;
}
VoxelSettings to_vs(const VS* v) {
  VoxelSettings s;
  s.tau_cut = v->tau_cut;
  s.sigma_cap = v->sigma_cap;
  return s;
}
GridRegion to_region(const Region* r) {
  GridRegion g;
  g.dims = {r->dims[0], r->dims[1], r->dims[2]};
  g.spacing = r->spacing;
  g.origin = Vec3(r->origin[0], r->origin[1], r->origin[2]);
  return g;
}
void put_stats(const RenderStats& s, Stats* out, double* ms) {
  if (out) {
    out->culled += s.culled;
    out->degenerate += s.degenerate;
    out->tile_pairs += s.tile_pairs;
    out->pixel_pairs += s.pixel_pairs;
  }
  if (ms) {
    ms[0] += s.forward_ms;
    ms[1] += s.backward_ms;
  }
}
void put_grads(const ParamGradients& g, double* gp, double* gl, double* gq, double* gr,
               double* pgn, uint8_t* vis) {
  const std::size_t n = g.positions.size();
  for (std::size_t i = 0; i < n; ++i) {
    for (int k = 0; k < 3; ++k) {
      gp[3 * i + k] = g.positions[i][k];
      gl[3 * i + k] = g.log_scales[i][k];
    }
    for (int k = 0; k < 4; ++k) gq[4 * i + k] = g.rotations[i][k];
    gr[i] = g.raw_densities[i];
    pgn[i] = g.pos_grad_norm[i];
    vis[i] = g.visible[i];
  }
}
}  // namespace

#define GUARD(...)                       \
  try {                                  \
    __VA_ARGS__;                         \
    return 0;                            \
  } catch (const contract_error& e) {    \
    g_err = e.what();                    \
    return 1;                            \
  } catch (const std::exception& e) {    \
    g_err = e.what();                    \
    return 2;                            \
  }

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { set_thread_count(n); }
int ref_thread_count() { return thread_count(); }

void* ref_cloud_create(int64_t n, const double* pos, const double* ls, const double* q,
                       const double* raw) {
  auto* c = new GaussianCloud();
  c->reserve(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    c->push_back(Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]),
                 Vec3(ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]),
                 Vec4(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]), raw[i]);
  }
  return c;
}
void ref_cloud_destroy(void* c) { delete static_cast<GaussianCloud*>(c); }

int ref_rasterize_view(void* cloud, const Geo* g, const double* angles, int n_angles, int view,
                       const RS* rs, double* image, Stats* stats, double* ms) {
  GUARD({
    RenderStats s;
    const Image img = rasterize_view(*static_cast<GaussianCloud*>(cloud), to_geom(g, angles, n_angles),
                                     static_cast<std::size_t>(view), to_rs(rs), &s);
    std::memcpy(image, img.values.data(), img.values.size() * sizeof(double));
    put_stats(s, stats, ms);
  })
}

int ref_rasterize_backward(void* cloud, const Geo* g, const double* angles, int n_angles, int view,
                           const double* grad_image, const RS* rs, double* gp, double* gl,
                           double* gq, double* gr, double* pgn, uint8_t* vis, double* ms) {
  GUARD({
    const ScanGeometry geom = to_geom(g, angles, n_angles);
    Image gi = Image::zeros(geom.n_u, geom.n_v);
    std::memcpy(gi.values.data(), grad_image, gi.values.size() * sizeof(double));
    RenderStats s;
    const ParamGradients pg = rasterize_backward(*static_cast<GaussianCloud*>(cloud), geom,
                                                 static_cast<std::size_t>(view), gi, to_rs(rs), &s);
    put_grads(pg, gp, gl, gq, gr, pgn, vis);
    put_stats(s, nullptr, ms);
  })
}

// project_cloud + bin_tiles for one view: per-splat bbox/flags and the CSR tile lists.
int ref_project_and_bin(void* cloud, const Geo* g, const double* angles, int n_angles, int view,
                        const RS* rs, int32_t* rect /*4N*/, uint8_t* culled, uint8_t* degenerate,
                        double* mean2d /*2N*/, double* conic /*4N*/, double* amplitude,
                        int64_t* tile_offsets, int32_t* tile_splats, int64_t* n_pairs) {
  GUARD({
    const GaussianCloud& c = *static_cast<GaussianCloud*>(cloud);
    const ScanGeometry geom = to_geom(g, angles, n_angles);
    const ViewFrame frame = view_frame(geom, static_cast<std::size_t>(view));
    const RasterSettings settings = to_rs(rs);
    const std::vector<Splat2D> splats = project_cloud(c, frame, geom, settings);
    for (std::size_t i = 0; i < splats.size(); ++i) {
      const Splat2D& s = splats[i];
      rect[4 * i] = s.u_min;
      rect[4 * i + 1] = s.u_max;
      rect[4 * i + 2] = s.v_min;
      rect[4 * i + 3] = s.v_max;
      culled[i] = s.culled;
      degenerate[i] = s.degenerate;
      mean2d[2 * i] = s.mean2d[0];
      mean2d[2 * i + 1] = s.mean2d[1];
      for (int k = 0; k < 4; ++k) conic[4 * i + k] = s.conic(k / 2, k % 2);
      amplitude[i] = s.amplitude;
    }
    const TileBins bins = bin_tiles(splats, geom.n_u, geom.n_v, settings.tile_size);
    int64_t acc = 0;
    for (std::size_t t = 0; t < bins.bins.size(); ++t) {
      if (tile_offsets) tile_offsets[t] = acc;
      for (const int32_t idx : bins.bins[t]) {
        if (tile_splats) tile_splats[acc] = idx;
        ++acc;
      }
    }
    if (tile_offsets) tile_offsets[bins.bins.size()] = acc;
    *n_pairs = acc;
  })
}

int ref_voxelize(void* cloud, const Region* r, const VS* vs, double* volume, Stats* stats,
                 double* ms) {
  GUARD({
    RenderStats s;
    const Volume v = voxelize(*static_cast<GaussianCloud*>(cloud), to_region(r), to_vs(vs), &s);
    std::memcpy(volume, v.values.data(), v.values.size() * sizeof(double));
    put_stats(s, stats, ms);
  })
}

int ref_voxelize_backward(void* cloud, const Region* r, const double* grad_volume, const VS* vs,
                          double* gp, double* gl, double* gq, double* gr, double* pgn,
                          uint8_t* vis, double* ms) {
  GUARD({
    const GridRegion region = to_region(r);
    Volume gvol = Volume::zeros(region.dims, region.spacing, region.origin);
    std::memcpy(gvol.values.data(), grad_volume, gvol.values.size() * sizeof(double));
    RenderStats s;
    const ParamGradients pg =
        voxelize_backward(*static_cast<GaussianCloud*>(cloud), region, gvol, to_vs(vs), &s);
    put_grads(pg, gp, gl, gq, gr, pgn, vis);
    put_stats(s, nullptr, ms);
  })
}

int ref_prepare_voxel_splats(void* cloud, const Region* r, const VS* vs, int32_t* lo, int32_t* hi,
                             uint8_t* skip) {
  GUARD({
    const std::vector<detail::VoxelSplat> sp =
        detail::prepare_voxel_splats(*static_cast<GaussianCloud*>(cloud), to_region(r), to_vs(vs));
    for (std::size_t i = 0; i < sp.size(); ++i) {
      for (int k = 0; k < 3; ++k) {
        lo[3 * i + k] = sp[i].lo[k];
        hi[3 * i + k] = sp[i].hi[k];
      }
      skip[i] = sp[i].skip;
    }
  })
}

// Harness generators from the reference (bench.hpp:33-52, synthetic.hpp:246-271).
int64_t ref_synthetic_cloud(int64_t count, double half_extent, double scale, double anisotropy,
                            double density, uint64_t seed, double* pos, double* ls, double* q,
                            double* raw) {
  SyntheticCloudConfig cfg;
  cfg.count = count;
  cfg.half_extent = half_extent;
  cfg.scale = scale;
  cfg.anisotropy = anisotropy;
  cfg.density = density;
  cfg.seed = seed;
  const GaussianCloud c = synthetic_cloud(cfg);
  for (std::size_t i = 0; i < c.size(); ++i) {
    for (int k = 0; k < 3; ++k) {
      pos[3 * i + k] = c.positions[i][k];
      ls[3 * i + k] = c.log_scales[i][k];
    }
    for (int k = 0; k < 4; ++k) q[4 * i + k] = c.rotations[i][k];
    raw[i] = c.raw_densities[i];
  }
  return static_cast<int64_t>(c.size());
}

// oracles::random_cloud (tests/oracles.hpp:168-184), the reference tests' fixture cloud.
int64_t ref_random_cloud(uint64_t seed, int count, double pos_range, double scale_lo,
                         double scale_hi, double* pos, double* ls, double* q, double* raw) {
  const GaussianCloud c = oracles::random_cloud(seed, count, pos_range, scale_lo, scale_hi);
  for (std::size_t i = 0; i < c.size(); ++i) {
    for (int k = 0; k < 3; ++k) {
      pos[3 * i + k] = c.positions[i][k];
      ls[3 * i + k] = c.log_scales[i][k];
    }
    for (int k = 0; k < 4; ++k) q[4 * i + k] = c.rotations[i][k];
    raw[i] = c.raw_densities[i];
  }
  return static_cast<int64_t>(c.size());
}

// The benchmark phantom cloud (harness, not a reference function), drawn with
// the reference's own Rng (rng.hpp:18-69) so the reference arm of bench.py builds its inputs
// without the product library. Same arithmetic as the product harness's
// gsct_host_make_cloud(kind 2): positions uniform inside the outer Shepp-Logan ellipsoid
// (semi-axes 0.69, 0.92, 0.81 of the half-side), log-scales ln(s0) + U(-0.3, 0.3) with
// s0 = 0.554 (V_fg / N)^(1/3), normalised N(0,1)^4 quaternions, raw density 0.15 U(0.2, 1).
int64_t ref_shepp_logan_cloud(int64_t count, double side, double sp, uint64_t seed, double* pos, double* ls,
                              double* q, double* raw) {
  Rng rng(seed);
  const double half = 0.5 * side * sp;
  const double ax = 0.69 * half, ay = 0.92 * half, az = 0.81 * half;
  const double vfg = 4.0 / 3.0 * M_PI * ax * ay * az;
  const double s0 = 0.554 * std::cbrt(vfg / static_cast<double>(count > 0 ? count : 1));
  for (int64_t i = 0; i < count; ++i) {
    double x, y, z;
    do {
      x = rng.uniform(-1.0, 1.0);
      y = rng.uniform(-1.0, 1.0);
      z = rng.uniform(-1.0, 1.0);
    } while (x * x + y * y + z * z > 1.0);
    pos[3 * i] = x * ax;
    pos[3 * i + 1] = y * ay;
    pos[3 * i + 2] = z * az;
    for (int k = 0; k < 3; ++k) ls[3 * i + k] = std::log(s0) + rng.uniform(-0.3, 0.3);
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
    for (int k = 0; k < 4; ++k) q[4 * i + k] = qq[k] / nrm;
    raw[i] = 0.15 * rng.uniform(0.2, 1.0);
  }
  return count;
}

void ref_default_geometry(int nx, int ny, int nz, double spacing, int n_views, int cone, int n_u,
                          int n_v, Geo* out, double* angles) {
  const Volume vol = Volume::zeros({nx, ny, nz}, spacing, Vec3::Zero());
  const ScanGeometry g = default_geometry(vol, static_cast<std::size_t>(n_views),
                                          cone ? BeamMode::cone : BeamMode::parallel, n_u, n_v);
  out->cone = cone;
  out->n_u = g.n_u;
  out->n_v = g.n_v;
  out->s_u = g.s_u;
  out->s_v = g.s_v;
  out->source_to_origin = g.source_to_origin;
  out->origin_to_detector = g.origin_to_detector;
  for (int i = 0; i < n_views; ++i) angles[i] = g.angles[static_cast<std::size_t>(i)];
}


constexpr std::array<int, 3> kOneVox{{1, 1, 1}};

// total_loss_recon (losses.hpp:613-637) with alpha_tv = 0 on one image: out3 = {l1, ssim,
// total}, grad[n_v * n_u] = d total / d rendered.
int ref_total_loss_recon(const double* rendered, const double* measured, int n_u, int n_v, double alpha_ssim,
                         double* grad, double* out3) {
  GUARD({
    Image r;
    Image m;
    r.n_u = m.n_u = n_u;
    r.n_v = m.n_v = n_v;
    r.values.assign(rendered, rendered + static_cast<std::size_t>(n_u) * n_v);
    m.values.assign(measured, measured + static_cast<std::size_t>(n_u) * n_v);
    LossWeights wts;
    wts.alpha_ssim = alpha_ssim;
    wts.alpha_tv = 0.0;
    const Volume sub = Volume::zeros(kOneVox, 1.0, Vec3::Zero());
    const ReconLoss L = total_loss_recon(r, m, sub, wts);
    out3[0] = L.l1;
    out3[1] = L.ssim;
    out3[2] = L.total;
    std::memcpy(grad, L.grad_image.values.data(), L.grad_image.values.size() * sizeof(double));
  });
}

// adam_step (optim.hpp:158-182) on a cloud (arrays updated in place) with moments in the
// same flat layouts; step / skipped in-out.
int ref_adam_step(int64_t n, double* pos, double* ls, double* q, double* raw, double* const* mv,
                  const double* gpos, const double* gls, const double* gq, const double* graw, const double* lrs,
                  int64_t* step, int64_t* skipped) {
  GUARD({
    GaussianCloud c;
    for (int64_t i = 0; i < n; ++i)
      c.push_back(Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]), Vec3(ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]),
                  Vec4(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]), raw[i]);
    OptimState st;
    st.init(static_cast<std::size_t>(n), 0);
    ParamGradients g;
    g.resize(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) {
        st.m_pos[i][a] = mv[0][3 * i + a];
        st.v_pos[i][a] = mv[1][3 * i + a];
        st.m_ls[i][a] = mv[2][3 * i + a];
        st.v_ls[i][a] = mv[3][3 * i + a];
        g.positions[i][a] = gpos[3 * i + a];
        g.log_scales[i][a] = gls[3 * i + a];
      }
      for (int a = 0; a < 4; ++a) {
        st.m_rot[i][a] = mv[4][4 * i + a];
        st.v_rot[i][a] = mv[5][4 * i + a];
        g.rotations[i][a] = gq[4 * i + a];
      }
      st.m_dens[i] = mv[6][i];
      st.v_dens[i] = mv[7][i];
      g.raw_densities[i] = graw[i];
    }
    st.step = *step;
    st.skipped_updates = *skipped;
    LearningRates lr;
    lr.position = lrs[0];
    lr.log_scale = lrs[1];
    lr.rotation = lrs[2];
    lr.density = lrs[3];
    adam_step(c, st, g, lr);
    for (int64_t i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) {
        pos[3 * i + a] = c.positions[i][a];
        ls[3 * i + a] = c.log_scales[i][a];
        mv[0][3 * i + a] = st.m_pos[i][a];
        mv[1][3 * i + a] = st.v_pos[i][a];
        mv[2][3 * i + a] = st.m_ls[i][a];
        mv[3][3 * i + a] = st.v_ls[i][a];
      }
      for (int a = 0; a < 4; ++a) {
        q[4 * i + a] = c.rotations[i][a];
        mv[4][4 * i + a] = st.m_rot[i][a];
        mv[5][4 * i + a] = st.v_rot[i][a];
      }
      raw[i] = c.raw_densities[i];
      mv[6][i] = st.m_dens[i];
      mv[7][i] = st.v_dens[i];
    }
    *step = st.step;
    *skipped = st.skipped_updates;
  });
}

// total_loss_fit (losses.hpp:648-664) on a volume (x fastest): out3 = {l1, ssim, total}
int ref_total_loss_fit(const double* rendered, const double* target, const int* dims, double alpha_ssim,
                       int streaming, double* grad, double* out3) {
  GUARD({
    const std::array<int, 3> d{{dims[0], dims[1], dims[2]}};
    Volume r = Volume::zeros(d, 1.0, Vec3::Zero());
    Volume t = Volume::zeros(d, 1.0, Vec3::Zero());
    std::memcpy(r.values.data(), rendered, r.values.size() * sizeof(double));
    std::memcpy(t.values.data(), target, t.values.size() * sizeof(double));
    const FitLoss L = total_loss_fit(r, t, alpha_ssim, streaming ? SsimPath::streaming : SsimPath::materialized);
    out3[0] = L.l1;
    out3[1] = L.ssim;
    out3[2] = L.total;
    std::memcpy(grad, L.grad.values.data(), L.grad.values.size() * sizeof(double));
  });
}

// tv3d (losses.hpp:530-595)
int ref_tv3d(const double* volume, const int* dims, double* grad, double* value) {
  GUARD({
    const std::array<int, 3> d{{dims[0], dims[1], dims[2]}};
    Volume v = Volume::zeros(d, 1.0, Vec3::Zero());
    std::memcpy(v.values.data(), volume, v.values.size() * sizeof(double));
    const Tv3dResult R = tv3d(v);
    *value = R.value;
    std::memcpy(grad, R.grad.values.data(), R.grad.values.size() * sizeof(double));
  });
}

// raymarch_project (synthetic.hpp:171-232): images[n_angles][n_v][n_u]
int ref_raymarch_project(const double* volume, const int* dims, double spacing, const double* origin, const Geo* g,
                         const double* angles, int n_angles, double* images) {
  GUARD({
    const std::array<int, 3> d{{dims[0], dims[1], dims[2]}};
    Volume v = Volume::zeros(d, spacing, Vec3(origin[0], origin[1], origin[2]));
    std::memcpy(v.values.data(), volume, v.values.size() * sizeof(double));
    const ProjectionSet P = raymarch_project(v, to_geom(g, angles, n_angles));
    const std::size_t npx = static_cast<std::size_t>(g->n_u) * g->n_v;
    for (int k = 0; k < n_angles; ++k)
      std::memcpy(images + k * npx, P.images[static_cast<std::size_t>(k)].values.data(), npx * sizeof(double));
  });
}

// adaptive_control (optim.hpp:201-317) of the unchanged reference on flat arrays. In:
// n rows of params / moments / accumulators, rng = {x[312], p} (Rng::restore_state text),
// cfg = {grad_threshold, prune_density, split_scale_fraction, scene_extent}, max_gaussians.
// Out (capacity rows): params / moments, the report {pruned, cloned, split, n_next} and the
// engine state after the call (in place; the reference leaves it unchanged, see the caller).
int ref_adaptive_control(int64_t n, const double* pos, const double* ls, const double* q, const double* raw,
                         const double* const* mv, const double* acc_norm, const double* acc_dir,
                         const int64_t* acc_count, uint64_t* rng, const double* cfg, int64_t max_gaussians,
                         int64_t capacity, double* opos, double* ols, double* oq, double* oraw, double* const* omv,
                         int64_t* report) {
  GUARD({
    GaussianCloud c;
    for (int64_t i = 0; i < n; ++i)
      c.push_back(Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]), Vec3(ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]),
                  Vec4(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]), raw[i]);
    OptimState st;
    st.init(static_cast<std::size_t>(n), 0);
    for (int64_t i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) {
        st.m_pos[i][a] = mv[0][3 * i + a];
        st.v_pos[i][a] = mv[1][3 * i + a];
        st.m_ls[i][a] = mv[2][3 * i + a];
        st.v_ls[i][a] = mv[3][3 * i + a];
        st.accum_grad_dir[i][a] = acc_dir[3 * i + a];
      }
      for (int a = 0; a < 4; ++a) {
        st.m_rot[i][a] = mv[4][4 * i + a];
        st.v_rot[i][a] = mv[5][4 * i + a];
      }
      st.m_dens[i] = mv[6][i];
      st.v_dens[i] = mv[7][i];
      st.accum_grad_norm[i] = acc_norm[i];
      st.accum_count[i] = acc_count[i];
    }
    {
      std::ostringstream os;
      for (int k = 0; k < 312; ++k) os << rng[k] << ' ';
      os << rng[312];
      st.rng.restore_state(os.str());
    }
    st.scene_extent = cfg[3];
    TrainConfig tc;
    tc.grad_threshold = cfg[0];
    tc.prune_density = cfg[1];
    tc.split_scale_fraction = cfg[2];
    tc.max_gaussians = static_cast<std::size_t>(max_gaussians);
    const AdaptiveReport r = adaptive_control(c, st, tc);
    const int64_t m = static_cast<int64_t>(c.size());
    report[0] = static_cast<int64_t>(r.pruned);
    report[1] = static_cast<int64_t>(r.cloned);
    report[2] = static_cast<int64_t>(r.split);
    report[3] = m;
    if (m > capacity) return 2;
    for (int64_t i = 0; i < m; ++i) {
      for (int a = 0; a < 3; ++a) {
        opos[3 * i + a] = c.positions[i][a];
        ols[3 * i + a] = c.log_scales[i][a];
        omv[0][3 * i + a] = st.m_pos[i][a];
        omv[1][3 * i + a] = st.v_pos[i][a];
        omv[2][3 * i + a] = st.m_ls[i][a];
        omv[3][3 * i + a] = st.v_ls[i][a];
      }
      for (int a = 0; a < 4; ++a) {
        oq[4 * i + a] = c.rotations[i][a];
        omv[4][4 * i + a] = st.m_rot[i][a];
        omv[5][4 * i + a] = st.v_rot[i][a];
      }
      oraw[i] = c.raw_densities[i];
      omv[6][i] = st.m_dens[i];
      omv[7][i] = st.v_dens[i];
    }
    std::istringstream in(st.rng.save_state());
    for (int k = 0; k < 313; ++k) in >> rng[k];
  });
}

// compress_model / decompress_model (io.hpp:319-425) of the unchanged reference. compress:
// out must hold 16 + 22 n bytes; *saturated (CompressStats). decompress: arrays of
// capacity rows; *n_out = decoded count (error 2 if it exceeds the capacity).
int ref_compress_model(int64_t n, const double* pos, const double* ls, const double* q, const double* raw,
                       uint8_t* out, int64_t* saturated) {
  GUARD({
    GaussianCloud c;
    for (int64_t i = 0; i < n; ++i)
      c.push_back(Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]), Vec3(ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]),
                  Vec4(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]), raw[i]);
    CompressStats st;
    const std::vector<std::uint8_t> b = compress_model(c, &st);
    std::memcpy(out, b.data(), b.size());
    *saturated = static_cast<int64_t>(st.saturated);
  });
}

int ref_decompress_model(const uint8_t* bytes, int64_t n_bytes, int64_t capacity, double* pos, double* ls, double* q,
                         double* raw, int64_t* n_out) {
  GUARD({
    const std::vector<std::uint8_t> b(bytes, bytes + n_bytes);
    const GaussianCloud c = decompress_model(b);
    const int64_t m = static_cast<int64_t>(c.size());
    *n_out = m;
    if (m > capacity) return 2;
    for (int64_t i = 0; i < m; ++i) {
      for (int a = 0; a < 3; ++a) {
        pos[3 * i + a] = c.positions[i][a];
        ls[3 * i + a] = c.log_scales[i][a];
      }
      for (int a = 0; a < 4; ++a) q[4 * i + a] = c.rotations[i][a];
      raw[i] = c.raw_densities[i];
    }
  });
}
}  // extern "C"
