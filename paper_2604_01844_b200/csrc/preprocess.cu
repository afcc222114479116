// fp64 per-splat kernels: the view-independent splat pre-pass, raster set-up (K1), raster
// chain-rule tail (K4b) + finalize, voxel set-up (K6), voxel chain-rule tail (K8b), and
// the projection parity hook.
// Compiled with --fmad=false so the arithmetic is the reference's, operation by operation
// (see splat_fp64.cuh): integer boxes and keys are bit-exact with the CPU oracle.
#include <cuda_runtime.h>

#include <algorithm>

#include "gsct_internal.cuh"

namespace gsct_dev {

namespace {

constexpr double kLog2eD = 1.4426950408889634074;

__device__ __forceinline__ void flag_error(DevStats* st, int64_t i, int code) {
  atomicMin(&st->error_key, (static_cast<unsigned long long>(i) << 2) | static_cast<unsigned>(code));
}

// Warp-aggregated add of small integer counters.
__device__ __forceinline__ void warp_add(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

__device__ __forceinline__ RasterRec empty_rec() {
  RasterRec r;
  r.urange = 0xFFFFu;  // u_min = 65535 > u_max = 0
  r.vrange = 0xFFFFu;
  r.mo_u = r.mo_v = r.A = r.B = r.C = r.amp = 0.f;
  return r;
}

// View-independent pre-pass, one thread per splat: activation, Sigma, det test, Sigma^-1
// (computed once instead of once per view; identical values, so boxes stay bit-exact).
// Writes the set-up twice: structure-of-arrays for the per-(view, splat) set-up kernel
// (coalesced field loads) and array-of-structs for the backward tail (lazy L1 re-reads
// keep its register pressure down).
__global__ void __launch_bounds__(128) k_splat_prepare(Cloud c, int64_t i0, int64_t i1, PreSplat* __restrict__ pre,
                                                       PreSplat* __restrict__ pre_aos,
                                                       DevStats* __restrict__ st) {
  const int64_t i = i0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= i1) return;
  PreSplat s;
  prepare_splat(c.pos, c.ls, c.q, c.raw, i, s);
  if (s.status) flag_error(st, i, s.status);
  pre_store(pre, c.n, i, s);
  pre_aos[i] = s;
}

// K1: one thread per (splat, view): project_full -> splat_bbox from the pre-pass, then the
// fp32 record, the binning tile count and the exact RenderStats counters.
// (launch bounds: 8 CTAs x 128 threads per SM -> <= 64 registers, 50% occupancy; the
// kernel is fp64-latency bound, profiles/)
#ifndef GSCT_PRE_MINB
#define GSCT_PRE_MINB 8
#endif
#ifndef GSCT_PRE_VIEWS
#define GSCT_PRE_VIEWS 8  // views per thread (the splat's set-up loaded once per thread)
#endif
constexpr int kPreViews = GSCT_PRE_VIEWS;
__global__ void __launch_bounds__(128, GSCT_PRE_MINB) k_raster_preprocess(const PreSplat* __restrict__ pre, int64_t n,
                                                           int64_t i0, int64_t i1, int n_views, const Frame* __restrict__ frames, Geo g,
                                                           RSet rs, int bin_ts,
                                                           RasterRec* __restrict__ rec,
                                                           uint32_t* __restrict__ tile_count,
                                                           DevStats* __restrict__ st,
                                                           unsigned long long* __restrict__ view_pairs,
                                                           WalkOut walk) {
  const int64_t i = i0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long n_culled = 0, n_degen = 0, n_tp = 0, n_pp = 0;
  PreSplat s;
  if (i < i1) pre_load(pre, n, i, s);  // once per thread, reused for its kPreViews views
  for (int vg = 0; vg < kPreViews; ++vg) {
  const int v = blockIdx.y * kPreViews + vg;
  uint32_t cnt = 0;
  if (i < i1 && v < n_views) {
    RasterRec r = empty_rec();
    if (s.status == 0) {
      Proj p;
      project_full(frames[v], g, s.pos, s.sigma, s.sigma_inv, s.det_ok != 0, s.density, rs, p);
      if (p.degenerate) {
        n_degen += 1;
      } else if (p.culled) {
        n_culled += 1;
      } else {
        const int u0 = p.rect[0], u1 = p.rect[1], v0 = p.rect[2], v1 = p.rect[3];
        r.urange = static_cast<uint32_t>(u0) | (static_cast<uint32_t>(u1) << 16);
        r.vrange = static_cast<uint32_t>(v0) | (static_cast<uint32_t>(v1) << 16);
        r.mo_u = static_cast<float>(p.mean2d[0] - static_cast<double>(u0));
        r.mo_v = static_cast<float>(p.mean2d[1] - static_cast<double>(v0));
        r.A = static_cast<float>(-0.5 * kLog2eD * p.conic[0]);
        r.B = static_cast<float>(-kLog2eD * p.conic[1]);
        r.C = static_cast<float>(-0.5 * kLog2eD * p.conic[3]);
        r.amp = static_cast<float>(p.amplitude);
        {  // chain safety over the 8-column / row-pair aligned bbox, carried in amp's sign
          const float dua = static_cast<float>((u0 & ~7) - u0) - r.mo_u;
          const float dub = static_cast<float>((u1 | 7) - u0) - r.mo_u;
          const float dva = static_cast<float>((v0 & ~1) - v0) - r.mo_v;
          const float dvb = static_cast<float>((v1 | 1) - v0) - r.mo_v;
          if (!raster_chain_safe(r.A, r.B, r.C, dua, dub, dva, dvb)) r.amp = copysignf(r.amp, -1.f);
        }
        // binning count at the kernel's tile size; stats at the requested tile size
        cnt = static_cast<uint32_t>((u1 / bin_ts - u0 / bin_ts + 1) * (v1 / bin_ts - v0 / bin_ts + 1));
        const int ts = rs.tile_size;
        n_tp += static_cast<unsigned long long>((u1 / ts - u0 / ts + 1)) *
                static_cast<unsigned long long>((v1 / ts - v0 / ts + 1));
        n_pp += static_cast<unsigned long long>(u1 - u0 + 1) * static_cast<unsigned long long>(v1 - v0 + 1);
      }
    }
    const int64_t item = static_cast<int64_t>(v) * n + i;
    rec[item] = r;
    if (tile_count) tile_count[item] = cnt;
    if (walk.count) {  // the backward's walk-order bucket and rank (order.cu)
      const uint32_t b = walk_bucket(r.urange, r.vrange, walk.view_base + v, walk.L);
      walk.slot[item] = make_uint2(b, atomicAdd(walk.count + b, 1u));
    }
  }
  // per-view pair totals (every lane of the warp shares the view: blockIdx.y)
  if (view_pairs && v < n_views) {
    const uint32_t ws = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && ws) atomicAdd(view_pairs + v, static_cast<unsigned long long>(ws));
  }
  }
  warp_add(&st->culled, n_culled);
  warp_add(&st->degenerate, n_degen);
  warp_add(&st->tile_pairs, n_tp);
  warp_add(&st->pixel_pairs, n_pp);
}

__global__ void k_debug_project(const PreSplat* __restrict__ pre, int64_t n, const Frame* __restrict__ frame,
                                Geo g, RSet rs, int32_t* rect, uint8_t* flags, double* mean2d, double* conic,
                                double* amplitude) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  PreSplat s;
    pre_load(pre, n, i, s);
  if (s.status) return;
  Proj p;
  project_full(*frame, g, s.pos, s.sigma, s.sigma_inv, s.det_ok != 0, s.density, rs, p);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    rect[4 * i + k] = p.rect[k];
    conic[4 * i + k] = p.conic[k];
  }
  flags[i] = static_cast<uint8_t>((p.culled ? 1 : 0) | (p.degenerate ? 2 : 0));
  mean2d[2 * i] = p.mean2d[0];
  mean2d[2 * i + 1] = p.mean2d[1];
  amplitude[i] = p.amplitude;
}

// K6: one thread per splat: prepare_voxel_splat in grid coordinates, clip to the window,
// fp32 record relative to the grid-clipped box corner, brick count, exact stats.
__global__ void __launch_bounds__(256) k_voxel_preprocess(Cloud c, VoxGrid grid, Window win,
                                                          double tau_cut, double sigma_cap,
                                                          VoxelRec* __restrict__ rec,
                                                          uint32_t* __restrict__ brick_count,
                                                          int32_t* lo_out, int32_t* hi_out,
                                                          uint8_t* skip_out, DevStats* st) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long n_culled = 0, n_pp = 0;
  if (i < c.n) {
    VoxelRec r;
    r.lox = r.loy = r.loz = 1.f;
    r.hix = r.hiy = r.hiz = 0.f;  // empty
    r.rho = r.Q00 = r.offx = r.offy = r.offz = r.Q11 = r.Q22 = r.Q01 = r.Q02 = r.Q12 = 0.f;
    uint32_t cnt = 0;
    int lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
    bool vis = false;
    Act a;
    const int err = activate(c.pos, c.ls, c.q, c.raw, i, a);
    if (err) {
      flag_error(st, i, err);
    } else {
      double sigma[9], A[9];
      covariance(a.scales, a.uq, sigma);
      vis = prepare_voxel_splat(a, sigma, grid, tau_cut, sigma_cap, A, lo, hi);
      // The record keeps the grid-clipped box (so per-voxel arithmetic does not depend on
      // the window: z-slabs reproduce the full-grid volume bit for bit); the window clip
      // only decides visibility, brick counts and stats.
      int wlo[3], whi[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        wlo[k] = lo[k] > win.lo[k] ? lo[k] : win.lo[k];
        whi[k] = hi[k] < win.hi[k] - 1 ? hi[k] : win.hi[k] - 1;
        vis = vis && wlo[k] <= whi[k];
      }
      if (vis) {
        r.lox = static_cast<float>(lo[0]);
        r.loy = static_cast<float>(lo[1]);
        r.loz = static_cast<float>(lo[2]);
        r.hix = static_cast<float>(hi[0]);
        r.hiy = static_cast<float>(hi[1]);
        r.hiz = static_cast<float>(hi[2]);
        r.rho = static_cast<float>(a.density);
        r.offx = static_cast<float>(a.pos[0] - (grid.origin[0] + grid.spacing * lo[0]));
        r.offy = static_cast<float>(a.pos[1] - (grid.origin[1] + grid.spacing * lo[1]));
        r.offz = static_cast<float>(a.pos[2] - (grid.origin[2] + grid.spacing * lo[2]));
        const double h = -0.5 * kLog2eD;
        r.Q00 = static_cast<float>(h * GM3(A, 0, 0));
        r.Q11 = static_cast<float>(h * GM3(A, 1, 1));
        r.Q22 = static_cast<float>(h * GM3(A, 2, 2));
        r.Q01 = static_cast<float>(2.0 * h * GM3(A, 0, 1));
        r.Q02 = static_cast<float>(2.0 * h * GM3(A, 0, 2));
        r.Q12 = static_cast<float>(2.0 * h * GM3(A, 1, 2));
        cnt = 1;
#pragma unroll
        for (int k = 0; k < 3; ++k)
          cnt *= static_cast<uint32_t>((whi[k] - win.lo[k]) / (k == 2 ? kBrickZ : kBrick) -
                                       (wlo[k] - win.lo[k]) / (k == 2 ? kBrickZ : kBrick) + 1);
        n_pp = static_cast<unsigned long long>(whi[0] - wlo[0] + 1) *
               static_cast<unsigned long long>(whi[1] - wlo[1] + 1) *
               static_cast<unsigned long long>(whi[2] - wlo[2] + 1);
      } else {
        n_culled = 1;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        lo[k] = wlo[k];
        hi[k] = whi[k];
      }
    }
    if (rec) rec[i] = r;
    if (brick_count) brick_count[i] = cnt;
    if (lo_out) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        lo_out[3 * i + k] = vis ? lo[k] : 0;
        hi_out[3 * i + k] = vis ? hi[k] : -1;
      }
      skip_out[i] = vis ? 0 : 1;
    }
  }
  warp_add(&st->culled, n_culled);
  warp_add(&st->pixel_pairs, n_pp);
}

// K8b: one thread per splat: from the fp32 voxel-loop moments (summed over all windows)
// to dL/d(raw parameters) in fp64, voxelizer.hpp:250-255 + covariance_backward.
// T: float (this call's own moments) or double (moments all-reduced across ranks in fp64).
template <class T>
__global__ void __launch_bounds__(128) k_voxel_tail(Cloud c, VoxGrid grid, double tau_cut,
                                                    double sigma_cap, const T* __restrict__ m,
                                                    double* __restrict__ g_pos,
                                                    double* __restrict__ g_ls, double* __restrict__ g_q,
                                                    double* __restrict__ g_raw,
                                                    double* __restrict__ g_pgn,
                                                    uint8_t* __restrict__ visible, DevStats* st) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= c.n) return;
  const int64_t n = c.n;
  double gp[3] = {0, 0, 0}, gl[3] = {0, 0, 0}, gq[4] = {0, 0, 0, 0}, gr = 0.0, pgn = 0.0;
  uint8_t vis = 0;
  Act a;
  const int err = activate(c.pos, c.ls, c.q, c.raw, i, a);
  if (err) {
    flag_error(st, i, err);
  } else {
    double sigma[9], A[9];
    int lo[3], hi[3];
    covariance(a.scales, a.uq, sigma);
    if (prepare_voxel_splat(a, sigma, grid, tau_cut, sigma_cap, A, lo, hi)) {
      vis = 1;
      const double M0 = m[0 * n + i];
      const double M1[3] = {m[1 * n + i], m[2 * n + i], m[3 * n + i]};
      // second moments: xx, yy, zz, xy, xz, yz
      const double sxx = m[4 * n + i], syy = m[5 * n + i], szz = m[6 * n + i];
      const double sxy = m[7 * n + i], sxz = m[8 * n + i], syz = m[9 * n + i];
      const double rho = a.density;
      double am1[3];
      mul3v(A, M1, am1);
#pragma unroll
      for (int k = 0; k < 3; ++k) gp[k] = rho * am1[k];
      const double hr = -0.5 * rho;
      const double gA[9] = {hr * sxx, hr * sxy, hr * sxz, hr * sxy, hr * syy,
                            hr * syz, hr * sxz, hr * syz, hr * szz};
      double negA[9], t[9], gsig[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) negA[k] = -A[k];
      mul33(negA, gA, t);
      mul33(t, A, gsig);
      gr = a.raw_density >= 0.0 ? M0 : 0.0;
      pgn = sqrt(dot3(gp, gp));
      covariance_backward(a.scales, a.uq, a.raw_q, gsig, gl, gq);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g_pos[3 * i + k] = gp[k];
    g_ls[3 * i + k] = gl[k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) g_q[4 * i + k] = gq[k];
  g_raw[i] = gr;
  g_pgn[i] = pgn;
  visible[i] = vis;
}

inline unsigned blocks_for(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

}  // namespace

void launch_splat_prepare(const Cloud& c, PreSplat* pre, PreSplat* pre_aos, DevStats* stats, cudaStream_t st,
                          int64_t i0, int64_t i1) {
  if (i1 < 0) i1 = c.n;
  if (i1 <= i0) return;
  k_splat_prepare<<<blocks_for(i1 - i0, 128), 128, 0, st>>>(c, i0, i1, pre, pre_aos, stats);
  count_launch();
}

void launch_raster_preprocess(const PreSplat* pre, int64_t n, const Frame* frames_dev, int n_views, const Geo& g,
                              const RSet& rs, int bin_ts, RasterRec* rec, uint32_t* tile_count,
                              DevStats* stats, cudaStream_t st, int64_t i0, int64_t i1,
                              unsigned long long* view_pairs, const WalkOut* walk) {
  if (i1 < 0) i1 = n;
  if (i1 <= i0 || n_views == 0) return;
  dim3 grid(blocks_for(i1 - i0, 128), static_cast<unsigned>((n_views + kPreViews - 1) / kPreViews));
  k_raster_preprocess<<<grid, 128, 0, st>>>(pre, n, i0, i1, n_views, frames_dev, g, rs, bin_ts, rec, tile_count,
                                            stats, tile_count ? view_pairs : nullptr, walk ? *walk : WalkOut{});
  count_launch();
}

__global__ void k_sum_u32(const uint32_t* __restrict__ counts, int64_t n, unsigned long long* __restrict__ total) {
  unsigned long long acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    acc += counts[i];
  warp_add(total, acc);
}

void launch_sum_u32(const uint32_t* counts, int64_t n, unsigned long long* total, cudaStream_t st) {
  if (n <= 0) return;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  k_sum_u32<<<blocks, 256, 0, st>>>(counts, n, total);
  count_launch();
}


void launch_debug_project(const PreSplat* pre, int64_t n, const Frame* frame_dev, const Geo& g, const RSet& rs,
                          int32_t* rect, uint8_t* flags, double* mean2d, double* conic, double* amplitude,
                          cudaStream_t st) {
  if (n == 0) return;
  k_debug_project<<<blocks_for(n, 128), 128, 0, st>>>(pre, n, frame_dev, g, rs, rect, flags, mean2d, conic,
                                                      amplitude);
  count_launch();
}

void launch_voxel_preprocess(const Cloud& c, const VoxGrid& grid, const Window& win,
                             double tau_cut, double sigma_cap, VoxelRec* rec,
                             uint32_t* brick_count, int32_t* lo_out, int32_t* hi_out,
                             uint8_t* skip_out, DevStats* stats, cudaStream_t st) {
  if (c.n == 0) return;
  k_voxel_preprocess<<<blocks_for(c.n, 256), 256, 0, st>>>(c, grid, win, tau_cut, sigma_cap, rec,
                                                           brick_count, lo_out, hi_out, skip_out,
                                                           stats);
  count_launch();
}

template <class T>
void launch_voxel_tail(const Cloud& c, const VoxGrid& grid, double tau_cut, double sigma_cap,
                       const T* moments, double* g_pos, double* g_ls, double* g_q,
                       double* g_raw, double* g_pgn, uint8_t* visible, DevStats* stats,
                       cudaStream_t st) {
  if (c.n == 0) return;
  k_voxel_tail<T><<<blocks_for(c.n, 128), 128, 0, st>>>(c, grid, tau_cut, sigma_cap, moments, g_pos,
                                                        g_ls, g_q, g_raw, g_pgn, visible, stats);
  count_launch();
}
template void launch_voxel_tail<float>(const Cloud&, const VoxGrid&, double, double, const float*, double*, double*,
                                       double*, double*, double*, uint8_t*, DevStats*, cudaStream_t);
template void launch_voxel_tail<double>(const Cloud&, const VoxGrid&, double, double, const double*, double*,
                                        double*, double*, double*, double*, uint8_t*, DevStats*, cudaStream_t);

__global__ void k_widen_f32(const float* __restrict__ a, double* __restrict__ b, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = static_cast<double>(a[i]);
}

// Sparse gradient rows (GSCT_HOST_ZEROED): a splat's row is kept when it is visible or has
// any non-zero entry (so the zero-filled host buffers end up equal to the dense output).
__global__ void k_grad_row_flags(const double* __restrict__ gp, const double* __restrict__ gl,
                                 const double* __restrict__ gq, const double* __restrict__ gr,
                                 const double* __restrict__ gn, const uint8_t* __restrict__ gv, int64_t n,
                                 uint32_t* __restrict__ flag) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool keep = gv[i] != 0 || gr[i] != 0.0 || gn[i] != 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) keep = keep || gp[3 * i + k] != 0.0 || gl[3 * i + k] != 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) keep = keep || gq[4 * i + k] != 0.0;
  flag[i] = keep ? 1u : 0u;
}
// rows[r] = {pos 3, log_scale 3, quat 4, raw, pos_grad_norm, visible}, idx[r] = splat (ascending)
__global__ void k_grad_rows(const double* __restrict__ gp, const double* __restrict__ gl,
                            const double* __restrict__ gq, const double* __restrict__ gr,
                            const double* __restrict__ gn, const uint8_t* __restrict__ gv, int64_t n,
                            const uint32_t* __restrict__ flag,
                            const uint32_t* __restrict__ pos, double* __restrict__ rows, uint32_t* __restrict__ idx,
                            uint32_t* __restrict__ count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == n - 1) *count = pos[i] + flag[i];
  if (!flag[i]) return;
  const uint32_t r = pos[i];
  double* o = rows + static_cast<int64_t>(r) * 13;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o[k] = gp[3 * i + k];
    o[3 + k] = gl[3 * i + k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) o[6 + k] = gq[4 * i + k];
  o[10] = gr[i];
  o[11] = gn[i];
  o[12] = gv[i] ? 1.0 : 0.0;
  idx[r] = static_cast<uint32_t>(i);
}

void launch_grad_row_flags(const double* gp, const double* gl, const double* gq, const double* gr, const double* gn,
                           const uint8_t* gv, int64_t n, uint32_t* flag, cudaStream_t st) {
  if (n <= 0) return;
  k_grad_row_flags<<<blocks_for(n, 256), 256, 0, st>>>(gp, gl, gq, gr, gn, gv, n, flag);
  count_launch();
}
void launch_grad_rows(const double* gp, const double* gl, const double* gq, const double* gr, const double* gn,
                      const uint8_t* gv, int64_t n, const uint32_t* flag, const uint32_t* pos, double* rows,
                      uint32_t* idx, uint32_t* count, cudaStream_t st) {
  if (n <= 0) return;
  k_grad_rows<<<blocks_for(n, 256), 256, 0, st>>>(gp, gl, gq, gr, gn, gv, n, flag, pos, rows, idx, count);
  count_launch();
}

void launch_widen_f32(const float* a, double* b, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_widen_f32<<<blocks_for(n, 256), 256, 0, st>>>(a, b, n);
  count_launch();
}

}  // namespace gsct_dev

namespace gsct_dev {
namespace {

// adam_update (optim.hpp:149-156), operation for operation: this TU is compiled without
// FMA contraction and double sqrt / division are IEEE-rounded, so with the host-side
// bias terms (std::pow) the update is bit-identical to the reference's.
__device__ __forceinline__ void adam_update(double& param, double& m, double& v, double grad, double lr,
                                            double bias1, double bias2) {
  constexpr double b1 = 0.9, b2 = 0.999, eps = 1e-15;
  m = b1 * m + (1.0 - b1) * grad;
  v = b2 * v + (1.0 - b2) * grad * grad;
  param -= lr * (m / bias1) / (sqrt(v / bias2) + eps);
}

// adam_step (optim.hpp:158-182): one thread per splat; splats with any non-finite
// gradient are skipped and counted; raw densities are re-projected to >= 0.
__global__ void k_adam_step(int64_t n, double* __restrict__ pos, double* __restrict__ ls, double* __restrict__ q,
                            double* __restrict__ raw, double* __restrict__ m_pos, double* __restrict__ v_pos,
                            double* __restrict__ m_ls, double* __restrict__ v_ls, double* __restrict__ m_rot,
                            double* __restrict__ v_rot, double* __restrict__ m_dens, double* __restrict__ v_dens,
                            const double* __restrict__ g_pos, const double* __restrict__ g_ls,
                            const double* __restrict__ g_q, const double* __restrict__ g_raw, double lr_pos,
                            double lr_ls, double lr_rot, double lr_dens, double bias1, double bias2,
                            unsigned long long* __restrict__ skipped) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  bool skip = false;
  if (i < n) {
    bool ok = isfinite(g_raw[i]);
#pragma unroll
    for (int a = 0; a < 3; ++a) ok = ok && isfinite(g_pos[3 * i + a]) && isfinite(g_ls[3 * i + a]);
#pragma unroll
    for (int a = 0; a < 4; ++a) ok = ok && isfinite(g_q[4 * i + a]);
    skip = !ok;
    if (ok) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        adam_update(pos[3 * i + a], m_pos[3 * i + a], v_pos[3 * i + a], g_pos[3 * i + a], lr_pos, bias1, bias2);
        adam_update(ls[3 * i + a], m_ls[3 * i + a], v_ls[3 * i + a], g_ls[3 * i + a], lr_ls, bias1, bias2);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
        adam_update(q[4 * i + a], m_rot[4 * i + a], v_rot[4 * i + a], g_q[4 * i + a], lr_rot, bias1, bias2);
      adam_update(raw[i], m_dens[i], v_dens[i], g_raw[i], lr_dens, bias1, bias2);
      if (raw[i] < 0.0) raw[i] = 0.0;
    }
  }
  const unsigned ball = __ballot_sync(0xffffffffu, skip);
  if ((threadIdx.x & 31) == 0 && ball) atomicAdd(skipped, static_cast<unsigned long long>(__popc(ball)));
}

}  // namespace

void launch_adam_step(int64_t n, double* pos, double* ls, double* q, double* raw, double* const* mv,
                      const double* g_pos, const double* g_ls, const double* g_q, const double* g_raw,
                      const double* lrs, double bias1, double bias2, unsigned long long* skipped, cudaStream_t st) {
  if (n == 0) return;
  k_adam_step<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
      n, pos, ls, q, raw, mv[0], mv[1], mv[2], mv[3], mv[4], mv[5], mv[6], mv[7], g_pos, g_ls, g_q, g_raw, lrs[0],
      lrs[1], lrs[2], lrs[3], bias1, bias2, skipped);
  count_launch();
}

}  // namespace gsct_dev

// ---------------------------------------------------------------------------------------
// Ray-marched volume projector: raymarch_project (synthetic.hpp:
// 171-232), the synthetic ground-truth generator -- trilinear samples at spacing/2 steps along
// every pixel's ray, independent of the splat rasterizer. One thread per (view, pixel); ray
// set-up, positions and the sum in fp64 (the reference's arithmetic), trilinear weights and
// voxel values in fp32 (the volume is fp32 on the device). Lives in this --fmad=false TU
// and divides where the reference divides, so ray entry/exit and the step count
// ceil((t1 - t0) / step) are the reference's exactly (a knife edge for axis-aligned rays).
// ---------------------------------------------------------------------------------------
namespace gsct_dev {
namespace {

struct VolDesc {
  int nx, ny, nz;
  double spacing, ox, oy, oz;
};

__global__ void __launch_bounds__(256) k_raymarch(const float* __restrict__ vol, VolDesc vd,
                                                  const Frame* __restrict__ frames, Geo g, int n_views,
                                                  float* __restrict__ images) {
  const int64_t npx = static_cast<int64_t>(g.n_u) * g.n_v;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= npx * n_views) return;
  const int view = static_cast<int>(gid / npx);
  const int64_t px = gid - view * npx;
  const int u = static_cast<int>(px % g.n_u), v = static_cast<int>(px / g.n_u);
  const Frame fr = frames[view];
  const double cu = 0.5 * (g.n_u - 1), cv = 0.5 * (g.n_v - 1);
  double pix[3], org[3], dir[3];
  for (int k = 0; k < 3; ++k)  // pixel_center_world (projector.hpp:47-53)
    pix[k] = fr.dc[k] + (u - cu) * g.s_u * fr.u[k] + (v - cv) * g.s_v * fr.v[k];
  if (g.cone) {
    double n2 = 0.0;
    for (int k = 0; k < 3; ++k) {
      org[k] = fr.src[k];
      dir[k] = pix[k] - fr.src[k];
      n2 += dir[k] * dir[k];
    }
    const double nrm = sqrt(n2);  // Eigen normalized(): v / v.norm()
    for (int k = 0; k < 3; ++k) dir[k] /= nrm;
  } else {
    for (int k = 0; k < 3; ++k) {
      org[k] = pix[k];
      dir[k] = fr.d[k];
    }
  }
  const double o3[3] = {vd.ox, vd.oy, vd.oz};
  const int n3[3] = {vd.nx, vd.ny, vd.nz};
  double t0 = -INFINITY, t1 = INFINITY;
  for (int a = 0; a < 3; ++a) {
    const double lo = o3[a] - 0.5 * vd.spacing, hi = o3[a] + vd.spacing * (n3[a] - 1) + 0.5 * vd.spacing;
    if (fabs(dir[a]) < 1e-300) {
      if (org[a] < lo || org[a] > hi) {
        t0 = 1.0;
        t1 = 0.0;
        break;
      }
      continue;
    }
    double ta = (lo - org[a]) / dir[a], tb = (hi - org[a]) / dir[a];
    if (ta > tb) {
      const double s = ta;
      ta = tb;
      tb = s;
    }
    t0 = fmax(t0, ta);
    t1 = fmin(t1, tb);
  }
  double value = 0.0;
  if (t1 > t0) {
    const double step = 0.5 * vd.spacing;
    const int64_t n_steps = max(static_cast<int64_t>(1), static_cast<int64_t>(ceil((t1 - t0) / step)));
    const double dt = (t1 - t0) / static_cast<double>(n_steps);
    for (int64_t i = 0; i < n_steps; ++i) {
      const double t = t0 + (static_cast<double>(i) + 0.5) * dt;
      double gc[3];
      for (int a = 0; a < 3; ++a) {  // sample_trilinear (core.hpp:320-339)
        const double w = org[a] + t * dir[a];
        gc[a] = fmin(fmax((w - o3[a]) / vd.spacing, 0.0), static_cast<double>(n3[a] - 1));
      }
      const int x0 = min(static_cast<int>(gc[0]), vd.nx - 2 >= 0 ? vd.nx - 2 : 0);
      const int y0 = min(static_cast<int>(gc[1]), vd.ny - 2 >= 0 ? vd.ny - 2 : 0);
      const int z0 = min(static_cast<int>(gc[2]), vd.nz - 2 >= 0 ? vd.nz - 2 : 0);
      const int x1 = min(x0 + 1, vd.nx - 1), y1 = min(y0 + 1, vd.ny - 1), z1 = min(z0 + 1, vd.nz - 1);
      const float tx = static_cast<float>(gc[0] - x0), ty = static_cast<float>(gc[1] - y0),
                  tz = static_cast<float>(gc[2] - z0);
      auto at = [&](int x, int y, int z) {
        return __ldg(vol + (static_cast<int64_t>(z) * vd.ny + y) * vd.nx + x);
      };
      const float c00 = fmaf(at(x1, y0, z0) - at(x0, y0, z0), tx, at(x0, y0, z0));
      const float c10 = fmaf(at(x1, y1, z0) - at(x0, y1, z0), tx, at(x0, y1, z0));
      const float c01 = fmaf(at(x1, y0, z1) - at(x0, y0, z1), tx, at(x0, y0, z1));
      const float c11 = fmaf(at(x1, y1, z1) - at(x0, y1, z1), tx, at(x0, y1, z1));
      const float c0 = fmaf(c10 - c00, ty, c00), c1 = fmaf(c11 - c01, ty, c01);
      value += static_cast<double>(fmaf(c1 - c0, tz, c0));
    }
    value *= dt;
  }
  images[gid] = static_cast<float>(value);
}

}  // namespace

void launch_raymarch(const float* vol, const int dims[3], double spacing, const double origin[3], const Frame* frames,
                     const Geo& g, int n_views, float* images, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(g.n_u) * g.n_v * n_views;
  if (total == 0) return;
  VolDesc vd{dims[0], dims[1], dims[2], spacing, origin[0], origin[1], origin[2]};
  k_raymarch<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(vol, vd, frames, g, n_views, images);
  count_launch();
}

}  // namespace gsct_dev
