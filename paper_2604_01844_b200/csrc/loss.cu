// Next-row kernels: the image loss of the reconstruction loop, L1 + SSIM2D
// (losses.hpp:28-45, 82-272, total_loss_recon 613-637 without the TV term), forward and
// gradient w.r.t. the rendered image, so the backward can start from device-resident
// grad images instead of a host round trip per view.
//
// Per view (image = n_v x n_u, u fastest):
//   l1   = mean |p - t|,                 dl1/dp = sign(p - t) / N   (sign(0) = 0)
//   ssim = 1 - mean over valid 11x11 windows of SSIM(window), Gaussian window sigma 1.5,
//          C1 = 1e-4, C2 = 9e-4 (unit data range), window centres fully inside the image;
//          dssim/dp = -1/N_out * [adj(ca) + adj(cb) * p + adj(cc) * t]   (losses.hpp:170-272)
//   grad = dl1/dp + alpha * dssim/dp,   total = l1 + alpha * ssim.
// Moments, SSIM points and sums are fp64 (the variance terms E[x^2] - E[x]^2 cancel);
// images and the gradient are fp32. Sums are per-tile partials combined in a fixed order
// (deterministic). Compiled with FMA contraction (tolerance-level parity, no keys).
#include <cuda_runtime.h>

#include "gsct_internal.cuh"

namespace gsct_dev {

namespace {

constexpr int kW = 11, kR = 5;  // SSIM window
constexpr int kT = 32;            // tile width (outputs / pixels)
constexpr int kTY = 16;           // tile height
constexpr int kH = kT + kW - 1;   // tile + halo, x (42)
constexpr int kHY = kTY + kW - 1; // tile + halo, y (26)
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

struct SsimWin {
  double w[kW];
};

// K9a: one CTA per 32x32 tile of valid window positions (outputs) and view: stages the
// 42x42 input region, separable 11-tap filtering of the five moment maps in fp64
// (horizontal then vertical), the per-window SSIM value and gradient coefficients
// (ssim_point, losses.hpp:173-196); writes ca/cb/cc maps (fp32) and a per-tile sum of s.
__global__ void __launch_bounds__(256) k_ssim_fwd(const float* __restrict__ pred, const float* __restrict__ targ,
                                                  int nu, int nv, SsimWin win, float* __restrict__ coef,
                                                  double* __restrict__ part_s) {
  __shared__ float sp[kHY][kH + 1], st[kHY][kH + 1];
  __shared__ double hs[5][kHY][kT];
  const int nuo = nu - (kW - 1), nvo = nv - (kW - 1);
  const int tx = blockIdx.x, ty = blockIdx.y, view = blockIdx.z;
  const int x0 = tx * kT, y0 = ty * kTY;
  const int64_t npx = static_cast<int64_t>(nu) * nv;
  const float* p = pred + view * npx;
  const float* t = targ + view * npx;
  for (int k = threadIdx.x; k < kHY * kH; k += blockDim.x) {
    const int r = k / kH, c = k % kH;
    const int x = x0 + c, y = y0 + r;
    const bool in = x < nu && y < nv;
    sp[r][c] = in ? p[static_cast<int64_t>(y) * nu + x] : 0.f;
    st[r][c] = in ? t[static_cast<int64_t>(y) * nu + x] : 0.f;
  }
  __syncthreads();
  // horizontal pass: rows 0..25, output columns 0..31
  for (int k = threadIdx.x; k < kHY * kT; k += blockDim.x) {
    const int r = k / kT, c = k % kT;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const double x = sp[r][c + j], y = st[r][c + j], w = win.w[j];
      a0 = fma(w, x, a0);
      a1 = fma(w, y, a1);
      a2 = fma(w, x * x, a2);
      a3 = fma(w, y * y, a3);
      a4 = fma(w, x * y, a4);
    }
    hs[0][r][c] = a0, hs[1][r][c] = a1, hs[2][r][c] = a2, hs[3][r][c] = a3, hs[4][r][c] = a4;
  }
  __syncthreads();
  double s_sum = 0.0;
  const int64_t nout = static_cast<int64_t>(nuo) * nvo;
  float* ca = coef + (view * 3 + 0) * nout;
  float* cb = coef + (view * 3 + 1) * nout;
  float* cc = coef + (view * 3 + 2) * nout;
  for (int k = threadIdx.x; k < kTY * kT; k += blockDim.x) {
    const int r = k / kT, c = k % kT;
    const int xo = x0 + c, yo = y0 + r;
    if (xo >= nuo || yo >= nvo) continue;
    double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const double w = win.w[j];
#pragma unroll
      for (int q = 0; q < 5; ++q) m[q] = fma(w, hs[q][r + j][c], m[q]);
    }
    // ssim_point (losses.hpp:173-196)
    const double mx = m[0], my = m[1];
    const double sx = m[2] - mx * mx, sy = m[3] - my * my, sxy = m[4] - mx * my;
    const double a1 = 2.0 * mx * my + kC1, a2 = 2.0 * sxy + kC2;
    const double b1 = mx * mx + my * my + kC1, b2 = sx + sy + kC2;
    const double inv_b1b2 = 1.0 / (b1 * b2);
    const double s = a1 * a2 * inv_b1b2;
    const double ds_dmx = 2.0 * my * a2 * inv_b1b2 - 2.0 * mx * s / b1;
    const double ds_dsx = -s / b2;
    const double ds_dsxy = 2.0 * a1 * inv_b1b2;
    const int64_t o = static_cast<int64_t>(yo) * nuo + xo;
    ca[o] = static_cast<float>(ds_dmx - 2.0 * ds_dsx * mx - ds_dsxy * my);
    cb[o] = static_cast<float>(2.0 * ds_dsx);
    cc[o] = static_cast<float>(ds_dsxy);
    s_sum += s;
  }
  // fixed-order block reduction: warp xor tree, then warp partials in order
  __shared__ double wsum[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s_sum += __shfl_xor_sync(0xffffffffu, s_sum, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s_sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) tot += wsum[w];
    part_s[(static_cast<int64_t>(view) * gridDim.y + ty) * gridDim.x + tx] = tot;
  }
}

// K9b: one CTA per 32x32 pixel tile and view: adjoint (transposed) filtering of the three
// coefficient maps over every window covering each pixel (ssim_adj_y / ssim_adj_x,
// losses.hpp:136-170), then grad = sign(d)/N + alpha * (-1/N_out) (A + B p + C t), and a
// per-tile sum of |p - t|.
__global__ void __launch_bounds__(256) k_ssim_bwd(const float* __restrict__ pred, const float* __restrict__ targ,
                                                  int nu, int nv, SsimWin win, const float* __restrict__ coef,
                                                  double alpha, float* __restrict__ grad,
                                                  double* __restrict__ part_l1) {
  __shared__ float cs[3][kHY][kH + 1];
  __shared__ double vs[3][kTY][kH];
  const int nuo = nu - (kW - 1), nvo = nv - (kW - 1);
  const int tx = blockIdx.x, ty = blockIdx.y, view = blockIdx.z;
  const int x0 = tx * kT, y0 = ty * kTY;
  const int64_t npx = static_cast<int64_t>(nu) * nv, nout = static_cast<int64_t>(nuo) * nvo;
  // windows c in [x0 - 10, x0 + 31], d in [y0 - 10, y0 + 15] (zero outside the valid range)
  for (int k = threadIdx.x; k < kHY * kH; k += blockDim.x) {
    const int r = k / kH, c = k % kH;
    const int xo = x0 - (kW - 1) + c, yo = y0 - (kW - 1) + r;
    const bool in = xo >= 0 && yo >= 0 && xo < nuo && yo < nvo;
    const int64_t o = static_cast<int64_t>(yo) * nuo + xo;
#pragma unroll
    for (int q = 0; q < 3; ++q) cs[q][r][c] = in ? coef[(view * 3 + q) * nout + o] : 0.f;
  }
  __syncthreads();
  // vertical adjoint: pixel rows 0..15 (y = y0 + r) sum windows d = y - 10 .. y, weight w[y - d]
  for (int k = threadIdx.x; k < kTY * kH; k += blockDim.x) {
    const int r = k / kH, c = k % kH;
    double a[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < kW; ++j) {  // window row index in smem: r + j, weight w[kW - 1 - j]
      const double w = win.w[kW - 1 - j];
#pragma unroll
      for (int q = 0; q < 3; ++q) a[q] = fma(w, static_cast<double>(cs[q][r + j][c]), a[q]);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) vs[q][r][c] = a[q];
  }
  __syncthreads();
  const double inv_out = 1.0 / static_cast<double>(nout), inv_in = 1.0 / static_cast<double>(npx);
  const float* p = pred + view * npx;
  const float* t = targ + view * npx;
  float* g = grad + view * npx;
  double l1 = 0.0;
  for (int k = threadIdx.x; k < kTY * kT; k += blockDim.x) {
    const int r = k / kT, c = k % kT;
    const int x = x0 + c, y = y0 + r;
    if (x >= nu || y >= nv) continue;
    double a[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const double w = win.w[kW - 1 - j];
#pragma unroll
      for (int q = 0; q < 3; ++q) a[q] = fma(w, vs[q][r][c + j], a[q]);
    }
    const int64_t i = static_cast<int64_t>(y) * nu + x;
    const double pv = p[i], tv = t[i], d = pv - tv;
    l1 += fabs(d);
    const double gl1 = d > 0.0 ? inv_in : (d < 0.0 ? -inv_in : 0.0);
    const double gs = -inv_out * (a[0] + a[1] * pv + a[2] * tv);
    g[i] = static_cast<float>(gl1 + alpha * gs);
  }
  __shared__ double wsum[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = l1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) tot += wsum[w];
    part_l1[(static_cast<int64_t>(view) * gridDim.y + ty) * gridDim.x + tx] = tot;
  }
}

// K9c: per view, the tile partials in tile order -> l1, ssim loss, total.
__global__ void k_loss_finish(const double* __restrict__ part_s, int tiles_s, const double* __restrict__ part_l1,
                              int tiles_p, int n_views, double n_out, double n_in, double alpha,
                              double* __restrict__ out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n_views) return;
  double s = 0.0, l = 0.0;
  for (int k = 0; k < tiles_s; ++k) s += part_s[static_cast<int64_t>(v) * tiles_s + k];
  for (int k = 0; k < tiles_p; ++k) l += part_l1[static_cast<int64_t>(v) * tiles_p + k];
  const double l1 = l / n_in, ssim = 1.0 - s / n_out;
  out[3 * v + 0] = l1;
  out[3 * v + 1] = ssim;
  out[3 * v + 2] = l1 + alpha * ssim;
}

}  // namespace

void launch_image_loss(const float* pred, const float* targ, int n_views, int nu, int nv, const double* window,
                       double alpha, float* coef, double* part_s, double* part_l1, float* grad, double* out3,
                       cudaStream_t st) {
  if (n_views == 0) return;
  SsimWin w;
  for (int k = 0; k < kW; ++k) w.w[k] = window[k];
  const int nuo = nu - (kW - 1), nvo = nv - (kW - 1);
  const dim3 go((nuo + kT - 1) / kT, (nvo + kTY - 1) / kTY, n_views);
  const dim3 gp((nu + kT - 1) / kT, (nv + kTY - 1) / kTY, n_views);
  k_ssim_fwd<<<go, 256, 0, st>>>(pred, targ, nu, nv, w, coef, part_s);
  k_ssim_bwd<<<gp, 256, 0, st>>>(pred, targ, nu, nv, w, coef, alpha, grad, part_l1);
  k_loss_finish<<<(n_views + 127) / 128, 128, 0, st>>>(part_s, static_cast<int>(go.x * go.y), part_l1,
                                                      static_cast<int>(gp.x * gp.y), n_views,
                                                      static_cast<double>(nuo) * nvo,
                                                      static_cast<double>(nu) * nv, alpha, out3);
  count_launch(3);
}

int64_t image_loss_partials(int n_views, int nu, int nv) {
  const int nuo = nu - (kW - 1), nvo = nv - (kW - 1);
  return static_cast<int64_t>(n_views) *
         (static_cast<int64_t>((nuo + kT - 1) / kT) * ((nvo + kTY - 1) / kTY) +
          static_cast<int64_t>((nu + kT - 1) / kT) * ((nv + kTY - 1) / kTY));
}

}  // namespace gsct_dev

// ---------------------------------------------------------------------------------------
// Volume-fit loss: total_loss_fit = L1 + alpha * SSIM3D
// (losses.hpp:275-516, 648-664) and TV3D (losses.hpp:530-595), forward + gradient.
// SSIM3D is computed as separable valid passes x -> y -> z over the five moment volumes
// (fp64), the SSIM point per window centre, then the transposed passes z -> y -> x of the
// three coefficient volumes; the reference's streaming and materialised paths are the same
// arithmetic (bit-equal), and this device version agrees with them to fp64 rounding.
// ---------------------------------------------------------------------------------------
namespace gsct_dev {
namespace {

struct Dims3 {
  int n[3];  // x, y, z extents of the array being filtered
};

// moments of (p, t): channels x, y, x^2, y^2, xy (fp64), full size
__global__ void k_vol_products(const float* __restrict__ p, const float* __restrict__ t, int64_t nvox,
                               double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nvox) return;
  const double x = p[i], y = t[i];
  out[i] = x;
  out[nvox + i] = y;
  out[2 * nvox + i] = x * x;
  out[3 * nvox + i] = y * y;
  out[4 * nvox + i] = x * y;
}

// One separable pass along `axis` over C channels. valid: out extent = in - 10,
// out[i] = sum_k w[k] in[i + k]; adjoint: out extent = in + 10, out[i] = sum over windows c
// covering i of w[i - c] in[c] (ascending c).
template <bool kAdjoint>
__global__ void k_vol_pass(const double* __restrict__ in, Dims3 din, int axis, int channels, SsimWin win,
                           double* __restrict__ out) {
  Dims3 dout = din;
  dout.n[axis] = kAdjoint ? din.n[axis] + (kW - 1) : din.n[axis] - (kW - 1);
  const int64_t nout = static_cast<int64_t>(dout.n[0]) * dout.n[1] * dout.n[2];
  const int64_t nin = static_cast<int64_t>(din.n[0]) * din.n[1] * din.n[2];
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= nout * channels) return;
  const int c = static_cast<int>(gid / nout);
  int64_t r = gid - c * nout;
  int idx[3];
  idx[0] = static_cast<int>(r % dout.n[0]);
  r /= dout.n[0];
  idx[1] = static_cast<int>(r % dout.n[1]);
  idx[2] = static_cast<int>(r / dout.n[1]);
  const int64_t stride = axis == 0 ? 1 : (axis == 1 ? din.n[0] : static_cast<int64_t>(din.n[0]) * din.n[1]);
  int base[3] = {idx[0], idx[1], idx[2]};
  const int i = idx[axis];
  double acc = 0.0;
  if (!kAdjoint) {
    base[axis] = i;
    const double* src = in + c * nin + (static_cast<int64_t>(base[2]) * din.n[1] + base[1]) * din.n[0] + base[0];
#pragma unroll
    for (int k = 0; k < kW; ++k) acc = fma(win.w[k], src[k * stride], acc);
  } else {
    const int lo = max(0, i - (kW - 1)), hi = min(din.n[axis] - 1, i);
    base[axis] = 0;
    const double* src = in + c * nin + (static_cast<int64_t>(base[2]) * din.n[1] + base[1]) * din.n[0] + base[0];
    for (int cc = lo; cc <= hi; ++cc) acc = fma(win.w[i - cc], src[cc * stride], acc);
  }
  out[c * nout + (static_cast<int64_t>(idx[2]) * dout.n[1] + idx[1]) * dout.n[0] + idx[0]] = acc;
}

// SSIM point per window centre: coefficient volumes (fp64) + per-block partial sums of s
__global__ void __launch_bounds__(256) k_vol_ssim_point(const double* __restrict__ m, int64_t nout,
                                                        double* __restrict__ coef, double* __restrict__ part) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (i < nout) {
    const double mx = m[i], my = m[nout + i];
    const double sx = m[2 * nout + i] - mx * mx, sy = m[3 * nout + i] - my * my, sxy = m[4 * nout + i] - mx * my;
    const double a1 = 2.0 * mx * my + kC1, a2 = 2.0 * sxy + kC2;
    const double b1 = mx * mx + my * my + kC1, b2 = sx + sy + kC2;
    const double inv_b1b2 = 1.0 / (b1 * b2);
    s = a1 * a2 * inv_b1b2;
    const double ds_dmx = 2.0 * my * a2 * inv_b1b2 - 2.0 * mx * s / b1;
    const double ds_dsx = -s / b2;
    const double ds_dsxy = 2.0 * a1 * inv_b1b2;
    coef[i] = ds_dmx - 2.0 * ds_dsx * mx - ds_dsxy * my;
    coef[nout + i] = 2.0 * ds_dsx;
    coef[2 * nout + i] = ds_dsxy;
  }
  __shared__ double ws[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) tot += ws[w];
    part[blockIdx.x] = tot;
  }
}

// grad = sign(d)/N + alpha * (-1/N_out) (A + B p + C t); per-block partial sums of |d|
__global__ void __launch_bounds__(256) k_vol_grad(const float* __restrict__ p, const float* __restrict__ t,
                                                  const double* __restrict__ adj, int64_t nvox, double inv_out,
                                                  double alpha, float* __restrict__ grad,
                                                  double* __restrict__ part) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double l1 = 0.0;
  if (i < nvox) {
    const double pv = p[i], tv = t[i], d = pv - tv;
    l1 = fabs(d);
    const double inv_in = 1.0 / static_cast<double>(nvox);
    const double gl1 = d > 0.0 ? inv_in : (d < 0.0 ? -inv_in : 0.0);
    double gs = 0.0;
    if (alpha > 0.0) gs = -inv_out * (adj[i] + adj[nvox + i] * pv + adj[2 * nvox + i] * tv);
    grad[i] = static_cast<float>(gl1 + alpha * gs);
  }
  __shared__ double ws[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = l1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) tot += ws[w];
    part[blockIdx.x] = tot;
  }
}

__global__ void k_sum_parts(const double* __restrict__ part, int64_t n, double* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) s += part[k];
    *out = s;
  }
}

// TV3D (losses.hpp:530-595): pass 1 = magnitudes 1/g and per-block sums of g over interior
// voxels; pass 2 = the gather of every term a voxel appears in.
__global__ void __launch_bounds__(256) k_tv_mag(const float* __restrict__ v, int nx, int ny, int nz,
                                                double* __restrict__ inv_mag, double* __restrict__ part) {
  const int mx = nx - 1, my = ny - 1, mz = nz - 1;
  const int64_t nint = static_cast<int64_t>(mx) * my * mz;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double g = 0.0;
  if (i < nint) {
    const int x = static_cast<int>(i % mx), y = static_cast<int>((i / mx) % my), z = static_cast<int>(i / (static_cast<int64_t>(mx) * my));
    const int64_t o = (static_cast<int64_t>(z) * ny + y) * nx + x;
    const double c = v[o];
    const double dx = v[o + 1] - c, dy = v[o + nx] - c, dz = v[o + static_cast<int64_t>(nx) * ny] - c;
    g = sqrt(dx * dx + dy * dy + dz * dz + 1e-8 * 1e-8);
    inv_mag[i] = 1.0 / g;
  }
  __shared__ double ws[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = g;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) tot += ws[w];
    part[blockIdx.x] = tot;
  }
}

__global__ void k_tv_grad(const float* __restrict__ v, int nx, int ny, int nz, const double* __restrict__ inv_mag,
                          float* __restrict__ grad) {
  const int mx = nx - 1, my = ny - 1, mz = nz - 1;
  const int64_t n = static_cast<int64_t>(nx) * ny * nz;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = static_cast<int>(i % nx), y = static_cast<int>((i / nx) % ny), z = static_cast<int>(i / (static_cast<int64_t>(nx) * ny));
  auto at = [&](int xx, int yy, int zz) { return static_cast<double>(v[(static_cast<int64_t>(zz) * ny + yy) * nx + xx]); };
  auto im = [&](int xx, int yy, int zz) { return inv_mag[(static_cast<int64_t>(zz) * my + yy) * mx + xx]; };
  const double c = at(x, y, z);
  double acc = 0.0;
  if (x < mx && y < my && z < mz) acc -= ((at(x + 1, y, z) - c) + (at(x, y + 1, z) - c) + (at(x, y, z + 1) - c)) * im(x, y, z);
  if (x > 0 && y < my && z < mz) acc += (c - at(x - 1, y, z)) * im(x - 1, y, z);
  if (y > 0 && x < mx && z < mz) acc += (c - at(x, y - 1, z)) * im(x, y - 1, z);
  if (z > 0 && x < mx && y < my) acc += (c - at(x, y, z - 1)) * im(x, y, z - 1);
  const double inv_n = 1.0 / (static_cast<double>(mx) * my * mz);
  grad[i] = static_cast<float>(acc * inv_n);
}

inline unsigned nblk(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

}  // namespace

int64_t volume_loss_scratch_doubles(const int dims[3]) {
  const int64_t n = static_cast<int64_t>(dims[0]) * dims[1] * dims[2];
  return 10 * n + 2 * nblk(n, 256) + 8;  // two 5-channel ping-pong buffers (>= 3-channel adjoints) + partials
}

void launch_volume_loss(const float* pred, const float* targ, const int dims[3], const double* window, double alpha,
                        double* scratch, float* grad, double* out3, cudaStream_t st) {
  SsimWin w;
  for (int k = 0; k < kW; ++k) w.w[k] = window[k];
  const int64_t n = static_cast<int64_t>(dims[0]) * dims[1] * dims[2];
  double* A = scratch;          // 5 n
  double* B = scratch + 5 * n;  // 5 n
  double* part_s = scratch + 10 * n;
  double* part_l = part_s + nblk(n, 256);
  double* sums = part_l + nblk(n, 256);  // {sum s, sum |d|}
  Dims3 d{{dims[0], dims[1], dims[2]}};
  const int64_t nout = static_cast<int64_t>(dims[0] - 10) * (dims[1] - 10) * (dims[2] - 10);
  if (alpha > 0.0) {
    k_vol_products<<<nblk(n, 256), 256, 0, st>>>(pred, targ, n, A);
    Dims3 d1 = d;
    d1.n[0] -= 10;
    k_vol_pass<false><<<nblk(5 * static_cast<int64_t>(d1.n[0]) * d1.n[1] * d1.n[2], 256), 256, 0, st>>>(A, d, 0, 5, w, B);
    Dims3 d2 = d1;
    d2.n[1] -= 10;
    k_vol_pass<false><<<nblk(5 * static_cast<int64_t>(d2.n[0]) * d2.n[1] * d2.n[2], 256), 256, 0, st>>>(B, d1, 1, 5, w, A);
    Dims3 d3 = d2;
    d3.n[2] -= 10;
    k_vol_pass<false><<<nblk(5 * nout, 256), 256, 0, st>>>(A, d2, 2, 5, w, B);
    k_vol_ssim_point<<<nblk(nout, 256), 256, 0, st>>>(B, nout, A, part_s);
    k_sum_parts<<<1, 32, 0, st>>>(part_s, static_cast<int64_t>(nblk(nout, 256)), sums);
    // adjoints z -> y -> x of the three coefficient volumes
    k_vol_pass<true><<<nblk(3 * static_cast<int64_t>(d2.n[0]) * d2.n[1] * d2.n[2], 256), 256, 0, st>>>(A, d3, 2, 3, w, B);
    k_vol_pass<true><<<nblk(3 * static_cast<int64_t>(d1.n[0]) * d1.n[1] * d1.n[2], 256), 256, 0, st>>>(B, d2, 1, 3, w, A);
    k_vol_pass<true><<<nblk(3 * n, 256), 256, 0, st>>>(A, d1, 0, 3, w, B);
    count_launch(9);
  }
  k_vol_grad<<<nblk(n, 256), 256, 0, st>>>(pred, targ, B, n, 1.0 / static_cast<double>(nout), alpha, grad, part_l);
  k_sum_parts<<<1, 32, 0, st>>>(part_l, static_cast<int64_t>(nblk(n, 256)), sums + 1);
  count_launch(2);
  (void)out3;
}

int64_t tv3d_scratch_doubles(const int dims[3]) {
  const int64_t nint = static_cast<int64_t>(dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1);
  return nint + nblk(nint, 256) + 2;
}

void launch_tv3d(const float* vol, const int dims[3], double* scratch, float* grad, cudaStream_t st) {
  const int64_t nint = static_cast<int64_t>(dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1);
  const int64_t n = static_cast<int64_t>(dims[0]) * dims[1] * dims[2];
  double* inv_mag = scratch;
  double* part = scratch + nint;
  double* sum = part + nblk(nint, 256);
  k_tv_mag<<<nblk(nint, 256), 256, 0, st>>>(vol, dims[0], dims[1], dims[2], inv_mag, part);
  k_sum_parts<<<1, 32, 0, st>>>(part, static_cast<int64_t>(nblk(nint, 256)), sum);
  k_tv_grad<<<nblk(n, 256), 256, 0, st>>>(vol, dims[0], dims[1], dims[2], inv_mag, grad);
  count_launch(3);
}

}  // namespace gsct_dev
