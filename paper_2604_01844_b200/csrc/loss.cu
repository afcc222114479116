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
