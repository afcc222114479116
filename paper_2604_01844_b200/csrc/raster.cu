// Rasterizer pair kernels (fp32): tile-pair emission (K2), tile ranges, the per-tile
// forward accumulation (K3) and the per-splat backward pixel loop (K4a).
//
// K3 follows rasterize_view (projector.hpp:321-347): every pixel sums the splats of its
// tile list in ascending splat index (the list order produced by the stable sort), only
// over pixels inside each splat's bbox, value amp * exp(-0.5 (a du^2 + c dv^2) - b du dv).
// K4a follows rasterize_backward's pixel loop (projector.hpp:399-420): each splat is
// owned by one warp that walks its own bbox; per-pixel terms are reduced with a fixed
// xor-shuffle tree, so gradients are bit-stable without atomics.
#include <cuda_runtime.h>

#include "gsct_internal.cuh"

namespace gsct_dev {

namespace {

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void k_emit_tile_pairs(const RasterRec* __restrict__ rec,
                                  const uint32_t* __restrict__ offsets,
                                  const uint32_t* __restrict__ counts, int64_t n, int n_views,
                                  int tiles_u, int n_tiles, int ts, uint32_t* __restrict__ keys,
                                  uint32_t* __restrict__ vals) {
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= n * n_views) return;
  const uint32_t cnt = counts[item];
  if (cnt == 0) return;
  const int v = static_cast<int>(item / n);
  const uint32_t i = static_cast<uint32_t>(item - static_cast<int64_t>(v) * n);
  const RasterRec r = rec[item];
  const int u0 = r.urange & 0xFFFF, u1 = r.urange >> 16;
  const int v0 = r.vrange & 0xFFFF, v1 = r.vrange >> 16;
  uint32_t off = offsets[item];
  const uint32_t base = static_cast<uint32_t>(v) * static_cast<uint32_t>(n_tiles);
  for (int tv = v0 / ts; tv <= v1 / ts; ++tv)
    for (int tu = u0 / ts; tu <= u1 / ts; ++tu) {
      keys[off] = base + static_cast<uint32_t>(tv * tiles_u + tu);
      vals[off] = i;
      ++off;
    }
}

__global__ void k_ranges(const uint32_t* __restrict__ keys, int64_t n_pairs,
                         uint32_t* __restrict__ start, uint32_t* __restrict__ end) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n_pairs) return;
  const uint32_t key = keys[k];
  if (k == 0 || keys[k - 1] != key) start[key] = static_cast<uint32_t>(k);
  if (k == n_pairs - 1 || keys[k + 1] != key) end[key] = static_cast<uint32_t>(k + 1);
}

// One CTA (256 threads) per 16x16 tile and view. Warp w owns an 8x4 pixel patch so that
// splat rectangles that miss the patch are skipped warp-uniformly.
__global__ void __launch_bounds__(256) k_raster_fwd(const RasterRec* __restrict__ rec,
                                                    const uint32_t* __restrict__ vals,
                                                    const uint32_t* __restrict__ start,
                                                    const uint32_t* __restrict__ end, int64_t n,
                                                    int n_u, int n_v, int tiles_u,
                                                    float* __restrict__ images) {
  __shared__ float4 s_rect[256];  // fu0, fu1, fv0, fv1
  __shared__ float4 s_par[256];   // mo_u, mo_v, A, B
  __shared__ float2 s_par2[256];  // C, amp
  const int tile = blockIdx.x;
  const int view = blockIdx.y;
  const int n_tiles = gridDim.x;
  const int tu = tile % tiles_u, tv = tile / tiles_u;
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  const int pu0 = tu * kTile + (w & 1) * 8, pv0 = tv * kTile + (w >> 1) * 4;
  const int px = pu0 + (l & 7), py = pv0 + (l >> 3);
  const float fu = static_cast<float>(px), fv = static_cast<float>(py);
  const float wu0 = static_cast<float>(pu0), wu1 = wu0 + 7.f;
  const float wv0 = static_cast<float>(pv0), wv1 = wv0 + 3.f;
  const uint32_t key = static_cast<uint32_t>(view) * n_tiles + tile;
  const uint32_t b = start[key], e = end[key];
  const RasterRec* __restrict__ vrec = rec + static_cast<int64_t>(view) * n;
  float acc = 0.f;
  for (uint32_t base = b; base < e; base += 256) {
    const int cnt = min(256u, e - base);
    __syncthreads();
    if (t < cnt) {
      const RasterRec r = vrec[vals[base + t]];
      s_rect[t] = make_float4(static_cast<float>(r.urange & 0xFFFF), static_cast<float>(r.urange >> 16),
                              static_cast<float>(r.vrange & 0xFFFF), static_cast<float>(r.vrange >> 16));
      s_par[t] = make_float4(r.mo_u, r.mo_v, r.A, r.B);
      s_par2[t] = make_float2(r.C, r.amp);
    }
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {
      const float4 rc = s_rect[j];
      if (rc.x > wu1 || rc.y < wu0 || rc.z > wv1 || rc.w < wv0) continue;  // warp-uniform
      const float4 p = s_par[j];
      const float2 p2 = s_par2[j];
      const float du = (fu - rc.x) - p.x;
      const float dv = (fv - rc.z) - p.y;
      const float ex = ex2_approx(fmaf(fmaf(p.z, du, p.w * dv), du, p2.x * dv * dv));
      if (fu >= rc.x && fu <= rc.y && fv >= rc.z && fv <= rc.w) acc = fmaf(p2.y, ex, acc);
    }
  }
  if (px < n_u && py < n_v)
    images[static_cast<int64_t>(view) * n_u * n_v + static_cast<int64_t>(py) * n_u + px] = acc;
}

// One warp per (view, splat) item, grid-stride. Lanes walk the bbox row-major in steps of
// 32 pixels. Moments of t = exp(e) * w: {t, t du, t dv, t du^2, t du dv, t dv^2}.
__global__ void __launch_bounds__(256) k_raster_bwd_pairs(const RasterRec* __restrict__ rec,
                                                          int64_t n_items, int64_t n, int n_u,
                                                          int n_v,
                                                          const float* __restrict__ grad,
                                                          float4* __restrict__ moments) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t item = warp; item < n_items; item += n_warps) {
    const RasterRec r = rec[item];
    const int u0 = r.urange & 0xFFFF, u1 = r.urange >> 16;
    const int v0 = r.vrange & 0xFFFF, v1 = r.vrange >> 16;
    const int W = u1 - u0 + 1, H = v1 - v0 + 1;
    if (W <= 0 || H <= 0) continue;
    const int view = static_cast<int>(item / n);
    const float* __restrict__ gi = grad + static_cast<int64_t>(view) * n_u * n_v;
    const int npix = W * H;
    int pu = lane % W, pv = lane / W;
    const int su = 32 % W, sv = 32 / W;
    float fpu = static_cast<float>(pu), fpv = static_cast<float>(pv);
    const float fsu = static_cast<float>(su), fsv = static_cast<float>(sv), fW = static_cast<float>(W);
    float m0 = 0.f, mu = 0.f, mv = 0.f, muu = 0.f, muv = 0.f, mvv = 0.f;
    for (int p = lane; p < npix; p += 32) {
      const float w = __ldg(gi + static_cast<int64_t>(v0 + pv) * n_u + (u0 + pu));
      const float du = fpu - r.mo_u, dv = fpv - r.mo_v;
      const float ex = ex2_approx(fmaf(fmaf(r.A, du, r.B * dv), du, r.C * dv * dv));
      const float tt = ex * w;
      m0 += tt;
      const float tu_ = tt * du, tv_ = tt * dv;
      mu += tu_;
      mv += tv_;
      muu = fmaf(tu_, du, muu);
      muv = fmaf(tu_, dv, muv);
      mvv = fmaf(tv_, dv, mvv);
      pu += su;
      pv += sv;
      fpu += fsu;
      fpv += fsv;
      if (pu >= W) {
        pu -= W;
        pv += 1;
        fpu -= fW;
        fpv += 1.f;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m0 += __shfl_xor_sync(0xffffffffu, m0, o);
      mu += __shfl_xor_sync(0xffffffffu, mu, o);
      mv += __shfl_xor_sync(0xffffffffu, mv, o);
      muu += __shfl_xor_sync(0xffffffffu, muu, o);
      muv += __shfl_xor_sync(0xffffffffu, muv, o);
      mvv += __shfl_xor_sync(0xffffffffu, mvv, o);
    }
    if (lane == 0) {
      moments[2 * item] = make_float4(m0, mu, mv, muu);
      moments[2 * item + 1] = make_float4(muv, mvv, 0.f, 0.f);
    }
  }
}

inline unsigned blocks_for(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

}  // namespace

void launch_emit_tile_pairs(const RasterRec* rec, const uint32_t* offsets, const uint32_t* counts,
                            int64_t n, int n_views, int ts, int tiles_u, int n_tiles, uint32_t* keys,
                            uint32_t* vals, cudaStream_t st) {
  const int64_t items = n * n_views;
  if (items == 0) return;
  k_emit_tile_pairs<<<blocks_for(items, 256), 256, 0, st>>>(rec, offsets, counts, n, n_views,
                                                            tiles_u, n_tiles, ts, keys, vals);
  count_launch();
}

void launch_ranges(const uint32_t* keys, int64_t n_pairs, uint32_t* start, uint32_t* end,
                   cudaStream_t st) {
  if (n_pairs == 0) return;
  k_ranges<<<blocks_for(n_pairs, 256), 256, 0, st>>>(keys, n_pairs, start, end);
  count_launch();
}

void launch_raster_fwd(const RasterRec* rec, const uint32_t* vals, const uint32_t* start,
                       const uint32_t* end, int64_t n, int n_views, int n_u, int n_v, int tiles_u,
                       int tiles_v, float* images, cudaStream_t st) {
  if (n_views == 0) return;
  dim3 grid(static_cast<unsigned>(tiles_u * tiles_v), static_cast<unsigned>(n_views));
  k_raster_fwd<<<grid, 256, 0, st>>>(rec, vals, start, end, n, n_u, n_v, tiles_u, images);
  count_launch();
}

void launch_raster_bwd_pairs(const RasterRec* rec, int64_t n, int n_views, int n_u, int n_v,
                             const float* grad_images, float* moments, unsigned int* /*work*/,
                             cudaStream_t st) {
  const int64_t items = n * n_views;
  if (items == 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (items + 7) / 8;  // 8 warps per block
  const unsigned blocks = static_cast<unsigned>(want < static_cast<int64_t>(sms) * 16 ? want : static_cast<int64_t>(sms) * 16);
  k_raster_bwd_pairs<<<blocks, 256, 0, st>>>(rec, items, n, n_u, n_v, grad_images,
                                             reinterpret_cast<float4*>(moments));
  count_launch();
}

}  // namespace gsct_dev
