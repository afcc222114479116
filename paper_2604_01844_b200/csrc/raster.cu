// Rasterizer pair kernels (fp32): tile-pair emission (K2), key ranges, the per-tile
// forward accumulation (K3), the backward walk-order keys and the per-item backward pixel
// walk (K4a).
//
// K3 follows rasterize_view (projector.hpp:321-347): every pixel sums the splats whose
// bbox covers it in ascending splat index (the list order produced by the stable sort),
// value amp * exp(-0.5 (a du^2 + c dv^2) - b du dv). K4a follows rasterize_backward's pixel
// loop (projector.hpp:399-420): each (view, splat) item is owned by ONE lane that walks its
// own bbox sequentially, so gradients are bit-stable without atomics or cross-lane trees.
//
// Both are issue-bound rather than HBM-bound (profiles/r1/raster): the designs minimise
// issue slots per splat-pixel pair (packed f32x2 arithmetic, multiplicative exp chains in
// the forward) and wasted lanes (per-lane record filtering in the forward, lane-per-item
// with shape-sorted work in the backward). See DESIGN.md section 4.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "gsct_internal.cuh"
#include "packed_f32.cuh"

namespace gsct_dev {

namespace {

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

// [start, end) of every key in the sorted key array: one thread per key, binary search
// (n_keys * log2(pairs) reads instead of a pass over all pairs).
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* __restrict__ a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void k_ranges(const uint32_t* __restrict__ keys, uint32_t n_pairs, uint32_t n_keys,
                         uint32_t* __restrict__ start, uint32_t* __restrict__ end) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_keys) return;
  start[k] = lower_bound_u32(keys, n_pairs, k);
  end[k] = lower_bound_u32(keys, n_pairs, k + 1);
}

// Packed keys-only binning (one view chunk, <= 256 super-tiles per view, < 2^24 splats):
// each pair is ONE u32 = super-tile << 24 | splat, emitted view-major in splat order, so a
// stable radix pass over bits 24..31 orders them (tile, view, splat) while moving 4 bytes per
// pair instead of a key + value. The (view, tile) counts the ranges need are histogrammed
// here (per-CTA shared-memory bins, flushed with integer atomics: order-free).
__global__ void __launch_bounds__(256) k_emit_tile_keys(const RasterRec* __restrict__ rec,
                                                        const uint32_t* __restrict__ offsets,
                                                        const uint32_t* __restrict__ counts, int64_t n, int n_views,
                                                        int tiles_u, int n_tiles, int ts, uint32_t* __restrict__ keys,
                                                        uint32_t* __restrict__ vt_count) {
  __shared__ uint32_t h[2][256];  // a CTA's 256 items span at most two views (n >= 256)
  const int64_t item0 = static_cast<int64_t>(blockIdx.x) * blockDim.x;
  const int vbase = static_cast<int>(item0 / n);
  for (int k = threadIdx.x; k < 512; k += blockDim.x) (&h[0][0])[k] = 0u;
  __syncthreads();
  const int64_t item = item0 + threadIdx.x;
  if (item < n * n_views) {
    const uint32_t cnt = counts[item];
    if (cnt) {
      const int v = static_cast<int>(item / n);
      const uint32_t i = static_cast<uint32_t>(item - static_cast<int64_t>(v) * n);
      const RasterRec r = rec[item];
      const int u0 = r.urange & 0xFFFF, u1 = r.urange >> 16;
      const int v0 = r.vrange & 0xFFFF, v1 = r.vrange >> 16;
      uint32_t off = offsets[item];
      for (int tv = v0 / ts; tv <= v1 / ts; ++tv)
        for (int tu = u0 / ts; tu <= u1 / ts; ++tu) {
          const uint32_t t = static_cast<uint32_t>(tv * tiles_u + tu);
          keys[off++] = (t << 24) | i;
          atomicAdd(&h[v - vbase][t], 1u);
        }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 2 * n_tiles; k += blockDim.x) {
    const int vv = vbase + k / n_tiles, t = k % n_tiles;
    const uint32_t c = h[k / n_tiles][t];
    if (c && vv < n_views) atomicAdd(&vt_count[vv * n_tiles + t], c);
  }
}

// Wide variant for > 256 tiles per view (2048^2: 4096 super-tiles, key = tile << 20 | splat):
// each CTA emits kWideItems consecutive items (so it still spans at most two views) into
// shared-memory bins of 2 x n_tiles counts, flushed once per CTA with integer atomics.
__global__ void __launch_bounds__(256) k_emit_tile_keys_wide(const RasterRec* __restrict__ rec,
                                                             const uint32_t* __restrict__ offsets,
                                                             const uint32_t* __restrict__ counts, int64_t n,
                                                             int n_views, int tiles_u, int n_tiles, int ts, int shift,
                                                             uint32_t* __restrict__ keys,
                                                             uint32_t* __restrict__ vt_count) {
  extern __shared__ uint32_t hw[];  // [2][n_tiles]
  const int64_t item0 = static_cast<int64_t>(blockIdx.x) * kWideItems;
  const int vbase = static_cast<int>(item0 / n);
  for (int k = threadIdx.x; k < 2 * n_tiles; k += blockDim.x) hw[k] = 0u;
  __syncthreads();
  const int64_t n_items = n * n_views;
  for (int it = threadIdx.x; it < kWideItems; it += blockDim.x) {
    const int64_t item = item0 + it;
    if (item >= n_items) break;
    const uint32_t cnt = counts[item];
    if (!cnt) continue;
    const int v = static_cast<int>(item / n);
    const uint32_t i = static_cast<uint32_t>(item - static_cast<int64_t>(v) * n);
    const RasterRec r = rec[item];
    const int u0 = r.urange & 0xFFFF, u1 = r.urange >> 16;
    const int v0 = r.vrange & 0xFFFF, v1 = r.vrange >> 16;
    uint32_t off = offsets[item];
    uint32_t* hv = hw + (v - vbase) * n_tiles;
    for (int tv = v0 / ts; tv <= v1 / ts; ++tv)
      for (int tu = u0 / ts; tu <= u1 / ts; ++tu) {
        const uint32_t t = static_cast<uint32_t>(tv * tiles_u + tu);
        keys[off++] = (t << shift) | i;
        atomicAdd(&hv[t], 1u);
      }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 2 * n_tiles; k += blockDim.x) {
    const int vv = vbase + k / n_tiles, t = k % n_tiles;
    const uint32_t c = hw[k];
    if (c && vv < n_views) atomicAdd(&vt_count[vv * n_tiles + t], c);
  }
}

// Ranges for > 256 tiles: one CTA of 1024 threads, tiles in rounds of 1024 with a running base.
__global__ void __launch_bounds__(1024) k_ranges_from_counts_wide(const uint32_t* __restrict__ vt_count, int n_views,
                                                                  int n_tiles, int key_stride,
                                                                  uint32_t* __restrict__ start,
                                                                  uint32_t* __restrict__ end) {
  __shared__ uint32_t tot[1024];
  __shared__ uint32_t round_base;
  if (threadIdx.x == 0) round_base = 0u;
  for (int r0 = 0; r0 < n_tiles; r0 += 1024) {
    const int t = r0 + threadIdx.x;
    uint32_t sum = 0;
    if (t < n_tiles)
      for (int v = 0; v < n_views; ++v) sum += vt_count[v * n_tiles + t];
    __syncthreads();
    tot[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const uint32_t x = threadIdx.x >= static_cast<unsigned>(o) ? tot[threadIdx.x - o] : 0u;
      __syncthreads();
      tot[threadIdx.x] += x;
      __syncthreads();
    }
    const uint32_t rb = round_base;
    if (t < n_tiles) {
      uint32_t base = rb + tot[threadIdx.x] - sum;
      for (int v = 0; v < n_views; ++v) {
        const uint32_t c = vt_count[v * n_tiles + t];
        start[v * key_stride + t] = base;
        end[v * key_stride + t] = base + c;
        base += c;
      }
    }
    __syncthreads();
    if (threadIdx.x == 1023) round_base = rb + tot[1023];
    __syncthreads();
  }
}

// [start, end) per (view, tile) of the (tile, view, splat)-ordered packed keys, from the
// counts: one CTA, thread t owns tile t (block scan of the tile totals, then the views).
__global__ void __launch_bounds__(256) k_ranges_from_counts(const uint32_t* __restrict__ vt_count, int n_views,
                                                            int n_tiles, int key_stride, uint32_t* __restrict__ start,
                                                            uint32_t* __restrict__ end) {
  __shared__ uint32_t tot[256];
  const int t = threadIdx.x;
  uint32_t sum = 0;
  if (t < n_tiles)
    for (int v = 0; v < n_views; ++v) sum += vt_count[v * n_tiles + t];
  tot[t] = sum;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {  // inclusive Hillis-Steele scan
    const uint32_t x = t >= o ? tot[t - o] : 0u;
    __syncthreads();
    tot[t] += x;
    __syncthreads();
  }
  if (t >= n_tiles) return;
  uint32_t base = tot[t] - sum;  // exclusive
  for (int v = 0; v < n_views; ++v) {
    const uint32_t c = vt_count[v * n_tiles + t];
    start[v * key_stride + t] = base;
    end[v * key_stride + t] = base + c;
    base += c;
  }
}

// [start, end) of every key after the one-pass binning: keys = view << tile_bits | tile
// sorted by tile only (stable), i.e. ascending in ord(key) = tile << 16 | view; binary
// search in that order, one thread per key.
__device__ __forceinline__ uint32_t swapped_ord(uint32_t key, int tile_bits) {
  return ((key & ((1u << tile_bits) - 1u)) << 16) | (key >> tile_bits);
}
__device__ __forceinline__ uint32_t lower_bound_swapped(const uint32_t* __restrict__ a, uint32_t n, uint32_t x,
                                                        int tile_bits) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (swapped_ord(__ldg(a + mid), tile_bits) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
__global__ void k_ranges_swapped(const uint32_t* __restrict__ keys, uint32_t n_pairs, uint32_t n_keys, int tile_bits,
                                 uint32_t* __restrict__ start, uint32_t* __restrict__ end) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_keys) return;
  const uint32_t o = swapped_ord(k, tile_bits);
  start[k] = lower_bound_swapped(keys, n_pairs, o, tile_bits);
  end[k] = lower_bound_swapped(keys, n_pairs, o + 1, tile_bits);
}

// Forward (K3): one warp per 32x16 half of a 32x32 super-tile and view; lane l owns the
// 2 x 8 pixel block at rows 2(l>>2), +1 and columns 8(l&3) .. +7, the two rows held in the
// halves of packed f32x2 registers. Records of the super-tile list (ascending splat index =
// the reference's per-pixel accumulation order) are staged 32 at a time in the warp's
// shared-memory slice; the staging lane also derives the per-splat ratio c = exp2(2A), a
// "chain-safe" flag and the 32-bit mask of lanes whose block the record's bbox meets. A
// 5-step xor-shuffle 32x32 bit transpose turns those masks into each lane's own list of
// records, so a lane only walks records that touch its block (in list order).
// Along a row the Gaussian is evaluated multiplicatively: with e(k) = E0 + k D + k(k-1) A,
//   g(k+1) = g(k) r(k),  r(k+1) = r(k) c,   g(0) = 2^E0,  r(0) = 2^D,
// i.e. 2 packed FMULs per pixel pair instead of one MUFU.EX2 per pixel; the column mask
// predicates the accumulation, row validity is folded into the amplitude. The chain is used
// when no value in the (8-column aligned) bbox window under/overflows fp32 (the flag);
// otherwise the splat takes the direct MUFU path. Both give amp * exp(e) to a few ulps.
struct __align__(16) StagedRec2 {
  float4 p;  // du_t = (tx0 - u0) - mo_u, dv_t = (ty0 - v0) - mo_v (block-origin offsets), A, B
  float4 q;  // C, amp, c = exp2(2A), chain-safe flag (1/0)
  uint4 m;   // column mask (32 columns), row mask (16 rows), lane mask, -
};

#ifndef GSCT_FWD_SAFE_BATCH
#define GSCT_FWD_SAFE_BATCH 1  // all-chain-safe batches skip the per-record safety branch
#endif
#ifndef GSCT_FWD_STAGE_A1E
#define GSCT_FWD_STAGE_A1E 1  // the staging lane pre-computes the chain step's record terms
#endif
#ifndef GSCT_FWD_PREFLAG
#define GSCT_FWD_PREFLAG 1  // chain-safety flag from the set-up instead of per staged record
#endif

#ifndef GSCT_FWD_UNROLL
#define GSCT_FWD_UNROLL 2  // unroll factor of the per-lane record walk (A/B on 2x4 blocks: 1 -> 3.50, 4 -> 3.15 ms;
                           // current kernel: 1 / 2 / 4 / 8 -> 2.51 / 2.50 / 2.53 / 2.54 ms)
#endif
constexpr int kFwdUnroll = GSCT_FWD_UNROLL;
// Accumulation: {row 0, row 1} per column with predicated packed FMAs (__ffma2_rn, which
// ptxas predicates in place; inline-asm FFMA2 under an `if` got a temporary + predicated MOV
// pairs; scalar FFMAs per row: A/B C2 3.22 vs 2.92 ms).

#ifndef GSCT_FWD_GROUPS
#define GSCT_FWD_GROUPS 2  // records staged per warp batch = 32 x groups (lane balance); A/B
                           // C2 (min blocks 7/8): G1 2.65 ms, G2 2.56, G3 2.98, G4 3.23 -- the
                           // refill logic and registers eat the balance gain beyond 2 groups
#endif
constexpr int kFwdGroups = GSCT_FWD_GROUPS;

// Stages one record (the staging lane's work, see StagedRec2); returns the lane mask.
__device__ __forceinline__ uint32_t stage_record(const RasterRec& r, int tx0, int ty0, StagedRec2* slot) {
  constexpr int kHW = 2 * kTile, kHH = kTile;
  const int u0 = r.urange & 0xFFFF, u1 = r.urange >> 16, v0 = r.vrange & 0xFFFF, v1 = r.vrange >> 16;
  const int c0 = max(u0 - tx0, 0), c1 = min(u1 - tx0, kHW - 1);
  const int r0 = max(v0 - ty0, 0), r1 = min(v1 - ty0, kHH - 1);
  if (c0 > c1 || r0 > r1) return 0u;
  StagedRec2 s;
  const float du_t = (static_cast<float>(tx0) - static_cast<float>(u0)) - r.mo_u;
  const float dv_t = (static_cast<float>(ty0) - static_cast<float>(v0)) - r.mo_v;
  const uint32_t cm = (c1 == 31 ? 0xFFFFFFFFu : ((2u << c1) - 1u)) & ~((1u << c0) - 1u);
  const uint32_t rm = ((2u << r1) - 1u) & ~((1u << r0) - 1u);
  // lane mask: column octets c0/8..c1/8 x row pairs r0/2..r1/2 (lane = 4 * pair + octet)
  const uint32_t octs = ((2u << (c1 >> 3)) - 1u) & ~((1u << (c0 >> 3)) - 1u);
  const uint32_t pairs = (0x11111111u >> (4 * (7 - (r1 >> 1)))) & (0x11111111u << (4 * (r0 >> 1)));
  const uint32_t lanes_rel = pairs * octs;
#if GSCT_FWD_PREFLAG
  // chain safety from the set-up (over the whole aligned bbox, amp's sign bit)
  const bool safe = !signbit(r.amp);
#else
  // chain-safety window: rows r0..r1 x 8-aligned columns
  const bool safe = raster_chain_safe(r.A, r.B, r.C, du_t + static_cast<float>(c0 & ~7),
                                      du_t + static_cast<float>(c1 | 7), dv_t + static_cast<float>(r0 & ~1),
                                      dv_t + static_cast<float>(r1 | 1));
#endif
  s.p = make_float4(du_t, dv_t, r.A, r.B);
  s.q = make_float4(r.C, fabsf(r.amp), ex2_approx(2.f * r.A), safe ? 1.f : 0.f);
#if GSCT_FWD_STAGE_A1E
  // the chain's column-step term A (2 du + 1) at du = du_t + lc is K1 + K2 lc (one FFMA per lane)
  s.m = make_uint4(cm, rm, __float_as_uint(r.A * fmaf(2.f, du_t, 1.f)), __float_as_uint(2.f * r.A));
#else
  s.m = make_uint4(cm, rm, lanes_rel, 0u);
#endif
  *slot = s;
  return lanes_rel;
}

// Batches of 32 x kFwdGroups records: the warp's loop runs max over lanes of the lane's
// record count in the batch, so bigger batches even out the per-lane counts (simulated on
// the C2 lists: lane efficiency 61% at 32 records, 73% at 128, 85% over whole lists).
#ifndef GSCT_FWD_MINB
#define GSCT_FWD_MINB 7  // 72 registers (G=2) without spills
#endif
__global__ void __launch_bounds__(128, GSCT_FWD_MINB) k_raster_fwd4(const RasterRec* __restrict__ rec,
                                                     const uint32_t* __restrict__ vals,
                                                     const uint32_t* __restrict__ start,
                                                     const uint32_t* __restrict__ end, int64_t n, int n_u,
                                                     int n_v, int stiles_u, int n_stiles, int key_stride,
                                                     float* __restrict__ images, int bulk_out, uint32_t vmask, const uint32_t* __restrict__ sched,
    int n_views) {
  constexpr int kHH = kTile;  // half-tile: 32 wide, 16 tall
  constexpr int kBatch = 32 * kFwdGroups;
  __shared__ StagedRec2 s_rec[4][kBatch];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int half, st, view;
  if (sched) {  // longest lists first (k_fwd_sched_*): 1-D grid over (view, super-tile, half)
    const int64_t w = static_cast<int64_t>(blockIdx.x) * 4 + warp;
    if (w >= 2 * static_cast<int64_t>(n_views) * n_stiles) return;
    const uint32_t it = __ldg(sched + (w >> 1));
    view = static_cast<int>(it / static_cast<uint32_t>(n_stiles));
    st = static_cast<int>(it - static_cast<uint32_t>(view) * n_stiles);
    half = 2 * st + static_cast<int>(w & 1);
  } else {
    half = blockIdx.x * 4 + warp;  // 2 halves per super-tile
    if (half >= 2 * n_stiles) return;
    st = half >> 1;
    view = blockIdx.y;
  }
  const int tx0 = (st % stiles_u) * kBinTile;
  const int ty0 = (st / stiles_u) * kBinTile + (half & 1) * kHH;
  if (ty0 >= n_v) return;
  const int lr = 2 * (lane >> 2), lc = 8 * (lane & 3);
  const float flr = static_cast<float>(lr), flc = static_cast<float>(lc);
  const uint32_t key = static_cast<uint32_t>(view) * key_stride + st;
  const uint32_t b = start[key], e = end[key];
  const RasterRec* __restrict__ vrec = rec + static_cast<int64_t>(view) * n;
  StagedRec2* sw = s_rec[warp];
  float2 acc[8];  // per column {row 0, row 1}
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = make_float2(0.f, 0.f);

  // records of the next batch and indices of the one after are prefetched across the
  // current batch's walk (two dependent loads kept off the critical path)
  uint32_t idx_next[kFwdGroups];
  RasterRec recs[kFwdGroups];
#pragma unroll
  for (int g = 0; g < kFwdGroups; ++g) {
    const uint32_t k = b + 32 * g + lane;
    if (k < e) recs[g] = vrec[__ldg(vals + k) & vmask];
    idx_next[g] = k + kBatch < e ? __ldg(vals + k + kBatch) & vmask : 0u;
  }
  for (uint32_t base = b; base < e; base += kBatch) {
    uint32_t todo[kFwdGroups];
    bool my_safe = true;  // every record this lane staged (and some lane walks) is chain-safe
#pragma unroll
    for (int g = 0; g < kFwdGroups; ++g) {
      const uint32_t rel = base + 32 * g + lane < e ? stage_record(recs[g], tx0, ty0, sw + 32 * g + lane) : 0u;
      if (rel) my_safe = my_safe && sw[32 * g + lane].q.w != 0.f;  // the staged flag (this lane's own write)
      todo[g] = warp_transpose32(rel, lane);
    }
    __syncwarp();
#pragma unroll
    for (int g = 0; g < kFwdGroups; ++g) {
      const uint32_t k = base + kBatch + 32 * g + lane;
      if (k < e) recs[g] = vrec[idx_next[g]];
      idx_next[g] = k + kBatch < e ? __ldg(vals + k + kBatch) & vmask : 0u;
    }
    // one flat loop over the lane's records of the whole batch, so lanes do not wait for
    // each other at group boundaries; a batch whose records are all chain-safe (the common
    // case) runs a copy of the loop without the per-record safety branch
    auto walk = [&](auto all_safe) {
#if GSCT_FWD_GROUPS == 1
    uint32_t cur = todo[0];
#pragma unroll kFwdUnroll
    while (cur) {
      const int j = __ffs(cur) - 1;
      cur &= cur - 1u;
#else
    // group words shifted in as they empty (a 64-bit find-first per record cost more)
    uint32_t cur = todo[0];
    int gbase = 0;
#pragma unroll
    for (int g = 1; g < kFwdGroups; ++g)
      if (cur == 0u) {
        cur = todo[g];
        gbase = 32 * g;
      }
    int gnext = gbase / 32 + 1;
#pragma unroll kFwdUnroll
    while (cur) {
      const int j = gbase + __ffs(cur) - 1;
      cur &= cur - 1u;
      if (cur == 0u) {
#pragma unroll
        for (int g = 1; g < kFwdGroups; ++g)
          if (cur == 0u && g >= gnext) {
            cur = todo[g];
            gbase = 32 * g;
            gnext = g + 1;
          }
      }
#endif
      const float4 p = sw[j].p;
      const float4 q = sw[j].q;
#if GSCT_FWD_STAGE_A1E
      const uint4 mm = sw[j].m;
#else
      const uint2 mm = make_uint2(sw[j].m.x, sw[j].m.y);
#endif
      const uint32_t mask = (mm.x >> lc) & 0xFFu;  // this lane's 8 columns
      const uint32_t rows = (mm.y >> lr) & 3u;     // this lane's 2 rows
      const float a0 = (rows & 1u) ? q.y : 0.f, a1 = (rows & 2u) ? q.y : 0.f;
      const float du0 = p.x + flc;
      const float dv0 = p.y + flr;
      const float bdu = p.w * du0, au2 = p.z * du0 * du0;
      const float2 A01 = make_float2(a0, a1);
      const float2 DV2 = make_float2(dv0, dv0 + 1.f);
      // accumulation inside each branch: no merge of the h registers after the branch
      // (a merged h[8] cost ~10 register-pair MOVs per record)
      if (decltype(all_safe)::value || q.w != 0.f) {
        const float2 E0 = __ffma2_rn(DV2, __ffma2_rn(make_float2(q.x, q.x), DV2, make_float2(bdu, bdu)),
                                     make_float2(au2, au2));
#if GSCT_FWD_STAGE_A1E
        const float a1e = fmaf(__uint_as_float(mm.w), flc, __uint_as_float(mm.z));
#else
        const float a1e = p.z * fmaf(2.f, du0, 1.f);
#endif
        const float2 D = __ffma2_rn(make_float2(p.w, p.w), DV2, make_float2(a1e, a1e));
        float2 h = make_float2(ex2_approx(E0.x), ex2_approx(E0.y));
        float2 rr = make_float2(ex2_approx(D.x), ex2_approx(D.y));
        const float2 c2 = make_float2(q.z, q.z);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (mask & (1u << k)) acc[k] = __ffma2_rn(h, A01, acc[k]);
          if (k < 7) h = __fmul2_rn(h, rr);
          if (k < 6) rr = __fmul2_rn(rr, c2);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float duk = du0 + static_cast<float>(k);
          const float bk = p.w * duk, ak = p.z * duk * duk;
          const float2 ek = __ffma2_rn(DV2, __ffma2_rn(make_float2(q.x, q.x), DV2, make_float2(bk, bk)),
                                       make_float2(ak, ak));
          const float2 h = make_float2(ex2_approx(ek.x), ex2_approx(ek.y));
          if (mask & (1u << k)) acc[k] = __ffma2_rn(h, A01, acc[k]);
        }
      }
    }
    };
#if GSCT_FWD_SAFE_BATCH
    if (__all_sync(0xffffffffu, my_safe))
      walk(std::integral_constant<bool, true>{});
    else
#endif
      walk(std::integral_constant<bool, false>{});
    __syncwarp();
  }
  const int px0 = tx0 + lc;
  if (bulk_out && tx0 + 2 * kTile <= n_u && (n_u & 3) == 0) {
    // host-mapped output: the half-tile goes through the warp's (now idle) staging smem and
    // leaves as one 128 B TMA bulk store per row (cp.async.bulk, async proxy); the warp only
    // waits until its smem has been read, not for the PCIe writes, so plain stores' PCIe
    // back-pressure no longer stalls the warp's exit
    float* so = reinterpret_cast<float*>(sw);  // 16 rows x 32 floats = 2 KB of the 3 KB slice
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      so[lr * 32 + lc + k] = acc[k].x;
      so[(lr + 1) * 32 + lc + k] = acc[k].y;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(so));
      for (int rr = 0; rr < kHH && ty0 + rr < n_v; ++rr) {
        float* dst = images + static_cast<int64_t>(view) * n_u * n_v + static_cast<int64_t>(ty0 + rr) * n_u + tx0;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(dst),
                     "r"(sbase + rr * 128u)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    return;
  }
  if (px0 >= n_u) return;
  float acc0[8], acc1[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    acc0[k] = acc[k].x;
    acc1[k] = acc[k].y;
  }
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int py = ty0 + lr + hh;
    if (py >= n_v) continue;
    const float* v = hh ? acc1 : acc0;
    float* rowp = images + static_cast<int64_t>(view) * n_u * n_v + static_cast<int64_t>(py) * n_u;
    if (((n_u & 3) == 0) && px0 + 8 <= n_u) {
      reinterpret_cast<float4*>(rowp + px0)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(rowp + px0)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (px0 + k < n_u) rowp[px0 + k] = v[k];
    }
  }
}

// Longest-first schedule of the forward's warps: (view, super-tile) pairs ordered by view
// group (groups of `vg` consecutive views), then by descending list length class
// (floor(log2(length))) inside the group -- an integer-atomic counting sort; the order inside
// a class is arbitrary: it only decides which warp starts when, never what a warp computes.
// Without it the longest lists (the phantom's centre, in every view) can start in the last
// wave and set the kernel's end. Across all views at once the records of every view are
// re-read from DRAM by tiles spread over the whole kernel (C2: 2.9 GB of DRAM reads instead
// of 1.2), which still costs less than the tail.
__global__ void k_fwd_sched_count(const uint32_t* __restrict__ start, const uint32_t* __restrict__ end, int n_views,
                                  int n_stiles, int key_stride, int vg, uint32_t* __restrict__ cls_cnt,
                                  uint32_t* __restrict__ slot) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(n_views) * n_stiles) return;
  const int v = static_cast<int>(i / n_stiles), t = static_cast<int>(i - static_cast<int64_t>(v) * n_stiles);
  const uint32_t key = static_cast<uint32_t>(v) * key_stride + t;
  const uint32_t len = end[key] - start[key];
  const uint32_t b = static_cast<uint32_t>(v / vg) * 32u + static_cast<uint32_t>(__clz(len | 1u));
  slot[i] = (b << 21) | atomicAdd(cls_cnt + b, 1u);  // ranks < 2^21, buckets < 2^11
}
__global__ void k_fwd_sched_scatter(const uint32_t* __restrict__ cls_cnt, int n_buckets,
                                    const uint32_t* __restrict__ slot, int64_t n, uint32_t* __restrict__ sched) {
  __shared__ uint32_t off[2048];
  __shared__ uint32_t wsum[32];
  // exclusive scan of the bucket counts (<= 2048), 256 threads x 8
  uint32_t v[8], run = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int bi = threadIdx.x * 8 + k;
    v[k] = bi < n_buckets ? cls_cnt[bi] : 0u;
    run += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < 8 ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < 8) wsum[lane] = w;
  }
  __syncthreads();
  uint32_t base = (warp ? wsum[warp - 1] : 0u) + x - run;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    off[threadIdx.x * 8 + k] = base;
    base += v[k];
  }
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t s = slot[i];
  sched[off[s >> 21] + (s & 0x001FFFFFu)] = static_cast<uint32_t>(i);
}

// Lane-per-item backward (K4a). The per-(view, splat) pixel loop is small (hundreds of
// pixels), so warp-cooperative schemes spend more instructions on lane mapping and the
// cross-lane moment reduction than on pixels. Here ONE LANE owns one item end to end: it
// walks the bbox rows, each row as 16-byte aligned float4 chunks of the grad image (VEC=4;
// the <= 3 columns left of u_min / right of u_max in the edge chunks are zeroed and add
// exact zeros), and accumulates per row, in packed f32x2 arithmetic over column pairs,
//   s0 = sum t, s1 = sum t k, s2 = sum t k^2,   t = exp2(A du^2 + B du dv + C dv^2) * w,
// with k = column - round(mean) (du = k - delta, |delta| <= 1/2) and the exponent evaluated
// directly as a quadratic in k (two packed FMAs per pixel pair, no error accumulation).
// Rows fold into the six moments {t, t du, t dv, t du^2, t du dv, t dv^2}. No shuffles,
// no shared memory; every item's result depends only on its own inputs (duplicated splats
// get bit-identical moments). Items are processed in `order` (sorted by bbox shape, see
// k_bwd_shape_keys) so the 32 lanes of a warp walk near-identical loop trip counts.
#ifndef GSCT_LD_NA
#define GSCT_LD_NA 0  // 1: grad-image row loads bypass L1 allocation (A/B: 3.77 vs 3.59 ms, off)
#endif
__device__ __forceinline__ void ldg_v8(const float* p, float (&w)[8]) {
#if GSCT_LD_NA
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#else
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#endif
               : "=f"(w[0]), "=f"(w[1]), "=f"(w[2]), "=f"(w[3]), "=f"(w[4]), "=f"(w[5]), "=f"(w[6]), "=f"(w[7])
               : "l"(p));
}

#ifndef GSCT_BWD_UNROLL
#define GSCT_BWD_UNROLL 1  // chunk-loop unroll (A/B: nested row/chunk loops 3.59 ms vs flat prefetching loop 3.93)
#endif
constexpr int kBwdUnroll = GSCT_BWD_UNROLL;
#ifndef GSCT_LANES_MINB
#define GSCT_LANES_MINB 4  // 64 registers: 32 resident warps per SM
#endif
template <int VEC>
__global__ void __launch_bounds__(256, GSCT_LANES_MINB) k_raster_bwd_lanes(const RasterRec* __restrict__ rec,
                                                          const uint32_t* __restrict__ order,
                                                          int64_t n_items, int64_t n, int n_u, int n_v,
                                                          const float* __restrict__ grad,
                                                          float* __restrict__ moments, double inv_n,
                                                          int view_offset) {
  constexpr int CW = VEC == 8 ? 8 : 4;  // columns per chunk
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n_items) return;
  const int64_t item = order ? static_cast<int64_t>(__ldg(order + t)) : t;
  const RasterRec r = rec[item];
  const int u0 = r.urange & 0xFFFF, u1 = r.urange >> 16;
  const int v0 = r.vrange & 0xFFFF, v1 = r.vrange >> 16;
  const int W = u1 - u0 + 1, H = v1 - v0 + 1;
  float4* dst = reinterpret_cast<float4*>(moments + (static_cast<int64_t>(view_offset) * n + item) * 8);
  if (W <= 0 || H <= 0) {  // culled or degenerate in this view: visibility flag 0 for the tail
    dst[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    dst[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  // view = item / n without a 64-bit integer division (exact: the quotient's fractional
  // part is >= 0.5/n away from an integer, far above the fp64 rounding error)
  const int view = static_cast<int>((static_cast<double>(item) + 0.5) * inv_n);
  const int ua = VEC > 1 ? (u0 & ~(VEC - 1)) : u0;  // aligned first column
  const int lead = u0 - ua;                         // extra columns left of the bbox
  const int ncol = lead + W;                        // columns walked, relative to ua
  const int nch = (ncol + CW - 1) / CW;             // chunks per row
  const float rmu = rintf(r.mo_u);
  const float delta = r.mo_u - rmu;
  const float fcm = static_cast<float>(lead) + rmu;  // k = column - fcm
  const f2_t A2 = f2_pack(r.A, r.A);
  const f2_t TWO2 = f2_pack(2.f, 2.f);
  const f2_t K0 = f2_pack(-fcm, 1.f - fcm);
  const float m2a_d = -2.f * r.A * delta, mb_d = -r.B * delta, a_dd = r.A * delta * delta;
  const float* __restrict__ prow = grad + static_cast<int64_t>(view) * n_u * n_v + static_cast<int64_t>(v0) * n_u + ua;
  float m0 = 0.f, mu = 0.f, mv = 0.f, muu = 0.f, muv = 0.f, mvv = 0.f;
  float dv = -r.mo_v;
  auto load = [&](const float* q, float (&w)[CW], int c) {
    if constexpr (VEC == 8) {
      ldg_v8(q, w);
    } else if constexpr (VEC == 4) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(q));
      w[0] = x.x, w[1] = x.y, w[2] = x.z, w[3] = x.w;
    } else {
#pragma unroll
      for (int k = 0; k < CW; ++k) w[k] = (k == 0 || c + k < ncol) ? __ldg(q + k) : 0.f;
    }
  };
  f2_t BP2, CP2;
  auto row_coeffs = [&]() {
    // E(k) = A k^2 + B' k + C'  (du = k - delta)
    const float bp = fmaf(r.B, dv, m2a_d);
    const float cp = fmaf(dv, fmaf(r.C, dv, mb_d), a_dd);
    BP2 = f2_pack(bp, bp);
    CP2 = f2_pack(cp, cp);
  };
  for (int row = 0; row < H; ++row, prow += n_u, dv += 1.f) {
    row_coeffs();
    f2_t s0 = f2_pack(0.f, 0.f), s1 = s0, s2 = s0;
    f2_t kA = K0;
#pragma unroll kBwdUnroll
    for (int j = 0; j < nch; ++j) {
      float w[CW];
      const int c = CW * j;
      load(prow + c, w, c);
      if (VEC > 1) {
        if (j == 0) {  // columns left of u_min
#pragma unroll
          for (int q = 0; q < CW - 1; ++q)
            if (q < lead) w[q] = 0.f;
        }
        if (j == nch - 1) {  // columns right of u_max
#pragma unroll
          for (int q = 1; q < CW; ++q)
            if (c + q >= ncol) w[q] = 0.f;
        }
      }
#pragma unroll
      for (int h = 0; h < CW / 2; ++h) {
        const f2_t e = f2_fma(f2_fma(A2, kA, BP2), kA, CP2);
        float e0, e1;
        f2_unpack(e, e0, e1);
        const f2_t tt = f2_mul(f2_pack(ex2_approx(e0), ex2_approx(e1)), f2_pack(w[2 * h], w[2 * h + 1]));
        s0 = f2_add(s0, tt);
        const f2_t tk = f2_mul(tt, kA);
        s1 = f2_add(s1, tk);
        s2 = f2_fma(tk, kA, s2);
        kA = f2_add(kA, TWO2);
      }
    }
    float t0, t1, t2;
    {
      float a, b;
      f2_unpack(s0, a, b);
      t0 = a + b;
      f2_unpack(s1, a, b);
      t1 = a + b;
      f2_unpack(s2, a, b);
      t2 = a + b;
    }
    // sum t du = t1 - delta t0;  sum t du^2 = t2 - 2 delta t1 + delta^2 t0
    const float su = fmaf(-delta, t0, t1);
    const float suu = fmaf(delta, fmaf(delta, t0, -2.f * t1), t2);
    m0 += t0;
    mu += su;
    mv = fmaf(dv, t0, mv);
    muu += suu;
    muv = fmaf(dv, su, muv);
    mvv = fmaf(dv * dv, t0, mvv);
  }
  // view-major slot (view_offset + view, i) = view_offset * n + item;
  // [m0 mu mv muu muv mvv visible=1 0]
  dst[0] = make_float4(m0, mu, mv, muu);
  dst[1] = make_float4(muv, mvv, 1.f, 0.f);
}

// Chain variant of K4a (the default for 32 B-aligned rows). Same ownership (one lane per
// (view, splat) item, bbox rows walked as 32 B chunks of 8 columns, edge columns zeroed),
// but the exponent along a row is a multiplicative chain over column PAIRS instead of one
// MUFU.EX2 per pixel: with the packed pair g = (2^e(k), 2^e(k+1)),
//   g(k+2) = g(k) r(k),  r(k+2) = r(k) c,  r(k) = 2^(e(k+2) - e(k)),  c = 2^(8A),
// (e(k+2) - e(k) = A (4 du + 4) + 2 B dv is linear in k), so a row costs 4 MUFU for its
// seeds and two packed FMULs per column pair. The per-chunk sums use compile-time column
// offsets (Y0 = sum t, Y1 = sum t k, Y2 = sum t k^2 for k = 0..7 in the chunk), folded into
// the row sums around the centred column k' = k - round(kappa) once per chunk. A record whose
// chain could leave the normal fp32 range over its walked window takes the direct path.
__device__ __forceinline__ bool raster_chain2_safe(float A, float B, float C, float dua, float dub, float dva,
                                                   float dvb) {
  const float emin = fminf(fminf(raster_quad_e(A, B, C, dua, dva), raster_quad_e(A, B, C, dua, dvb)),
                           fminf(raster_quad_e(A, B, C, dub, dva), raster_quad_e(A, B, C, dub, dvb)));
  const float da = A * fmaf(4.f, dua, 4.f), db = A * fmaf(4.f, dub, 4.f);
  const float b2a = 2.f * B * dva, b2b = 2.f * B * dvb;
  const float dmax = fmaxf(fmaxf(fabsf(da + b2a), fabsf(da + b2b)), fmaxf(fabsf(db + b2a), fabsf(db + b2b)));
  return emin > -100.f && dmax < 100.f && A > -12.f;
}

#ifndef GSCT_CHAIN_MINB
#define GSCT_CHAIN_MINB 3
#endif
#ifndef GSCT_CHAIN_UNROLL
#define GSCT_CHAIN_UNROLL 1
#endif
#ifndef GSCT_CHAIN_MINB4_MAX_PX
#define GSCT_CHAIN_MINB4_MAX_PX (1 << 20)  // images up to 1M pixels: the 64-register walk
#endif
constexpr int kChainUnroll = GSCT_CHAIN_UNROLL;

// Row source of the chain walk: a grad-image row in global memory (32 B-aligned chunks,
// ld.global.nc.v8). (A shared-memory tile source -- one CTA per 64x64 region staging its grad
// tile -- was slower: lane-per-item gathers from shared memory bank-conflict.)
struct GlobalRows {
  const float* p;
  int stride;
  __device__ __forceinline__ void load(int off, float (&w)[8]) const { ldg_v8(p + off, w); }
  __device__ __forceinline__ void next() { p += stride; }
};

// One (view, splat) item's pixel walk (K4a arithmetic, see above): rows of `row` starting at
// the walked column ua = u0 - lead; writes the 6 moments + visibility to dst.
template <class Rows>
__device__ __forceinline__ void bwd_walk(const RasterRec& r, int lead, int W, int H, Rows row, float4* dst) {
  const int ncol = lead + W;
  const int nch = (ncol + 7) >> 3;
  // walked column k = 0 .. 8 nch - 1 (absolute ua + k); du = k - kap
  const float kap = static_cast<float>(lead) + r.mo_u;
  const float kr = rintf(kap);
  const float dl = kap - kr;  // du = k' - dl, k' = k - kr
  const float A = r.A, B = r.B, C = r.C;
  const bool safe = raster_chain2_safe(A, B, C, -kap, static_cast<float>(8 * nch + 1) - kap, -r.mo_v,
                                       static_cast<float>(H - 1) - r.mo_v);
  float m0 = 0.f, mu = 0.f, mv = 0.f, muu = 0.f, muv = 0.f, mvv = 0.f;
  float dv = -r.mo_v;
  const f2_t c2 = f2_bc(ex2_approx(8.f * A));
  const f2_t KO0 = f2_pack(0.f, 1.f);
  // edge-column masks of the first and last chunk as packed 0/1 pairs (per item, all rows)
  f2_t MF[4], ML[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const int q0 = 2 * h, q1 = 2 * h + 1, last = 8 * (nch - 1);
    const bool f0 = q0 >= lead && (nch > 1 || q0 < ncol), f1 = q1 >= lead && (nch > 1 || q1 < ncol);
    MF[h] = f2_pack(f0 ? 1.f : 0.f, f1 ? 1.f : 0.f);
    ML[h] = f2_pack(last + q0 < ncol ? 1.f : 0.f, last + q1 < ncol ? 1.f : 0.f);
  }
  for (int rw = 0; rw < H; ++rw, row.next(), dv += 1.f) {
    f2_t X0 = f2_bc(0.f), X1 = X0, X2 = X0;
    if (safe) {
      const float du0 = -kap;
      const float bdv = B * dv, cdv2 = C * dv * dv;
      const float e0 = fmaf(fmaf(A, du0, bdv), du0, cdv2);
      const float e1 = fmaf(fmaf(A, du0 + 1.f, bdv), du0 + 1.f, cdv2);
      const float d0 = fmaf(A, fmaf(4.f, du0, 4.f), 2.f * bdv);
      const float d1 = fmaf(4.f, A, d0);
      f2_t g = f2_pack(ex2_approx(e0), ex2_approx(e1));
      f2_t rr = f2_pack(ex2_approx(d0), ex2_approx(d1));
      // BE = (k'(col 0 of the chunk), k'(col 1)); per chunk, with tt_h the pair (2h, 2h+1):
      //   Y0 = sum_h tt_h, Z = sum_h h tt_h, Q = sum_h h^2 tt_h
      //   sum t k' = BE Y0 + 2 Z,  sum t k'^2 = BE (BE Y0 + 4 Z) + 4 Q
      f2_t BE = f2_add(f2_bc(-kr), KO0);
      // one 8-column chunk; kMask: first / last chunk (edge columns zeroed by the 0/1 pairs)
      auto chunk = [&](int off, const f2_t* M, auto masked) {
        float w[8];
        row.load(off, w);
        f2_t W0 = f2_pack(w[0], w[1]), W1 = f2_pack(w[2], w[3]), W2 = f2_pack(w[4], w[5]),
             W3 = f2_pack(w[6], w[7]);
        if constexpr (decltype(masked)::value) {
          W0 = f2_mul(W0, M[0]), W1 = f2_mul(W1, M[1]), W2 = f2_mul(W2, M[2]), W3 = f2_mul(W3, M[3]);
        }
        const f2_t t0 = f2_mul(g, W0);
        g = f2_mul(g, rr);
        rr = f2_mul(rr, c2);
        const f2_t t1 = f2_mul(g, W1);
        g = f2_mul(g, rr);
        rr = f2_mul(rr, c2);
        const f2_t t2 = f2_mul(g, W2);
        g = f2_mul(g, rr);
        rr = f2_mul(rr, c2);
        const f2_t t3 = f2_mul(g, W3);
        g = f2_mul(g, rr);
        rr = f2_mul(rr, c2);
        const f2_t Y0 = f2_add(f2_add(t0, t1), f2_add(t2, t3));
        const f2_t Z = f2_fma(t3, f2_bc(3.f), f2_fma(t2, f2_bc(2.f), t1));
        const f2_t Q = f2_fma(t3, f2_bc(9.f), f2_fma(t2, f2_bc(4.f), t1));
        X0 = f2_add(X0, Y0);
        X1 = f2_fma(BE, Y0, f2_fma(Z, f2_bc(2.f), X1));
        X2 = f2_fma(BE, f2_fma(Z, f2_bc(4.f), f2_mul(BE, Y0)), f2_fma(Q, f2_bc(4.f), X2));
        BE = f2_add(BE, f2_bc(8.f));
      };
      using yes = std::integral_constant<bool, true>;
      using no = std::integral_constant<bool, false>;
      chunk(0, MF, yes{});
#pragma unroll kChainUnroll
      for (int j = 1; j < nch - 1; ++j) chunk(8 * j, nullptr, no{});
      if (nch > 1) chunk(8 * (nch - 1), ML, yes{});
    } else {
      // direct path: one exp2 per pixel (the quadratic in k' evaluated per column pair)
      float b = -kr;
      const f2_t A2 = f2_bc(A);
      const float bp = fmaf(B, dv, -2.f * A * dl), cp = fmaf(dv, fmaf(C, dv, -B * dl), A * dl * dl);
      const f2_t BP2 = f2_bc(bp), CP2 = f2_bc(cp);
#pragma unroll 1
      for (int j = 0; j < nch; ++j, b += 8.f) {
        float w[8];
        row.load(8 * j, w);
        f2_t kA = f2_add(f2_bc(b), KO0);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          // E(k') = A k'^2 + B' k' + C'  (du = k' - dl)
          const f2_t e = f2_fma(f2_fma(A2, kA, BP2), kA, CP2);
          float e0, e1;
          f2_unpack(e, e0, e1);
          f2_t wp = f2_pack(w[2 * h], w[2 * h + 1]);
          if (j == 0)
            wp = f2_mul(wp, MF[h]);
          else if (j == nch - 1)
            wp = f2_mul(wp, ML[h]);
          const f2_t tt = f2_mul(f2_pack(ex2_approx(e0), ex2_approx(e1)), wp);
          X0 = f2_add(X0, tt);
          const f2_t tk = f2_mul(tt, kA);
          X1 = f2_add(X1, tk);
          X2 = f2_fma(tk, kA, X2);
          kA = f2_add(kA, f2_bc(2.f));
        }
      }
    }
    float t0, t1, t2;
    {
      float a, c;
      f2_unpack(X0, a, c);
      t0 = a + c;
      f2_unpack(X1, a, c);
      t1 = a + c;
      f2_unpack(X2, a, c);
      t2 = a + c;
    }
    // sum t du = t1 - dl t0;  sum t du^2 = t2 - 2 dl t1 + dl^2 t0
    const float su = fmaf(-dl, t0, t1);
    const float suu = fmaf(dl, fmaf(dl, t0, -2.f * t1), t2);
    m0 += t0;
    mu += su;
    mv = fmaf(dv, t0, mv);
    muu += suu;
    muv = fmaf(dv, su, muv);
    mvv = fmaf(dv * dv, t0, mvv);
  }
  dst[0] = make_float4(m0, mu, mv, muu);
  dst[1] = make_float4(muv, mvv, 1.f, 0.f);
}

// MINB: resident CTAs per SM the registers are capped for (3: 80 registers, 4: 64 with a few
// spilled bytes -- A/B: C2 (512^2) 2.365 vs 2.418 ms, C5 (2048^2) 56.1 vs 55.7 ms).
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_raster_bwd_chain(const RasterRec* __restrict__ rec,
                                                                           const uint32_t* __restrict__ order,
                                                                           int64_t n_items, int64_t n, int n_u,
                                                                           int n_v, const float* __restrict__ grad,
                                                                           float* __restrict__ moments, double inv_n,
                                                                           int view_offset) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n_items) return;
  const int64_t item = order ? static_cast<int64_t>(__ldg(order + t)) : t;
  const RasterRec r = rec[item];
  const int u0 = r.urange & 0xFFFF, u1 = r.urange >> 16;
  const int v0 = r.vrange & 0xFFFF, v1 = r.vrange >> 16;
  const int W = u1 - u0 + 1, H = v1 - v0 + 1;
  float4* dst = reinterpret_cast<float4*>(moments + (static_cast<int64_t>(view_offset) * n + item) * 8);
  if (W <= 0 || H <= 0) {
    dst[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    dst[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const int view = static_cast<int>((static_cast<double>(item) + 0.5) * inv_n);
  const int ua = u0 & ~7;
  const GlobalRows rows{grad + static_cast<int64_t>(view) * n_u * n_v + static_cast<int64_t>(v0) * n_u + ua, n_u};
  bwd_walk(r, u0 - ua, W, H, rows, dst);
}

// Spatial walk-order keys for the chain backward: a coarse shape class (chunks per row
// clamped to 4, rows / 4 clamped to 15: near-uniform trip counts in a warp) then the bbox's
// top row and left column, so the 32 lanes of a warp walk items whose rows coincide and whose
// 32 B row chunks share 128 B lines (simulated on C2 records: L1 wavefronts per row-chunk load
// 28.7 -> 7.9 at near-equal trip-count uniformity; the top row must be exact, the column can be
// coarse: 24 key bits at C2 and C5). Layouts as k_bwd_shape_keys (view-major or shape-major);
// pos = (v0 >> vs) << ub | (u0 >> us).
#ifndef GSCT_BWD_KEY24
#define GSCT_BWD_KEY24 1  // 1: 6-bit shape class, 24-bit keys at C2/C5; 0: 8-bit class, 32-bit keys
#endif
constexpr int kShape2Bits = GSCT_BWD_KEY24 ? 6 : 8;
__global__ void k_bwd_spatial_keys(const RasterRec* __restrict__ rec, int64_t n_items, int64_t n, int vs, int us,
                                   int ub, int pos_bits, int view_bits, int view_major, uint32_t* __restrict__ keys,
                                   uint32_t* __restrict__ vals) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const RasterRec r = rec[i];
  const int u0 = r.urange & 0xFFFF, u1 = r.urange >> 16;
  const int v0 = r.vrange & 0xFFFF, v1 = r.vrange >> 16;
  const int W = u1 - u0 + 1, H = v1 - v0 + 1;
  const uint32_t view = static_cast<uint32_t>(i / n);
  const int sp_bits = kShape2Bits + pos_bits;
  uint32_t key = view_major ? (view << sp_bits) | ((1u << sp_bits) - 1u)
                            : (sp_bits + view_bits >= 32 ? 0xFFFFFFFFu : (1u << (sp_bits + view_bits)) - 1u);
  if (W > 0 && H > 0) {
    const int nch = ((u0 & 7) + W + 7) >> 3;
    const uint32_t shape = GSCT_BWD_KEY24
                               ? (static_cast<uint32_t>(min(nch, 4) - 1) << 4) | static_cast<uint32_t>(min(H >> 2, 15))
                               : (static_cast<uint32_t>(min(nch, 7)) << 5) | static_cast<uint32_t>(min(H >> 1, 31));
    const uint32_t pos = (static_cast<uint32_t>(v0 >> vs) << ub) | static_cast<uint32_t>(u0 >> us);
    key = view_major ? (view << sp_bits) | (shape << pos_bits) | pos
                     : (shape << (view_bits + pos_bits)) | (view << pos_bits) | pos;
  }
  keys[i] = key;
  vals[i] = static_cast<uint32_t>(i);
}

// Bbox-shape sort keys for the lane-per-item backward: (chunks per row, rows), each clamped
// to 6 bits, so a warp's 32 items have near-identical loop trip counts. Empty items sort
// last. Values = item index (the stable sort keeps index order inside a shape class).
// Walk-order keys, two layouts chosen per call (bwd_view_major):
//   shape-major (shape, view, region): a shape class of all views at a time;
//   view-major (view, shape, region): a warp's lanes walk one image and every view is one
//     contiguous range of the order (so chunked host grad images can share one sort).
// A/B: C2 (512^2 images) view-major 3.44 ms vs 3.55; C5 (2048^2) 72.9 vs 67.7 ms.
// Rejected: dropping the view from the key (16 / 15 bits, 2 radix passes; C2 3.82 / 3.93 ms)
// and coarse-shape row-band orders (3.81 ms).
#ifndef GSCT_REGION_BITS
#define GSCT_REGION_BITS 0  // 0: adaptive (below)
#endif
// shape = chunks per row (5 bits) | rows (6 bits)
constexpr int kShapeBits = 11;
__global__ void k_bwd_shape_keys(const RasterRec* __restrict__ rec, int64_t n_items, int64_t n, int vec,
                                 int region_shift, int region_bits, int view_bits, int view_major,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const RasterRec r = rec[i];
  const int u0 = r.urange & 0xFFFF, u1 = r.urange >> 16;
  const int v0 = r.vrange & 0xFFFF, v1 = r.vrange >> 16;
  const int W = u1 - u0 + 1, H = v1 - v0 + 1;
  const uint32_t view = static_cast<uint32_t>(i / n);
  const int sr_bits = kShapeBits + region_bits;
  // empty items sort last (view-major: last within their own view, so each view's n items
  // stay one contiguous range)
  uint32_t key = view_major ? (view << sr_bits) | ((1u << sr_bits) - 1u) : (1u << (sr_bits + view_bits)) - 1u;
  if (W > 0 && H > 0) {
    const int cw = vec == 8 ? 8 : 4;
    const int lead = vec > 1 ? (u0 & (vec - 1)) : 0;
    const int nch = (lead + W + cw - 1) / cw;
    constexpr int hb = kShapeBits - 5;
    const uint32_t shape = (static_cast<uint32_t>(min(nch, 31)) << hb) | static_cast<uint32_t>(min(H, (1 << hb) - 1));
    const int half = region_bits / 2;
    const uint32_t ru = min(u0 >> region_shift, (1 << half) - 1), rv = min(v0 >> region_shift, (1 << half) - 1);
    const uint32_t region = (rv << half) | ru;
    key = view_major ? (view << sr_bits) | (shape << region_bits) | region
                     : (shape << (view_bits + region_bits)) | (view << region_bits) | region;
  }
  keys[i] = key;
  vals[i] = static_cast<uint32_t>(i);
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

void launch_emit_tile_keys(const RasterRec* rec, const uint32_t* offsets, const uint32_t* counts, int64_t n,
                           int n_views, int ts, int tiles_u, int n_tiles, uint32_t* keys, uint32_t* vt_count,
                           cudaStream_t st) {
  const int64_t items = n * n_views;
  if (items == 0) return;
  k_emit_tile_keys<<<blocks_for(items, 256), 256, 0, st>>>(rec, offsets, counts, n, n_views, tiles_u, n_tiles, ts,
                                                           keys, vt_count);
  count_launch();
}

void launch_ranges_from_counts(const uint32_t* vt_count, int n_views, int n_tiles, int key_stride, uint32_t* start,
                               uint32_t* end, cudaStream_t st) {
  k_ranges_from_counts<<<1, 256, 0, st>>>(vt_count, n_views, n_tiles, key_stride, start, end);
  count_launch();
}

void launch_emit_tile_keys_wide(const RasterRec* rec, const uint32_t* offsets, const uint32_t* counts, int64_t n,
                                int n_views, int ts, int tiles_u, int n_tiles, int shift, uint32_t* keys,
                                uint32_t* vt_count, cudaStream_t st) {
  const int64_t items = n * n_views;
  if (items == 0) return;
  const size_t smem = 2 * static_cast<size_t>(n_tiles) * sizeof(uint32_t);
  k_emit_tile_keys_wide<<<blocks_for(items, kWideItems), 256, smem, st>>>(
      rec, offsets, counts, n, n_views, tiles_u, n_tiles, ts, shift, keys, vt_count);
  count_launch();
}

void launch_ranges_from_counts_wide(const uint32_t* vt_count, int n_views, int n_tiles, int key_stride,
                                    uint32_t* start, uint32_t* end, cudaStream_t st) {
  k_ranges_from_counts_wide<<<1, 1024, 0, st>>>(vt_count, n_views, n_tiles, key_stride, start, end);
  count_launch();
}

void launch_ranges_swapped(const uint32_t* keys, int64_t n_pairs, uint32_t n_keys, int tile_bits, uint32_t* start,
                          uint32_t* end, cudaStream_t st) {
  if (n_keys == 0) return;
  k_ranges_swapped<<<blocks_for(n_keys, 256), 256, 0, st>>>(keys, static_cast<uint32_t>(n_pairs), n_keys, tile_bits,
                                                            start, end);
  count_launch();
}

void launch_ranges(const uint32_t* keys, int64_t n_pairs, uint32_t n_keys, uint32_t* start, uint32_t* end,
                   cudaStream_t st) {
  if (n_keys == 0) return;
  k_ranges<<<blocks_for(n_keys, 256), 256, 0, st>>>(keys, static_cast<uint32_t>(n_pairs), n_keys, start, end);
  count_launch();
}

#ifndef GSCT_BWD_CHAIN
#define GSCT_BWD_CHAIN 1  // chain backward + spatial walk order for 32 B-aligned rows
#endif
#ifndef GSCT_BWD_VEC
#define GSCT_BWD_VEC 8  // widest grad-image row load of the lane-per-item backward (8: 32 B)
#endif
int bwd_vec(int n_u, const float* grad_images) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(grad_images);
  if (GSCT_BWD_VEC >= 8 && n_u % 8 == 0 && a % 32 == 0) return 8;
  if (n_u % 4 == 0 && a % 16 == 0) return 4;
  return 1;
}

#ifndef GSCT_VIEW_MAJOR_MAX_PX
#define GSCT_VIEW_MAJOR_MAX_PX (1 << 20)  // view-major walk order up to 1M-pixel (4 MB) images
#endif
bool bwd_view_major(int n_u, int n_v) { return static_cast<int64_t>(n_u) * n_v <= GSCT_VIEW_MAJOR_MAX_PX; }

bool bwd_chain_applies(int vec) { return GSCT_BWD_CHAIN && vec == 8; }

int launch_bwd_shape_keys(const RasterRec* rec, int64_t n, int n_views, int n_u, int n_v, int vec,
                          uint32_t* keys, uint32_t* vals, cudaStream_t st) {
  const int64_t n_items = n * n_views;
  if (n_items == 0) return kShapeBits;
  int view_bits = 0, region_bits = 0, region_shift = 0;
  const int side = n_u > n_v ? n_u : n_v;
  while ((1 << view_bits) < n_views) ++view_bits;
  // 2^(bits/2) x 2^(bits/2) detector regions: the finest regions of >= 32 px that keep the
  // key within 24 bits (three radix passes). A/B (shape-major): C2 (512^2, 75 views) 6 bits
  // 3.54 ms vs 8 bits 3.60; C5 (2048^2, 8 views) 6 bits 73.5 ms, 10 bits 67.7, 12 bits 66.4;
  // (view-major, C2) 2 / 4 / 6 / 8 bits: 3.63 / 3.55 / 3.44 / 3.53 ms
  if (GSCT_BWD_CHAIN && vec == 8) {
    auto bits_of = [](int x) {
      int b = 0;
      while (x > 0) ++b, x >>= 1;
      return b;
    };
    // 24 key bits (three radix passes) when the exact top row and >= 1 column bit fit
    int budget = (GSCT_BWD_KEY24 ? 24 : 32) - kShape2Bits - view_bits;
    if (budget < bits_of(n_v - 1) + 1) budget = 32 - kShape2Bits - view_bits;
    int vs = 0, us = 0;
    while (bits_of((n_v - 1) >> vs) + bits_of((n_u - 1) >> us) > budget) {
      if (bits_of((n_u - 1) >> us) > 2)
        ++us;
      else
        ++vs;
    }
    const int ub = bits_of((n_u - 1) >> us), pos_bits = bits_of((n_v - 1) >> vs) + ub;
    k_bwd_spatial_keys<<<blocks_for(n_items, 256), 256, 0, st>>>(rec, n_items, n, vs, us, ub, pos_bits, view_bits,
                                                                 bwd_view_major(n_u, n_v) ? 1 : 0, keys, vals);
    count_launch();
    return kShape2Bits + view_bits + pos_bits;
  }
  region_bits = GSCT_REGION_BITS;
  if (region_bits == 0) {
    region_bits = 2;
    while (region_bits + 2 <= 24 - kShapeBits - view_bits && (side >> ((region_bits + 2) / 2)) >= 32) region_bits += 2;
  }
  while ((side >> region_shift) > (1 << (region_bits / 2))) ++region_shift;
  k_bwd_shape_keys<<<blocks_for(n_items, 256), 256, 0, st>>>(rec, n_items, n, vec, region_shift, region_bits,
                                                             view_bits, bwd_view_major(n_u, n_v) ? 1 : 0, keys,
                                                             vals);
  count_launch();
  return kShapeBits + view_bits + region_bits;  // key bits
}

void launch_raster_bwd_lanes(const RasterRec* rec, const uint32_t* order, int64_t n, int n_views, int n_u,
                             int n_v, const float* grad_images, float* moments, int view_offset,
                             cudaStream_t st) {
  const int64_t items = n * n_views;
  if (items == 0) return;
  const int vec = bwd_vec(n_u, grad_images);
  if (GSCT_BWD_CHAIN && vec == 8)
    if (static_cast<int64_t>(n_u) * n_v <= GSCT_CHAIN_MINB4_MAX_PX)
      k_raster_bwd_chain<4><<<blocks_for(items, 256), 256, 0, st>>>(rec, order, items, n, n_u, n_v, grad_images,
                                                                     moments, 1.0 / static_cast<double>(n), view_offset);
    else
      k_raster_bwd_chain<GSCT_CHAIN_MINB><<<blocks_for(items, 256), 256, 0, st>>>(
          rec, order, items, n, n_u, n_v, grad_images, moments, 1.0 / static_cast<double>(n), view_offset);
  else if (vec == 8)
    k_raster_bwd_lanes<8><<<blocks_for(items, 256), 256, 0, st>>>(rec, order, items, n, n_u, n_v, grad_images,
                                                                  moments, 1.0 / static_cast<double>(n), view_offset);
  else if (vec == 4)
    k_raster_bwd_lanes<4><<<blocks_for(items, 256), 256, 0, st>>>(rec, order, items, n, n_u, n_v, grad_images,
                                                                  moments, 1.0 / static_cast<double>(n), view_offset);
  else
    k_raster_bwd_lanes<1><<<blocks_for(items, 256), 256, 0, st>>>(rec, order, items, n, n_u, n_v, grad_images,
                                                                  moments, 1.0 / static_cast<double>(n), view_offset);
  count_launch();
}

#ifndef GSCT_FWD_LPT
#define GSCT_FWD_LPT 1  // longest lists first (k_fwd_sched_*; A/B C2 forward 2.52 -> 2.26 ms)
#endif
void launch_fwd_schedule(const uint32_t* start, const uint32_t* end, int n_views, int n_lists, int key_stride,
                         int view_group, uint32_t* ws, cudaStream_t st) {
  const int64_t items = static_cast<int64_t>(n_views) * n_lists;
  if (items == 0) return;
  const int vg = view_group < 1 ? 1 : view_group;
  const int n_buckets = ((n_views + vg - 1) / vg) * 32;  // <= 2048 (callers keep n_views / vg <= 64)
  uint32_t* cnt = ws;
  uint32_t* slot = ws + 2048;
  cudaMemsetAsync(cnt, 0, static_cast<size_t>(n_buckets) * sizeof(uint32_t), st);
  k_fwd_sched_count<<<blocks_for(items, 256), 256, 0, st>>>(start, end, n_views, n_lists, key_stride, vg, cnt, slot);
  count_launch();
  k_fwd_sched_scatter<<<blocks_for(items, 256), 256, 0, st>>>(cnt, n_buckets, slot, items, slot + items);
  count_launch();
}

void launch_raster_fwd_super(const RasterRec* rec, const uint32_t* vals, const uint32_t* start,
                             const uint32_t* end, int64_t n, int n_views, int n_u, int n_v, int stiles_u,
                             int stiles_v, int key_stride, float* images, cudaStream_t st, int bulk_out,
                             uint32_t vmask, uint32_t* sched_ws) {
  if (n_views == 0) return;
  const int n_stiles = stiles_u * stiles_v;
  const int64_t items = static_cast<int64_t>(n_views) * n_stiles;
  uint32_t* sched = nullptr;
  // over all views of the launch (A/B C2: 2.25 ms; per 7-view groups that keep the records
  // L2-resident 2.49; none 2.52). Not for host-mapped images: there the kernel's PCIe stores
  // follow the schedule and scattered host writes cost more than the tail (C2 e2e 8.36 vs 7.87 ms)
#ifndef GSCT_FWD_LPT_DEV_VG
#define GSCT_FWD_LPT_DEV_VG 0  // > 0: device images scheduled longest-first within groups of this many views
#endif
#ifndef GSCT_FWD_LPT_HOST_VG
#define GSCT_FWD_LPT_HOST_VG 0  // > 0: host-mapped images scheduled longest-first within groups of this many views
#endif
  if (GSCT_FWD_LPT && sched_ws && (!bulk_out || GSCT_FWD_LPT_HOST_VG > 0)) {  // sched_ws: 2048 + 2 * items words
    const int vg = bulk_out ? std::min(GSCT_FWD_LPT_HOST_VG, n_views)
                            : (GSCT_FWD_LPT_DEV_VG > 0 ? std::min(GSCT_FWD_LPT_DEV_VG, n_views) : n_views);
    if ((n_views + vg - 1) / vg <= 64) {
      launch_fwd_schedule(start, end, n_views, n_stiles, key_stride, vg, sched_ws, st);
      sched = sched_ws + 2048 + items;
    }
  }
  // one warp per 32x16 half-super-tile (A/B at C2: 2x4-px lane blocks 3.65 ms, 2x8 2.96 ms,
  // 4x8 3.34 ms; CTA-shared staging with block barriers was slower still)
  if (sched) {
    k_raster_fwd4<<<blocks_for(2 * items, 4), 128, 0, st>>>(rec, vals, start, end, n, n_u, n_v, stiles_u, n_stiles,
                                                           key_stride, images, bulk_out, vmask, sched, n_views);
  } else {
    dim3 g4(static_cast<unsigned>((2 * n_stiles + 3) / 4), static_cast<unsigned>(n_views));
    k_raster_fwd4<<<g4, 128, 0, st>>>(rec, vals, start, end, n, n_u, n_v, stiles_u, n_stiles, key_stride, images,
                                      bulk_out, vmask, nullptr, n_views);
  }
  count_launch();
}

}  // namespace gsct_dev
