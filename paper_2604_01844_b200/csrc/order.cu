// Hand-written ordering primitives of the hot path (no library sort):
//
//  * exclusive scan of u32 counts (3 kernels: per-block sums, one-CTA scan of the block sums,
//    per-block scan + base), used for the binning offsets and the bucket starts;
//  * the raster backward's walk order (K4a): a counting sort of the (view, splat) items into
//    spatial buckets (shape class, top row, column band), see launch_bwd_walk_order.
//
// The walk order only schedules the items (every item is processed exactly once by one lane,
// whatever its position), so ranks inside a bucket come from integer atomics: the order may
// differ run to run, the gradients never do.
#include <cuda_runtime.h>

#include <cstdint>

#include "gsct_internal.cuh"

namespace gsct_dev {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanPerThread = 8;  // load8 / store8
constexpr int kScanTile = kScanThreads * kScanPerThread;  // 8192 items per block

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// 8 consecutive u32 per thread as one 32 B access (the arrays are 256 B aligned and every
// thread's first index is a multiple of 8); scalar guarded tail
__device__ __forceinline__ void load8(const uint32_t* a, int64_t i, int64_t n, uint32_t (&v)[8]) {
  if (i + 8 <= n) {
    asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(a + i));
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = i + k < n ? a[i + k] : 0u;
  }
}
__device__ __forceinline__ void store8(uint32_t* a, int64_t i, int64_t n, const uint32_t (&v)[8]) {
  if (i + 8 <= n) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a + i), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (i + k < n) a[i + k] = v[k];
  }
}

// Exclusive block scan of one value per thread (1024 threads = 32 warps); returns the
// block total. Ends with a barrier so the shared words can be reused by the next call.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t& excl) {
  __shared__ uint32_t wbase[32];
  __shared__ uint32_t wtotal;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t inc = warp_incl_scan(x, lane);
  if (lane == 31) wbase[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = wbase[lane];
    const uint32_t wi = warp_incl_scan(w, lane);
    wbase[lane] = wi - w;
    if (lane == 31) wtotal = wi;
  }
  __syncthreads();
  excl = wbase[warp] + inc - x;
  const uint32_t total = wtotal;
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_block_sums(const uint32_t* in, int64_t n,
                                                                  uint32_t* __restrict__ sums) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanPerThread;
  uint32_t v[kScanPerThread];
  load8(in, base, n, v);
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) s += v[k];
  uint32_t excl;
  const uint32_t total = block_excl_scan(s, excl);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_sums(uint32_t* __restrict__ sums, int n_blocks) {
  // one CTA: exclusive scan of <= kScanTile block sums, in place
  const int base = threadIdx.x * kScanPerThread;
  uint32_t v[kScanPerThread];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    v[k] = base + k < n_blocks ? sums[base + k] : 0u;
    s += v[k];
  }
  uint32_t excl;
  block_excl_scan(s, excl);
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    if (base + k < n_blocks) sums[base + k] = excl;
    excl += v[k];
  }
}

// in == out allowed (each thread reads its items before the block barriers, then writes them)
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const uint32_t* in, int64_t n,
                                                             const uint32_t* __restrict__ sums, uint32_t* out) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanPerThread;
  uint32_t v[kScanPerThread];
  load8(in, base, n, v);
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) s += v[k];
  uint32_t excl;
  block_excl_scan(s, excl);
  excl += sums[blockIdx.x];
  uint32_t o[kScanPerThread];
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    o[k] = excl;
    excl += v[k];
  }
  store8(out, base, n, o);
}

// ---- backward walk order (buckets: gsct_internal.cuh walk_bucket) ----------------------
__global__ void k_walk_count(const RasterRec* __restrict__ rec, int64_t n_items, int64_t n, WalkLayout L,
                             uint32_t* __restrict__ count, uint2* __restrict__ slot) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const int view = static_cast<int>(i / n);
  const uint2 uv = *reinterpret_cast<const uint2*>(rec + i);
  const uint32_t b = walk_bucket(uv.x, uv.y, view, L);
  slot[i] = make_uint2(b, atomicAdd(count + b, 1u));
}

__global__ void k_walk_scatter(const uint2* __restrict__ slot, int64_t n_items, const uint32_t* __restrict__ start,
                               uint32_t* __restrict__ order) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const uint2 s = slot[i];
  order[start[s.x] + s.y] = static_cast<uint32_t>(i);
}

inline unsigned blocks_for(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

}  // namespace

int64_t scan_workspace_u32(int64_t n) {
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  return nb + (nb + kScanTile - 1) / kScanTile + 2;
}

void launch_exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* block_sums, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb > kScanTile) {  // > 67M items: two-level recursion on the block sums
    k_scan_block_sums<<<static_cast<unsigned>(nb), kScanThreads, 0, st>>>(in, n, block_sums);
    count_launch();
    launch_exclusive_scan_u32(block_sums, block_sums, nb, block_sums + nb, st);
  } else {
    k_scan_block_sums<<<static_cast<unsigned>(nb), kScanThreads, 0, st>>>(in, n, block_sums);
    count_launch();
    k_scan_sums<<<1, kScanThreads, 0, st>>>(block_sums, static_cast<int>(nb));
    count_launch();
  }
  k_scan_apply<<<static_cast<unsigned>(nb), kScanThreads, 0, st>>>(in, n, block_sums, out);
  count_launch();
}

#ifndef GSCT_WALK_CAP_LOG2
#define GSCT_WALK_CAP_LOG2 25  // bucket table of at most 2^this words (rows coarsened beyond; A/B
                               // 2^26 / 2^27: C5 backward 52.8 / 53.2 ms vs 52.5, 1024^2 set-up +
                               // order + backward within +-0.05 ms -- finer rows buy nothing)
#endif
WalkLayout walk_layout(int n_views, int n_u, int n_v) {
  WalkLayout L;
  // column bands (the top row must be exact for shared lines, the column can be coarse); rows
  // exact while the bucket table stays <= 2^25 words. Band width A/B (backward ms): 512^2
  // 64 px 2.348 / 32 px 2.369 / 128 px 2.416; 1024^2 256 px (8 bands) 10.95 / 64 px 11.00 /
  // 32 px 10.88; 2048^2 256 px 55.70 / 128 px 54.99 / 64 px 53.79 / 32 px 52.52
  const int band_px = n_u > 512 ? GSCT_WALK_BAND_PX_WIDE : GSCT_WALK_BAND_PX;
  while ((1 << L.us) < band_px || ((n_u - 1) >> L.us) + 1 > GSCT_WALK_BANDS) ++L.us;
  L.nu = ((n_u - 1) >> L.us) + 1;
  auto total = [&]() { return static_cast<int64_t>(n_views) * L.shapes * (((n_v - 1) >> L.vs) + 1) * L.nu; };
  while (total() > (int64_t(1) << GSCT_WALK_CAP_LOG2) && L.vs < 16) ++L.vs;
  L.nv = ((n_v - 1) >> L.vs) + 1;
  return L;
}

int64_t walk_buckets(const WalkLayout& L, int n_views) {
  return static_cast<int64_t>(n_views) * L.shapes * L.nv * L.nu;
}

void launch_walk_count(const RasterRec* rec, int64_t n, int n_views, const WalkLayout& L, uint32_t* counts,
                       uint2* slots, cudaStream_t st) {
  const int64_t items = n * n_views;
  if (items == 0) return;
  k_walk_count<<<blocks_for(items, 256), 256, 0, st>>>(rec, items, n, L, counts, slots);
  count_launch();
}

void launch_walk_scatter(const uint32_t* counts, uint32_t* starts, int64_t n_buckets, const uint2* slots,
                         int64_t items, uint32_t* block_sums, uint32_t* order, cudaStream_t st) {
  if (items == 0) return;
  launch_exclusive_scan_u32(counts, starts, n_buckets, block_sums, st);
  k_walk_scatter<<<blocks_for(items, 256), 256, 0, st>>>(slots, items, starts, order);
  count_launch();
}

}  // namespace gsct_dev
