// Internal types and kernel-launch wrappers shared by the CUDA translation units of
// libgsct_b200.so. Nothing here crosses the C ABI (include/gsct_cuda.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "splat_fp64.cuh"

namespace gsct_dev {

constexpr int kTile = 16;       // reference default tile (projector.hpp:67); the raster
                                // kernel is specialised for it, other sizes are rejected
constexpr int kBinTile = 32;   // forward binning granularity (32x32 super-tiles of 4 tiles)
constexpr int kBrick = 8;       // voxel brick edge in x and y
constexpr int kBrickZ = 16;     // voxel brick depth (a brick = 8 x 8 x 16 voxels = one warp)
constexpr float kLog2e = 1.4426950408889634f;

// Device counters written by the set-up kernels (order-independent integer sums).
struct DevStats {
  unsigned long long culled, degenerate, tile_pairs, pixel_pairs;
  unsigned long long error_key;  // min over (splat << 2 | code), ~0 if none
};

// Per (view, splat) raster record, fp32, 32 B. Coordinates are relative to the splat's
// integer bbox corner (computed in fp64, then rounded) so fp32 per-pixel offsets are
// exact-to-rounding at 2048^2 detectors. Exponent coefficients are pre-scaled by log2(e):
//   exp(e) = exp2(A du^2 + B du dv + C dv^2), A=-a/2*log2e, B=-b*log2e, C=-c/2*log2e.
struct __align__(16) RasterRec {
  uint32_t urange;  // u_min | u_max << 16   (empty: u_min > u_max)
  uint32_t vrange;  // v_min | v_max << 16
  float mo_u, mo_v; // mean2d - (u_min, v_min)
  float A, B, C, amp;  // amp's sign bit set: the forward's exp chain is not safe over the
                       // record's aligned bbox (raster_chain_safe) -> direct exp2 path
};
static_assert(sizeof(RasterRec) == 32, "RasterRec must be 32 B");

// Per splat voxel record, fp32, 64 B. lo/hi: inclusive box in grid indices (already
// clipped to the call's window), as exact floats. off = p - (origin + spacing*lo) (fp64,
// rounded). q(d) coefficients pre-scaled by -0.5*log2e; cross terms carry the factor 2:
//   exp(-q/2) = exp2(Q00 dx^2 + Q11 dy^2 + Q22 dz^2 + Q01 dx dy + Q02 dx dz + Q12 dy dz).
struct __align__(16) VoxelRec {
  float lox, loy, loz, rho;
  float hix, hiy, hiz, Q00;
  float offx, offy, offz, Q11;
  float Q22, Q01, Q02, Q12;
};
static_assert(sizeof(VoxelRec) == 64, "VoxelRec must be 64 B");

// Chain safety of a raster record over a window of offsets du in [dua, dub] (8-column
// aligned), dv in [dva, dvb] (row-pair aligned): the multiplicative exp chain of the forward
// (g <- g r, r <- r c) stays finite and normal when no exponent in the window is below -100
// and no per-column step exceeds 100 in magnitude. The exponent A du^2 + B du dv + C dv^2
// is negative semi-definite, so its minimum over a box is at a corner; the step
// A (2 du + 1) + B dv is linear, so its extremes are at corners too -- a flag computed over
// a box holds for every sub-box.
__device__ __forceinline__ float raster_quad_e(float A, float B, float C, float du, float dv) {
  return fmaf(fmaf(A, du, B * dv), du, C * dv * dv);
}
__device__ __forceinline__ bool raster_chain_safe(float A, float B, float C, float dua, float dub, float dva,
                                                  float dvb) {
  const float emin = fminf(fminf(raster_quad_e(A, B, C, dua, dva), raster_quad_e(A, B, C, dua, dvb)),
                           fminf(raster_quad_e(A, B, C, dub, dva), raster_quad_e(A, B, C, dub, dvb)));
  const float da = A * fmaf(2.f, dua, 1.f), db = A * fmaf(2.f, dub, 1.f);
  const float dmax = fmaxf(fmaxf(fabsf(fmaf(B, dva, da)), fabsf(fmaf(B, dvb, da))),
                           fmaxf(fabsf(fmaf(B, dva, db)), fabsf(fmaf(B, dvb, db))));
  return emin > -100.f && dmax < 100.f && A > -25.f;
}

// Walk-order buckets of the raster backward (K4a, order.cu): view-major over a call's views,
// then a coarse bbox shape class (chunks per row 1..4+ x rows / 4; near-uniform loop trip
// counts in a warp), the exact top row (>> vs) and a column band (>> us): the lanes of a warp
// then walk coinciding rows with 32 B chunks in shared 128 B lines. Empty items: the last
// class of their view.
#ifndef GSCT_WALK_HCLASSES
#define GSCT_WALK_HCLASSES 16  // row-count classes per chunk count (H >> GSCT_WALK_HSHIFT, clamped)
#endif
#ifndef GSCT_WALK_HSHIFT
#define GSCT_WALK_HSHIFT 2
#endif
#ifndef GSCT_WALK_BANDS
#define GSCT_WALK_BANDS 64  // at most this many column bands per row
#endif
#ifndef GSCT_WALK_BAND_PX
#define GSCT_WALK_BAND_PX 64  // column band width (pixels, power of two), detectors <= 512 wide
#endif
#ifndef GSCT_WALK_BAND_PX_WIDE
#define GSCT_WALK_BAND_PX_WIDE 32  // ... wider detectors (their top rows are coarsened by the 2^25 cap)
#endif
struct WalkLayout {
  int shapes = 4 * GSCT_WALK_HCLASSES + 1;  // shape classes + the empty class
  int vs = 0, us = 0;
  int nv = 1, nu = 1;  // row / column bands
};
__device__ __forceinline__ uint32_t walk_bucket(uint32_t urange, uint32_t vrange, int view, const WalkLayout& L) {
  const int u0 = urange & 0xFFFF, u1 = urange >> 16;
  const int v0 = vrange & 0xFFFF, v1 = vrange >> 16;
  const int W = u1 - u0 + 1, H = v1 - v0 + 1;
  int shape = L.shapes - 1, pv = 0, pu = 0;
  if (W > 0 && H > 0) {
    const int nch = ((u0 & 7) + W + 7) >> 3;
    shape = (min(nch, 4) - 1) * GSCT_WALK_HCLASSES + min(H >> GSCT_WALK_HSHIFT, GSCT_WALK_HCLASSES - 1);
#ifndef GSCT_WALK_BIG_FIRST
#define GSCT_WALK_BIG_FIRST 1  // largest shape classes first in each view (no long items in the last wave)
#endif
    if (GSCT_WALK_BIG_FIRST) shape = L.shapes - 2 - shape;
    pv = min(v0 >> L.vs, L.nv - 1);
    pu = min(u0 >> L.us, L.nu - 1);
  }
  return (static_cast<uint32_t>(view * L.shapes + shape) * static_cast<uint32_t>(L.nv) + static_cast<uint32_t>(pv)) *
             static_cast<uint32_t>(L.nu) +
         static_cast<uint32_t>(pu);
}
// optional output of the set-up kernel: per item its walk bucket and rank in it
struct WalkOut {
  uint32_t* count = nullptr;  // [buckets], zeroed by the caller
  uint2* slot = nullptr;      // [items of the launch]: (bucket, rank)
  int view_base = 0;          // global view index of the launch's view 0
  WalkLayout L;
};

struct Cloud {
  int64_t n;
  const double* pos;
  const double* ls;
  const double* q;
  const double* raw;
};

struct Window {
  int lo[3], hi[3];  // [lo, hi)
};

// ---- launch wrappers (defined in preprocess.cu / raster.cu / voxel.cu) ----
// pre: structure-of-arrays set-up (pre_store/pre_load); pre_aos: the same, array-of-structs
void launch_splat_prepare(const Cloud& c, PreSplat* pre, PreSplat* pre_aos, DevStats* stats, cudaStream_t st,
                          int64_t i0 = 0, int64_t i1 = -1);  // splats [i0, i1), -1 = n
// view_pairs (optional): per-view 64-bit sums of tile_count, accumulated with atomics
void launch_raster_preprocess(const PreSplat* pre, int64_t n, const Frame* frames_dev, int n_views,
                              const Geo& g, const RSet& rs, int bin_ts, RasterRec* rec,
                              uint32_t* tile_count, DevStats* stats, cudaStream_t st, int64_t i0 = 0,
                              int64_t i1 = -1, unsigned long long* view_pairs = nullptr,
                              const WalkOut* walk = nullptr);
// order.cu: exclusive scan of u32 (in == out allowed); block_sums needs scan_workspace_u32(n) words
int64_t scan_workspace_u32(int64_t n);
void launch_exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* block_sums, cudaStream_t st);
// raster backward walk order by a counting sort into spatial buckets (shape class, top row,
// column band): counts[walk_order_buckets(...)], slots[items], block_sums[scan_workspace_u32(buckets)]
WalkLayout walk_layout(int n_views, int n_u, int n_v);
int64_t walk_buckets(const WalkLayout& L, int n_views);
// buckets + ranks from records (when the set-up did not produce them)
void launch_walk_count(const RasterRec* rec, int64_t n, int n_views, const WalkLayout& L, uint32_t* counts,
                       uint2* slots, cudaStream_t st);
// counts -> bucket starts, then order[start[b] + rank] = item (counts kept: the order can be
// rebuilt from the same slots)
void launch_walk_scatter(const uint32_t* counts, uint32_t* starts, int64_t n_buckets, const uint2* slots,
                         int64_t items, uint32_t* block_sums, uint32_t* order, cudaStream_t st);
// *total += sum of counts[0, n) (64-bit)
void launch_sum_u32(const uint32_t* counts, int64_t n, unsigned long long* total, cudaStream_t st);
// (tail.cu) acc: fp64 [11][N] view sum (g_pos 3, g_sigma 6, g_raw, sum |dL/dmean2d|);
// moments: view-major [n_views][N] x 8 fp32 {t, t du, t dv, t du^2, t du dv, t dv^2,
// visible, 0} covering every view of the call
void launch_raster_tail(const PreSplat* pre_aos, int64_t n, int64_t i0, int64_t i1, const Frame* frames_dev,
                        int n_views, const Geo& g, const RSet& rs, const float* moments, double* acc,
                        uint8_t* visible, cudaStream_t st);  // splats [i0, i1)
void launch_raster_finalize(const Cloud& c, int64_t i0, int64_t i1, const double* acc, double* g_pos,
                            double* g_ls, double* g_q, double* g_raw, double* g_pgn, cudaStream_t st,
                            int bulk_out = 0);  // 1: gradient arrays host-mapped, 16 B aligned
void launch_debug_project(const PreSplat* pre, int64_t n, const Frame* frame_dev, const Geo& g,
                          const RSet& rs, int32_t* rect, uint8_t* flags, double* mean2d,
                          double* conic, double* amplitude, cudaStream_t st);
void launch_voxel_preprocess(const Cloud& c, const VoxGrid& grid, const Window& win,
                             double tau_cut, double sigma_cap, VoxelRec* rec,
                             uint32_t* brick_count, int32_t* lo_out, int32_t* hi_out,
                             uint8_t* skip_out, DevStats* stats, cudaStream_t st);
template <class T>
void launch_voxel_tail(const Cloud& c, const VoxGrid& grid, double tau_cut, double sigma_cap,
                       const T* moments, double* g_pos, double* g_ls, double* g_q,
                       double* g_raw, double* g_pgn, uint8_t* visible, DevStats* stats,
                       cudaStream_t st);
// b[i] = (double)a[i]
void launch_widen_f32(const float* a, double* b, int64_t n, cudaStream_t st);
// sparse gradient rows (GSCT_HOST_ZEROED outputs)
void launch_grad_row_flags(const double* gp, const double* gl, const double* gq, const double* gr, const double* gn,
                           const uint8_t* gv, int64_t n, uint32_t* flag, cudaStream_t st);
void launch_grad_rows(const double* gp, const double* gl, const double* gq, const double* gr, const double* gn,
                      const uint8_t* gv, int64_t n, const uint32_t* flag, const uint32_t* pos, double* rows,
                      uint32_t* idx, uint32_t* count, cudaStream_t st);  // rows: 13 doubles

void launch_emit_tile_pairs(const RasterRec* rec, const uint32_t* offsets,
                            const uint32_t* counts, int64_t n, int n_views, int ts, int tiles_u,
                            int n_tiles, uint32_t* keys, uint32_t* vals, cudaStream_t st);
void launch_ranges(const uint32_t* keys, int64_t n_pairs, uint32_t n_keys, uint32_t* start,
                   uint32_t* end, cudaStream_t st);
// keys = view << tile_bits | tile, sorted by the tile bits only (view order < 2^16 kept)
void launch_ranges_swapped(const uint32_t* keys, int64_t n_pairs, uint32_t n_keys, int tile_bits,
                           uint32_t* start, uint32_t* end, cudaStream_t st);
// forward over 32x32 super-tile lists (keys = view * n_stiles + super-tile)
// Longest-first order of n_views x n_lists lists [start, end) (list (v, t) at key v * key_stride + t)
// inside groups of view_group consecutive views (ceil(n_views / view_group) <= 64): ws needs
// 2048 + 2 * items words; the order (item = v * n_lists + t) lands at ws + 2048 + items.
void launch_fwd_schedule(const uint32_t* start, const uint32_t* end, int n_views, int n_lists, int key_stride,
                         int view_group, uint32_t* ws, cudaStream_t st);
void launch_raster_fwd_super(const RasterRec* rec, const uint32_t* vals, const uint32_t* start,
                             const uint32_t* end, int64_t n, int n_views, int n_u, int n_v, int stiles_u,
                             int stiles_v, int key_stride, float* images, cudaStream_t st, int bulk_out,
                             uint32_t vmask, uint32_t* sched_ws = nullptr);  // 2048 + 2 * views * super-tiles words  // splat = vals[k] & vmask (packed keys)
// packed keys-only binning (tile << 24 | splat) with (view, tile) counts, and its ranges
void launch_emit_tile_keys(const RasterRec* rec, const uint32_t* offsets, const uint32_t* counts, int64_t n,
                           int n_views, int ts, int tiles_u, int n_tiles, uint32_t* keys, uint32_t* vt_count,
                           cudaStream_t st);
void launch_ranges_from_counts(const uint32_t* vt_count, int n_views, int n_tiles, int key_stride, uint32_t* start,
                               uint32_t* end, cudaStream_t st);
// > 256 tiles per view (key = tile << shift | splat, CTA-level shared-memory counts); a CTA
// emits kWideItems consecutive items, so n >= kWideItems keeps it within two views
constexpr int kWideItems = 4096;
constexpr int kWideMinItems = kWideItems;
void launch_emit_tile_keys_wide(const RasterRec* rec, const uint32_t* offsets, const uint32_t* counts, int64_t n,
                                int n_views, int ts, int tiles_u, int n_tiles, int shift, uint32_t* keys,
                                uint32_t* vt_count, cudaStream_t st);
void launch_ranges_from_counts_wide(const uint32_t* vt_count, int n_views, int n_tiles, int key_stride,
                                    uint32_t* start, uint32_t* end, cudaStream_t st);
// lane-per-item backward: shape sort keys, then the pixel walk in `order`
int bwd_vec(int n_u, const float* grad_images);  // 8, 4 or 1 floats per row load
// true when the walk-order keys of an n_u x n_v detector are view-major (each view a
// contiguous range of the order)
bool bwd_view_major(int n_u, int n_v);
// the chain backward (k_raster_bwd_chain + spatial walk order) runs for this row-load width
bool bwd_chain_applies(int vec);
// returns the number of key bits to sort on
int launch_bwd_shape_keys(const RasterRec* rec, int64_t n, int n_views, int n_u, int n_v, int vec,
                          uint32_t* keys, uint32_t* vals, cudaStream_t st);
void launch_raster_bwd_lanes(const RasterRec* rec, const uint32_t* order, int64_t n, int n_views, int n_u,
                             int n_v, const float* grad_images, float* moments, int view_offset,
                             cudaStream_t st);

void launch_emit_brick_pairs(const VoxelRec* rec, const uint32_t* offsets,
                             const uint32_t* counts, int64_t n, const Window& win, int nbx,
                             int nby, uint32_t* keys, uint32_t* vals, cudaStream_t st);
void launch_voxel_fwd(const VoxelRec* rec, const uint32_t* vals, const uint32_t* start,
                      const uint32_t* end, const Window& win, int nbx, int nby, int nbz,
                      float spacing, float* volume, cudaStream_t st, uint32_t* sched_ws = nullptr);
// lane-per-splat voxel backward: row-load width (8 or 1), walk-order keys (returns key
// bits), the pixel walk
int voxel_bwd_vec(const Window& win, const float* grad_volume);
int launch_voxel_lane_keys(const VoxelRec* rec, int64_t n, const Window& win, int vec, uint32_t* keys,
                           uint32_t* vals, cudaStream_t st);
// voxels_per_splat: full-grid voxels / splats (stands in for the box size: lanes per splat)
void launch_voxel_bwd_lanes(const VoxelRec* rec, const uint32_t* order, int64_t n, const Window& win,
                            float spacing, const float* grad_volume, float* moments, cudaStream_t st,
                            double voxels_per_splat);
// (loss.cu) fused L1 + SSIM2D image loss: coef = 3 * n_views * n_out fp32 scratch,
// part_s / part_l1 = per-tile partials (image_loss_partials total), out3[3 * n_views] =
// {l1, ssim loss, total} per view (device), grad = d total / d pred (fp32, device)
void launch_image_loss(const float* pred, const float* targ, int n_views, int nu, int nv, const double* window,
                       double alpha, float* coef, double* part_s, double* part_l1, float* grad, double* out3,
                       cudaStream_t st);
int64_t image_loss_partials(int n_views, int nu, int nv);
// (loss.cu) volume-fit loss L1 + alpha * SSIM3D and TV3D; the scalar sums land at the end of
// the scratch ({sum s, sum |d|} / {sum g}), the caller forms the means
int64_t volume_loss_scratch_doubles(const int dims[3]);
void launch_volume_loss(const float* pred, const float* targ, const int dims[3], const double* window, double alpha,
                        double* scratch, float* grad, double* out3, cudaStream_t st);
int64_t tv3d_scratch_doubles(const int dims[3]);
// (loss.cu) raymarch_project: images[n_views][n_v][n_u] (fp32) of an fp32 volume
void launch_raymarch(const float* vol, const int dims[3], double spacing, const double origin[3], const Frame* frames,
                     const Geo& g, int n_views, float* images, cudaStream_t st);
void launch_tv3d(const float* vol, const int dims[3], double* scratch, float* grad, cudaStream_t st);
// (preprocess.cu) adam_step; mv = {m_pos, v_pos, m_ls, v_ls, m_rot, v_rot, m_dens, v_dens},
// lrs = {position, log_scale, rotation, density}
void launch_adam_step(int64_t n, double* pos, double* ls, double* q, double* raw, double* const* mv,
                      const double* g_pos, const double* g_ls, const double* g_q, const double* g_raw,
                      const double* lrs, double bias1, double bias2, unsigned long long* skipped, cudaStream_t st);

// (control.cu) adaptive control: accumulate_control_stats; classify (activate, max density,
// prune / eligible flags, budget, clone / split, output rows -- small_host (pinned) receives
// {max density bits, first activation error key, survivors, cloned, split}); the mt19937_64
// draws (state_dev = {x[312], p}); the spliced output rows. mv = the 8 Adam moment arrays.
void launch_ctrl_accumulate(int64_t n, const uint8_t* visible, const double* pgn, const double* g_pos,
                            double* acc_norm, double* acc_dir, int64_t* acc_count, cudaStream_t st);
size_t ctrl_scratch_bytes(int64_t n);
cudaError_t launch_ctrl_classify(const Cloud& c, double prune_density, double grad_threshold, double split_below,
                                 int64_t max_gaussians, const double* acc_norm, const int64_t* acc_count,
                                 void* scratch, unsigned long long* small_host, cudaStream_t st);
void launch_mt_generate(unsigned long long* state_dev, unsigned long long* out, int64_t count, cudaStream_t st);
void launch_ctrl_write(const Cloud& c, const double* const* mv_in, const double* acc_dir, void* scratch,
                       const unsigned long long* draws, double log_1p6, double* pos, double* ls, double* q,
                       double* raw, double* const* mv_out, cudaStream_t st);

// (codec.cu) FGSC body: 11 binary16 words per splat; counters = {saturated, error key}
void launch_fgsc_encode(const Cloud& c, uint16_t* body, unsigned long long* counters, cudaStream_t st);
void launch_fgsc_decode(const uint16_t* body, int64_t n, const double* log_table, double* pos, double* ls, double* q,
                        double* raw, cudaStream_t st);

// Launch accounting (gsct_ctx_launch_count).
extern thread_local int64_t* g_launch_counter;
inline void count_launch(int k = 1) {
  if (g_launch_counter) *g_launch_counter += k;
}

}  // namespace gsct_dev
