/* gsct_cuda.h — C ABI of the B200-native FaCT-GS hot paths (libgsct_b200.so).
 *
 * Plain C: pointers, sizes and POD structs only; no C++ or torch types cross this
 * boundary. Every entry point replaces one reference operator of the header-only C++
 * library `gsct` (reference paths below are relative to /root/reference):
 *
 *   gsct_rasterize_fwd  <- gsct::rasterize_view      proj/include/gsct/projector.hpp:308-360
 *   gsct_rasterize_bwd  <- gsct::rasterize_backward  proj/include/gsct/projector.hpp:371-482
 *                          (+ ParamGradients::add over views, proj/include/gsct/core.hpp:152-162)
 *   gsct_voxelize_fwd   <- gsct::voxelize / voxelize_full  proj/include/gsct/voxelizer.hpp:162-206
 *   gsct_voxelize_bwd   <- gsct::voxelize_backward    proj/include/gsct/voxelizer.hpp:214-263
 *   gsct_debug_project  <- gsct::project_cloud        proj/include/gsct/projector.hpp:292-303
 *   gsct_debug_tile_pairs <- gsct::bin_tiles          proj/include/gsct/projector.hpp:266-286
 *   gsct_debug_fwd_bins <- gsct::bin_tiles (tile 32)  the forward's own super-tile lists
 *   gsct_debug_voxel_boxes <- detail::prepare_voxel_splats proj/include/gsct/voxelizer.hpp:145-155
 *   gsct_host_*         <- harness/utility functions (rng.hpp, bench.hpp, synthetic.hpp,
 *                          voxelizer.hpp:76-93 sample_subvolume, projector.hpp:29-43 view_frame)
 *
 * Semantics follow the reference: per pixel / voxel, splats accumulate in ascending splat
 * index (projector.hpp:305-307, voxelizer.hpp:159-161); backward gradients are owned per
 * splat and reduced in a fixed order, so every result is bit-stable run to run; culled and
 * degenerate splats are counted, not errors. Invalid input returns GSCT_ERR_CONTRACT with
 * the reference's message (gsct::contract_error, common.hpp:15-31), naming the lowest
 * offending splat index for non-finite parameters or zero quaternions (core.hpp:86-90).
 *
 * Numerics: per-splat set-up (activation, covariance, projection, line-integral factor,
 * dilation, conic, integer bounding boxes, tile/brick keys, chain rule) runs in fp64 in the
 * reference's operation order, so boxes and keys are bit-exact; per-pair work (exp of the
 * quadratic form, accumulation) is fp32. Images and volumes are fp32; gradients fp64.
 *
 * Layouts: cloud arrays are the reference's AoS doubles (GaussianCloud vectors):
 *   pos[3N], log_scale[3N], quat[4N] (w,x,y,z), raw_density[N].
 * Images: [n_views][n_v][n_u] (u fastest, core.hpp:237). Volumes: x fastest, then y, z
 * (core.hpp:300-302). Pointers flagged GSCT_HOST are copied through the context's pinned
 * staging; GSCT_DEVICE pointers are used in place (device-resident fast path).
 */
#ifndef GSCT_CUDA_H
#define GSCT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSCT_ABI_VERSION 2

enum gsct_status {
  GSCT_OK = 0,
  GSCT_ERR_CONTRACT = 1, /* maps to gsct::contract_error */
  GSCT_ERR_CUDA = 2,
  GSCT_ERR_OOM = 3,
  GSCT_ERR_PARSE = 4     /* maps to gsct::parse_error; the message ends "(byte offset N)" */
};

/* GSCT_HOST_ZEROED (gradient outputs only): host buffers the caller has zero-filled, so a call
 * whose gradients are sparse (gsct_voxelize_bwd over a sub-region: only the splats whose box
 * meets it have entries) transfers and writes only those splats' rows; elsewhere = GSCT_HOST. */
enum gsct_location { GSCT_HOST = 0, GSCT_DEVICE = 1, GSCT_HOST_ZEROED = 2 };

typedef struct gsct_ctx_s* gsct_ctx;
typedef struct gsct_group_s* gsct_group;

/* ScanGeometry minus the angle list (core.hpp:203-222). */
typedef struct {
  int cone; /* 0 parallel, 1 cone (BeamMode) */
  int n_u, n_v;
  double s_u, s_v;
  double source_to_origin, origin_to_detector;
} gsct_geometry;

/* RasterSettings (projector.hpp:64-71). bounding: 0 rect_density_aware, 1 square. */
typedef struct {
  double tau_cut, sigma_cap, dilation_px2;
  int tile_size, dilate, bounding;
} gsct_raster_settings;

/* VoxelSettings (voxelizer.hpp:99-102). */
typedef struct {
  double tau_cut, sigma_cap;
} gsct_voxel_settings;

/* The grid bounding boxes are computed in: a GridRegion's dims/spacing/origin
 * (voxelizer.hpp:43-71; origin = world centre of voxel (0,0,0)). */
typedef struct {
  int dims[3];
  double spacing;
  double origin[3];
} gsct_grid;

/* Sub-box [lo, hi) of the grid that a call produces (z-slab sharding). NULL = whole grid.
 * Boxes stay in grid coordinates and are clipped, so slabs tile the full-grid result. */
typedef struct {
  int lo[3], hi[3];
} gsct_window;

/* RenderStats (projector.hpp:73-80); accumulated with += like the reference. */
typedef struct {
  int64_t culled, degenerate, tile_pairs, pixel_pairs;
  double forward_ms, backward_ms;
} gsct_stats;

typedef struct {
  int64_t n;
  const double* pos;
  const double* log_scale;
  const double* quat;
  const double* raw_density;
  int location; /* gsct_location */
} gsct_cloud;

/* ParamGradients (core.hpp:135-150): overwritten (not accumulated) by the call. */
typedef struct {
  double* pos;           /* 3N */
  double* log_scale;     /* 3N */
  double* quat;          /* 4N */
  double* raw_density;   /* N */
  double* pos_grad_norm; /* N */
  uint8_t* visible;      /* N */
  int location;
} gsct_grads;

/* ---- context ---------------------------------------------------------------- */
int gsct_ctx_create(int device, gsct_ctx* out);
void gsct_ctx_destroy(gsct_ctx ctx);
const char* gsct_ctx_last_error(gsct_ctx ctx);
/* Run on an external CUDA stream (cudaStream_t as void*), e.g. torch's current stream. */
int gsct_ctx_set_stream(gsct_ctx ctx, void* stream);
void* gsct_ctx_stream(gsct_ctx ctx);
/* async != 0: calls only enqueue work (no host sync, no *_ms timing); device-side
 * stats/errors are collected by gsct_ctx_synchronize. Default: synchronous (reference). */
int gsct_ctx_set_async(gsct_ctx ctx, int async);
/* save != 0: gsct_rasterize_fwd keeps its per-(view, splat) set-up records and the next
 * gsct_rasterize_bwd called with the same cloud pointers/size, geometry, angles and
 * settings reuses them instead of recomputing (autograd-style saved state). The caller
 * guarantees the cloud contents did not change in between. Default 0: every call
 * recomputes, as the reference does (projector.hpp:393). */
int gsct_ctx_set_save_for_backward(gsct_ctx ctx, int save);
int gsct_ctx_synchronize(gsct_ctx ctx, gsct_stats* stats_accum);
/* Bytes of device workspace currently held (grow-only arena). */
size_t gsct_ctx_workspace_bytes(gsct_ctx ctx);
/* Number of kernels this context has launched (for the bench's gpu_launches claim). */
int64_t gsct_ctx_launch_count(gsct_ctx ctx);
int gsct_abi_version(void);

/* Per-phase device timing (CUDA events on the context stream around each phase's
 * launches; RenderStats-style tracing, projector.hpp:73-80). Off by default. */
enum gsct_phase {
  GSCT_PH_RASTER_SETUP = 0, /* K1: fp64 projection + bbox + record */
  GSCT_PH_RASTER_BIN,       /* K2: scan + key emission + radix sort + tile ranges */
  GSCT_PH_RASTER_FWD,       /* K3: per-tile forward accumulation */
  GSCT_PH_RASTER_BWD,       /* K4a: per-splat backward pixel loop */
  GSCT_PH_RASTER_TAIL,      /* K4b: fp64 chain rule + view sum */
  GSCT_PH_VOXEL_SETUP,      /* K6 */
  GSCT_PH_VOXEL_BIN,        /* brick scan + emission + sort + ranges */
  GSCT_PH_VOXEL_FWD,        /* K7 */
  GSCT_PH_VOXEL_BWD,        /* K8a */
  GSCT_PH_VOXEL_TAIL,       /* K8b */
  GSCT_PH_RASTER_ORDER,     /* K4a walk order: keys + radix sort (split from RASTER_BWD) */
  GSCT_NUM_PHASES
};
int gsct_ctx_set_profiling(gsct_ctx ctx, int on);
/* Synchronizes, returns accumulated milliseconds and launch counts per phase, resets. */
int gsct_ctx_phase_times(gsct_ctx ctx, double ms[GSCT_NUM_PHASES], int64_t counts[GSCT_NUM_PHASES]);

/* On-box throughput microbenchmarks (roofline denominators): kind 0 = MUFU ex2.approx.f32
 * per second, kind 1 = FP32 FFMA per second, over the whole device. */
int gsct_microbench(gsct_ctx ctx, int kind, double* ops_per_second);

/* ---- rasterizer ---------------------------------------------------------------- */
/* Forward projection of n_views views (angles: host array, radians) into
 * images[n_views][n_v][n_u] (fp32). One call == n_views calls of rasterize_view. */
int gsct_rasterize_fwd(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_geometry* geom,
                       const double* angles, int n_views, const gsct_raster_settings* rs,
                       float* images, int images_location, gsct_stats* stats);

/* Backward of the same views: grads = sum over views (ascending view order, fp64) of
 * rasterize_backward(view, grad_images[view]); pos_grad_norm sums the per-view |dL/dmean2d|,
 * visible ORs (exactly ParamGradients::add over the per-view results). */
int gsct_rasterize_bwd(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_geometry* geom,
                       const double* angles, int n_views, const gsct_raster_settings* rs,
                       const float* grad_images, int grad_location, gsct_grads* out,
                       gsct_stats* stats);

/* ---- voxelizer ----------------------------------------------------------------- */
/* volume: window dims (x fastest), fp32. */
int gsct_voxelize_fwd(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_grid* grid,
                      const gsct_window* window, const gsct_voxel_settings* vs, float* volume,
                      int volume_location, gsct_stats* stats);

int gsct_voxelize_bwd(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_grid* grid,
                      const gsct_window* window, const gsct_voxel_settings* vs,
                      const float* grad_volume, int grad_location, gsct_grads* out,
                      gsct_stats* stats);

/* Split backward for z-slab sharding by a caller with its own collectives: per-splat
 * partial sums over the window (moments: device fp64 [10][N]: sum t, sum t*d (3),
 * sum t*d_i*d_j (6; xx,yy,zz,xy,xz,yz), t = exp(-q/2) * w, d in world units; each splat's
 * window sum is formed in fp32, then widened), reduced across ranks by the caller (fp64
 * all-reduce sum), then finished per splat in fp64. With a group attached to the context
 * (gsct_ctx_set_group) gsct_voxelize_bwd does this reduction itself. */
int gsct_voxelize_bwd_moments(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_grid* grid,
                              const gsct_window* window, const gsct_voxel_settings* vs,
                              const float* grad_volume, int grad_location, double* moments_dev);
int gsct_voxelize_bwd_finish(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_grid* grid,
                             const gsct_voxel_settings* vs, const double* moments_dev,
                             gsct_grads* out);

/* ---- multi-GPU: one NCCL communicator per context -------------------
 * Rank 0 makes an id (gsct_group_new_id), the caller distributes its 128 bytes to every
 * rank over its own channel (MPI, torch.distributed, a file), and every rank creates its
 * group on its context's device (collective: all ranks must call) and attaches it. With a
 * group attached:
 *   gsct_rasterize_bwd  -- each rank passes ITS views (e.g. round-robin view shards); the
 *       fp64 per-splat view sums are all-reduced on the context stream before the final
 *       chain rule, so every rank gets (bit-identical) gradients summed over ALL ranks'
 *       views = ParamGradients::add over every view (core.hpp:152-162). A rank with no views
 *       (n_views == 0) still takes part. gsct_rasterize_fwd is unchanged (images stay
 *       rank-local).
 *   gsct_voxelize_fwd   -- window NULL: rank r computes z-slab [r nz/P, (r+1) nz/P) of the
 *       full grid and the slabs are all-gathered, so every rank holds voxelize_full's
 *       volume (slabs tile it bit for bit); window given: that window only, no exchange.
 *   gsct_voxelize_bwd   -- window NULL: rank r walks its z-slab of the (full-grid) grad
 *       volume; window given: that window (ranks pass disjoint windows). The per-splat
 *       moments are all-reduced in fp64 before the fp64 finish; pos_grad_norm is formed
 *       after the reduction (voxelizer.hpp:250-255).
 * All collectives are enqueued on the context stream (no host synchronisation beyond the
 * call's own). NCCL (libnccl.so.2) is loaded at the first gsct_group_* call. */
typedef struct {
  unsigned char bytes[128]; /* ncclUniqueId */
} gsct_group_id;
int gsct_group_new_id(gsct_ctx ctx, gsct_group_id* out);
int gsct_group_create(gsct_ctx ctx, const gsct_group_id* id, int n_ranks, int rank, gsct_group* out);
/* Attach (g != NULL) or detach (NULL) a group; the group's device must be the context's. */
int gsct_ctx_set_group(gsct_ctx ctx, gsct_group g);
int gsct_group_info(gsct_group g, int* rank, int* n_ranks);
void gsct_group_destroy(gsct_group g);

/* ---- next-row operators ----------------------------------------------- */
/* Image loss of the reconstruction loop: total_loss_recon (losses.hpp:613-637) with
 * alpha_tv = 0, i.e. L1 (losses.hpp:28-45) + alpha_ssim * SSIM2D (losses.hpp:214-272) per
 * view. losses[3 * n_views] (host): {l1, ssim loss (1 - mean SSIM), total} per view;
 * grad_images = d total / d rendered (fp32, same [n_views][n_v][n_u] layout as the images,
 * ready for gsct_rasterize_bwd). location applies to rendered, measured and grad_images. */
int gsct_image_loss(gsct_ctx ctx, const float* rendered, const float* measured, int n_views, int n_u,
                    int n_v, double alpha_ssim, float* grad_images, int location, double* losses);

/* Volume-fit loss total_loss_fit (losses.hpp:648-664): L1 + alpha_ssim * SSIM3D (11^3
 * Gaussian window, losses.hpp:275-516) on a volume of dims {nx, ny, nz} (x fastest);
 * out3 (host) = {l1, ssim loss, total}; grad = d total / d rendered (fp32). */
int gsct_volume_loss(gsct_ctx ctx, const float* rendered, const float* target, const int dims[3],
                     double alpha_ssim, float* grad, int location, double* out3);
/* TV3D (losses.hpp:530-595): isotropic forward-difference TV, mean over interior voxels;
 * *value (host) and grad (fp32, same layout). */
int gsct_tv3d(gsct_ctx ctx, const float* volume, const int dims[3], float* grad, int location,
              double* value);

/* Ray-marched line integrals of a voxel volume (raymarch_project, synthetic.hpp:171-232):
 * the synthetic ground-truth generator, trilinear samples at spacing/2 along every pixel ray.
 * volume: fp32, grid dims (x fastest), grid->origin = centre of voxel (0,0,0);
 * images[n_views][n_v][n_u] fp32. */
int gsct_raymarch_project(gsct_ctx ctx, const float* volume, const gsct_grid* grid, int volume_location,
                          const gsct_geometry* geom, const double* angles, int n_views, float* images,
                          int images_location);

/* Adam (optim.hpp:133-182): beta1 0.9, beta2 0.999, eps 1e-15; splats with a non-finite
 * gradient are skipped and counted; raw densities re-projected to >= 0. Parameters (the
 * cloud arrays, updated in place), moments and gradients are device arrays (fp64). The
 * update is bit-identical to the reference's adam_step. */
typedef struct {
  double position, log_scale, rotation, density;
} gsct_learning_rates;
typedef struct {
  double *m_pos, *v_pos;  /* 3N each */
  double *m_ls, *v_ls;    /* 3N */
  double *m_rot, *v_rot;  /* 4N */
  double *m_dens, *v_dens;/* N */
  int64_t step;           /* incremented by the call (OptimState::step) */
  int64_t skipped_updates;/* accumulated (OptimState::skipped_updates) */
} gsct_adam_state;
int gsct_adam_step(gsct_ctx ctx, gsct_cloud* params, gsct_adam_state* state, const gsct_grads* grads,
                   const gsct_learning_rates* lrs);

/* Adaptive density control (optim.hpp:185-317) and its accumulators
 * (accumulate_control_stats, optim.hpp:366-373): the OptimState arrays that track the cloud
 * size besides the Adam moments. Device arrays. */
typedef struct {
  double* grad_norm; /* N: summed |dL/dmean2d| over visible view-steps (accum_grad_norm) */
  double* grad_dir;  /* 3N: summed dL/dposition (accum_grad_dir) */
  int64_t* count;    /* N: visible view-steps (accum_count) */
} gsct_control_accum;
/* std::mt19937_64 engine state of gsct::Rng (rng.hpp:18-69) in libstdc++'s layout: the 312
 * state words then the position p -- the numbers Rng::save_state writes, in order. */
typedef struct {
  uint64_t x[312];
  uint64_t p;
} gsct_rng_state;
/* TrainConfig's adaptive-control fields (optim.hpp:38-41) + OptimState::scene_extent. */
typedef struct {
  double grad_threshold, prune_density, split_scale_fraction, scene_extent;
  int64_t max_gaussians;
} gsct_control_config;
typedef struct {
  int64_t pruned, cloned, split; /* AdaptiveReport (optim.hpp:188-192) */
  int64_t n_next;                /* rows written to the output cloud */
} gsct_adaptive_report;
/* accumulate_control_stats: for every splat with grads->visible set, grad_norm +=
 * pos_grad_norm, grad_dir += grads->pos, count += 1. grads device-resident. */
int gsct_accumulate_control_stats(gsct_ctx ctx, int64_t n, const gsct_grads* grads, gsct_control_accum* acc);
/* adaptive_control: prune, then clone / split in index order under the max_gaussians cap;
 * survivors, clones and split children are spliced in index order into out_cloud /
 * out_state (device arrays of at least `capacity` rows, distinct from the inputs), fresh
 * rows with zero moments; out_acc (capacity rows) is zeroed for the n_next rows; step and
 * skipped_updates carry over. The split children draw 12 engine outputs each from rng
 * (host) in index order; like the reference -- which draws from state.rng and then replaces
 * the state with a copy taken before the draws (optim.hpp:244, 301, 315) -- the caller's
 * engine state is left unchanged. The
 * required capacity is max(n, max_gaussians); a smaller one that the result does not fit
 * is a contract error. Non-finite parameters / zero quaternions are contract errors, as in
 * activate (core.hpp:80-97). */
int gsct_adaptive_control(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_adam_state* state,
                          const gsct_control_accum* acc, const gsct_rng_state* rng,
                          const gsct_control_config* cfg, int64_t capacity, gsct_cloud* out_cloud,
                          gsct_adam_state* out_state, gsct_control_accum* out_acc, gsct_adaptive_report* report);

/* Compressed model (io.hpp:319-425): "FGSC", u32 version 1, u64 count, then 22 bytes per
 * splat = 11 little-endian binary16 (half.hpp) of the ACTIVATED position, scales, unit
 * quaternion (quantize-then-renormalise fixed point) and density. bytes: 16 + 22 N, at
 * `location` (2-byte aligned). *saturated = values clipped to +-65504 (CompressStats); like
 * the reference, a warning goes to stderr when any were. Non-finite parameters / zero
 * quaternions are contract errors (activate). */
int gsct_compress_model(gsct_ctx ctx, const gsct_cloud* cloud, uint8_t* bytes, int location, int64_t* saturated);
/* decompress_model: header errors (truncation, magic, version, size) are GSCT_ERR_PARSE with
 * the reference's messages. out->n must equal the header's count (bytes 8..15, little
 * endian); out arrays (pos, log_scale, quat, raw_density) at out->location. Log-scales of
 * scales floored at 2^-24; unit quaternions (zero -> identity); densities clamped at 0. */
int gsct_decompress_model(gsct_ctx ctx, const uint8_t* bytes, int64_t n_bytes, int location, gsct_cloud* out);

/* ---- parity hooks (bit-exactness checks against the CPU oracle) ------------------ */
/* Per splat for one view: rect[4N] (u_min,u_max,v_min,v_max), flags[N] (bit0 culled,
 * bit1 degenerate), mean2d[2N], conic[4N] (row-major), amplitude[N]; host outputs. */
int gsct_debug_project(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_geometry* geom,
                       double angle, const gsct_raster_settings* rs, int32_t* rect,
                       uint8_t* flags, double* mean2d, double* conic, double* amplitude);
/* The forward's OWN binning (the code gsct_rasterize_fwd runs: 32x32 super-tiles, the
 * packed / key+value plan, view chunks and <= 2^30-pair binning ranges) exported as CSR:
 * offsets[n_views * n_stiles + 1] over (view, super-tile) in view-major, tile row-major
 * order, splats[] the ascending splat list of each. n_stiles = ceil(n_u/32) * ceil(n_v/32).
 * *n_pairs is set; splats written only if capacity suffices. Compare with bin_tiles
 * (projector.hpp:266-286) at tile_size 32. */
int gsct_debug_fwd_bins(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_geometry* geom, const double* angles,
                        int n_views, const gsct_raster_settings* rs, int64_t* offsets, uint32_t* splats,
                        int64_t capacity, int64_t* n_pairs);
/* Sorted (key, value) pairs of the binning of n_views views: key = view*n_tiles + tile,
 * value = splat; *n_pairs is set; arrays written only if capacity suffices. */
int gsct_debug_tile_pairs(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_geometry* geom,
                          const double* angles, int n_views, const gsct_raster_settings* rs,
                          uint32_t* keys, uint32_t* values, int64_t capacity, int64_t* n_pairs);
/* lo[3N], hi[3N] inclusive grid indices (clipped to the window), skip[N]. */
int gsct_debug_voxel_boxes(gsct_ctx ctx, const gsct_cloud* cloud, const gsct_grid* grid,
                           const gsct_window* window, const gsct_voxel_settings* vs,
                           int32_t* lo, int32_t* hi, uint8_t* skip);

/* ---- host-side harness (no GPU needed) ------------------------------------------ */
/* view_frame (projector.hpp:29-43): u[3], v[3], d[3], detector_center[3], source[3], focal. */
void gsct_host_view_frame(const gsct_geometry* geom, double angle, double frame[16]);
/* default_angles / default_geometry (synthetic.hpp:236-271). */
void gsct_host_default_geometry(const int dims[3], double spacing, int n_views, int cone,
                                int n_u, int n_v, gsct_geometry* out, double* angles);
/* Rng (rng.hpp:18-69): mt19937_64 with the reference's uniform/normal mappings. */
void* gsct_host_rng_create(uint64_t seed);
void gsct_host_rng_destroy(void* rng);
double gsct_host_rng_uniform(void* rng, double lo, double hi);
double gsct_host_rng_normal(void* rng);
int64_t gsct_host_rng_uniform_int(void* rng, int64_t n);
void gsct_host_rng_get_state(void* rng, gsct_rng_state* out);
void gsct_host_rng_set_state(void* rng, const gsct_rng_state* in);
/* sample_subvolume (voxelizer.hpp:76-93): writes offset[3], dims[3]; returns 0 or 1 (error). */
int gsct_host_sample_subvolume(const int parent_dims[3], const int sub_dims[3], void* rng,
                               int offset[3], int dims[3]);
/* Seeded clouds written into caller arrays (pos, log_scale, quat, raw):
 *   kind 0: synthetic_cloud (bench.hpp:33-52): p0=half_extent p1=scale p2=anisotropy p3=density
 *   kind 1: random_cloud (tests/oracles.hpp:168-184): p0=pos_range p1=scale_lo p2=scale_hi
 *   kind 2: modified 3D Shepp-Logan phantom cloud: p0=grid side (voxels),
 *           p1=spacing; positions uniform in the outer ellipsoid, 1-NN-like scales. */
int gsct_host_make_cloud(int kind, int64_t count, uint64_t seed, const double* params,
                         double* pos, double* log_scale, double* quat, double* raw);
/* Element conversions of host arrays on the library's host worker pool (the C++ adapter's
 * fp64 <-> fp32 image / volume conversions; GSCT_HOSTIO_THREADS threads, serial below 64k
 * elements): dst[i] = (float)src[i];  dst[i] = scale * (double)src[i]. */
void gsct_host_f64_to_f32(const double* src, float* dst, int64_t n);
void gsct_host_f32_to_f64(const float* src, double* dst, int64_t n, double scale);

#ifdef __cplusplus
}
#endif
#endif /* GSCT_CUDA_H */
