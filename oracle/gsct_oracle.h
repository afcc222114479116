/* TEST INFRASTRUCTURE ONLY — CPU restatement (plain C) of the FaCT-GS reference hot
 * path, used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker. Nothing in the product path (paper_2604_01844_b200/) may link or call it.
 *
 * Every function follows the reference C++ line by line, with the arithmetic order of
 * the Eigen-subset shim (oracle/shim/Eigen/Dense: sequential reductions, Eigen cofactor
 * inverse/determinant, Eigen closed-form 3x3 eigenvalues). It is pinned bit-for-bit
 * against the reference itself compiled from /root/reference (oracle/_ref, see
 * tests/test_oracle_vs_ref.py) and against the reference's own known-answer tests
 * (tests/test_oracle_known_answers.py). Single-threaded, fp64 throughout.
 *
 * Layouts: cloud SoA doubles pos[3N], log_scale[3N], quat[4N] (w,x,y,z), raw[N];
 * images u fastest (v*n_u+u); volumes x fastest ((z*ny+y)*nx+x).
 * Return codes: 0 ok, 1 contract error (message via orc_last_error()).
 */
#ifndef GSCT_ORACLE_H
#define GSCT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int cone;           /* BeamMode::cone */
  int n_u, n_v;
  double s_u, s_v;
  double source_to_origin, origin_to_detector;
} orc_geometry;

typedef struct {
  double tau_cut, sigma_cap, dilation_px2;
  int tile_size, dilate, bounding; /* bounding: 0 rect_density_aware, 1 square */
} orc_raster_settings;

typedef struct {
  double tau_cut, sigma_cap;
} orc_voxel_settings;

typedef struct {
  int dims[3];
  double spacing;
  double origin[3];
} orc_region;

typedef struct {
  int64_t culled, degenerate, tile_pairs, pixel_pairs;
} orc_stats;

/* One projected splat (projector.hpp:126-141 SplatProjection + Splat2D). */
typedef struct {
  double mean2d[2];
  double cov2d[4];  /* row-major */
  double conic[4];  /* row-major */
  double amplitude;
  int u_min, u_max, v_min, v_max;
  int culled, degenerate;
} orc_splat2d;

typedef struct {
  double pos[3], scales[3], unit_quat[4], density;
} orc_act;

const char* orc_last_error(void);

int orc_activate(const double* pos, const double* ls, const double* q, const double* raw,
                 int64_t i, orc_act* out);
void orc_covariance(const double scales[3], const double unit_quat[4], double sigma[9]);

/* view_frame (projector.hpp:29-43): u,v,d,det_center,source (3 each), focal. */
void orc_view_frame(const orc_geometry* g, double theta, double frame[16]);

int orc_splat_bbox(double g_peak, const double cov2d[4], const double mean2d[2], double tau,
                   int n_u, int n_v, int rect[4], double sigma_cap, int mode);

/* project_cloud (projector.hpp:292-303) for one view angle. */
int orc_project_cloud(int64_t n, const double* pos, const double* ls, const double* q,
                      const double* raw, const orc_geometry* g, double theta,
                      const orc_raster_settings* rs, orc_splat2d* out);

/* bin_tiles (projector.hpp:266-286) as CSR: tile_offsets[n_tiles+1], tile_splats[pairs].
 * Pass tile_splats == NULL to only count. Returns pair count (>=0). */
int64_t orc_bin_tiles(int64_t n, const orc_splat2d* splats, int n_u, int n_v, int tile_size,
                      int64_t* tile_offsets, int32_t* tile_splats);

int orc_rasterize_view(int64_t n, const double* pos, const double* ls, const double* q,
                       const double* raw, const orc_geometry* g, double theta,
                       const orc_raster_settings* rs, double* image, orc_stats* stats);

/* grads: g_pos[3N], g_ls[3N], g_q[4N], g_raw[N], pos_grad_norm[N], visible[N] */
int orc_rasterize_backward(int64_t n, const double* pos, const double* ls, const double* q,
                           const double* raw, const orc_geometry* g, double theta,
                           const double* grad_image, const orc_raster_settings* rs,
                           double* g_pos, double* g_ls, double* g_q, double* g_raw,
                           double* pos_grad_norm, uint8_t* visible);

/* prepare_voxel_splat (voxelizer.hpp:117-143): lo[3], hi[3], skip, sigma_inv[9] (row-major). */
int orc_prepare_voxel_splats(int64_t n, const double* pos, const double* ls, const double* q,
                             const double* raw, const orc_region* region,
                             const orc_voxel_settings* vs, int32_t* lo, int32_t* hi,
                             uint8_t* skip, double* sigma_inv);

/* Eigen closed-form max eigenvalue of a symmetric 3x3 (row-major). */
double orc_max_eigenvalue_3x3(const double m[9]);

int orc_voxelize(int64_t n, const double* pos, const double* ls, const double* q,
                 const double* raw, const orc_region* region, const orc_voxel_settings* vs,
                 double* volume, orc_stats* stats);

int orc_voxelize_backward(int64_t n, const double* pos, const double* ls, const double* q,
                          const double* raw, const orc_region* region,
                          const double* grad_volume, const orc_voxel_settings* vs,
                          double* g_pos, double* g_ls, double* g_q, double* g_raw,
                          double* pos_grad_norm, uint8_t* visible);

/* covariance_backward (core.hpp:170-191); grad_sigma row-major 3x3. */
void orc_covariance_backward(const double scales[3], const double unit_quat[4],
                             const double raw_quat[4], const double grad_sigma[9],
                             double grad_log_scales[3], double grad_raw_quat[4]);

#ifdef __cplusplus
}
#endif
#endif
