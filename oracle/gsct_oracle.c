/* TEST INFRASTRUCTURE ONLY — see gsct_oracle.h. CPU restatement of the reference
 * hot path (/root/reference/proj/include/gsct/{core,projector,voxelizer}.hpp).
 * Compile with -O2 -ffp-contract=off (no FMA contraction, no fast-math) so the
 * arithmetic matches the reference built with the Eigen-subset shim bit-for-bit. */
#include "gsct_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(const char* msg, long long idx) {
  if (idx >= 0)
    snprintf(g_err, sizeof g_err, "%s %lld", msg, idx);
  else
    snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

/* ---- fixed-size helpers, row-major storage, Eigen-shim reduction order ---- */
#define M(a, i, j) ((a)[(i)*3 + (j)])

static double dot3(const double* a, const double* b) {
  double acc = a[0] * b[0];
  acc += a[1] * b[1];
  acc += a[2] * b[2];
  return acc;
}
static double norm3(const double* a) { return sqrt(dot3(a, a)); }
static double norm4(const double* a) {
  double acc = a[0] * a[0];
  acc += a[1] * a[1];
  acc += a[2] * a[2];
  acc += a[3] * a[3];
  return sqrt(acc);
}
/* c = a*b, 3x3 */
static void mul33(const double* a, const double* b, double* c) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = M(a, i, 0) * M(b, 0, j);
      acc += M(a, i, 1) * M(b, 1, j);
      acc += M(a, i, 2) * M(b, 2, j);
      t[i * 3 + j] = acc;
    }
  memcpy(c, t, sizeof t);
}
static void mul3v(const double* a, const double* v, double* out) {
  double t[3];
  for (int i = 0; i < 3; ++i) {
    double acc = M(a, i, 0) * v[0];
    acc += M(a, i, 1) * v[1];
    acc += M(a, i, 2) * v[2];
    t[i] = acc;
  }
  memcpy(out, t, sizeof t);
}
/* Determinant.h: det3_helper sums */
static double det3(const double* m) {
  const double h012 = M(m, 0, 0) * (M(m, 1, 1) * M(m, 2, 2) - M(m, 1, 2) * M(m, 2, 1));
  const double h102 = M(m, 0, 1) * (M(m, 1, 0) * M(m, 2, 2) - M(m, 1, 2) * M(m, 2, 0));
  const double h201 = M(m, 0, 2) * (M(m, 1, 0) * M(m, 2, 1) - M(m, 1, 1) * M(m, 2, 0));
  return h012 - h102 + h201;
}
static double cof3(const double* m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return M(m, i1, j1) * M(m, i2, j2) - M(m, i1, j2) * M(m, i2, j1);
}
/* InverseImpl.h compute_inverse<.,.,3> */
static void inv3(const double* m, double* r) {
  const double c00 = cof3(m, 0, 0), c10 = cof3(m, 1, 0), c20 = cof3(m, 2, 0);
  double det = c00 * M(m, 0, 0);
  det += c10 * M(m, 1, 0);
  det += c20 * M(m, 2, 0);
  const double invdet = 1.0 / det;
  double t[9];
  M(t, 1, 0) = cof3(m, 0, 1) * invdet;
  M(t, 1, 1) = cof3(m, 1, 1) * invdet;
  M(t, 2, 0) = cof3(m, 0, 2) * invdet;
  M(t, 1, 2) = cof3(m, 2, 1) * invdet;
  M(t, 2, 1) = cof3(m, 1, 2) * invdet;
  M(t, 2, 2) = cof3(m, 2, 2) * invdet;
  M(t, 0, 0) = c00 * invdet;
  M(t, 0, 1) = c10 * invdet;
  M(t, 0, 2) = c20 * invdet;
  memcpy(r, t, sizeof t);
}
static double det2(const double* m) { return m[0] * m[3] - m[2] * m[1]; }
static void inv2(const double* m, double* r) {
  const double invdet = 1.0 / det2(m);
  double t[4];
  t[0] = m[3] * invdet;
  t[2] = -m[2] * invdet;
  t[1] = -m[1] * invdet;
  t[3] = m[0] * invdet;
  memcpy(r, t, sizeof t);
}
/* c(2x2) = a(2x2) * b(2x2) */
static void mul22(const double* a, const double* b, double* c) {
  double t[4];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      double acc = a[i * 2 + 0] * b[0 * 2 + j];
      acc += a[i * 2 + 1] * b[1 * 2 + j];
      t[i * 2 + j] = acc;
    }
  memcpy(c, t, sizeof t);
}
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* projector.hpp:91-95 */
static double max_eig2(const double* m) {
  const double half_trace = 0.5 * (m[0] + m[3]);
  const double half_gap = 0.5 * (m[0] - m[3]);
  return half_trace + sqrt(half_gap * half_gap + m[1] * m[2]);
}

/* ---- core.hpp ---- */

/* core.hpp:80-97 */
int orc_activate(const double* pos, const double* ls, const double* q, const double* raw,
                 int64_t i, orc_act* out) {
  const double* p = pos + 3 * i;
  const double* l = ls + 3 * i;
  const double* qq = q + 4 * i;
  const double rho = raw[i];
  int fin = isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]) && isfinite(l[0]) &&
            isfinite(l[1]) && isfinite(l[2]) && isfinite(qq[0]) && isfinite(qq[1]) &&
            isfinite(qq[2]) && isfinite(qq[3]) && isfinite(rho);
  if (!fin) return fail("activate: non-finite parameter in splat", (long long)i);
  const double norm = norm4(qq);
  if (!(norm > 0.0)) return fail("activate: zero quaternion in splat", (long long)i);
  for (int k = 0; k < 3; ++k) {
    out->pos[k] = p[k];
    out->scales[k] = exp(l[k]);
  }
  for (int k = 0; k < 4; ++k) out->unit_quat[k] = qq[k] / norm;
  out->density = dmax(rho, 0.0);
  return 0;
}

/* core.hpp:100-107 */
static void rotation_matrix(const double* q, double* R) {
  const double r = q[0], x = q[1], y = q[2], z = q[3];
  M(R, 0, 0) = 1 - 2 * (y * y + z * z);
  M(R, 0, 1) = 2 * (x * y - r * z);
  M(R, 0, 2) = 2 * (x * z + r * y);
  M(R, 1, 0) = 2 * (x * y + r * z);
  M(R, 1, 1) = 1 - 2 * (x * x + z * z);
  M(R, 1, 2) = 2 * (y * z - r * x);
  M(R, 2, 0) = 2 * (x * z - r * y);
  M(R, 2, 1) = 2 * (y * z + r * x);
  M(R, 2, 2) = 1 - 2 * (x * x + y * y);
}

/* core.hpp:111-115: N = R diag(s); Sigma = N N^T */
void orc_covariance(const double scales[3], const double unit_quat[4], double sigma[9]) {
  double R[9], N[9];
  rotation_matrix(unit_quat, R);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M(N, i, j) = M(R, i, j) * scales[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = M(N, i, 0) * M(N, j, 0);
      acc += M(N, i, 1) * M(N, j, 1);
      acc += M(N, i, 2) * M(N, j, 2);
      M(sigma, i, j) = acc;
    }
}

/* core.hpp:170-191 */
void orc_covariance_backward(const double scales[3], const double uq[4], const double raw_quat[4],
                             const double G[9], double g_ls[3], double g_q[4]) {
  double rot[9], n_mat[9], G2[9], grad_n[9], rt_gn[9], grad_rot[9];
  rotation_matrix(uq, rot);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M(n_mat, i, j) = M(rot, i, j) * scales[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M(G2, i, j) = M(G, i, j) + M(G, j, i);
  mul33(G2, n_mat, grad_n);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = M(rot, 0, i) * M(grad_n, 0, j);
      acc += M(rot, 1, i) * M(grad_n, 1, j);
      acc += M(rot, 2, i) * M(grad_n, 2, j);
      M(rt_gn, i, j) = acc;
    }
  for (int k = 0; k < 3; ++k) g_ls[k] = scales[k] * M(rt_gn, k, k);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M(grad_rot, i, j) = M(grad_n, i, j) * scales[j];
  const double r = uq[0], x = uq[1], y = uq[2], z = uq[3];
  const double d_r[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
  const double d_x[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * r, 2 * z, 2 * r, -4 * x};
  const double d_y[9] = {-4 * y, 2 * x, 2 * r, 2 * x, 0, 2 * z, -2 * r, 2 * z, -4 * y};
  const double d_z[9] = {-4 * z, -2 * r, 2 * x, 2 * r, -4 * z, 2 * y, 2 * x, 2 * y, 0};
  const double* dm[4] = {d_r, d_x, d_y, d_z};
  double gu[4];
  for (int k = 0; k < 4; ++k) {
    /* cwiseProduct(...).sum() in column-major storage order */
    double acc = M(grad_rot, 0, 0) * M(dm[k], 0, 0);
    for (int c = 0; c < 3; ++c)
      for (int rr = 0; rr < 3; ++rr) {
        if (c == 0 && rr == 0) continue;
        acc += M(grad_rot, rr, c) * M(dm[k], rr, c);
      }
    gu[k] = acc;
  }
  const double norm = norm4(raw_quat);
  double dd = uq[0] * gu[0];
  dd += uq[1] * gu[1];
  dd += uq[2] * gu[2];
  dd += uq[3] * gu[3];
  for (int k = 0; k < 4; ++k) g_q[k] = (gu[k] - uq[k] * dd) / norm;
}

/* ---- projector.hpp ---- */

/* projector.hpp:29-43 */
void orc_view_frame(const orc_geometry* g, double theta, double f[16]) {
  memset(f, 0, 16 * sizeof(double));
  double* u = f;
  double* v = f + 3;
  double* d = f + 6;
  double* dc = f + 9;
  double* src = f + 12;
  d[0] = cos(theta);
  d[1] = sin(theta);
  d[2] = 0.0;
  u[0] = -sin(theta);
  u[1] = cos(theta);
  u[2] = 0.0;
  v[0] = 0.0;
  v[1] = 0.0;
  v[2] = 1.0;
  if (g->cone) {
    for (int k = 0; k < 3; ++k) {
      src[k] = -g->source_to_origin * d[k];
      dc[k] = g->origin_to_detector * d[k];
    }
    f[15] = g->source_to_origin + g->origin_to_detector;
  }
}

/* projector.hpp:101-117 */
int orc_splat_bbox(double g_peak, const double cov2d[4], const double mean2d[2], double tau,
                   int n_u, int n_v, int rect[4], double sigma_cap, int mode) {
  if (!(g_peak > tau)) return 0;
  const double cap = sigma_cap * sqrt(dmax(max_eig2(cov2d), 0.0));
  double hu = cap, hv = cap;
  if (mode == 0) {
    const double r = sqrt(2.0 * log(g_peak / tau));
    hu = dmin(r * sqrt(dmax(cov2d[0], 0.0)), cap);
    hv = dmin(r * sqrt(dmax(cov2d[3], 0.0)), cap);
  }
  int a = (int)ceil(mean2d[0] - hu), b = (int)floor(mean2d[0] + hu);
  int c = (int)ceil(mean2d[1] - hv), d = (int)floor(mean2d[1] + hv);
  rect[0] = a > 0 ? a : 0;
  rect[1] = b < n_u - 1 ? b : n_u - 1;
  rect[2] = c > 0 ? c : 0;
  rect[3] = d < n_v - 1 ? d : n_v - 1;
  return !(rect[1] < rect[0] || rect[3] < rect[2]);
}

/* projector.hpp:126-141 (the fields the backward pass reuses) */
typedef struct {
  orc_splat2d s;
  double sigma[9], sigma_inv[9], ad[3], beta, mu, k, cov_px[4], density, d_ray[3];
  double t_cam[3], jac[6], dist;
} proj_t;

/* projector.hpp:143-236 */
static void project_full(const double* fr, const orc_geometry* g, const double* position,
                         const double* cov3d, double density, const orc_raster_settings* rs,
                         proj_t* p) {
  const double* fu = fr;
  const double* fv = fr + 3;
  const double* fd = fr + 6;
  const double* fdc = fr + 9;
  const double* fsrc = fr + 12;
  const double focal = fr[15];
  memset(p, 0, sizeof *p);
  memcpy(p->sigma, cov3d, sizeof p->sigma);
  p->density = density;
  p->beta = 1.0;
  p->k = 1.0;
  for (int i = 0; i < 3; ++i) M(p->sigma_inv, i, i) = 1.0;
  p->cov_px[0] = p->cov_px[3] = 1.0;
  p->d_ray[0] = 1.0;
  orc_splat2d* s = &p->s;
  s->cov2d[0] = s->cov2d[3] = 1.0;
  s->conic[0] = s->conic[3] = 1.0;
  s->u_min = 0;
  s->u_max = -1;
  s->v_min = 0;
  s->v_max = -1;
  s->culled = 1;
  s->degenerate = 0;

  const double d3 = det3(cov3d);
  if (!(d3 > 0.0) || !isfinite(d3)) {
    s->degenerate = 1;
    return;
  }
  inv3(cov3d, p->sigma_inv);
  const double cu = 0.5 * (g->n_u - 1);
  const double cv = 0.5 * (g->n_v - 1);
  if (!g->cone) {
    double rel[3], muc[3], mvc[3], tmp[3];
    memcpy(p->d_ray, fd, sizeof p->d_ray);
    for (int k = 0; k < 3; ++k) rel[k] = position[k] - fdc[k];
    s->mean2d[0] = dot3(rel, fu) / g->s_u + cu;
    s->mean2d[1] = dot3(rel, fv) / g->s_v + cv;
    for (int k = 0; k < 3; ++k) {
      muc[k] = fu[k] / g->s_u;
      mvc[k] = fv[k] / g->s_v;
    }
    mul3v(cov3d, muc, tmp);
    p->cov_px[0] = dot3(muc, tmp);
    mul3v(cov3d, mvc, tmp);
    p->cov_px[1] = p->cov_px[2] = dot3(muc, tmp);
    p->cov_px[3] = dot3(mvc, tmp);
  } else {
    double rel[3];
    for (int k = 0; k < 3; ++k) rel[k] = position[k] - fsrc[k];
    p->dist = norm3(rel);
    p->t_cam[0] = dot3(rel, fu);
    p->t_cam[1] = dot3(rel, fv);
    p->t_cam[2] = dot3(rel, fd);
    const double tz = p->t_cam[2];
    if (!(tz > 1e-9 * focal)) {
      s->degenerate = 1;
      return;
    }
    for (int k = 0; k < 3; ++k) p->d_ray[k] = rel[k] / p->dist;
    const double f = focal;
    s->mean2d[0] = f * p->t_cam[0] / (tz * g->s_u) + cu;
    s->mean2d[1] = f * p->t_cam[1] / (tz * g->s_v) + cv;
    double* J = p->jac; /* 2x3 row-major */
    J[0] = f / (g->s_u * tz);
    J[2] = -f * p->t_cam[0] / (g->s_u * tz * tz);
    J[4] = f / (g->s_v * tz);
    J[5] = -f * p->t_cam[1] / (g->s_v * tz * tz);
    double rot[9];
    for (int k = 0; k < 3; ++k) {
      M(rot, 0, k) = fu[k];
      M(rot, 1, k) = fv[k];
      M(rot, 2, k) = fd[k];
    }
    double T[6], A[6];
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = J[i * 3 + 0] * M(rot, 0, j);
        acc += J[i * 3 + 1] * M(rot, 1, j);
        acc += J[i * 3 + 2] * M(rot, 2, j);
        T[i * 3 + j] = acc;
      }
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = T[i * 3 + 0] * M(cov3d, 0, j);
        acc += T[i * 3 + 1] * M(cov3d, 1, j);
        acc += T[i * 3 + 2] * M(cov3d, 2, j);
        A[i * 3 + j] = acc;
      }
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) {
        double acc = A[i * 3 + 0] * T[j * 3 + 0];
        acc += A[i * 3 + 1] * T[j * 3 + 1];
        acc += A[i * 3 + 2] * T[j * 3 + 2];
        p->cov_px[i * 2 + j] = acc;
      }
  }
  mul3v(p->sigma_inv, p->d_ray, p->ad);
  p->beta = dot3(p->d_ray, p->ad);
  if (!(p->beta > 0.0) || !isfinite(p->beta)) {
    s->degenerate = 1;
    return;
  }
  p->mu = sqrt(2.0 * M_PI / p->beta);

  double cr[4];
  memcpy(cr, p->cov_px, sizeof cr);
  if (rs->dilate) {
    cr[0] += rs->dilation_px2;
    cr[3] += rs->dilation_px2;
    const double det_raw = dmax(det2(p->cov_px), 0.0);
    p->k = sqrt(det_raw / det2(cr));
  }
  const double dt2 = det2(cr);
  const double lam_max = max_eig2(cr);
  const double lam_min = dt2 / dmax(lam_max, DBL_MIN);
  if (!(dt2 > 0.0) || !(lam_max / lam_min < 1e12) || !isfinite(dt2)) {
    s->degenerate = 1;
    return;
  }
  memcpy(s->cov2d, cr, sizeof cr);
  s->conic[0] = cr[3] / dt2;
  s->conic[1] = -cr[1] / dt2;
  s->conic[2] = -cr[2] / dt2;
  s->conic[3] = cr[0] / dt2;
  s->amplitude = p->mu * density * p->k;
  int rect[4];
  if (orc_splat_bbox(s->amplitude, s->cov2d, s->mean2d, rs->tau_cut, g->n_u, g->n_v, rect,
                     rs->sigma_cap, rs->bounding)) {
    s->u_min = rect[0];
    s->u_max = rect[1];
    s->v_min = rect[2];
    s->v_max = rect[3];
    s->culled = 0;
  } else {
    s->culled = 1;
  }
}

static int validate_geometry(const orc_geometry* g) {
  if (!(g->n_u >= 1 && g->n_v >= 1)) return fail("ScanGeometry: detector must be at least 1x1", -1);
  if (!(g->s_u > 0.0 && g->s_v > 0.0)) return fail("ScanGeometry: pixel spacing must be positive", -1);
  if (g->cone && !(g->source_to_origin > 0.0 && g->origin_to_detector > 0.0))
    return fail("ScanGeometry: cone distances must be positive", -1);
  return 0;
}

/* projector.hpp:292-303 */
int orc_project_cloud(int64_t n, const double* pos, const double* ls, const double* q,
                      const double* raw, const orc_geometry* g, double theta,
                      const orc_raster_settings* rs, orc_splat2d* out) {
  double fr[16];
  orc_view_frame(g, theta, fr);
  for (int64_t i = 0; i < n; ++i) {
    orc_act act;
    if (orc_activate(pos, ls, q, raw, i, &act)) return 1;
    double sigma[9];
    orc_covariance(act.scales, act.unit_quat, sigma);
    proj_t p;
    project_full(fr, g, act.pos, sigma, act.density, rs, &p);
    out[i] = p.s;
  }
  return 0;
}

/* projector.hpp:266-286 */
int64_t orc_bin_tiles(int64_t n, const orc_splat2d* splats, int n_u, int n_v, int tile_size,
                      int64_t* tile_offsets, int32_t* tile_splats) {
  const int tiles_u = (n_u + tile_size - 1) / tile_size;
  const int tiles_v = (n_v + tile_size - 1) / tile_size;
  const int64_t n_tiles = (int64_t)tiles_u * tiles_v;
  int64_t* counts = (int64_t*)calloc((size_t)n_tiles + 1, sizeof(int64_t));
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      if (!tile_splats) break;
      int64_t acc = 0;
      for (int64_t t = 0; t < n_tiles; ++t) {
        tile_offsets[t] = acc;
        acc += counts[t];
        counts[t] = tile_offsets[t];
      }
      tile_offsets[n_tiles] = acc;
    }
    for (int64_t i = 0; i < n; ++i) {
      const orc_splat2d* s = &splats[i];
      if (s->culled || s->degenerate) continue;
      const int tu0 = s->u_min / tile_size, tu1 = s->u_max / tile_size;
      const int tv0 = s->v_min / tile_size, tv1 = s->v_max / tile_size;
      for (int tv = tv0; tv <= tv1; ++tv)
        for (int tu = tu0; tu <= tu1; ++tu) {
          const int64_t t = (int64_t)tv * tiles_u + tu;
          if (pass == 0)
            counts[t]++;
          else
            tile_splats[counts[t]++] = (int32_t)i;
        }
    }
  }
  int64_t total = 0;
  if (!tile_splats) {
    for (int64_t t = 0; t < n_tiles; ++t) total += counts[t];
    if (tile_offsets) {
      int64_t acc = 0;
      for (int64_t t = 0; t < n_tiles; ++t) {
        tile_offsets[t] = acc;
        acc += counts[t];
      }
      tile_offsets[n_tiles] = acc;
    }
  } else {
    total = tile_offsets[n_tiles];
  }
  free(counts);
  return total;
}

/* projector.hpp:308-360 */
int orc_rasterize_view(int64_t n, const double* pos, const double* ls, const double* q,
                       const double* raw, const orc_geometry* g, double theta,
                       const orc_raster_settings* rs, double* image, orc_stats* stats) {
  if (validate_geometry(g)) return 1;
  if (!isfinite(theta)) return fail("ScanGeometry: non-finite angle", -1);
  if (rs->tile_size < 1) return fail("bin_tiles: tile size must be at least 1", -1);
  orc_splat2d* sp = (orc_splat2d*)malloc(sizeof(orc_splat2d) * (size_t)(n > 0 ? n : 1));
  if (orc_project_cloud(n, pos, ls, q, raw, g, theta, rs, sp)) {
    free(sp);
    return 1;
  }
  const int ts = rs->tile_size;
  const int tiles_u = (g->n_u + ts - 1) / ts, tiles_v = (g->n_v + ts - 1) / ts;
  const int64_t n_tiles = (int64_t)tiles_u * tiles_v;
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_tiles + 1));
  const int64_t pairs = orc_bin_tiles(n, sp, g->n_u, g->n_v, ts, off, NULL);
  int32_t* lists = (int32_t*)malloc(sizeof(int32_t) * (size_t)(pairs > 0 ? pairs : 1));
  orc_bin_tiles(n, sp, g->n_u, g->n_v, ts, off, lists);
  memset(image, 0, sizeof(double) * (size_t)g->n_u * (size_t)g->n_v);
  int64_t evals = 0;
  for (int64_t t = 0; t < n_tiles; ++t) {
    const int tu = (int)(t % tiles_u), tv = (int)(t / tiles_u);
    const int px_u0 = tu * ts, px_v0 = tv * ts;
    const int px_u1 = g->n_u - 1 < px_u0 + ts - 1 ? g->n_u - 1 : px_u0 + ts - 1;
    const int px_v1 = g->n_v - 1 < px_v0 + ts - 1 ? g->n_v - 1 : px_v0 + ts - 1;
    for (int64_t k = off[t]; k < off[t + 1]; ++k) {
      const orc_splat2d* s = &sp[lists[k]];
      const int u0 = px_u0 > s->u_min ? px_u0 : s->u_min;
      const int u1 = px_u1 < s->u_max ? px_u1 : s->u_max;
      const int v0 = px_v0 > s->v_min ? px_v0 : s->v_min;
      const int v1 = px_v1 < s->v_max ? px_v1 : s->v_max;
      const double a = s->conic[0], b = s->conic[1], c = s->conic[3];
      for (int v = v0; v <= v1; ++v) {
        const double dv = v - s->mean2d[1];
        for (int u = u0; u <= u1; ++u) {
          const double du = u - s->mean2d[0];
          const double e = -0.5 * (a * du * du + c * dv * dv) - b * du * dv;
          image[(size_t)v * g->n_u + u] += s->amplitude * exp(e);
        }
        evals += (u1 - u0 + 1);
      }
    }
  }
  if (stats) {
    for (int64_t i = 0; i < n; ++i) {
      stats->culled += sp[i].culled && !sp[i].degenerate;
      stats->degenerate += sp[i].degenerate;
    }
    stats->tile_pairs += pairs;
    stats->pixel_pairs += evals;
  }
  free(lists);
  free(off);
  free(sp);
  return 0;
}

/* projector.hpp:371-482 */
int orc_rasterize_backward(int64_t n, const double* pos, const double* ls, const double* q,
                           const double* raw, const orc_geometry* g, double theta,
                           const double* grad_image, const orc_raster_settings* rs,
                           double* g_pos, double* g_ls, double* g_q, double* g_raw,
                           double* pos_grad_norm, uint8_t* visible) {
  double fr[16];
  orc_view_frame(g, theta, fr);
  memset(g_pos, 0, sizeof(double) * 3 * (size_t)n);
  memset(g_ls, 0, sizeof(double) * 3 * (size_t)n);
  memset(g_q, 0, sizeof(double) * 4 * (size_t)n);
  memset(g_raw, 0, sizeof(double) * (size_t)n);
  memset(pos_grad_norm, 0, sizeof(double) * (size_t)n);
  memset(visible, 0, (size_t)n);
  double cam_rot[9];
  for (int k = 0; k < 3; ++k) {
    M(cam_rot, 0, k) = fr[k];
    M(cam_rot, 1, k) = fr[3 + k];
    M(cam_rot, 2, k) = fr[6 + k];
  }
  for (int64_t i = 0; i < n; ++i) {
    orc_act act;
    if (orc_activate(pos, ls, q, raw, i, &act)) return 1;
    double sigma[9];
    orc_covariance(act.scales, act.unit_quat, sigma);
    proj_t p;
    project_full(fr, g, act.pos, sigma, act.density, rs, &p);
    const orc_splat2d* s = &p.s;
    if (s->culled || s->degenerate) continue;
    visible[i] = 1;

    double g_amp = 0.0, gm[2] = {0.0, 0.0}, gc[4] = {0.0, 0.0, 0.0, 0.0};
    const double a = s->conic[0], b = s->conic[1], c = s->conic[3];
    for (int v = s->v_min; v <= s->v_max; ++v) {
      const double dv = v - s->mean2d[1];
      for (int u = s->u_min; u <= s->u_max; ++u) {
        const double du = u - s->mean2d[0];
        const double e = -0.5 * (a * du * du + c * dv * dv) - b * du * dv;
        const double w = grad_image[(size_t)v * g->n_u + u];
        if (w == 0.0) continue;
        const double expo = exp(e);
        g_amp += expo * w;
        const double ge = s->amplitude * expo * w;
        gm[0] += ge * (a * du + b * dv);
        gm[1] += ge * (b * du + c * dv);
        gc[0] += ge * (-0.5 * du * du);
        gc[1] += ge * (-0.5 * du * dv);
        gc[2] += ge * (-0.5 * dv * du);
        gc[3] += ge * (-0.5 * dv * dv);
      }
    }
    const double g_mu = act.density * p.k * g_amp;
    const double g_rho = p.mu * p.k * g_amp;
    const double g_k = p.mu * act.density * g_amp;

    double negc[4] = {-s->conic[0], -s->conic[1], -s->conic[2], -s->conic[3]};
    double tmp2[4], gcov[4];
    mul22(negc, gc, tmp2);
    mul22(tmp2, s->conic, gcov);
    if (rs->dilate) {
      const double det_raw = det2(p.cov_px);
      if (det_raw > 0.0) {
        double ci[4];
        inv2(p.cov_px, ci);
        const double sc = g_k * (p.k / 2.0);
        for (int k = 0; k < 4; ++k) gcov[k] += sc * (ci[k] - s->conic[k]);
      }
    }
    const double g_beta = -g_mu * p.mu / (2.0 * p.beta);
    double gsig[9];
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) M(gsig, r, cc) = -g_beta * (p.ad[r] * p.ad[cc]);
    double gp[3] = {0.0, 0.0, 0.0};
    if (!g->cone) {
      double mc[6]; /* 3x2 row-major: col0 = u/s_u, col1 = v/s_v */
      for (int k = 0; k < 3; ++k) {
        mc[k * 2 + 0] = fr[k] / g->s_u;
        mc[k * 2 + 1] = fr[3 + k] / g->s_v;
      }
      double A[6];
      for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 2; ++cc) {
          double acc = mc[r * 2 + 0] * gcov[0 * 2 + cc];
          acc += mc[r * 2 + 1] * gcov[1 * 2 + cc];
          A[r * 2 + cc] = acc;
        }
      for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc) {
          double acc = A[r * 2 + 0] * mc[cc * 2 + 0];
          acc += A[r * 2 + 1] * mc[cc * 2 + 1];
          M(gsig, r, cc) += acc;
        }
      for (int k = 0; k < 3; ++k) gp[k] = gm[0] * mc[k * 2 + 0] + gm[1] * mc[k * 2 + 1];
    } else {
      const double* J = p.jac;
      double T[6];
      for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 3; ++j) {
          double acc = J[r * 3 + 0] * M(cam_rot, 0, j);
          acc += J[r * 3 + 1] * M(cam_rot, 1, j);
          acc += J[r * 3 + 2] * M(cam_rot, 2, j);
          T[r * 3 + j] = acc;
        }
      double A[6]; /* 3x2 = T^T gcov */
      for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 2; ++cc) {
          double acc = T[0 * 3 + r] * gcov[0 * 2 + cc];
          acc += T[1 * 3 + r] * gcov[1 * 2 + cc];
          A[r * 2 + cc] = acc;
        }
      for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc) {
          double acc = A[r * 2 + 0] * T[0 * 3 + cc];
          acc += A[r * 2 + 1] * T[1 * 3 + cc];
          M(gsig, r, cc) += acc;
        }
      double G2[4] = {gcov[0] + gcov[0], gcov[1] + gcov[2], gcov[2] + gcov[1], gcov[3] + gcov[3]};
      double C1[6], gT[6], gJ[6];
      for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 3; ++j) {
          double acc = G2[r * 2 + 0] * T[0 * 3 + j];
          acc += G2[r * 2 + 1] * T[1 * 3 + j];
          C1[r * 3 + j] = acc;
        }
      for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 3; ++j) {
          double acc = C1[r * 3 + 0] * M(sigma, 0, j);
          acc += C1[r * 3 + 1] * M(sigma, 1, j);
          acc += C1[r * 3 + 2] * M(sigma, 2, j);
          gT[r * 3 + j] = acc;
        }
      for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 3; ++j) {
          double acc = gT[r * 3 + 0] * M(cam_rot, j, 0);
          acc += gT[r * 3 + 1] * M(cam_rot, j, 1);
          acc += gT[r * 3 + 2] * M(cam_rot, j, 2);
          gJ[r * 3 + j] = acc;
        }
      const double f = fr[15], tz = p.t_cam[2];
      const double su = g->s_u, sv = g->s_v;
      double gt[3];
      for (int k = 0; k < 3; ++k) gt[k] = J[0 * 3 + k] * gm[0] + J[1 * 3 + k] * gm[1];
      gt[0] += gJ[0 * 3 + 2] * (-f / (su * tz * tz));
      gt[1] += gJ[1 * 3 + 2] * (-f / (sv * tz * tz));
      gt[2] += gJ[0 * 3 + 0] * (-f / (su * tz * tz)) +
               gJ[0 * 3 + 2] * (2.0 * f * p.t_cam[0] / (su * tz * tz * tz)) +
               gJ[1 * 3 + 1] * (-f / (sv * tz * tz)) +
               gJ[1 * 3 + 2] * (2.0 * f * p.t_cam[1] / (sv * tz * tz * tz));
      for (int k = 0; k < 3; ++k) {
        double acc = M(cam_rot, 0, k) * gt[0];
        acc += M(cam_rot, 1, k) * gt[1];
        acc += M(cam_rot, 2, k) * gt[2];
        gp[k] = acc;
      }
      double gd[3];
      for (int k = 0; k < 3; ++k) gd[k] = 2.0 * g_beta * p.ad[k];
      const double dd = dot3(p.d_ray, gd);
      for (int k = 0; k < 3; ++k) gp[k] += (gd[k] - p.d_ray[k] * dd) / p.dist;
    }
    for (int k = 0; k < 3; ++k) g_pos[3 * i + k] = gp[k];
    g_raw[i] = raw[i] >= 0.0 ? g_rho : 0.0;
    pos_grad_norm[i] = sqrt(gm[0] * gm[0] + gm[1] * gm[1]);
    orc_covariance_backward(act.scales, act.unit_quat, q + 4 * i, gsig, g_ls + 3 * i, g_q + 4 * i);
  }
  return 0;
}

/* ---- voxelizer.hpp ---- */

/* Eigen direct_selfadjoint_eigenvalues<.,3> (see oracle/shim/Eigen/Dense); returns max. */
double orc_max_eigenvalue_3x3(const double* mat) {
  double trace = M(mat, 0, 0);
  trace += M(mat, 1, 1);
  trace += M(mat, 2, 2);
  const double shift = trace / 3.0;
  double m[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M(m, i, j) = i >= j ? M(mat, i, j) : M(mat, j, i);
  for (int i = 0; i < 3; ++i) M(m, i, i) -= shift;
  /* cwiseAbs().maxCoeff() in column-major order */
  double scale = fabs(M(m, 0, 0));
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) {
      const double v = fabs(M(m, r, c));
      if (v > scale) scale = v;
    }
  if (scale > 0.0)
    for (int k = 0; k < 9; ++k) m[k] /= scale;
  const double s_inv3 = 1.0 / 3.0;
  const double s_sqrt3 = sqrt(3.0);
  const double c0 = M(m, 0, 0) * M(m, 1, 1) * M(m, 2, 2) + 2.0 * M(m, 1, 0) * M(m, 2, 0) * M(m, 2, 1) -
                    M(m, 0, 0) * M(m, 2, 1) * M(m, 2, 1) - M(m, 1, 1) * M(m, 2, 0) * M(m, 2, 0) -
                    M(m, 2, 2) * M(m, 1, 0) * M(m, 1, 0);
  const double c1 = M(m, 0, 0) * M(m, 1, 1) - M(m, 1, 0) * M(m, 1, 0) + M(m, 0, 0) * M(m, 2, 2) -
                    M(m, 2, 0) * M(m, 2, 0) + M(m, 1, 1) * M(m, 2, 2) - M(m, 2, 1) * M(m, 2, 1);
  const double c2 = M(m, 0, 0) + M(m, 1, 1) + M(m, 2, 2);
  const double c2_over_3 = c2 * s_inv3;
  double a_over_3 = (c2 * c2_over_3 - c1) * s_inv3;
  a_over_3 = dmax(a_over_3, 0.0);
  const double half_b = 0.5 * (c0 + c2_over_3 * (2.0 * c2_over_3 * c2_over_3 - c1));
  double qq = a_over_3 * a_over_3 * a_over_3 - half_b * half_b;
  qq = dmax(qq, 0.0);
  const double rho = sqrt(a_over_3);
  const double theta = atan2(sqrt(qq), half_b) * s_inv3;
  const double cos_theta = cos(theta);
  const double sin_theta = sin(theta);
  double e[3];
  e[0] = c2_over_3 - rho * (cos_theta + s_sqrt3 * sin_theta);
  e[1] = c2_over_3 - rho * (cos_theta - s_sqrt3 * sin_theta);
  e[2] = c2_over_3 + 2.0 * rho * cos_theta;
  for (int k = 0; k < 3; ++k) e[k] = e[k] * scale + shift;
  double mx = e[0];
  if (e[1] > mx) mx = e[1];
  if (e[2] > mx) mx = e[2];
  return mx;
}

typedef struct {
  double pos[3], sigma_inv[9], density;
  int lo[3], hi[3], skip;
} vsplat_t;

/* voxelizer.hpp:117-143 */
static void prepare_voxel_splat(const orc_act* act, const double* sigma, const orc_region* rg,
                                const orc_voxel_settings* vs, vsplat_t* out) {
  memset(out, 0, sizeof *out);
  memcpy(out->pos, act->pos, sizeof out->pos);
  out->density = act->density;
  for (int k = 0; k < 3; ++k) {
    M(out->sigma_inv, k, k) = 1.0;
    out->lo[k] = 0;
    out->hi[k] = -1;
  }
  out->skip = 1;
  if (!(act->density > vs->tau_cut)) return;
  const double det = det3(sigma);
  if (!(det > 0.0) || !isfinite(det)) return;
  inv3(sigma, out->sigma_inv);
  const double lam_max = orc_max_eigenvalue_3x3(sigma);
  const double cap = vs->sigma_cap * sqrt(dmax(lam_max, 0.0));
  const double r = sqrt(2.0 * log(act->density / vs->tau_cut));
  int overlap = 1;
  for (int a = 0; a < 3; ++a) {
    const double h = dmin(r * sqrt(dmax(M(sigma, a, a), 0.0)), cap);
    const double gg = (act->pos[a] - rg->origin[a]) / rg->spacing;
    const int lo = (int)ceil(gg - h / rg->spacing);
    const int hi = (int)floor(gg + h / rg->spacing);
    out->lo[a] = lo > 0 ? lo : 0;
    out->hi[a] = hi < rg->dims[a] - 1 ? hi : rg->dims[a] - 1;
    overlap = overlap && out->lo[a] <= out->hi[a];
  }
  out->skip = !overlap;
}

int orc_prepare_voxel_splats(int64_t n, const double* pos, const double* ls, const double* q,
                             const double* raw, const orc_region* region,
                             const orc_voxel_settings* vs, int32_t* lo, int32_t* hi,
                             uint8_t* skip, double* sigma_inv) {
  for (int64_t i = 0; i < n; ++i) {
    orc_act act;
    if (orc_activate(pos, ls, q, raw, i, &act)) return 1;
    double sigma[9];
    orc_covariance(act.scales, act.unit_quat, sigma);
    vsplat_t v;
    prepare_voxel_splat(&act, sigma, region, vs, &v);
    for (int k = 0; k < 3; ++k) {
      lo[3 * i + k] = v.lo[k];
      hi[3 * i + k] = v.hi[k];
    }
    skip[i] = (uint8_t)v.skip;
    if (sigma_inv) memcpy(sigma_inv + 9 * i, v.sigma_inv, sizeof v.sigma_inv);
  }
  return 0;
}

/* voxelizer.hpp:162-199 */
int orc_voxelize(int64_t n, const double* pos, const double* ls, const double* q,
                 const double* raw, const orc_region* rg, const orc_voxel_settings* vs,
                 double* out, orc_stats* stats) {
  vsplat_t* sp = (vsplat_t*)malloc(sizeof(vsplat_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    orc_act act;
    if (orc_activate(pos, ls, q, raw, i, &act)) {
      free(sp);
      return 1;
    }
    double sigma[9];
    orc_covariance(act.scales, act.unit_quat, sigma);
    prepare_voxel_splat(&act, sigma, rg, vs, &sp[i]);
  }
  const int nx = rg->dims[0], ny = rg->dims[1], nz = rg->dims[2];
  memset(out, 0, sizeof(double) * (size_t)nx * ny * nz);
  int64_t evals = 0;
  for (int z = 0; z < nz; ++z) {
    for (int64_t i = 0; i < n; ++i) {
      const vsplat_t* v = &sp[i];
      if (v->skip || z < v->lo[2] || z > v->hi[2]) continue;
      const double* A = v->sigma_inv;
      const double dz = rg->origin[2] + rg->spacing * z - v->pos[2];
      for (int y = v->lo[1]; y <= v->hi[1]; ++y) {
        const double dy = rg->origin[1] + rg->spacing * y - v->pos[1];
        for (int x = v->lo[0]; x <= v->hi[0]; ++x) {
          const double dx = rg->origin[0] + rg->spacing * x - v->pos[0];
          const double qq = M(A, 0, 0) * dx * dx + M(A, 1, 1) * dy * dy + M(A, 2, 2) * dz * dz +
                            2.0 * (M(A, 0, 1) * dx * dy + M(A, 0, 2) * dx * dz + M(A, 1, 2) * dy * dz);
          out[((size_t)z * ny + y) * nx + x] += v->density * exp(-0.5 * qq);
        }
        evals += v->hi[0] - v->lo[0] + 1;
      }
    }
  }
  if (stats) {
    for (int64_t i = 0; i < n; ++i) stats->culled += sp[i].skip;
    stats->pixel_pairs += evals;
  }
  free(sp);
  return 0;
}

/* voxelizer.hpp:214-263 */
int orc_voxelize_backward(int64_t n, const double* pos, const double* ls, const double* q,
                          const double* raw, const orc_region* rg, const double* gv,
                          const orc_voxel_settings* vs, double* g_pos, double* g_ls,
                          double* g_q, double* g_raw, double* pos_grad_norm, uint8_t* visible) {
  memset(g_pos, 0, sizeof(double) * 3 * (size_t)n);
  memset(g_ls, 0, sizeof(double) * 3 * (size_t)n);
  memset(g_q, 0, sizeof(double) * 4 * (size_t)n);
  memset(g_raw, 0, sizeof(double) * (size_t)n);
  memset(pos_grad_norm, 0, sizeof(double) * (size_t)n);
  memset(visible, 0, (size_t)n);
  const int nx = rg->dims[0], ny = rg->dims[1];
  for (int64_t i = 0; i < n; ++i) {
    orc_act act;
    if (orc_activate(pos, ls, q, raw, i, &act)) return 1;
    double sigma[9];
    orc_covariance(act.scales, act.unit_quat, sigma);
    vsplat_t v;
    prepare_voxel_splat(&act, sigma, rg, vs, &v);
    if (v.skip) continue;
    visible[i] = 1;
    const double* A = v.sigma_inv;
    double g_rho = 0.0, gp[3] = {0, 0, 0}, gA[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int z = v.lo[2]; z <= v.hi[2]; ++z)
      for (int y = v.lo[1]; y <= v.hi[1]; ++y)
        for (int x = v.lo[0]; x <= v.hi[0]; ++x) {
          const double w = gv[((size_t)z * ny + y) * nx + x];
          if (w == 0.0) continue;
          const double idx[3] = {(double)x, (double)y, (double)z};
          double delta[3], ad[3];
          for (int k = 0; k < 3; ++k) delta[k] = rg->origin[k] + rg->spacing * idx[k] - v.pos[k];
          mul3v(A, delta, ad);
          const double expo = exp(-0.5 * dot3(delta, ad));
          g_rho += expo * w;
          const double ge = v.density * expo * w;
          for (int k = 0; k < 3; ++k) gp[k] += ge * ad[k];
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) M(gA, r, c) -= 0.5 * ge * (delta[r] * delta[c]);
        }
    double negA[9], t[9], gsig[9];
    for (int k = 0; k < 9; ++k) negA[k] = -A[k];
    mul33(negA, gA, t);
    mul33(t, A, gsig);
    for (int k = 0; k < 3; ++k) g_pos[3 * i + k] = gp[k];
    g_raw[i] = raw[i] >= 0.0 ? g_rho : 0.0;
    pos_grad_norm[i] = norm3(gp);
    orc_covariance_backward(act.scales, act.unit_quat, q + 4 * i, gsig, g_ls + 3 * i, g_q + 4 * i);
  }
  return 0;
}
