// Per-splat fp64 set-up and chain rule, executed on the device one thread per
// (splat, view). This translation-unit fragment is only included from
// preprocess.cu, which is compiled with --fmad=false: every reduction below is written
// in the reference's operation order (Eigen fixed-size products: sequential in k; Eigen
// cofactor determinant/inverse; Eigen closed-form 3x3 eigenvalues), so integer bounding
// boxes and tile/brick keys are bit-exact with the CPU reference.
//
// Reference: /root/reference/proj/include/gsct/core.hpp:80-191 (activate, covariance,
// covariance_backward), projector.hpp:91-236 (max_eigenvalue_2x2, splat_bbox,
// project_full), projector.hpp:422-474 (rasterize_backward chain rule),
// voxelizer.hpp:117-143 (prepare_voxel_splat), voxelizer.hpp:250-255 (voxel chain rule).
#pragma once
#include <cfloat>
#include <cstdint>

namespace gsct_dev {

// Matrices are row-major double[9] / double[4]; index helper.
#define GM3(a, i, j) ((a)[(i)*3 + (j)])

struct Frame {  // view_frame(): u, v, d, detector centre, source, focal
  double u[3], v[3], d[3], dc[3], src[3], focal;
};

struct Geo {
  int cone, n_u, n_v;
  double s_u, s_v;
};

struct RSet {
  double tau_cut, sigma_cap, dilation_px2;
  int tile_size, dilate, bounding;
};

__device__ __forceinline__ double dmax_(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double dmin_(double a, double b) { return (b < a) ? b : a; }

__device__ __forceinline__ double dot3(const double* a, const double* b) {
  double acc = a[0] * b[0];
  acc += a[1] * b[1];
  acc += a[2] * b[2];
  return acc;
}
__device__ __forceinline__ double norm4(const double* a) {
  double acc = a[0] * a[0];
  acc += a[1] * a[1];
  acc += a[2] * a[2];
  acc += a[3] * a[3];
  return sqrt(acc);
}
__device__ __forceinline__ void mul33(const double* a, const double* b, double* c) {
  double t[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double acc = GM3(a, i, 0) * GM3(b, 0, j);
      acc += GM3(a, i, 1) * GM3(b, 1, j);
      acc += GM3(a, i, 2) * GM3(b, 2, j);
      t[i * 3 + j] = acc;
    }
#pragma unroll
  for (int k = 0; k < 9; ++k) c[k] = t[k];
}
__device__ __forceinline__ void mul3v(const double* a, const double* v, double* out) {
  double t[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double acc = GM3(a, i, 0) * v[0];
    acc += GM3(a, i, 1) * v[1];
    acc += GM3(a, i, 2) * v[2];
    t[i] = acc;
  }
  out[0] = t[0];
  out[1] = t[1];
  out[2] = t[2];
}
// Eigen Determinant.h (3x3): sum of det3_helper terms.
__device__ __forceinline__ double det3(const double* m) {
  const double h012 = GM3(m, 0, 0) * (GM3(m, 1, 1) * GM3(m, 2, 2) - GM3(m, 1, 2) * GM3(m, 2, 1));
  const double h102 = GM3(m, 0, 1) * (GM3(m, 1, 0) * GM3(m, 2, 2) - GM3(m, 1, 2) * GM3(m, 2, 0));
  const double h201 = GM3(m, 0, 2) * (GM3(m, 1, 0) * GM3(m, 2, 1) - GM3(m, 1, 1) * GM3(m, 2, 0));
  return h012 - h102 + h201;
}
__device__ __forceinline__ double cof3(const double* m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return GM3(m, i1, j1) * GM3(m, i2, j2) - GM3(m, i1, j2) * GM3(m, i2, j1);
}
// Eigen InverseImpl.h compute_inverse<.,.,3> (adjugate / det, det from column 0).
__device__ __forceinline__ void inv3(const double* m, double* r) {
  const double c00 = cof3(m, 0, 0), c10 = cof3(m, 1, 0), c20 = cof3(m, 2, 0);
  double det = c00 * GM3(m, 0, 0);
  det += c10 * GM3(m, 1, 0);
  det += c20 * GM3(m, 2, 0);
  const double invdet = 1.0 / det;
  double t[9];
  GM3(t, 1, 0) = cof3(m, 0, 1) * invdet;
  GM3(t, 1, 1) = cof3(m, 1, 1) * invdet;
  GM3(t, 2, 0) = cof3(m, 0, 2) * invdet;
  GM3(t, 1, 2) = cof3(m, 2, 1) * invdet;
  GM3(t, 2, 1) = cof3(m, 1, 2) * invdet;
  GM3(t, 2, 2) = cof3(m, 2, 2) * invdet;
  GM3(t, 0, 0) = c00 * invdet;
  GM3(t, 0, 1) = c10 * invdet;
  GM3(t, 0, 2) = c20 * invdet;
#pragma unroll
  for (int k = 0; k < 9; ++k) r[k] = t[k];
}
__device__ __forceinline__ double det2(const double* m) { return m[0] * m[3] - m[2] * m[1]; }
__device__ __forceinline__ void inv2(const double* m, double* r) {
  const double invdet = 1.0 / det2(m);
  const double t0 = m[3] * invdet, t2 = -m[2] * invdet, t1 = -m[1] * invdet, t3 = m[0] * invdet;
  r[0] = t0;
  r[1] = t1;
  r[2] = t2;
  r[3] = t3;
}
__device__ __forceinline__ void mul22(const double* a, const double* b, double* c) {
  double t[4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double acc = a[i * 2 + 0] * b[0 * 2 + j];
      acc += a[i * 2 + 1] * b[1 * 2 + j];
      t[i * 2 + j] = acc;
    }
  c[0] = t[0];
  c[1] = t[1];
  c[2] = t[2];
  c[3] = t[3];
}
// projector.hpp:91-95
__device__ __forceinline__ double max_eig2(const double* m) {
  const double half_trace = 0.5 * (m[0] + m[3]);
  const double half_gap = 0.5 * (m[0] - m[3]);
  return half_trace + sqrt(half_gap * half_gap + m[1] * m[2]);
}

struct Act {
  double pos[3], scales[3], uq[4], density, raw_q[4], raw_density;
};

// core.hpp:80-97. Returns 0 ok, 1 non-finite, 2 zero quaternion.
__device__ __forceinline__ int activate(const double* __restrict__ pos,
                                        const double* __restrict__ ls,
                                        const double* __restrict__ q,
                                        const double* __restrict__ raw, int64_t i, Act& a) {
  const double p0 = pos[3 * i], p1 = pos[3 * i + 1], p2 = pos[3 * i + 2];
  const double l0 = ls[3 * i], l1 = ls[3 * i + 1], l2 = ls[3 * i + 2];
  const double q0 = q[4 * i], q1 = q[4 * i + 1], q2 = q[4 * i + 2], q3 = q[4 * i + 3];
  const double rho = raw[i];
  const bool fin = isfinite(p0) && isfinite(p1) && isfinite(p2) && isfinite(l0) && isfinite(l1) &&
                   isfinite(l2) && isfinite(q0) && isfinite(q1) && isfinite(q2) && isfinite(q3) &&
                   isfinite(rho);
  if (!fin) return 1;
  a.raw_q[0] = q0;
  a.raw_q[1] = q1;
  a.raw_q[2] = q2;
  a.raw_q[3] = q3;
  const double norm = norm4(a.raw_q);
  if (!(norm > 0.0)) return 2;
  a.pos[0] = p0;
  a.pos[1] = p1;
  a.pos[2] = p2;
  a.scales[0] = exp(l0);
  a.scales[1] = exp(l1);
  a.scales[2] = exp(l2);
  a.uq[0] = q0 / norm;
  a.uq[1] = q1 / norm;
  a.uq[2] = q2 / norm;
  a.uq[3] = q3 / norm;
  a.raw_density = rho;
  a.density = dmax_(rho, 0.0);
  return 0;
}

// core.hpp:100-107
__device__ __forceinline__ void rotation_matrix(const double* q, double* R) {
  const double r = q[0], x = q[1], y = q[2], z = q[3];
  GM3(R, 0, 0) = 1 - 2 * (y * y + z * z);
  GM3(R, 0, 1) = 2 * (x * y - r * z);
  GM3(R, 0, 2) = 2 * (x * z + r * y);
  GM3(R, 1, 0) = 2 * (x * y + r * z);
  GM3(R, 1, 1) = 1 - 2 * (x * x + z * z);
  GM3(R, 1, 2) = 2 * (y * z - r * x);
  GM3(R, 2, 0) = 2 * (x * z - r * y);
  GM3(R, 2, 1) = 2 * (y * z + r * x);
  GM3(R, 2, 2) = 1 - 2 * (x * x + y * y);
}

// core.hpp:111-115
__device__ __forceinline__ void covariance(const double* s, const double* uq, double* sigma) {
  double R[9], N[9];
  rotation_matrix(uq, R);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) GM3(N, i, j) = GM3(R, i, j) * s[j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double acc = GM3(N, i, 0) * GM3(N, j, 0);
      acc += GM3(N, i, 1) * GM3(N, j, 1);
      acc += GM3(N, i, 2) * GM3(N, j, 2);
      GM3(sigma, i, j) = acc;
    }
}

// core.hpp:170-191
__device__ __forceinline__ void covariance_backward(const double* s, const double* uq,
                                                    const double* raw_q, const double* G,
                                                    double* g_ls, double* g_q) {
  double rot[9], n_mat[9], G2[9], grad_n[9], grad_rot[9];
  rotation_matrix(uq, rot);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      GM3(n_mat, i, j) = GM3(rot, i, j) * s[j];
      GM3(G2, i, j) = GM3(G, i, j) + GM3(G, j, i);
    }
  mul33(G2, n_mat, grad_n);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double acc = GM3(rot, 0, k) * GM3(grad_n, 0, k);
    acc += GM3(rot, 1, k) * GM3(grad_n, 1, k);
    acc += GM3(rot, 2, k) * GM3(grad_n, 2, k);
    g_ls[k] = s[k] * acc;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) GM3(grad_rot, i, j) = GM3(grad_n, i, j) * s[j];
  const double r = uq[0], x = uq[1], y = uq[2], z = uq[3];
  const double dm[4][9] = {{0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0},
                           {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * r, 2 * z, 2 * r, -4 * x},
                           {-4 * y, 2 * x, 2 * r, 2 * x, 0, 2 * z, -2 * r, 2 * z, -4 * y},
                           {-4 * z, -2 * r, 2 * x, 2 * r, -4 * z, 2 * y, 2 * x, 2 * y, 0}};
  double gu[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // cwiseProduct(...).sum() in Eigen's column-major storage order
    double acc = GM3(grad_rot, 0, 0) * dm[k][0];
    acc += GM3(grad_rot, 1, 0) * dm[k][3];
    acc += GM3(grad_rot, 2, 0) * dm[k][6];
    acc += GM3(grad_rot, 0, 1) * dm[k][1];
    acc += GM3(grad_rot, 1, 1) * dm[k][4];
    acc += GM3(grad_rot, 2, 1) * dm[k][7];
    acc += GM3(grad_rot, 0, 2) * dm[k][2];
    acc += GM3(grad_rot, 1, 2) * dm[k][5];
    acc += GM3(grad_rot, 2, 2) * dm[k][8];
    gu[k] = acc;
  }
  const double norm = norm4(raw_q);
  double dd = uq[0] * gu[0];
  dd += uq[1] * gu[1];
  dd += uq[2] * gu[2];
  dd += uq[3] * gu[3];
#pragma unroll
  for (int k = 0; k < 4; ++k) g_q[k] = (gu[k] - uq[k] * dd) / norm;
}

// projector.hpp:101-117; returns true when visible (not culled).
__device__ __forceinline__ bool splat_bbox(double g_peak, const double* cov2d,
                                           const double* mean2d, double tau, int n_u, int n_v,
                                           int* rect, double sigma_cap, int mode) {
  if (!(g_peak > tau)) return false;
  const double cap = sigma_cap * sqrt(dmax_(max_eig2(cov2d), 0.0));
  double hu = cap, hv = cap;
  if (mode == 0) {
    const double r = sqrt(2.0 * log(g_peak / tau));
    hu = dmin_(r * sqrt(dmax_(cov2d[0], 0.0)), cap);
    hv = dmin_(r * sqrt(dmax_(cov2d[3], 0.0)), cap);
  }
  const int a = (int)ceil(mean2d[0] - hu), b = (int)floor(mean2d[0] + hu);
  const int c = (int)ceil(mean2d[1] - hv), d = (int)floor(mean2d[1] + hv);
  rect[0] = a > 0 ? a : 0;
  rect[1] = b < n_u - 1 ? b : n_u - 1;
  rect[2] = c > 0 ? c : 0;
  rect[3] = d < n_v - 1 ? d : n_v - 1;
  return !(rect[1] < rect[0] || rect[3] < rect[2]);
}

// detail::SplatProjection (projector.hpp:126-141)
struct Proj {
  double mean2d[2], cov2d[4], conic[4], amplitude;
  int rect[4];
  bool culled, degenerate;
  double ad[3], beta, mu, k, cov_px[4], d_ray[3];
  double t_cam[3], jac[6], dist;
  // backward tail only (project_full<false>): reciprocals shared with raster_chain_rule
  double itz, inv_dist, rb;  // 1 / t_cam.z, 1 / dist, 1 / sqrt(beta)
};

// detail::project_full (projector.hpp:143-236)
// The view-independent part (det Sigma > 0 check and Sigma^-1, projector.hpp:151-156) is
// hoisted into prepare_splat(); its results are passed in (sigma_inv, det_ok).
// kBox = false (backward tail): the bounding box, the eigenvalue-ratio test and the cull
// are skipped -- the caller already knows the splat is visible in this view.
template <bool kBox = true>
__device__ __forceinline__ void project_full(const Frame& fr, const Geo& g, const double* position,
                                             const double* cov3d, const double* sigma_inv, bool det_ok,
                                             double density, const RSet& rs, Proj& p) {
  p.beta = 1.0;
  p.k = 1.0;
  p.mu = 0.0;
  p.dist = 0.0;
  p.amplitude = 0.0;
  p.culled = true;
  p.degenerate = false;
  p.rect[0] = 0;
  p.rect[1] = -1;
  p.rect[2] = 0;
  p.rect[3] = -1;
  p.mean2d[0] = p.mean2d[1] = 0.0;
#pragma unroll
  for (int k = 0; k < 6; ++k) p.jac[k] = 0.0;
  p.t_cam[0] = p.t_cam[1] = p.t_cam[2] = 0.0;

  if (!det_ok) {
    p.degenerate = true;
    return;
  }
  const double cu = 0.5 * (g.n_u - 1);
  const double cv = 0.5 * (g.n_v - 1);
  if (!g.cone) {
    double rel[3], muc[3], mvc[3], tmp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      p.d_ray[k] = fr.d[k];
      rel[k] = position[k] - fr.dc[k];
    }
    p.mean2d[0] = dot3(rel, fr.u) / g.s_u + cu;
    p.mean2d[1] = dot3(rel, fr.v) / g.s_v + cv;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      muc[k] = fr.u[k] / g.s_u;
      mvc[k] = fr.v[k] / g.s_v;
    }
    mul3v(cov3d, muc, tmp);
    p.cov_px[0] = dot3(muc, tmp);
    mul3v(cov3d, mvc, tmp);
    p.cov_px[1] = p.cov_px[2] = dot3(muc, tmp);
    p.cov_px[3] = dot3(mvc, tmp);
  } else {
    double rel[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) rel[k] = position[k] - fr.src[k];
    if (kBox) {
      p.dist = sqrt(dot3(rel, rel));
    } else {  // one rsqrt for the distance and its reciprocal
      const double d2 = dot3(rel, rel);
      p.inv_dist = rsqrt(d2);
      p.dist = d2 * p.inv_dist;
    }
    p.t_cam[0] = dot3(rel, fr.u);
    p.t_cam[1] = dot3(rel, fr.v);
    p.t_cam[2] = dot3(rel, fr.d);
    const double tz = p.t_cam[2];
    if (!(tz > 1e-9 * fr.focal)) {
      p.degenerate = true;
      return;
    }
    const double f = fr.focal;
    double* J = p.jac;
    if (kBox) {
#pragma unroll
      for (int k = 0; k < 3; ++k) p.d_ray[k] = rel[k] / p.dist;
      p.mean2d[0] = f * p.t_cam[0] / (tz * g.s_u) + cu;
      p.mean2d[1] = f * p.t_cam[1] / (tz * g.s_v) + cv;
      J[0] = f / (g.s_u * tz);
      J[2] = -f * p.t_cam[0] / (g.s_u * tz * tz);
      J[4] = f / (g.s_v * tz);
      J[5] = -f * p.t_cam[1] / (g.s_v * tz * tz);
    } else {  // backward tail: tolerance-level arithmetic, reciprocals instead of divisions
#pragma unroll
      for (int k = 0; k < 3; ++k) p.d_ray[k] = rel[k] * p.inv_dist;
      const double itz = 1.0 / tz;
      p.itz = itz;
      // 1 / s_u, 1 / s_v depend on kernel parameters only (hoisted out of the view loop)
      const double fu = f * (1.0 / g.s_u) * itz, fv = f * (1.0 / g.s_v) * itz;
      J[0] = fu;
      J[2] = -fu * p.t_cam[0] * itz;
      J[4] = fv;
      J[5] = -fv * p.t_cam[1] * itz;
    }
    const double* rows[3] = {fr.u, fr.v, fr.d};
    double T[6], A[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double acc = J[i * 3 + 0] * rows[0][j];
        acc += J[i * 3 + 1] * rows[1][j];
        acc += J[i * 3 + 2] * rows[2][j];
        T[i * 3 + j] = acc;
      }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double acc = T[i * 3 + 0] * GM3(cov3d, 0, j);
        acc += T[i * 3 + 1] * GM3(cov3d, 1, j);
        acc += T[i * 3 + 2] * GM3(cov3d, 2, j);
        A[i * 3 + j] = acc;
      }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double acc = A[i * 3 + 0] * T[j * 3 + 0];
        acc += A[i * 3 + 1] * T[j * 3 + 1];
        acc += A[i * 3 + 2] * T[j * 3 + 2];
        p.cov_px[i * 2 + j] = acc;
      }
  }
  mul3v(sigma_inv, p.d_ray, p.ad);
  p.beta = dot3(p.d_ray, p.ad);
  if (!(p.beta > 0.0) || !isfinite(p.beta)) {
    p.degenerate = true;
    return;
  }
  if (kBox) {
    p.mu = sqrt(2.0 * 3.14159265358979323846 / p.beta);
  } else {
    p.rb = rsqrt(p.beta);
    p.mu = 2.5066282746310002 * p.rb;  // sqrt(2 pi / beta)
  }

  double cr[4] = {p.cov_px[0], p.cov_px[1], p.cov_px[2], p.cov_px[3]};
  if (rs.dilate) {
    cr[0] += rs.dilation_px2;
    cr[3] += rs.dilation_px2;
  }
  const double dt2 = det2(cr);
  double rdt = 0.0;  // tail: 1 / sqrt(dt2) (the visible item has dt2 > 0)
  if (!kBox) rdt = rsqrt(dt2);
  if (rs.dilate) {
    const double det_raw = dmax_(det2(p.cov_px), 0.0);
    p.k = kBox ? sqrt(det_raw / dt2) : sqrt(det_raw) * rdt;
  }
  if (kBox) {
    const double lam_max = max_eig2(cr);
    const double lam_min = dt2 / dmax_(lam_max, DBL_MIN);
    if (!(dt2 > 0.0) || !(lam_max / lam_min < 1e12) || !isfinite(dt2)) {
      p.degenerate = true;
      return;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) p.cov2d[k] = cr[k];
  {
    // the conic feeds only the fp32 record and the gradients (never the integer box), so one
    // reciprocal replaces the reference's four divisions (<= 1 ulp apart)
    const double idt = kBox ? 1.0 / dt2 : rdt * rdt;
    p.conic[0] = cr[3] * idt;
    p.conic[1] = -cr[1] * idt;
    p.conic[2] = -cr[2] * idt;
    p.conic[3] = cr[0] * idt;
  }
  p.amplitude = p.mu * density * p.k;
  if (!kBox) {
    p.culled = false;
    return;
  }
  p.culled = !splat_bbox(p.amplitude, p.cov2d, p.mean2d, rs.tau_cut, g.n_u, g.n_v, p.rect,
                         rs.sigma_cap, rs.bounding);
  if (p.culled) {
    p.rect[0] = 0;
    p.rect[1] = -1;
    p.rect[2] = 0;
    p.rect[3] = -1;
  }
}

// rasterize_backward chain rule (projector.hpp:422-472) from the pixel-loop sums, up to
// dL/dSigma: gm = dL/dmean2d, gc = dL/dconic (row-major 2x2), g_amp = dL/damplitude.
// Outputs g_pos, g_sigma (row-major 3x3) and the gated density gradient; the map
// dL/dSigma -> d(log_scale, raw quat) (covariance_backward, core.hpp:170-191) is linear in
// dL/dSigma and applied once per splat to the view sum.
__device__ __forceinline__ void raster_chain_rule(const Frame& fr, const Geo& g, const RSet& rs,
                                                  double density, double raw_density,
                                                  const double* sigma, const Proj& p, double g_amp,
                                                  const double* gm, const double* gc, double* g_pos,
                                                  double* g_sigma, double& g_raw) {
  const double g_mu = density * p.k * g_amp;
  const double g_rho = p.mu * p.k * g_amp;
  const double g_k = p.mu * density * g_amp;

  const double negc[4] = {-p.conic[0], -p.conic[1], -p.conic[2], -p.conic[3]};
  double tmp2[4], gcov[4];
  mul22(negc, gc, tmp2);
  mul22(tmp2, p.conic, gcov);
  if (rs.dilate) {
    const double det_raw = det2(p.cov_px);
    if (det_raw > 0.0) {
      double ci[4];
      inv2(p.cov_px, ci);
      const double sc = g_k * (p.k / 2.0);
#pragma unroll
      for (int k = 0; k < 4; ++k) gcov[k] += sc * (ci[k] - p.conic[k]);
    }
  }
  const double g_beta = -g_mu * p.mu * (0.5 * p.rb * p.rb);  // -g_mu mu / (2 beta)
  double gsig[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) GM3(gsig, r, c) = -g_beta * (p.ad[r] * p.ad[c]);
  double gp[3];
  if (!g.cone) {
    double mc[6];
    const double isu = 1.0 / g.s_u, isv = 1.0 / g.s_v;  // kernel-parameter reciprocals (hoisted)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      mc[k * 2 + 0] = fr.u[k] * isu;
      mc[k * 2 + 1] = fr.v[k] * isv;
    }
    double A[6];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        double acc = mc[r * 2 + 0] * gcov[0 * 2 + c];
        acc += mc[r * 2 + 1] * gcov[1 * 2 + c];
        A[r * 2 + c] = acc;
      }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double acc = A[r * 2 + 0] * mc[c * 2 + 0];
        acc += A[r * 2 + 1] * mc[c * 2 + 1];
        GM3(gsig, r, c) += acc;
      }
#pragma unroll
    for (int k = 0; k < 3; ++k) gp[k] = gm[0] * mc[k * 2 + 0] + gm[1] * mc[k * 2 + 1];
  } else {
    const double* J = p.jac;
    const double* rows[3] = {fr.u, fr.v, fr.d};
    double T[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double acc = J[r * 3 + 0] * rows[0][j];
        acc += J[r * 3 + 1] * rows[1][j];
        acc += J[r * 3 + 2] * rows[2][j];
        T[r * 3 + j] = acc;
      }
    double A[6];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        double acc = T[0 * 3 + r] * gcov[0 * 2 + c];
        acc += T[1 * 3 + r] * gcov[1 * 2 + c];
        A[r * 2 + c] = acc;
      }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double acc = A[r * 2 + 0] * T[0 * 3 + c];
        acc += A[r * 2 + 1] * T[1 * 3 + c];
        GM3(gsig, r, c) += acc;
      }
    const double G2[4] = {gcov[0] + gcov[0], gcov[1] + gcov[2], gcov[2] + gcov[1],
                          gcov[3] + gcov[3]};
    double C1[6], gT[6], gJ[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double acc = G2[r * 2 + 0] * T[0 * 3 + j];
        acc += G2[r * 2 + 1] * T[1 * 3 + j];
        C1[r * 3 + j] = acc;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double acc = C1[r * 3 + 0] * GM3(sigma, 0, j);
        acc += C1[r * 3 + 1] * GM3(sigma, 1, j);
        acc += C1[r * 3 + 2] * GM3(sigma, 2, j);
        gT[r * 3 + j] = acc;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double acc = gT[r * 3 + 0] * rows[j][0];
        acc += gT[r * 3 + 1] * rows[j][1];
        acc += gT[r * 3 + 2] * rows[j][2];
        gJ[r * 3 + j] = acc;
      }
    const double f = fr.focal;
    const double su = g.s_u, sv = g.s_v;
    double gt[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) gt[k] = J[0 * 3 + k] * gm[0] + J[1 * 3 + k] * gm[1];
    // (tail-only code, tolerance-level: reciprocals instead of divisions)
    const double itz = p.itz;
    const double fu2 = -f * (1.0 / su) * itz * itz, fv2 = -f * (1.0 / sv) * itz * itz;
    gt[0] += gJ[0 * 3 + 2] * fu2;
    gt[1] += gJ[1 * 3 + 2] * fv2;
    gt[2] += gJ[0 * 3 + 0] * fu2 + gJ[0 * 3 + 2] * (-2.0 * fu2 * p.t_cam[0] * itz) + gJ[1 * 3 + 1] * fv2 +
             gJ[1 * 3 + 2] * (-2.0 * fv2 * p.t_cam[1] * itz);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double acc = rows[0][k] * gt[0];
      acc += rows[1][k] * gt[1];
      acc += rows[2][k] * gt[2];
      gp[k] = acc;
    }
    double gd[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) gd[k] = 2.0 * g_beta * p.ad[k];
    const double dd = dot3(p.d_ray, gd);
    const double inv_dist = p.inv_dist;
#pragma unroll
    for (int k = 0; k < 3; ++k) gp[k] += (gd[k] - p.d_ray[k] * dd) * inv_dist;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) g_pos[k] = gp[k];
#pragma unroll
  for (int k = 0; k < 9; ++k) g_sigma[k] = gsig[k];
  g_raw = raw_density >= 0.0 ? g_rho : 0.0;
}

// Eigen direct_selfadjoint_eigenvalues<.,3> (SelfAdjointEigenSolver::computeDirect);
// returns eigenvalues().maxCoeff().
__device__ __forceinline__ double max_eig3(const double* mat) {
  double trace = GM3(mat, 0, 0);
  trace += GM3(mat, 1, 1);
  trace += GM3(mat, 2, 2);
  const double shift = trace / 3.0;
  double m[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) GM3(m, i, j) = i >= j ? GM3(mat, i, j) : GM3(mat, j, i);
#pragma unroll
  for (int i = 0; i < 3; ++i) GM3(m, i, i) -= shift;
  double scale = fabs(GM3(m, 0, 0));
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const double v = fabs(GM3(m, r, c));
      if (v > scale) scale = v;
    }
  if (scale > 0.0) {
#pragma unroll
    for (int k = 0; k < 9; ++k) m[k] /= scale;
  }
  const double s_inv3 = 1.0 / 3.0;
  const double s_sqrt3 = sqrt(3.0);
  const double c0 = GM3(m, 0, 0) * GM3(m, 1, 1) * GM3(m, 2, 2) +
                    2.0 * GM3(m, 1, 0) * GM3(m, 2, 0) * GM3(m, 2, 1) -
                    GM3(m, 0, 0) * GM3(m, 2, 1) * GM3(m, 2, 1) -
                    GM3(m, 1, 1) * GM3(m, 2, 0) * GM3(m, 2, 0) -
                    GM3(m, 2, 2) * GM3(m, 1, 0) * GM3(m, 1, 0);
  const double c1 = GM3(m, 0, 0) * GM3(m, 1, 1) - GM3(m, 1, 0) * GM3(m, 1, 0) +
                    GM3(m, 0, 0) * GM3(m, 2, 2) - GM3(m, 2, 0) * GM3(m, 2, 0) +
                    GM3(m, 1, 1) * GM3(m, 2, 2) - GM3(m, 2, 1) * GM3(m, 2, 1);
  const double c2 = GM3(m, 0, 0) + GM3(m, 1, 1) + GM3(m, 2, 2);
  const double c2_over_3 = c2 * s_inv3;
  double a_over_3 = (c2 * c2_over_3 - c1) * s_inv3;
  a_over_3 = dmax_(a_over_3, 0.0);
  const double half_b = 0.5 * (c0 + c2_over_3 * (2.0 * c2_over_3 * c2_over_3 - c1));
  double qq = a_over_3 * a_over_3 * a_over_3 - half_b * half_b;
  qq = dmax_(qq, 0.0);
  const double rho = sqrt(a_over_3);
  const double theta = atan2(sqrt(qq), half_b) * s_inv3;
  const double cos_theta = cos(theta);
  const double sin_theta = sin(theta);
  double e0 = c2_over_3 - rho * (cos_theta + s_sqrt3 * sin_theta);
  double e1 = c2_over_3 - rho * (cos_theta - s_sqrt3 * sin_theta);
  double e2 = c2_over_3 + 2.0 * rho * cos_theta;
  e0 = e0 * scale + shift;
  e1 = e1 * scale + shift;
  e2 = e2 * scale + shift;
  double mx = e0;
  if (e1 > mx) mx = e1;
  if (e2 > mx) mx = e2;
  return mx;
}

// View-independent per-splat set-up shared by every view of a call: activation
// (core.hpp:80-97), Sigma (core.hpp:111-115) and the determinant test + Sigma^-1 of
// project_full (projector.hpp:151-156). Symmetric matrices stored as full row-major 3x3.
struct PreSplat {
  double pos[3];
  double sigma[9];
  double sigma_inv[9];
  double density;
  double raw_density;
  int det_ok;  // det Sigma > 0 and finite
  int status;  // 0 ok, 1 non-finite parameter, 2 zero quaternion
};

// PreSplat buffers are stored structure-of-arrays (same total size as n PreSplat structs):
// double field f of splat i at d[f * n + i] (23 doubles: pos, sigma, sigma_inv, density,
// raw_density), then det_ok and status as int arrays. A warp's loads of one field are one
// coalesced 256 B request instead of 32 strided 184 B structs.
constexpr int kPreDoubles = 23;
static_assert(sizeof(PreSplat) == kPreDoubles * 8 + 8, "PreSplat layout");
__device__ __forceinline__ void pre_store(PreSplat* buf, int64_t n, int64_t i, const PreSplat& s) {
  double* d = reinterpret_cast<double*>(buf);
  const double* src = reinterpret_cast<const double*>(&s);
#pragma unroll
  for (int f = 0; f < kPreDoubles; ++f) d[f * n + i] = src[f];
  int* ip = reinterpret_cast<int*>(d + kPreDoubles * n);
  ip[i] = s.det_ok;
  ip[n + i] = s.status;
}
__device__ __forceinline__ void pre_load(const PreSplat* buf, int64_t n, int64_t i, PreSplat& s) {
  const double* d = reinterpret_cast<const double*>(buf);
  double* dst = reinterpret_cast<double*>(&s);
#pragma unroll
  for (int f = 0; f < kPreDoubles; ++f) dst[f] = __ldg(d + f * n + i);
  const int* ip = reinterpret_cast<const int*>(d + kPreDoubles * n);
  s.det_ok = __ldg(ip + i);
  s.status = __ldg(ip + n + i);
}

__device__ __forceinline__ void prepare_splat(const double* __restrict__ pos, const double* __restrict__ ls,
                                              const double* __restrict__ q, const double* __restrict__ raw,
                                              int64_t i, PreSplat& s) {
  Act a;
  s.status = activate(pos, ls, q, raw, i, a);
  s.det_ok = 0;
  if (s.status) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) s.pos[k] = a.pos[k];
  s.density = a.density;
  s.raw_density = a.raw_density;
  covariance(a.scales, a.uq, s.sigma);
  const double d3 = det3(s.sigma);
  s.det_ok = (d3 > 0.0) && isfinite(d3);
  if (s.det_ok) inv3(s.sigma, s.sigma_inv);
}

struct VoxGrid {
  int dims[3];
  double spacing;
  double origin[3];
};

// detail::prepare_voxel_splat (voxelizer.hpp:117-143). Boxes in grid indices,
// clipped to the grid (the caller clips further to a window).
__device__ __forceinline__ bool prepare_voxel_splat(const Act& act, const double* sigma,
                                                    const VoxGrid& rg, double tau_cut,
                                                    double sigma_cap, double* sigma_inv,
                                                    int* lo, int* hi) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    lo[k] = 0;
    hi[k] = -1;
  }
  if (!(act.density > tau_cut)) return false;
  const double det = det3(sigma);
  if (!(det > 0.0) || !isfinite(det)) return false;
  inv3(sigma, sigma_inv);
  const double lam_max = max_eig3(sigma);
  const double cap = sigma_cap * sqrt(dmax_(lam_max, 0.0));
  const double r = sqrt(2.0 * log(act.density / tau_cut));
  bool overlap = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double h = dmin_(r * sqrt(dmax_(GM3(sigma, a, a), 0.0)), cap);
    const double gg = (act.pos[a] - rg.origin[a]) / rg.spacing;
    const int l = (int)ceil(gg - h / rg.spacing);
    const int u = (int)floor(gg + h / rg.spacing);
    lo[a] = l > 0 ? l : 0;
    hi[a] = u < rg.dims[a] - 1 ? u : rg.dims[a] - 1;
    overlap = overlap && lo[a] <= hi[a];
  }
  return overlap;
}

}  // namespace gsct_dev
