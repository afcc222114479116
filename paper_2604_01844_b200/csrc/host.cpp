// Host-side (CPU) part of libgsct_b200.so: view frames, default scan geometry, the seeded
// RNG with the reference's output mappings, sub-volume sampling and the benchmark cloud
// generators. Compiled with -ffp-contract=off so view frames are bit-identical to the
// reference's (glibc cos/sin), which keeps tile keys bit-exact.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <sstream>
#include <string>

#include "../../include/gsct_cuda.h"

namespace {

// rng.hpp:18-69 — std::mt19937_64 state transitions are fixed by the standard; the
// uniform/normal/uniform_int mappings are the reference's explicit ones.
class Rng {
 public:
  explicit Rng(uint64_t seed) : engine_(seed) {}
  uint64_t next() { return engine_(); }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  int64_t uniform_int(int64_t n) {
    const uint64_t un = static_cast<uint64_t>(n);
    const uint64_t limit = UINT64_MAX - UINT64_MAX % un;
    uint64_t r = next();
    while (r >= limit) r = next();
    return static_cast<int64_t>(r % un);
  }
  double normal() {
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
  std::string save_state() const {
    std::ostringstream out;
    out << engine_;
    return out.str();
  }
  void restore_state(const std::string& s) {
    std::istringstream in(s);
    in >> engine_;
  }

 private:
  std::mt19937_64 engine_;
};

double norm4(const double* q) {
  double acc = q[0] * q[0];
  acc += q[1] * q[1];
  acc += q[2] * q[2];
  acc += q[3] * q[3];
  return std::sqrt(acc);
}

void normalize4(double* q) {  // Eigen normalize(): divide by the norm when non-zero
  double zz = q[0] * q[0];
  zz += q[1] * q[1];
  zz += q[2] * q[2];
  zz += q[3] * q[3];
  if (zz > 0.0) {
    const double s = std::sqrt(zz);
    for (int k = 0; k < 4; ++k) q[k] /= s;
  }
}

}  // namespace

extern "C" {

// projector.hpp:29-43
void gsct_host_view_frame(const gsct_geometry* g, double theta, double f[16]) {
  for (int k = 0; k < 16; ++k) f[k] = 0.0;
  double* u = f;
  double* v = f + 3;
  double* d = f + 6;
  double* dc = f + 9;
  double* src = f + 12;
  d[0] = std::cos(theta);
  d[1] = std::sin(theta);
  d[2] = 0.0;
  u[0] = -std::sin(theta);
  u[1] = std::cos(theta);
  u[2] = 0.0;
  v[2] = 1.0;
  if (g->cone) {
    for (int k = 0; k < 3; ++k) {
      src[k] = -g->source_to_origin * d[k];
      dc[k] = g->origin_to_detector * d[k];
    }
    f[15] = g->source_to_origin + g->origin_to_detector;
  }
}

// synthetic.hpp:236-271 (default_angles, default_geometry; automatic cone distances)
void gsct_host_default_geometry(const int dims[3], double spacing, int n_views, int cone, int n_u,
                                int n_v, gsct_geometry* out, double* angles) {
  const double span = cone ? 2.0 * M_PI : M_PI;
  for (int i = 0; i < n_views; ++i)
    angles[i] = span * static_cast<double>(i) / static_cast<double>(n_views);
  out->cone = cone;
  out->n_u = n_u;
  out->n_v = n_v;
  const double width_xy = std::hypot(dims[0] * spacing, dims[1] * spacing) * 1.05;
  const double height = dims[2] * spacing * 1.05;
  if (cone) {
    const double radius = 0.5 * std::hypot(width_xy, height);
    out->source_to_origin = 4.0 * radius;
    out->origin_to_detector = 2.0 * radius;
    const double mag = (out->source_to_origin + out->origin_to_detector) / out->source_to_origin;
    out->s_u = mag * width_xy / n_u;
    out->s_v = mag * height / n_v;
  } else {
    out->source_to_origin = 0.0;
    out->origin_to_detector = 0.0;
    out->s_u = width_xy / n_u;
    out->s_v = height / n_v;
  }
}

void* gsct_host_rng_create(uint64_t seed) { return new Rng(seed); }
void gsct_host_rng_destroy(void* r) { delete static_cast<Rng*>(r); }
double gsct_host_rng_uniform(void* r, double lo, double hi) { return static_cast<Rng*>(r)->uniform(lo, hi); }
double gsct_host_rng_normal(void* r) { return static_cast<Rng*>(r)->normal(); }
int64_t gsct_host_rng_uniform_int(void* r, int64_t n) {
  if (n <= 0) return -1;
  return static_cast<Rng*>(r)->uniform_int(n);
}
// The engine's text form (Rng::save_state / restore_state): x[0..311] then p, libstdc++.
void gsct_host_rng_get_state(void* r, gsct_rng_state* out) {
  std::istringstream in(static_cast<Rng*>(r)->save_state());
  for (auto& w : out->x) in >> w;
  in >> out->p;
}
void gsct_host_rng_set_state(void* r, const gsct_rng_state* st) {
  std::ostringstream os;
  for (auto w : st->x) os << w << ' ';
  os << st->p;
  static_cast<Rng*>(r)->restore_state(os.str());
}

// voxelizer.hpp:76-93
int gsct_host_sample_subvolume(const int parent_dims[3], const int sub_dims[3], void* rng, int offset[3],
                               int dims[3]) {
  for (int a = 0; a < 3; ++a) {
    dims[a] = sub_dims[a];
    if (dims[a] > parent_dims[a]) {
      std::fprintf(stderr, "gsct: warning: sub-volume dim %d (%d) exceeds parent (%d); clamping\n", a, dims[a],
                   parent_dims[a]);
      dims[a] = parent_dims[a];
    }
    if (dims[a] < 1) return 1;
  }
  for (int a = 0; a < 3; ++a)
    offset[a] = static_cast<int>(static_cast<Rng*>(rng)->uniform_int(parent_dims[a] - dims[a] + 1));
  return 0;
}

int gsct_host_make_cloud(int kind, int64_t count, uint64_t seed, const double* p, double* pos,
                         double* ls, double* q, double* raw) {
  Rng rng(seed);
  if (kind == 0) {
    // bench.hpp:33-52 synthetic_cloud
    // The reference draws through Vec3(rng.uniform(), ...) / Vec4(rng.normal(), ...)
    // constructor calls, whose argument evaluation order C++ leaves unspecified; the GCC
    // build of the reference evaluates them right to left, so components are drawn last
    // to first here to reproduce the reference's clouds bit for bit.
    const double he = p[0], scale = p[1], aniso = p[2], density = p[3];
    for (int64_t i = 0; i < count; ++i) {
      pos[3 * i + 2] = rng.uniform(-he, he);
      pos[3 * i + 1] = rng.uniform(-he, he);
      pos[3 * i] = rng.uniform(-he, he);
      const double l = std::log(scale);
      ls[3 * i] = ls[3 * i + 1] = ls[3 * i + 2] = l;
      double qq[4] = {1, 0, 0, 0};
      if (aniso > 1.0) {
        ls[3 * i] += std::log(aniso);
        qq[3] = rng.normal();
        qq[2] = rng.normal();
        qq[1] = rng.normal();
        qq[0] = rng.normal();
        if (norm4(qq) == 0.0) {
          qq[0] = 1;
          qq[1] = qq[2] = qq[3] = 0;
        }
        normalize4(qq);
      }
      for (int k = 0; k < 4; ++k) q[4 * i + k] = qq[k];
      raw[i] = density;
    }
    return 0;
  }
  if (kind == 1) {
    // tests/oracles.hpp:168-184 random_cloud
    const double pr = p[0], slo = p[1], shi = p[2];
    for (int64_t i = 0; i < count; ++i) {  // same right-to-left draw order as above
      pos[3 * i + 2] = rng.uniform(-pr, pr);
      pos[3 * i + 1] = rng.uniform(-pr, pr);
      pos[3 * i] = rng.uniform(-pr, pr);
      ls[3 * i + 2] = std::log(rng.uniform(slo, shi));
      ls[3 * i + 1] = std::log(rng.uniform(slo, shi));
      ls[3 * i] = std::log(rng.uniform(slo, shi));
      double qq[4];
      qq[3] = rng.normal();
      qq[2] = rng.normal();
      qq[1] = rng.normal();
      qq[0] = rng.normal();
      if (norm4(qq) == 0.0) {
        qq[0] = 1;
        qq[1] = qq[2] = qq[3] = 0;
      }
      normalize4(qq);
      for (int k = 0; k < 4; ++k) q[4 * i + k] = qq[k];
      raw[i] = rng.uniform(0.2, 1.5);
    }
    return 0;
  }
  if (kind == 2) {
    // Modified 3D Shepp-Logan cloud: positions uniform inside the outer
    // ellipsoid (semi-axes 0.69, 0.92, 0.81 of the half-side), isotropic-ish 1-NN scales
    // s0 = 0.554 (V_fg / N)^(1/3) with U(-0.3, 0.3) log jitter per axis, random
    // orientation, raw density 0.15 * U(0.2, 1.0) (init.hpp:412 k = 0.15).
    const double side = p[0], sp = p[1];
    const double half = 0.5 * side * sp;
    const double ax = 0.69 * half, ay = 0.92 * half, az = 0.81 * half;
    const double vfg = 4.0 / 3.0 * M_PI * ax * ay * az;
    const double s0 = 0.554 * std::cbrt(vfg / static_cast<double>(count > 0 ? count : 1));
    for (int64_t i = 0; i < count; ++i) {
      double x, y, z;
      do {
        x = rng.uniform(-1.0, 1.0);
        y = rng.uniform(-1.0, 1.0);
        z = rng.uniform(-1.0, 1.0);
      } while (x * x + y * y + z * z > 1.0);
      pos[3 * i] = x * ax;
      pos[3 * i + 1] = y * ay;
      pos[3 * i + 2] = z * az;
      for (int k = 0; k < 3; ++k) ls[3 * i + k] = std::log(s0) + rng.uniform(-0.3, 0.3);
      double qq[4] = {rng.normal(), rng.normal(), rng.normal(), rng.normal()};
      if (norm4(qq) == 0.0) {
        qq[0] = 1;
        qq[1] = qq[2] = qq[3] = 0;
      }
      normalize4(qq);
      for (int k = 0; k < 4; ++k) q[4 * i + k] = qq[k];
      raw[i] = 0.15 * rng.uniform(0.2, 1.0);
    }
    return 0;
  }
  return 1;
}

}  // extern "C"
