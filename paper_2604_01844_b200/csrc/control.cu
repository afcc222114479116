// Adaptive density control on device: accumulate_control_stats
// (optim.hpp:366-373) and adaptive_control (optim.hpp:201-317) -- prune / clone / split with
// the Adam moments and the densification accumulators kept in lockstep, plus the reference
// Rng's std::mt19937_64 stream (rng.hpp:18-69) generated on device for the split children.
//
// Compiled with --fmad=false (like preprocess.cu): the decisions (prune, the clone/split
// threshold, the cap) compare fp64 values computed operation for operation as the reference
// does, so which splats are pruned / cloned / split and the output row order are bit-exact;
// child positions go through CUDA's log/cos (<= 2 ulp from glibc's), hence agree to ~1e-15
// relative rather than bit for bit.
//
// Plan (all per-splat work is one thread per splat, order-independent):
//   1. k_ctrl_activate: activate(); max activated density (atomicMax on the bits of a
//      non-negative double is exact and order-free); first failing splat (atomicMin).
//   2. k_ctrl_flags: prune / eligible flags; exclusive scans give survivors and, per
//      eligible splat, its rank in index order.
//   3. k_ctrl_ops: the reference's sequential budget loop is "the first `budget` eligible
//      splats in index order", i.e. rank < budget; rows per splat {prune 0, keep 1, clone 2,
//      split 2}; scans give each splat's output row and each split its index k.
//   4. k_mt_generate: 12 engine draws per split (2 children x 3 normals x 2 uniforms) from
//      the caller's engine state, in stream order; split k owns draws [12k, 12k + 12).
//   5. k_ctrl_write: rows spliced in index order (copy / fresh), fresh rows with zero moments.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "gsct_internal.cuh"

namespace gsct_dev {

namespace {

enum : uint8_t { kKeep = 0, kPrune = 1, kClone = 2, kSplit = 3 };

inline unsigned blocks_for(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

__global__ void __launch_bounds__(256) k_ctrl_accumulate(int64_t n, const uint8_t* __restrict__ visible,
                                                         const double* __restrict__ pgn,
                                                         const double* __restrict__ g_pos,
                                                         double* __restrict__ acc_norm,
                                                         double* __restrict__ acc_dir,
                                                         int64_t* __restrict__ acc_count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !visible[i]) return;
  acc_norm[i] += pgn[i];
#pragma unroll
  for (int a = 0; a < 3; ++a) acc_dir[3 * i + a] += g_pos[3 * i + a];
  acc_count[i] += 1;
}

__global__ void __launch_bounds__(256) k_ctrl_activate(Cloud c, unsigned long long* __restrict__ max_bits,
                                                       unsigned long long* __restrict__ err_key) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= c.n) return;
  Act a;
  const int st = activate(c.pos, c.ls, c.q, c.raw, i, a);
  if (st) {
    atomicMin(err_key, (static_cast<unsigned long long>(i) << 2) | static_cast<unsigned long long>(st));
    return;
  }
  // density >= 0 (max(rho, 0)); + 0.0 folds -0 into +0 so the bit order is the value order
  atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(a.density + 0.0)));
}

__global__ void __launch_bounds__(256) k_ctrl_flags(Cloud c, const unsigned long long* __restrict__ max_bits,
                                                    double prune_density, double grad_threshold,
                                                    const double* __restrict__ acc_norm,
                                                    const int64_t* __restrict__ acc_count, int* __restrict__ keep,
                                                    int* __restrict__ elig) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= c.n) return;
  const double max_density = __longlong_as_double(static_cast<long long>(*max_bits));
  const double prune_below = prune_density * max_density;
  const double rho = c.raw[i];
  const double density = rho < 0.0 ? 0.0 : rho;  // std::max(rho, 0.0) for the comparison
  const bool pruned = density < prune_below;
  bool e = false;
  if (!pruned && acc_count[i] != 0) {
    const double mean_grad = acc_norm[i] / static_cast<double>(acc_count[i]);
    e = mean_grad > grad_threshold;
  }
  keep[i] = pruned ? 0 : 1;
  elig[i] = e ? 1 : 0;
}

// totals: {survivors, cloned, split}
__global__ void __launch_bounds__(256) k_ctrl_ops(Cloud c, const int* __restrict__ keep,
                                                  const int* __restrict__ keep_off, const int* __restrict__ elig,
                                                  const int* __restrict__ elig_rank, int64_t max_gaussians,
                                                  double split_below, uint8_t* __restrict__ op, int* __restrict__ rows,
                                                  int* __restrict__ splitf, unsigned long long* __restrict__ totals) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n = c.n;
  if (i >= n) return;
  const int64_t survivors = static_cast<int64_t>(keep_off[n - 1]) + keep[n - 1];
  const int64_t budget = max_gaussians - survivors;
  uint8_t o = keep[i] ? kKeep : kPrune;
  if (elig[i] && static_cast<int64_t>(elig_rank[i]) < budget) {
    Act a;
    activate(c.pos, c.ls, c.q, c.raw, i, a);
    const double max_scale = dmax_(dmax_(a.scales[0], a.scales[1]), a.scales[2]);
    o = max_scale < split_below ? kClone : kSplit;
    atomicAdd(&totals[o == kClone ? 1 : 2], 1ull);
  }
  if (i == 0) atomicAdd(&totals[0], static_cast<unsigned long long>(survivors));
  op[i] = o;
  rows[i] = o == kPrune ? 0 : (o == kKeep ? 1 : 2);
  splitf[i] = o == kSplit ? 1 : 0;
}

// std::mt19937_64 (the standard's parameters): n 312, m 156, r 31, a 0xB5026F5AA96619E9,
// tempering (u 29, d 0x5555555555555555), (s 17, b 0x71D67FFFEDA60000),
// (t 37, c 0xFFF7EEE000000000), l 43. state = {x[0..311], p} as libstdc++ keeps it (the
// text form Rng::save_state writes). One CTA: the twist in three data-parallel phases.
constexpr int kMtN = 312, kMtM = 156;
constexpr unsigned long long kMtA = 0xB5026F5AA96619E9ull, kUpper = ~0ull << 31, kLower = (1ull << 31) - 1;

__device__ __forceinline__ unsigned long long mt_mix(unsigned long long y) { return (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull); }

__global__ void __launch_bounds__(320) k_mt_generate(unsigned long long* __restrict__ state,
                                                     unsigned long long* __restrict__ out, int64_t count) {
  __shared__ unsigned long long x[kMtN];
  const int t = threadIdx.x;
  if (t < kMtN) x[t] = state[t];
  int p = static_cast<int>(state[kMtN]);
  __syncthreads();
  int64_t done = 0;
  while (done < count) {
    if (p >= kMtN) {
      // phase A (k < n - m): old x[k], x[k + 1], x[k + m]; phase B (n - m <= k < n - 1):
      // old x[k], x[k + 1] and NEW x[k - (n - m)]; k = n - 1: old x[n - 1], NEW x[0], x[m - 1]
      unsigned long long ya = 0, yb = 0, old_last = 0;
      if (t < kMtN - kMtM) {
        ya = x[t + kMtM] ^ mt_mix((x[t] & kUpper) | (x[t + 1] & kLower));
      } else if (t < kMtN - 1) {
        yb = (x[t] & kUpper) | (x[t + 1] & kLower);
      } else if (t == kMtN - 1) {
        old_last = x[t];
      }
      __syncthreads();
      if (t < kMtN - kMtM) x[t] = ya;
      __syncthreads();
      if (t >= kMtN - kMtM && t < kMtN - 1) {
        x[t] = x[t - (kMtN - kMtM)] ^ mt_mix(yb);
      } else if (t == kMtN - 1) {
        x[t] = x[kMtM - 1] ^ mt_mix((old_last & kUpper) | (x[0] & kLower));
      }
      __syncthreads();
      p = 0;
    }
    const int64_t take = min(static_cast<int64_t>(kMtN - p), count - done);
    for (int k = t; k < take; k += blockDim.x) {
      unsigned long long y = x[p + k];
      y ^= (y >> 29) & 0x5555555555555555ull;
      y ^= (y << 17) & 0x71D67FFFEDA60000ull;
      y ^= (y << 37) & 0xFFF7EEE000000000ull;
      y ^= y >> 43;
      out[done + k] = y;
    }
    p += static_cast<int>(take);
    done += take;
  }
  __syncthreads();
  if (t < kMtN) state[t] = x[t];
  if (t == 0) state[kMtN] = static_cast<unsigned long long>(p);
}

// Rng::normal (rng.hpp:41-46) from two consecutive draws.
__device__ __forceinline__ double rng_normal(unsigned long long d0, unsigned long long d1) {
  const double u1 = 1.0 - static_cast<double>(d0 >> 11) * 0x1.0p-53;
  const double u2 = static_cast<double>(d1 >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

struct CtrlOut {
  double *pos, *ls, *q, *raw;
  double *m_pos, *v_pos, *m_ls, *v_ls, *m_rot, *v_rot, *m_dens, *v_dens;
};
struct CtrlIn {
  const double *m_pos, *v_pos, *m_ls, *v_ls, *m_rot, *v_rot, *m_dens, *v_dens;
};

__device__ __forceinline__ void put_params(const CtrlOut& o, int64_t r, const double* p, const double* l,
                                           const double* q, double raw) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    o.pos[3 * r + a] = p[a];
    o.ls[3 * r + a] = l[a];
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) o.q[4 * r + a] = q[a];
  o.raw[r] = raw;
}

__device__ __forceinline__ void put_moments(const CtrlOut& o, int64_t r, const CtrlIn* in, int64_t i) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    o.m_pos[3 * r + a] = in ? in->m_pos[3 * i + a] : 0.0;
    o.v_pos[3 * r + a] = in ? in->v_pos[3 * i + a] : 0.0;
    o.m_ls[3 * r + a] = in ? in->m_ls[3 * i + a] : 0.0;
    o.v_ls[3 * r + a] = in ? in->v_ls[3 * i + a] : 0.0;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    o.m_rot[4 * r + a] = in ? in->m_rot[4 * i + a] : 0.0;
    o.v_rot[4 * r + a] = in ? in->v_rot[4 * i + a] : 0.0;
  }
  o.m_dens[r] = in ? in->m_dens[i] : 0.0;
  o.v_dens[r] = in ? in->v_dens[i] : 0.0;
}

// The split children's normals: `Vec3 z(rng.normal(), rng.normal(), rng.normal())`
// (optim.hpp:301) -- the order the three constructor arguments are evaluated in is the
// compiler's; GCC on x86-64 evaluates them right to left, so z[2] takes the first normal.
#ifndef GSCT_SPLIT_ARG_ORDER_RTL
#define GSCT_SPLIT_ARG_ORDER_RTL 1
#endif

__global__ void __launch_bounds__(256) k_ctrl_write(Cloud c, CtrlIn in, const double* __restrict__ acc_dir,
                                                    const uint8_t* __restrict__ op, const int* __restrict__ row_off,
                                                    const int* __restrict__ split_idx,
                                                    const unsigned long long* __restrict__ draws,
                                                    double log_1p6, CtrlOut o) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= c.n) return;
  const uint8_t k = op[i];
  if (k == kPrune) return;
  const int64_t r = row_off[i];
  double p[3], l[3], q[4];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    p[a] = c.pos[3 * i + a];
    l[a] = c.ls[3 * i + a];
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) q[a] = c.q[4 * i + a];
  const double raw = c.raw[i];
  if (k == kKeep || k == kClone) {
    put_params(o, r, p, l, q, raw);
    put_moments(o, r, &in, i);
  }
  if (k == kKeep) return;
  Act act;
  activate(c.pos, c.ls, c.q, c.raw, i, act);
  if (k == kClone) {
    // optim.hpp:284-295: the copy nudged along the summed descent direction
    const double d0 = acc_dir[3 * i], d1 = acc_dir[3 * i + 1], d2 = acc_dir[3 * i + 2];
    const double norm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    double np[3] = {p[0], p[1], p[2]};
    if (norm > 0.0) {
      const double nudge = 0.5 * ((act.scales[0] + act.scales[1] + act.scales[2]) / 3.0);
      np[0] -= (d0 / norm) * nudge;
      np[1] -= (d1 / norm) * nudge;
      np[2] -= (d2 / norm) * nudge;
    }
    put_params(o, r + 1, np, l, q, raw);
    put_moments(o, r + 1, nullptr, 0);
    return;
  }
  // split (optim.hpp:296-305): two children, scales / 1.6, positions sampled from the parent
  double R[9];
  rotation_matrix(act.uq, R);
  const double cl[3] = {l[0] - log_1p6, l[1] - log_1p6, l[2] - log_1p6};
  const unsigned long long* d = draws + 12 * static_cast<int64_t>(split_idx[i]);
#pragma unroll
  for (int child = 0; child < 2; ++child) {
    double z[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int slot = GSCT_SPLIT_ARG_ORDER_RTL ? 2 - s : s;
      z[slot] = rng_normal(d[6 * child + 2 * s], d[6 * child + 2 * s + 1]);
    }
    const double w0 = act.scales[0] * z[0], w1 = act.scales[1] * z[1], w2 = act.scales[2] * z[2];
    double cp[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) cp[a] = p[a] + ((R[3 * a] * w0 + R[3 * a + 1] * w1) + R[3 * a + 2] * w2);
    put_params(o, r + child, cp, cl, q, raw);
    put_moments(o, r + child, nullptr, 0);
  }
}

}  // namespace

void launch_ctrl_accumulate(int64_t n, const uint8_t* visible, const double* pgn, const double* g_pos,
                            double* acc_norm, double* acc_dir, int64_t* acc_count, cudaStream_t st) {
  if (n == 0) return;
  k_ctrl_accumulate<<<blocks_for(n, 256), 256, 0, st>>>(n, visible, pgn, g_pos, acc_norm, acc_dir, acc_count);
  count_launch();
}

size_t ctrl_scratch_bytes(int64_t n) {
  size_t scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan, static_cast<int*>(nullptr), static_cast<int*>(nullptr),
                                static_cast<int>(n));
  return 8 * static_cast<size_t>(n) * sizeof(int) + static_cast<size_t>(n) + 64 + 256 + scan;
}

namespace {
struct CtrlScratch {
  int *keep, *keep_off, *elig, *elig_rank, *rows, *row_off, *splitf, *split_idx;
  uint8_t* op;
  unsigned long long* small;  // {max_bits, err_key, survivors, cloned, split}
  void* scan_tmp;
  size_t scan_bytes;
};
CtrlScratch carve(void* base, int64_t n) {
  CtrlScratch s;
  const size_t un = static_cast<size_t>(n);
  char* p = static_cast<char*>(base);
  s.small = reinterpret_cast<unsigned long long*>(p);
  p += 64;
  int* ints = reinterpret_cast<int*>(p);
  s.keep = ints;
  s.keep_off = ints + un;
  s.elig = ints + 2 * un;
  s.elig_rank = ints + 3 * un;
  s.rows = ints + 4 * un;
  s.row_off = ints + 5 * un;
  s.splitf = ints + 6 * un;
  s.split_idx = ints + 7 * un;
  p += 8 * un * sizeof(int);
  s.op = reinterpret_cast<uint8_t*>(p);
  p += un;
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  s.scan_tmp = p;
  s.scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, s.scan_bytes, static_cast<int*>(nullptr), static_cast<int*>(nullptr),
                                static_cast<int>(n));
  return s;
}
}  // namespace

#define CTRL_CK(call)                  \
  do {                                 \
    const cudaError_t e_ = (call);     \
    if (e_ != cudaSuccess) return e_;  \
  } while (0)

cudaError_t launch_ctrl_classify(const Cloud& c, double prune_density, double grad_threshold, double split_below,
                                 int64_t max_gaussians, const double* acc_norm, const int64_t* acc_count,
                                 void* scratch, unsigned long long* small_host, cudaStream_t st) {
  const int64_t n = c.n;
  CtrlScratch s = carve(scratch, n);
  CTRL_CK(cudaMemsetAsync(s.small, 0, 64, st));
  CTRL_CK(cudaMemsetAsync(s.small + 1, 0xff, sizeof(unsigned long long), st));
  const unsigned b = blocks_for(n, 256);
  k_ctrl_activate<<<b, 256, 0, st>>>(c, s.small, s.small + 1);
  k_ctrl_flags<<<b, 256, 0, st>>>(c, s.small, prune_density, grad_threshold, acc_norm, acc_count, s.keep, s.elig);
  const int ni = static_cast<int>(n);
  size_t tb = s.scan_bytes;
  CTRL_CK(cub::DeviceScan::ExclusiveSum(s.scan_tmp, tb, s.keep, s.keep_off, ni, st));
  CTRL_CK(cub::DeviceScan::ExclusiveSum(s.scan_tmp, tb, s.elig, s.elig_rank, ni, st));
  k_ctrl_ops<<<b, 256, 0, st>>>(c, s.keep, s.keep_off, s.elig, s.elig_rank, max_gaussians, split_below, s.op, s.rows,
                                s.splitf, s.small + 2);
  CTRL_CK(cub::DeviceScan::ExclusiveSum(s.scan_tmp, tb, s.rows, s.row_off, ni, st));
  CTRL_CK(cub::DeviceScan::ExclusiveSum(s.scan_tmp, tb, s.splitf, s.split_idx, ni, st));
  count_launch(3);
  return cudaMemcpyAsync(small_host, s.small, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
}

void launch_mt_generate(unsigned long long* state_dev, unsigned long long* out, int64_t count, cudaStream_t st) {
  k_mt_generate<<<1, 320, 0, st>>>(state_dev, out, count);
  count_launch();
}

void launch_ctrl_write(const Cloud& c, const double* const* mv_in, const double* acc_dir, void* scratch,
                       const unsigned long long* draws, double log_1p6, double* pos, double* ls, double* q,
                       double* raw, double* const* mv_out, cudaStream_t st) {
  const int64_t n = c.n;
  CtrlScratch s = carve(scratch, n);
  CtrlIn in{mv_in[0], mv_in[1], mv_in[2], mv_in[3], mv_in[4], mv_in[5], mv_in[6], mv_in[7]};
  CtrlOut o{pos, ls, q, raw, mv_out[0], mv_out[1], mv_out[2], mv_out[3], mv_out[4], mv_out[5], mv_out[6], mv_out[7]};
  k_ctrl_write<<<blocks_for(n, 256), 256, 0, st>>>(c, in, acc_dir, s.op, s.row_off, s.split_idx, draws, log_1p6, o);
  count_launch();
}

}  // namespace gsct_dev
