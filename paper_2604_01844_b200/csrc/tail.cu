// Raster backward tail (K4b) and finalize, fp64. Unlike preprocess.cu this translation unit
// is compiled WITH FMA contraction: nothing here feeds an integer box or key, results only
// need to agree with the reference within the gradient tolerance, and contracted DFMAs
// halve the fp64 instruction count of the (latency-bound) chain rule.
#include <cuda_runtime.h>

#include "gsct_internal.cuh"

namespace gsct_dev {

namespace {

// Four lanes per splat (8 splats per warp): lane q of a group takes views q, q+4, q+8, ...
// of ALL views of the call (75 views -> 19/19/19/18, no idle rounds), re-derives the fp64
// projection without the box / eigen tests (visibility comes from the pixel-loop flag),
// turns the fp32 moments into dL/d(amp, mean2d, conic) and runs the reference chain rule
// (projector.hpp:422-472) up to dL/dSigma. The four per-lane view sums are combined with a
// fixed 2-step xor tree inside the aligned group, so a splat's result depends only on its
// own inputs (ParamGradients::add up to fp64 reassociation; duplicates stay identical).
// acc layout [11][N]: g_pos(3), g_sigma(00,01,02,11,12,22), g_raw, sum |dL/dmean2d|.
#ifndef GSCT_TAIL_PAD
#define GSCT_TAIL_PAD 1
#endif
struct PaddedFrame {
  Frame f;
#if GSCT_TAIL_PAD
  double pad[GSCT_TAIL_PAD];
#endif
};

#ifndef GSCT_TAIL_SPRE
#define GSCT_TAIL_SPRE 1
#endif
struct PaddedPre {
  PreSplat p;
  double pad;
};
static_assert(sizeof(PreSplat) % sizeof(double) == 0, "PreSplat: whole doubles");

#ifndef GSCT_TAIL_LANES
#define GSCT_TAIL_LANES 4  // lanes per splat (each takes every L-th view); A/B C2 2/4/8: 0.737/0.731/0.810 ms
#endif
constexpr int kTL = GSCT_TAIL_LANES, kTLog = kTL == 8 ? 3 : (kTL == 4 ? 2 : (kTL == 2 ? 1 : 0));
constexpr int kTSplats = 128 / kTL;  // splats per 128-thread block

#ifndef GSCT_TAIL_MINB
#define GSCT_TAIL_MINB 4  // 128 registers
#endif
__global__ void __launch_bounds__(128, GSCT_TAIL_MINB) k_raster_tail(const PreSplat* __restrict__ pre /* AoS */, int64_t n,
                                                     int64_t i0, int64_t i1,
                                                     const Frame* __restrict__ frames_g, int n_views,
                                                     Geo g, RSet rs, const float4* __restrict__ moments,
                                                     int frames_in_smem, double* __restrict__ acc,
                                                     uint8_t* __restrict__ visible) {
  // smem frames padded to 17 doubles: the 4 lanes of a group read 4 different views, which
  // at the natural 128 B stride would all hit the same banks (4-way conflicts)
  extern __shared__ PaddedFrame s_frames[];
  if (frames_in_smem)
    for (int k = threadIdx.x; k < n_views; k += blockDim.x) s_frames[k].f = frames_g[k];
#if GSCT_TAIL_SPRE
  // the block's 32 splat set-ups staged in shared memory at a 200 B stride (8 distinct
  // splats per warp access: conflict-free banks), instead of 8 L1 lines per field load
  __shared__ PaddedPre s_pre[kTSplats];
  {
    const int64_t first = i0 + static_cast<int64_t>(blockIdx.x) * kTSplats;
    const int cnt = i1 - first < kTSplats ? static_cast<int>(i1 - first) : kTSplats;
    const double* src = reinterpret_cast<const double*>(pre + first);
    constexpr int kD = sizeof(PreSplat) / sizeof(double);
    for (int k = threadIdx.x; k < cnt * kD; k += blockDim.x)
      reinterpret_cast<double*>(&s_pre[k / kD].p)[k % kD] = src[k];
  }
#endif
  __syncthreads();
  const auto frame = [&](int vw) -> const Frame& { return frames_in_smem ? s_frames[vw].f : frames_g[vw]; };
  const int q = threadIdx.x & (kTL - 1);
  const int64_t i = i0 + ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> kTLog);
  const bool live = i < i1;
  double v[11];
#pragma unroll
  for (int k = 0; k < 11; ++k) v[k] = 0.0;
  bool vis = false;
  if (live) {
#if GSCT_TAIL_SPRE
    const PreSplat& s = s_pre[threadIdx.x >> kTLog].p;
#else
    const PreSplat& s = pre[i];  // array-of-structs copy (fields re-read from L1 as needed)
#endif
    if (s.status == 0) {
      for (int vw = q; vw < n_views; vw += kTL) {
        const int64_t item = static_cast<int64_t>(vw) * n + i;
        const float4 m1 = moments[2 * item + 1];
        if (m1.z == 0.f) continue;  // culled or degenerate in this view
        const float4 m0 = moments[2 * item];
        Proj p;
        const Frame& fr = frame(vw);
        project_full<false>(fr, g, s.pos, s.sigma, s.sigma_inv, s.det_ok != 0, s.density, rs, p);
        if (p.degenerate) continue;
        vis = true;
        // m0 = {sum t, sum t du, sum t dv, sum t du^2}, m1 = {sum t du dv, sum t dv^2, 1, -}
        const double amp = p.amplitude;
        const double a_ = p.conic[0], b_ = p.conic[1], c_ = p.conic[3];
        const double Mu = m0.y, Mv = m0.z;
        double gm[2], gc[4];
        gm[0] = amp * (a_ * Mu + b_ * Mv);
        gm[1] = amp * (b_ * Mu + c_ * Mv);
        gc[0] = -0.5 * amp * static_cast<double>(m0.w);
        gc[1] = -0.5 * amp * static_cast<double>(m1.x);
        gc[2] = gc[1];
        gc[3] = -0.5 * amp * static_cast<double>(m1.y);
        double gp[3], gs[9], gr;
        raster_chain_rule(fr, g, rs, s.density, s.raw_density, s.sigma, p, static_cast<double>(m0.x), gm,
                          gc, gp, gs, gr);
        v[0] += gp[0];
        v[1] += gp[1];
        v[2] += gp[2];
        v[3] += gs[0];
        v[4] += gs[1];
        v[5] += gs[2];
        v[6] += gs[4];
        v[7] += gs[5];
        v[8] += gs[8];
        v[9] += gr;
        v[10] += sqrt(gm[0] * gm[0] + gm[1] * gm[1]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 11; ++k) {
#pragma unroll
    for (int o = 1; o < kTL; o <<= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  const unsigned ball = __ballot_sync(0xffffffffu, vis);
  if (live && q == 0) {
#pragma unroll
    for (int k = 0; k < 11; ++k) acc[k * n + i] = v[k];
    visible[i] = static_cast<uint8_t>(((ball >> (threadIdx.x & 31)) & ((1u << kTL) - 1u)) != 0u);
  }
}

// Per-splat finalize: covariance_backward (core.hpp:170-191) of the summed dL/dSigma.
// bulk_out (host-mapped gradients): the block's 128 splats are staged in shared memory and
// leave as five contiguous TMA bulk stores (cp.async.bulk), so the strided per-splat stores
// do not cross PCIe one by one (a block whose byte counts are not 16-byte multiples --
// only an odd-sized last block -- stores directly).
__global__ void __launch_bounds__(128) k_raster_finalize(Cloud c, int64_t i0, int64_t i1,
                                                         const double* __restrict__ acc,
                                                         double* __restrict__ g_pos, double* __restrict__ g_ls,
                                                         double* __restrict__ g_q, double* __restrict__ g_raw,
                                                         double* __restrict__ g_pgn, int bulk_out) {
  __shared__ double s_out[128 * 12];
  const int64_t b0 = i0 + static_cast<int64_t>(blockIdx.x) * blockDim.x;
  const int64_t i = b0 + threadIdx.x;
  const int cnt = i1 - b0 < 128 ? static_cast<int>(i1 - b0) : 128;
  const bool bulk = bulk_out && (cnt % 2) == 0;
  const int64_t n = c.n;
  if (i < i1) {
    double gl[3] = {0, 0, 0}, gq[4] = {0, 0, 0, 0};
    Act a;
    if (activate(c.pos, c.ls, c.q, c.raw, i, a) == 0) {
      const double s00 = acc[3 * n + i], s01 = acc[4 * n + i], s02 = acc[5 * n + i];
      const double s11 = acc[6 * n + i], s12 = acc[7 * n + i], s22 = acc[8 * n + i];
      const double gsig[9] = {s00, s01, s02, s01, s11, s12, s02, s12, s22};
      covariance_backward(a.scales, a.uq, a.raw_q, gsig, gl, gq);
    }
    if (bulk) {
      const int t = threadIdx.x;
      double* sp = s_out;                // pos   [cnt][3]
      double* sl = s_out + 3 * cnt;      // ls    [cnt][3]
      double* sq = s_out + 6 * cnt;      // quat  [cnt][4]
      double* sr = s_out + 10 * cnt;     // raw   [cnt]
      double* sn = s_out + 11 * cnt;     // |dL/dmean2d| [cnt]
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        sp[3 * t + k] = acc[k * n + i];
        sl[3 * t + k] = gl[k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) sq[4 * t + k] = gq[k];
      sr[t] = acc[9 * n + i];
      sn[t] = acc[10 * n + i];
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        g_pos[3 * i + k] = acc[k * n + i];
        g_ls[3 * i + k] = gl[k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) g_q[4 * i + k] = gq[k];
      g_raw[i] = acc[9 * n + i];
      g_pgn[i] = acc[10 * n + i];
    }
  }
  if (!bulk) return;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(s_out));
    const uint32_t c8 = static_cast<uint32_t>(cnt) * 8u;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g_pos + 3 * b0), "r"(sb),
                 "r"(3u * c8) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g_ls + 3 * b0),
                 "r"(sb + 3u * c8), "r"(3u * c8) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g_q + 4 * b0),
                 "r"(sb + 6u * c8), "r"(4u * c8) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g_raw + b0),
                 "r"(sb + 10u * c8), "r"(c8) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g_pgn + b0),
                 "r"(sb + 11u * c8), "r"(c8) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

inline unsigned blocks_for(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

}  // namespace

void launch_raster_tail(const PreSplat* pre, int64_t n, int64_t i0, int64_t i1, const Frame* frames_dev,
                        int n_views, const Geo& g, const RSet& rs, const float* moments, double* acc,
                        uint8_t* visible, cudaStream_t st) {
  if (i1 <= i0) return;
  const size_t smem = static_cast<size_t>(n_views) * sizeof(PaddedFrame);
  const bool in_smem = smem <= 24 * 1024;
  k_raster_tail<<<blocks_for((i1 - i0) * kTL, 128), 128, in_smem ? smem : 0, st>>>(
      pre, n, i0, i1, frames_dev, n_views, g, rs, reinterpret_cast<const float4*>(moments), in_smem ? 1 : 0, acc,
      visible);
  count_launch();
}

void launch_raster_finalize(const Cloud& c, int64_t i0, int64_t i1, const double* acc, double* g_pos, double* g_ls,
                            double* g_q, double* g_raw, double* g_pgn, cudaStream_t st, int bulk_out) {
  if (i1 <= i0) return;
  k_raster_finalize<<<blocks_for(i1 - i0, 128), 128, 0, st>>>(c, i0, i1, acc, g_pos, g_ls, g_q, g_raw, g_pgn,
                                                              bulk_out);
  count_launch();
}

}  // namespace gsct_dev
