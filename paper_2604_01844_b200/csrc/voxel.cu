// Voxelizer pair kernels (fp32): brick-pair emission (K6b), the per-brick forward sum
// (K7), the backward walk-order keys and the per-splat backward voxel walk (K8a).
//
// K7 follows voxelize (voxelizer.hpp:162-199): each voxel sums, in ascending splat index,
// rho * exp(-q/2) of every splat whose box contains it. Instead of the reference's
// "every z slice scans all N splats" (an O(n_z * N) skip scan), splats are binned into
// 8x8x8 bricks with a stable sort, so each brick visits only its own ascending list.
// K8a follows voxelize_backward's loop (voxelizer.hpp:235-249): ONE LANE owns a splat and
// walks its own box sequentially, so gradients are bit-stable without atomics.
#include <cuda_runtime.h>

#include <type_traits>

#include "gsct_internal.cuh"
#include "packed_f32.cuh"

namespace gsct_dev {

namespace {

__global__ void k_emit_brick_pairs(const VoxelRec* __restrict__ rec,
                                   const uint32_t* __restrict__ offsets,
                                   const uint32_t* __restrict__ counts, int64_t n, Window win,
                                   int nbx, int nby, uint32_t* __restrict__ keys,
                                   uint32_t* __restrict__ vals) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (counts[i] == 0) return;
  const VoxelRec r = rec[i];
  // record boxes are grid-clipped; bin only the part inside the window
  const int x0 = max(static_cast<int>(r.lox), win.lo[0]), x1 = min(static_cast<int>(r.hix), win.hi[0] - 1);
  const int y0 = max(static_cast<int>(r.loy), win.lo[1]), y1 = min(static_cast<int>(r.hiy), win.hi[1] - 1);
  const int z0 = max(static_cast<int>(r.loz), win.lo[2]), z1 = min(static_cast<int>(r.hiz), win.hi[2] - 1);
  const int bx0 = (x0 - win.lo[0]) / kBrick, bx1 = (x1 - win.lo[0]) / kBrick;
  const int by0 = (y0 - win.lo[1]) / kBrick, by1 = (y1 - win.lo[1]) / kBrick;
  const int bz0 = (z0 - win.lo[2]) / kBrickZ, bz1 = (z1 - win.lo[2]) / kBrickZ;
  uint32_t off = offsets[i];
  for (int bz = bz0; bz <= bz1; ++bz)
    for (int by = by0; by <= by1; ++by)
      for (int bx = bx0; bx <= bx1; ++bx) {
        keys[off] = static_cast<uint32_t>((bz * nby + by) * nbx + bx);
        vals[off] = static_cast<uint32_t>(i);
        ++off;
      }
}



// Warp-cooperative form of k_emit_brick_pairs: the 32 splats of a warp hold a contiguous run
// of the pair array (offsets are the exclusive scan of the counts in splat order), so the
// warp writes that run with coalesced stores -- pair p of the run goes to the lane whose
// prefix covers p, decoded into its (bz, by, bx) in the same bz-by-bx order -- instead of
// every lane storing its own run (32 scattered runs per store instruction).
__global__ void __launch_bounds__(256) k_emit_brick_pairs_warp(const VoxelRec* __restrict__ rec,
                                                               const uint32_t* __restrict__ offsets,
                                                               const uint32_t* __restrict__ counts, int64_t n,
                                                               Window win, int nbx, int nby,
                                                               uint32_t* __restrict__ keys,
                                                               uint32_t* __restrict__ vals) {
  __shared__ int s_box[8][32][4];  // per warp, per lane: run start (in the warp's run), bx0, by0 | nx, bz0 | ny
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t c = 0;
  int bx0 = 0, by0 = 0, bz0 = 0, nx = 1, ny = 1;
  if (i < n) {
    c = counts[i];
    if (c) {
      const VoxelRec r = rec[i];
      // record boxes are grid-clipped; bin only the part inside the window
      const int x0 = max(static_cast<int>(r.lox), win.lo[0]), x1 = min(static_cast<int>(r.hix), win.hi[0] - 1);
      const int y0 = max(static_cast<int>(r.loy), win.lo[1]), y1 = min(static_cast<int>(r.hiy), win.hi[1] - 1);
      const int z0 = max(static_cast<int>(r.loz), win.lo[2]);
      bx0 = (x0 - win.lo[0]) / kBrick;
      by0 = (y0 - win.lo[1]) / kBrick;
      bz0 = (z0 - win.lo[2]) / kBrickZ;
      nx = (x1 - win.lo[0]) / kBrick - bx0 + 1;
      ny = (y1 - win.lo[1]) / kBrick - by0 + 1;
    }
  }
  uint32_t ex = c;  // inclusive warp scan, then exclusive
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, ex, o);
    if (lane >= o) ex += y;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, ex, 31);
  ex -= c;
  const uint32_t base = __shfl_sync(0xffffffffu, i < n ? offsets[i] : 0u, 0);
  s_box[w][lane][0] = static_cast<int>(ex);
  s_box[w][lane][1] = bx0;
  s_box[w][lane][2] = by0 | (nx << 16);
  s_box[w][lane][3] = bz0 | (ny << 16);
  __syncwarp();
  const int64_t i0 = i - lane;
  for (uint32_t p = lane; p < total; p += 32) {
    // owner: the last lane whose run starts at or before p (lanes with empty runs share
    // their start with the next lane and are skipped by taking the last such lane)
    int lo = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
      if (static_cast<uint32_t>(s_box[w][lo + step][0]) <= p) lo += step;
    const int j = static_cast<int>(p - static_cast<uint32_t>(s_box[w][lo][0]));
    const int b1 = s_box[w][lo][1], b2 = s_box[w][lo][2], b3 = s_box[w][lo][3];
    const int onx = b2 >> 16, ony = b3 >> 16;
    const int nxy = onx * ony;
    const int bz = j / nxy, rem = j - bz * nxy;
    const int by = rem / onx, bx = rem - by * onx;
    keys[base + p] = static_cast<uint32_t>(((bz + (b3 & 0xFFFF)) * nby + by + (b2 & 0xFFFF)) * nbx + bx + b1);
    vals[base + p] = static_cast<uint32_t>(i0 + lo);
  }
}

__device__ __forceinline__ float vox_e(const VoxelRec& r, float dx, float dy, float dz) {
  // Q00 dx^2 + Q11 dy^2 + Q22 dz^2 + Q01 dx dy + Q02 dx dz + Q12 dy dz
  return fmaf(dx, fmaf(r.Q00, dx, fmaf(r.Q01, dy, r.Q02 * dz)), fmaf(dy, fmaf(r.Q11, dy, r.Q12 * dz), r.Q22 * dz * dz));
}

struct __align__(16) StagedVox {
  float4 p;  // dx_b, dy_b (offsets of the brick origin voxel), z0 - lo_z (exact), rho
  float4 q;  // Q00, Q11, Q22, Q01
  float4 r;  // Q02, Q12, c = exp2(2 Q00 sp^2), chain-safe flag
  uint4 m;   // x mask | y mask << 8, lane mask, lane of the exact-peak row (or ~0), bits of off_z
};

// Forward (K7): one WARP per 8 x 8 x 16 brick (4 per CTA); lane l owns four x-rows of 8
// voxels: y = 2(l & 3), +1 (the halves of packed f32x2 registers) at z = 2(l >> 2), +1. The
// brick's splat list (ascending index = the reference's per-voxel order) is staged 32
// records at a time in warp-private shared memory; each lane walks only the records whose
// box meets its rows (32x32 warp bit transpose of the staged lane masks), so a staged
// record's set-up is shared by up to 32 voxels of the lane. Along x the Gaussian is a 1-D
// quadratic in the exponent, evaluated multiplicatively (g <- g r, r <- r c: 2 packed FMULs
// per voxel pair, one MUFU pair per row pair to start), with a per-record safety flag (no
// fp32 under/overflow anywhere in the brick window) falling back to direct exp2; the rows
// holding an exactly-on-lattice centre also use the direct path so the peak voxel is
// rho * exp2(0) = rho exactly (test_voxelizer.cpp:16-22).
#ifndef GSCT_VFWD_PACK
#define GSCT_VFWD_PACK 1  // staged record fields ordered so the walk loads 56 of its 64 bytes
#endif
#ifndef GSCT_VFWD_PLAIN_BATCH
#define GSCT_VFWD_PLAIN_BATCH 1
#endif
#ifndef GSCT_VFWD_MINB
#define GSCT_VFWD_MINB 7  // 72 registers, 7 CTAs/SM (A/B 512^3 before the packed staging: 5 CTAs 1.011 ms,
                          // 6 0.976, 7 1.001, 8 1.096; with it: 6 0.945, 7 0.936 -- 1024^3 5.67 / 5.61)
#endif
#ifndef GSCT_VFWD_UNROLL
#define GSCT_VFWD_UNROLL 1  // (2: 0.985 ms with 6 CTAs)
#endif
constexpr int kVfwdUnroll = GSCT_VFWD_UNROLL;
__global__ void __launch_bounds__(128, GSCT_VFWD_MINB) k_voxel_fwd2(const VoxelRec* __restrict__ rec,
                                                   const uint32_t* __restrict__ vals,
                                                   const uint32_t* __restrict__ start,
                                                   const uint32_t* __restrict__ end, Window win,
                                                   int nbx, int nby, int n_bricks, float sp,
                                                   float* __restrict__ volume, const uint32_t* __restrict__ sched) {
  __shared__ StagedVox s_rec[4][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * 4 + warp;
  if (w >= n_bricks) return;
  const int brick = sched ? static_cast<int>(__ldg(sched + w)) : w;  // longest lists first
  const int bx = brick % nbx, by = (brick / nbx) % nby, bz = brick / (nbx * nby);
  const int gx0 = win.lo[0] + bx * kBrick, gy0 = win.lo[1] + by * kBrick, gz0 = win.lo[2] + bz * kBrickZ;
  const int yp = lane & 3, zp = lane >> 2;
  const float fy = static_cast<float>(2 * yp) * sp;
  const uint32_t b = start[brick], e = end[brick];
  StagedVox* sw = s_rec[warp];
  float2 acc[2][8];  // [z][x] {y row 0, y row 1}
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[0][k] = acc[1][k] = make_float2(0.f, 0.f);
  for (uint32_t base = b; base < e; base += 32) {
    const int cnt = min(32u, e - base);
    uint32_t lanes_rel = 0u;
    bool my_plain = true;  // the staged record is chain-safe and has no lattice-exact peak here
    if (lane < cnt) {
      const VoxelRec r = rec[vals[base + lane]];
      StagedVox s;
      const int ilx = static_cast<int>(r.lox), ily = static_cast<int>(r.loy), ilz = static_cast<int>(r.loz);
      const int x_lo = max(ilx - gx0, 0), x_hi = min(static_cast<int>(r.hix) - gx0, kBrick - 1);
      const int y_lo = max(ily - gy0, 0), y_hi = min(static_cast<int>(r.hiy) - gy0, kBrick - 1);
      const int z_lo = max(ilz - gz0, 0), z_hi = min(static_cast<int>(r.hiz) - gz0, kBrickZ - 1);
      const uint32_t xm = ((2u << x_hi) - 1u) & ~((1u << x_lo) - 1u);
      const uint32_t ym = ((2u << y_hi) - 1u) & ~((1u << y_lo) - 1u);
      const uint32_t zm = ((2u << z_hi) - 1u) & ~((1u << z_lo) - 1u);
      const uint32_t ypairs = ((2u << (y_hi >> 1)) - 1u) & ~((1u << (y_lo >> 1)) - 1u);
      const uint32_t zpairs = (0x11111111u >> (4 * (7 - (z_hi >> 1)))) & (0x11111111u << (4 * (z_lo >> 1)));
      lanes_rel = zpairs * ypairs;
      const float dxb = fmaf(static_cast<float>(gx0 - ilx), sp, -r.offx);
      const float dyb = fmaf(static_cast<float>(gy0 - ily), sp, -r.offy);
      // z offsets are formed per lane from the absolute slice index (fmaf(z - lo, sp, -off)),
      // and the safety window spans the whole box in z, so z-slab windows reproduce the
      // full-grid volume bit for bit
      const float fgz = static_cast<float>(gz0 - ilz);
      // chain-safety window: x 0..7, rows (y_lo & ~1) .. (y_hi | 1), the whole box in z
      const float xa = dxb, xb = dxb + 7.f * sp, xc = dxb + 6.f * sp;
      const float ya = dyb + static_cast<float>(y_lo & ~1) * sp, yb = dyb + static_cast<float>(y_hi | 1) * sp;
      const float za = -r.offz, zb = fmaf(static_cast<float>(static_cast<int>(r.hiz) - ilz), sp, -r.offz);
      float emin = fminf(fminf(fminf(vox_e(r, xa, ya, za), vox_e(r, xa, ya, zb)), fminf(vox_e(r, xa, yb, za), vox_e(r, xa, yb, zb))),
                         fminf(fminf(vox_e(r, xb, ya, za), vox_e(r, xb, ya, zb)), fminf(vox_e(r, xb, yb, za), vox_e(r, xb, yb, zb))));
      // D(x) = e(x + sp) - e(x) = Q00 (2 x sp + sp^2) + (Q01 y + Q02 z) sp: linear, extremes at corners
      float dmax = 0.f;
#pragma unroll
      for (int cx = 0; cx < 2; ++cx)
#pragma unroll
        for (int cy = 0; cy < 2; ++cy)
#pragma unroll
          for (int cz = 0; cz < 2; ++cz) {
            const float x = cx ? xc : xa, y = cy ? yb : ya, z = cz ? zb : za;
            dmax = fmaxf(dmax, fabsf(fmaf(r.Q00, fmaf(2.f * x, sp, sp * sp), fmaf(r.Q01, y, r.Q02 * z) * sp)));
          }
      const float c2e = 2.f * r.Q00 * sp * sp;
      const bool safe = emin > -100.f && dmax < 100.f && c2e > -60.f;
      // exactly-on-lattice centre inside this brick -> that lane takes the direct path
      uint32_t peak = 0xFFFFFFFFu;
      const float cxf = r.offx / sp, cyf = r.offy / sp, czf = r.offz / sp;
      if (cxf == rintf(cxf) && cyf == rintf(cyf) && czf == rintf(czf)) {
        const int px = ilx + static_cast<int>(cxf) - gx0, py = ily + static_cast<int>(cyf) - gy0,
                  pz = ilz + static_cast<int>(czf) - gz0;
        if (px >= 0 && px < kBrick && py >= 0 && py < kBrick && pz >= 0 && pz < kBrickZ)
          peak = static_cast<uint32_t>((pz >> 1) * 4 + (py >> 1));  // the lane owning that row
      }
      s.p = make_float4(dxb, dyb, fgz, r.rho);
      s.q = make_float4(r.Q00, r.Q11, r.Q22, r.Q01);
#if GSCT_VFWD_PACK
      // the walk reads p, q, r and the first half of m (masks, peak): 56 of the 64 bytes
      s.r = make_float4(r.Q02, r.Q12, ex2_approx(c2e), r.offz);
      s.m = make_uint4(xm | (ym << 8) | (zm << 16), peak, safe ? 1u : 0u, lanes_rel);
#else
      s.r = make_float4(r.Q02, r.Q12, ex2_approx(c2e), safe ? 1.f : 0.f);
      s.m = make_uint4(xm | (ym << 8) | (zm << 16), lanes_rel, peak, __float_as_uint(r.offz));
#endif
      sw[lane] = s;
      my_plain = safe && peak == 0xFFFFFFFFu;
    }
    __syncwarp();
    uint32_t todo = warp_transpose32(lanes_rel, lane);
    // a batch of only plain records (the common case) walks without the direct-path branch
    auto walk = [&](auto plain) {
#pragma unroll kVfwdUnroll
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1u;
      const float4 p = sw[j].p;
      const float4 q = sw[j].q;
      const float4 rr4 = sw[j].r;
#if GSCT_VFWD_PACK
      const uint2 m = *reinterpret_cast<const uint2*>(&sw[j].m);  // masks, peak lane
      const float offz = rr4.w;
#else
      const uint4 m = sw[j].m;
      const float offz = __uint_as_float(m.w);
#endif
      const uint32_t xm = m.x & 0xFFu;
      const uint32_t rows = (m.x >> (8 + 2 * yp)) & 3u;
      const f2_t RHO = f2_pack((rows & 1u) ? p.w : 0.f, (rows & 2u) ? p.w : 0.f);
      const float dy0 = p.y + fy, dx0 = p.x;
      const f2_t DY = f2_pack(dy0, dy0 + sp);
#if GSCT_VFWD_PACK
      const bool direct = !decltype(plain)::value && (sw[j].m.z == 0u || m.y == static_cast<uint32_t>(lane));
#else
      const bool direct = !decltype(plain)::value && (rr4.w == 0.f || m.z == static_cast<uint32_t>(lane));
#endif
      // the exponent / chain arithmetic stays in inline-asm packed ops (never contracted, so a
      // voxel's value does not depend on which lane or unrolled z step computes it: z-slab
      // windows stay bit-identical); only the accumulation uses the __fadd2_rn builtin, which
      // ptxas predicates in place per x bit (a C-level `if` around an asm add left a
      // temporary + predicated MOV pairs)
      const auto accum = [&](float2& a, f2_t g) {
        float lo, hi;
        f2_unpack(g, lo, hi);
        a = __fadd2_rn(a, make_float2(lo, hi));
      };
#pragma unroll
      for (int zz = 0; zz < 2; ++zz) {
        if (!((m.x >> (16 + 2 * zp + zz)) & 1u)) continue;
        const float dz = fmaf(p.z + static_cast<float>(2 * zp + zz), sp, -offz);
        // e(dx) = Q00 dx^2 + L dx + K,  L = Q01 dy + Q02 dz,  K = Q11 dy^2 + Q12 dy dz + Q22 dz^2
        const f2_t L = f2_fma(f2_bc(q.w), DY, f2_bc(rr4.x * dz));
        const f2_t K = f2_fma(DY, f2_fma(f2_bc(q.y), DY, f2_bc(rr4.y * dz)), f2_bc(q.z * dz * dz));
        if (!direct) {
          const f2_t E0 = f2_fma(L, f2_bc(dx0), f2_add(K, f2_bc(q.x * dx0 * dx0)));
          const f2_t D0 = f2_fma(L, f2_bc(sp), f2_bc(q.x * fmaf(2.f * dx0, sp, sp * sp)));
          float e0, e1, d0, d1;
          f2_unpack(E0, e0, e1);
          f2_unpack(D0, d0, d1);
          f2_t g = f2_mul(f2_pack(ex2_approx(e0), ex2_approx(e1)), RHO);
          f2_t ratio = f2_pack(ex2_approx(d0), ex2_approx(d1));
          const f2_t C2 = f2_bc(rr4.z);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (xm & (1u << k)) accum(acc[zz][k], g);
            if (k < 7) g = f2_mul(g, ratio);
            if (k < 6) ratio = f2_mul(ratio, C2);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float dx = fmaf(static_cast<float>(k), sp, dx0);
            const f2_t ek = f2_fma(f2_add(f2_bc(q.x * dx), L), f2_bc(dx), K);
            float e0, e1;
            f2_unpack(ek, e0, e1);
            const f2_t g = f2_mul(f2_pack(ex2_approx(e0), ex2_approx(e1)), RHO);
            if (xm & (1u << k)) accum(acc[zz][k], g);
          }
        }
      }
    }
    };
#if GSCT_VFWD_PLAIN_BATCH
    if (__all_sync(0xffffffffu, my_plain))
      walk(std::integral_constant<bool, true>{});
    else
#endif
      walk(std::integral_constant<bool, false>{});
    __syncwarp();
  }
  const int wx = win.hi[0] - win.lo[0], wy = win.hi[1] - win.lo[1];
  const int x0 = gx0 - win.lo[0];
#pragma unroll
  for (int zz = 0; zz < 2; ++zz) {
    const int z = gz0 + 2 * zp + zz;
    if (z >= win.hi[2]) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int y = gy0 + 2 * yp + h;
      if (y >= win.hi[1]) continue;
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = h ? acc[zz][k].y : acc[zz][k].x;
      float* row = volume + (static_cast<int64_t>(z - win.lo[2]) * wy + (y - win.lo[1])) * wx;
      if ((wx & 3) == 0 && x0 + 8 <= wx) {
        reinterpret_cast<float4*>(row + x0)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(row + x0)[1] = make_float4(v[4], v[5], v[6], v[7]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (x0 + k < wx) row[x0 + k] = v[k];
      }
    }
  }
}

#ifndef GSCT_VOX_LANES
#define GSCT_VOX_LANES 4  // lanes per splat in the voxel backward (A/B at 512^3: 1 2.37, 2 2.02, 4 1.93, 8 2.05 ms)
#endif
constexpr int kVoxLanes = GSCT_VOX_LANES;
#ifndef GSCT_VLD_NA
#define GSCT_VLD_NA 1  // grad-volume row loads bypass L1 allocation (A/B: 2.36 vs 2.54 ms at 512^3)
#endif
#ifndef GSCT_VLD_L2PF
#define GSCT_VLD_L2PF 0  // 1: L2::256B prefetch-size hint on the grad-volume row loads
#endif
__device__ __forceinline__ void ldg_v8(const float* p, float (&w)[8]) {
#if GSCT_VLD_NA && GSCT_VLD_L2PF
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#elif GSCT_VLD_NA
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#else
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#endif
               : "=f"(w[0]), "=f"(w[1]), "=f"(w[2]), "=f"(w[3]), "=f"(w[4]), "=f"(w[5]), "=f"(w[6]), "=f"(w[7])
               : "l"(p));
}

// Voxel backward v2 (K8a): ONE LANE per splat (the raster backward's lane-per-item scheme).
// The lane walks the (window-clipped) box as x-rows of 32-byte aligned 8-voxel chunks of
// the grad volume (VEC = 8; VEC = 1 scalar fallback for unaligned windows; voxels outside
// the box in the edge chunks are zeroed), accumulating per row, in packed f32x2 over voxel
// pairs, s0 = sum t, s1 = sum t k, s2 = sum t k^2 with t = exp2(e) * w and
// dx = sp k - delta (k = x - round(centre), |delta| <= sp/2). The exponent along the row is a
// quadratic in k evaluated directly. Rows fold into the ten moments
// {t, t dx, t dy, t dz, t dx^2, t dy^2, t dz^2, t dx dy, t dx dz, t dy dz}. No shuffles; each
// splat's sums depend only on its own inputs. Splats run in `order` (detector-region major,
// then box shape) so warps see uniform trip counts and the grad volume stays L2-resident.
template <int VEC>
#ifndef GSCT_VBWD_MINB
#define GSCT_VBWD_MINB 4
#endif
__global__ void __launch_bounds__(256, GSCT_VBWD_MINB) k_voxel_bwd_lanes(const VoxelRec* __restrict__ rec,
                                                            const uint32_t* __restrict__ order, int64_t n,
                                                            Window win, float sp, const float* __restrict__ grad,
                                                            float* __restrict__ mom) {
  constexpr int CW = VEC == 8 ? 8 : 4;
  // kVoxLanes lanes per splat (an aligned group): lane q walks the slices z = q, q + kVoxLanes,
  // ... of the box; the group's ten sums are combined by a fixed xor tree at the end
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t t = tid / kVoxLanes;
  const int q = static_cast<int>(tid % kVoxLanes);
  const bool live = t < n;
  const int64_t i = live ? (order ? static_cast<int64_t>(__ldg(order + t)) : t) : 0;
  const VoxelRec r = rec[i];
  const int x0 = max(static_cast<int>(r.lox), win.lo[0]), y0 = max(static_cast<int>(r.loy), win.lo[1]),
            z0 = max(static_cast<int>(r.loz), win.lo[2]);
  const int W = min(static_cast<int>(r.hix), win.hi[0] - 1) - x0 + 1,
            H = min(static_cast<int>(r.hiy), win.hi[1] - 1) - y0 + 1,
            D = live ? min(static_cast<int>(r.hiz), win.hi[2] - 1) - z0 + 1 : 0;
  const bool empty = W <= 0 || H <= 0 || D <= 0;  // moments were zero-filled
  const int wx = win.hi[0] - win.lo[0], wy = win.hi[1] - win.lo[1];
  const int xa = VEC > 1 ? x0 - ((x0 - win.lo[0]) & (VEC - 1)) : x0;  // aligned first column
  const int lead = x0 - xa, ncol = lead + W, nch = (ncol + CW - 1) / CW;
  // k = x - xc (xc = round of the centre's x index); dx = (x - lo) sp - off = sp k - delta
  const float cxf = r.lox + r.offx / sp;
  const float xc = rintf(cxf);
  const float delta = fmaf(r.lox - xc, sp, r.offx);  // off - (xc - lo) sp
  const float fk0 = static_cast<float>(xa) - xc;      // k of the first walked column
  const float sp2 = sp * sp;
  const f2_t A2 = f2_bc(r.Q00 * sp2);
  const f2_t TWO2 = f2_bc(2.f);
  const f2_t K0 = f2_pack(fk0, fk0 + 1.f);
  const float* __restrict__ gz = grad + (static_cast<int64_t>(z0 - win.lo[2]) * wy + (y0 - win.lo[1])) * wx +
                                 (xa - win.lo[0]);
  float m[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) m[k] = 0.f;
  for (int zz = q; zz < (empty ? 0 : D); zz += kVoxLanes) {
    const float dz = fmaf(static_cast<float>(z0 + zz) - r.loz, sp, -r.offz);
    const float* __restrict__ prow = gz + static_cast<int64_t>(zz) * wy * wx;
    for (int yy = 0; yy < H; ++yy, prow += wx) {
      const float dy = fmaf(static_cast<float>(y0 + yy) - r.loy, sp, -r.offy);
      // e(dx) = Q00 dx^2 + L dx + K;  in k: A' k^2 + B' k + C'
      const float L = fmaf(r.Q01, dy, r.Q02 * dz);
      const float K = fmaf(dy, fmaf(r.Q11, dy, r.Q12 * dz), r.Q22 * dz * dz);
      const float bp = sp * fmaf(-2.f * r.Q00, delta, L);
      const float cp = fmaf(delta, fmaf(r.Q00, delta, -L), K);
      const f2_t BP2 = f2_bc(bp), CP2 = f2_bc(cp);
      f2_t s0 = f2_bc(0.f), s1 = s0, s2 = s0;
      f2_t kA = K0;
      for (int j = 0; j < nch; ++j) {
        float w[CW];
        const int c = CW * j;
        if constexpr (VEC == 8) {
          ldg_v8(prow + c, w);
        } else {
#pragma unroll
          for (int q = 0; q < CW; ++q) w[q] = (c + q < ncol) ? __ldg(prow + c + q) : 0.f;
        }
        if (VEC > 1) {
          if (j == 0) {  // columns left of the box
#pragma unroll
            for (int q = 0; q < CW - 1; ++q)
              if (q < lead) w[q] = 0.f;
          }
          if (j == nch - 1) {  // columns right of the box
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
      // sum t dx = sp t1 - delta t0;  sum t dx^2 = sp^2 t2 - 2 sp delta t1 + delta^2 t0
      const float sx = fmaf(sp, t1, -delta * t0);
      const float sxx = fmaf(sp2, t2, delta * fmaf(delta, t0, -2.f * sp * t1));
      m[0] += t0;
      m[1] += sx;
      m[2] = fmaf(dy, t0, m[2]);
      m[3] = fmaf(dz, t0, m[3]);
      m[4] += sxx;
      m[5] = fmaf(dy * dy, t0, m[5]);
      m[6] = fmaf(dz * dz, t0, m[6]);
      m[7] = fmaf(dy, sx, m[7]);
      m[8] = fmaf(dz, sx, m[8]);
      m[9] = fmaf(dy * dz, t0, m[9]);
    }
  }
#pragma unroll
  for (int k = 0; k < 10; ++k) {
#pragma unroll
    for (int o = 1; o < kVoxLanes; o <<= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
  }
  if (live && !empty && q == 0) {
#pragma unroll
    for (int k = 0; k < 10; ++k) mom[static_cast<int64_t>(k) * n + i] = m[k];
  }
}

// Voxel backward, chain variant (the default for 32 B-aligned rows): the ownership of
// k_voxel_bwd_lanes (kVoxLanes lanes per splat over interleaved z-slices, x-rows as 32 B chunks,
// a fixed xor tree at the end) with the raster chain backward's arithmetic: along an x-row the
// exponent e(k) = A' k^2 + B' k + C' (k = x - round(centre x)) is a multiplicative chain over
// voxel PAIRS, g(k+2) = g(k) r(k), r(k+2) = r(k) c with r(k) = 2^(e(k+2) - e(k)),
// c = 2^(8 A') -- 4 MUFU per row instead of one per voxel -- and per-chunk sums with
// compile-time column offsets. Edge voxels of the first / last chunk are zeroed by 0/1 pairs
// computed once per splat. A splat whose chain could leave the normal fp32 range over its
// walked box (quadratic minimum and step extremes at the box corners) takes the direct path.
__device__ __forceinline__ float vox_q(const VoxelRec& r, float dx, float dy, float dz) {
  return fmaf(dx, fmaf(r.Q00, dx, fmaf(r.Q01, dy, r.Q02 * dz)), fmaf(dy, fmaf(r.Q11, dy, r.Q12 * dz), r.Q22 * dz * dz));
}

#ifndef GSCT_VCHAIN_MINB
#define GSCT_VCHAIN_MINB 3
#endif
#ifndef GSCT_VCHAIN_PIPE
#define GSCT_VCHAIN_PIPE 0
#endif
#ifndef GSCT_VBWD_YLANES
#define GSCT_VBWD_YLANES 1  // lanes interleave y-rows of a slice (A/B: 1024^3 25.5 -> 11.8 ms, 512^3 1.774 vs 1.786)
#endif
template <int LANES>
__global__ void __launch_bounds__(256, GSCT_VCHAIN_MINB) k_voxel_bwd_chain(const VoxelRec* __restrict__ rec,
                                                                           const uint32_t* __restrict__ order,
                                                                           int64_t n, Window win, float sp,
                                                                           const float* __restrict__ grad,
                                                                           float* __restrict__ mom) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t t = tid / LANES;
  const int q = static_cast<int>(tid % LANES);
  const bool live = t < n;
  const int64_t i = live ? (order ? static_cast<int64_t>(__ldg(order + t)) : t) : 0;
  const VoxelRec r = rec[i];
  const int x0 = max(static_cast<int>(r.lox), win.lo[0]), y0 = max(static_cast<int>(r.loy), win.lo[1]),
            z0 = max(static_cast<int>(r.loz), win.lo[2]);
  const int W = min(static_cast<int>(r.hix), win.hi[0] - 1) - x0 + 1,
            H = min(static_cast<int>(r.hiy), win.hi[1] - 1) - y0 + 1,
            D = live ? min(static_cast<int>(r.hiz), win.hi[2] - 1) - z0 + 1 : 0;
  const bool empty = W <= 0 || H <= 0 || D <= 0;  // moments were zero-filled
  const int wx = win.hi[0] - win.lo[0], wy = win.hi[1] - win.lo[1];
  const int xa = x0 - ((x0 - win.lo[0]) & 7);  // aligned first column
  const int lead = x0 - xa, ncol = lead + W, nch = (ncol + 7) >> 3;
  const float cxf = r.lox + r.offx / sp;
  const float xc = rintf(cxf);
  const float delta = fmaf(r.lox - xc, sp, r.offx);  // dx = sp k - delta
  const float fk0 = static_cast<float>(xa) - xc;      // k of the first walked column
  const float sp2 = sp * sp;
  const float Ap = r.Q00 * sp2;  // e(k) = Ap k^2 + B' k + C'
  // chain safety over the walked box: k in [fk0, fk0 + 8 nch + 1], the box's y / z offsets
  bool safe = false;
  if (!empty) {
    const float dxa = fmaf(sp, fk0, -delta), dxb = fmaf(sp, fk0 + static_cast<float>(8 * nch + 1), -delta);
    const float dya = fmaf(static_cast<float>(y0) - r.loy, sp, -r.offy), dyb = dya + sp * static_cast<float>(H - 1);
    const float dza = fmaf(static_cast<float>(z0) - r.loz, sp, -r.offz), dzb = dza + sp * static_cast<float>(D - 1);
    float emin = 0.f, dmax = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float dx = (c & 1) ? dxb : dxa, dy = (c & 2) ? dyb : dya, dz = (c & 4) ? dzb : dza;
      emin = fminf(emin, vox_q(r, dx, dy, dz));
      // e(k+2) - e(k) in dx units: Q00 (4 sp dx + 4 sp^2) + 2 sp (Q01 dy + Q02 dz)
      const float d2 = fmaf(r.Q00, fmaf(4.f * sp, dx, 4.f * sp2), 2.f * sp * fmaf(r.Q01, dy, r.Q02 * dz));
      dmax = fmaxf(dmax, fabsf(d2));
    }
    safe = emin > -100.f && dmax < 100.f && Ap > -12.f;
  }
  const f2_t c2 = f2_bc(ex2_approx(8.f * Ap));
  const f2_t KO0 = f2_pack(0.f, 1.f);
  f2_t MF[4], ML[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const int a = 2 * h, b = 2 * h + 1, last = 8 * (nch - 1);
    const bool f0 = a >= lead && (nch > 1 || a < ncol), f1 = b >= lead && (nch > 1 || b < ncol);
    MF[h] = f2_pack(f0 ? 1.f : 0.f, f1 ? 1.f : 0.f);
    ML[h] = f2_pack(last + a < ncol ? 1.f : 0.f, last + b < ncol ? 1.f : 0.f);
  }
  const float* __restrict__ gz = grad + (static_cast<int64_t>(z0 - win.lo[2]) * wy + (y0 - win.lo[1])) * wx +
                                 (xa - win.lo[0]);
  float m[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) m[k] = 0.f;
#if GSCT_VBWD_YLANES
  // lane q walks rows q, q+4, ... of every z-slice: the lanes of a splat read neighbouring rows
  // of one slice (one 2 MB page) instead of four slices megabytes apart
  for (int zz = 0; zz < (empty ? 0 : D); ++zz) {
    const float dz = fmaf(static_cast<float>(z0 + zz) - r.loz, sp, -r.offz);
    const float* __restrict__ prow = gz + static_cast<int64_t>(zz) * wy * wx + static_cast<int64_t>(q) * wx;
    for (int yy = q; yy < H; yy += LANES, prow += LANES * wx) {
#else
  for (int zz = q; zz < (empty ? 0 : D); zz += LANES) {
    const float dz = fmaf(static_cast<float>(z0 + zz) - r.loz, sp, -r.offz);
    const float* __restrict__ prow = gz + static_cast<int64_t>(zz) * wy * wx;
    for (int yy = 0; yy < H; ++yy, prow += wx) {
#endif
      const float dy = fmaf(static_cast<float>(y0 + yy) - r.loy, sp, -r.offy);
      const float L = fmaf(r.Q01, dy, r.Q02 * dz);
      const float K = fmaf(dy, fmaf(r.Q11, dy, r.Q12 * dz), r.Q22 * dz * dz);
      const float bp = sp * fmaf(-2.f * r.Q00, delta, L);
      const float cp = fmaf(delta, fmaf(r.Q00, delta, -L), K);
      f2_t X0 = f2_bc(0.f), X1 = X0, X2 = X0;
      f2_t BE = f2_add(f2_bc(fk0), KO0);  // (k of the chunk's column 0, column 1)
      if (safe) {
        const float e0 = fmaf(fmaf(Ap, fk0, bp), fk0, cp);
        const float e1 = fmaf(fmaf(Ap, fk0 + 1.f, bp), fk0 + 1.f, cp);
        const float d0 = fmaf(Ap, fmaf(4.f, fk0, 4.f), 2.f * bp);
        const float d1 = fmaf(4.f, Ap, d0);
        f2_t g = f2_pack(ex2_approx(e0), ex2_approx(e1));
        f2_t rr = f2_pack(ex2_approx(d0), ex2_approx(d1));
        auto chunk = [&](const float (&w)[8], const f2_t* M, auto masked) {
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
#if GSCT_VCHAIN_PIPE
        // the next chunk's load is issued before the current chunk's arithmetic: two 32 B
        // loads in flight per lane (the walk at 1024^3 is L2 / DRAM latency-bound)
        float wa[8], wb[8];
        ldg_v8(prow, wa);
        if (nch > 1) ldg_v8(prow + 8, wb);
        chunk(wa, MF, yes{});
#pragma unroll 2
        for (int j = 1; j < nch - 1; ++j) {
#pragma unroll
          for (int k = 0; k < 8; ++k) wa[k] = wb[k];
          ldg_v8(prow + 8 * (j + 1), wb);
          chunk(wa, nullptr, no{});
        }
        if (nch > 1) chunk(wb, ML, yes{});
#else
        {
          float w[8];
          ldg_v8(prow, w);
          chunk(w, MF, yes{});
        }
#pragma unroll 1
        for (int j = 1; j < nch - 1; ++j) {
          float w[8];
          ldg_v8(prow + 8 * j, w);
          chunk(w, nullptr, no{});
        }
        if (nch > 1) {
          float w[8];
          ldg_v8(prow + 8 * (nch - 1), w);
          chunk(w, ML, yes{});
        }
#endif
      } else {
        const f2_t A2 = f2_bc(Ap), BP2 = f2_bc(bp), CP2 = f2_bc(cp);
#pragma unroll 1
        for (int j = 0; j < nch; ++j) {
          float w[8];
          ldg_v8(prow + 8 * j, w);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const f2_t e = f2_fma(f2_fma(A2, BE, BP2), BE, CP2);
            float e0, e1;
            f2_unpack(e, e0, e1);
            f2_t wp = f2_pack(w[2 * h], w[2 * h + 1]);
            if (j == 0)
              wp = f2_mul(wp, MF[h]);
            else if (j == nch - 1)
              wp = f2_mul(wp, ML[h]);
            const f2_t tt = f2_mul(f2_pack(ex2_approx(e0), ex2_approx(e1)), wp);
            X0 = f2_add(X0, tt);
            const f2_t tk = f2_mul(tt, BE);
            X1 = f2_add(X1, tk);
            X2 = f2_fma(tk, BE, X2);
            BE = f2_add(BE, f2_bc(2.f));
          }
        }
      }
      float t0, t1, t2;
      {
        float a, b;
        f2_unpack(X0, a, b);
        t0 = a + b;
        f2_unpack(X1, a, b);
        t1 = a + b;
        f2_unpack(X2, a, b);
        t2 = a + b;
      }
      // sum t dx = sp t1 - delta t0;  sum t dx^2 = sp^2 t2 - 2 sp delta t1 + delta^2 t0
      const float sx = fmaf(sp, t1, -delta * t0);
      const float sxx = fmaf(sp2, t2, delta * fmaf(delta, t0, -2.f * sp * t1));
      m[0] += t0;
      m[1] += sx;
      m[2] = fmaf(dy, t0, m[2]);
      m[3] = fmaf(dz, t0, m[3]);
      m[4] += sxx;
      m[5] = fmaf(dy * dy, t0, m[5]);
      m[6] = fmaf(dz * dz, t0, m[6]);
      m[7] = fmaf(dy, sx, m[7]);
      m[8] = fmaf(dz, sx, m[8]);
      m[9] = fmaf(dy * dz, t0, m[9]);
    }
  }
#pragma unroll
  for (int k = 0; k < 10; ++k) {
#pragma unroll
    for (int o = 1; o < LANES; o <<= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
  }
  if (live && !empty && q == 0) {
#pragma unroll
    for (int k = 0; k < 10; ++k) mom[static_cast<int64_t>(k) * n + i] = m[k];
  }
}

#ifndef GSCT_VREGION_SHIFT
#define GSCT_VREGION_SHIFT 6  // walk-order regions of 2^6 = 64 voxels per side
#endif
constexpr int kVRegionShift = GSCT_VREGION_SHIFT;
// Walk order for the lane-per-splat backward: 64^3 region of the box corner (L2 locality of
// the grad volume), then box shape (chunks per row, y-z rows / 16) for uniform warp trip
// counts. Returns the key bits through *bits.
__global__ void k_voxel_lane_keys(const VoxelRec* __restrict__ rec, int64_t n, Window win, int nrx, int nry,
                                  int vec, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const VoxelRec r = rec[i];
  const int x0 = max(static_cast<int>(r.lox), win.lo[0]), y0 = max(static_cast<int>(r.loy), win.lo[1]),
            z0 = max(static_cast<int>(r.loz), win.lo[2]);
  const int W = min(static_cast<int>(r.hix), win.hi[0] - 1) - x0 + 1,
            H = min(static_cast<int>(r.hiy), win.hi[1] - 1) - y0 + 1,
            D = min(static_cast<int>(r.hiz), win.hi[2] - 1) - z0 + 1;
  uint32_t key = 0xFFFFFFFFu;  // empty boxes last
  if (W > 0 && H > 0 && D > 0) {
    const int cw = vec == 8 ? 8 : 4;
    const int lead = vec > 1 ? ((x0 - win.lo[0]) & (vec - 1)) : 0;
    const uint32_t nch = min((lead + W + cw - 1) / cw, 7);
    const uint32_t rows = min((H * D) >> 4, 63);
    const uint32_t region = static_cast<uint32_t>(
        (((z0 - win.lo[2]) >> kVRegionShift) * nry + ((y0 - win.lo[1]) >> kVRegionShift)) * nrx +
        ((x0 - win.lo[0]) >> kVRegionShift));
    key = (region << 9) | (nch << 6) | rows;
  }
  keys[i] = key;
  vals[i] = static_cast<uint32_t>(i);
}

inline unsigned blocks_for(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

}  // namespace

void launch_emit_brick_pairs(const VoxelRec* rec, const uint32_t* offsets, const uint32_t* counts,
                             int64_t n, const Window& win, int nbx, int nby, uint32_t* keys,
                             uint32_t* vals, cudaStream_t st) {
  if (n == 0) return;
#ifndef GSCT_VEMIT_WARP
#define GSCT_VEMIT_WARP 1  // coalesced warp-cooperative brick-pair emission
#endif
  if (GSCT_VEMIT_WARP)
    k_emit_brick_pairs_warp<<<blocks_for(n, 256), 256, 0, st>>>(rec, offsets, counts, n, win, nbx, nby, keys, vals);
  else
    k_emit_brick_pairs<<<blocks_for(n, 256), 256, 0, st>>>(rec, offsets, counts, n, win, nbx, nby, keys, vals);
  count_launch();
}

#ifndef GSCT_VFWD_LPT
#define GSCT_VFWD_LPT 0  // 1: longest brick lists first (A/B 512^3: 1.08 vs 0.98 ms -- the z-major brick order keeps records L2-resident)
#endif
void launch_voxel_fwd(const VoxelRec* rec, const uint32_t* vals, const uint32_t* start,
                      const uint32_t* end, const Window& win, int nbx, int nby, int nbz,
                      float spacing, float* volume, cudaStream_t st, uint32_t* sched_ws) {
  const int64_t bricks = static_cast<int64_t>(nbx) * nby * nbz;
  if (bricks == 0) return;
  const uint32_t* sched = nullptr;
  if (GSCT_VFWD_LPT && sched_ws) {  // the forward raster's longest-first schedule over the brick lists
    launch_fwd_schedule(start, end, 1, static_cast<int>(bricks), static_cast<int>(bricks), 1, sched_ws, st);
    sched = sched_ws + 2048 + bricks;
  }
  k_voxel_fwd2<<<static_cast<unsigned>((bricks + 3) / 4), 128, 0, st>>>(
      rec, vals, start, end, win, nbx, nby, static_cast<int>(bricks), spacing, volume, sched);
  count_launch();
}


int voxel_bwd_vec(const Window& win, const float* grad_volume) {
  const int wx = win.hi[0] - win.lo[0];
  return (wx % 8 == 0 && reinterpret_cast<uintptr_t>(grad_volume) % 32 == 0) ? 8 : 1;
}

int launch_voxel_lane_keys(const VoxelRec* rec, int64_t n, const Window& win, int vec, uint32_t* keys,
                           uint32_t* vals, cudaStream_t st) {
  const int rs = kVRegionShift, rm = (1 << kVRegionShift) - 1;
  const int nrx = (win.hi[0] - win.lo[0] + rm) >> rs, nry = (win.hi[1] - win.lo[1] + rm) >> rs,
            nrz = (win.hi[2] - win.lo[2] + rm) >> rs;
  int rb = 0;
  while ((int64_t(1) << rb) < int64_t(nrx) * nry * nrz) ++rb;
  if (n > 0) {
    k_voxel_lane_keys<<<blocks_for(n, 256), 256, 0, st>>>(rec, n, win, nrx, nry, vec, keys, vals);
    count_launch();
  }
  return 9 + rb + 1;  // + 1: the all-ones key of empty boxes sorts after every region
}

void launch_voxel_bwd_lanes(const VoxelRec* rec, const uint32_t* order, int64_t n, const Window& win,
                            float spacing, const float* grad_volume, float* moments, cudaStream_t st,
                            double vps) {
  if (n == 0) return;
#ifndef GSCT_VBWD_CHAIN
#define GSCT_VBWD_CHAIN 1
#endif
#ifndef GSCT_VBWD_WIDE_VPS
#define GSCT_VBWD_WIDE_VPS 768  // grid voxels per splat above which 8 lanes share a splat
#endif
  // Large boxes (coarse clouds in big grids: 1024^3 / 1M splats ~ 1074 voxels per splat) walk
  // faster with 8 lanes per splat (A/B: 10.9 vs 11.8 ms at 1024^3), small ones with 4 (512^3 /
  // 500k ~ 268: 1.78 vs 1.90 ms); the full grid's voxels per splat stand in for the box size
  // (a z-slab window of the same grid takes the same choice).
  if (GSCT_VBWD_CHAIN && voxel_bwd_vec(win, grad_volume) == 8 && vps > GSCT_VBWD_WIDE_VPS)
    k_voxel_bwd_chain<8><<<blocks_for(n * 8, 256), 256, 0, st>>>(rec, order, n, win, spacing, grad_volume, moments);
  else if (GSCT_VBWD_CHAIN && voxel_bwd_vec(win, grad_volume) == 8)
    k_voxel_bwd_chain<kVoxLanes><<<blocks_for(n * kVoxLanes, 256), 256, 0, st>>>(rec, order, n, win, spacing,
                                                                                grad_volume, moments);
  else if (voxel_bwd_vec(win, grad_volume) == 8)
    k_voxel_bwd_lanes<8><<<blocks_for(n * kVoxLanes, 256), 256, 0, st>>>(rec, order, n, win, spacing, grad_volume,
                                                                        moments);
  else
    k_voxel_bwd_lanes<1><<<blocks_for(n * kVoxLanes, 256), 256, 0, st>>>(rec, order, n, win, spacing, grad_volume,
                                                                        moments);
  count_launch();
}


}  // namespace gsct_dev
