// Voxelizer pair kernels (fp32): brick-pair emission (K6b), the per-brick forward sum
// (K7) and the per-splat backward voxel loop (K8a).
//
// K7 follows voxelize (voxelizer.hpp:162-199): each voxel sums, in ascending splat index,
// rho * exp(-q/2) of every splat whose box contains it. Instead of the reference's
// "every z slice scans all N splats" (an O(n_z * N) skip scan), splats are binned into
// 8x8x8 bricks with a stable sort, so each brick visits only its own ascending list.
// K8a follows voxelize_backward's loop (voxelizer.hpp:235-249): one warp per splat walks
// its own box; per-voxel terms are reduced with a fixed xor-shuffle tree.
#include <cuda_runtime.h>

#include "gsct_internal.cuh"

namespace gsct_dev {

namespace {

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

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
  const int bz0 = (z0 - win.lo[2]) / kBrick, bz1 = (z1 - win.lo[2]) / kBrick;
  uint32_t off = offsets[i];
  for (int bz = bz0; bz <= bz1; ++bz)
    for (int by = by0; by <= by1; ++by)
      for (int bx = bx0; bx <= bx1; ++bx) {
        keys[off] = static_cast<uint32_t>((bz * nby + by) * nbx + bx);
        vals[off] = static_cast<uint32_t>(i);
        ++off;
      }
}

// One CTA (256 threads) per 8x8x8 brick: warp w owns z-slice w (8x8 voxels), each lane
// two voxels (x, y) and (x, y + 4).
__global__ void __launch_bounds__(256) k_voxel_fwd(const VoxelRec* __restrict__ rec,
                                                   const uint32_t* __restrict__ vals,
                                                   const uint32_t* __restrict__ start,
                                                   const uint32_t* __restrict__ end, Window win,
                                                   int nbx, int nby, float sp,
                                                   float* __restrict__ volume) {
  __shared__ float4 s_r[256][4];
  const int brick = blockIdx.x;
  const int bx = brick % nbx, by = (brick / nbx) % nby, bz = brick / (nbx * nby);
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  const int x = win.lo[0] + bx * kBrick + (l & 7);
  const int y0 = win.lo[1] + by * kBrick + (l >> 3);
  const int z = win.lo[2] + bz * kBrick + w;
  const float fx = static_cast<float>(x), fy0 = static_cast<float>(y0), fy1 = fy0 + 4.f;
  const float fz = static_cast<float>(z);
  const float wx0 = static_cast<float>(win.lo[0] + bx * kBrick), wx1 = wx0 + 7.f;
  const float wy0 = static_cast<float>(win.lo[1] + by * kBrick), wy1 = wy0 + 7.f;
  const uint32_t b = start[brick], e = end[brick];
  float acc0 = 0.f, acc1 = 0.f;
  for (uint32_t base = b; base < e; base += 256) {
    const int cnt = min(256u, e - base);
    __syncthreads();
    if (t < cnt) {
      const float4* src = reinterpret_cast<const float4*>(rec + vals[base + t]);
      s_r[t][0] = src[0];
      s_r[t][1] = src[1];
      s_r[t][2] = src[2];
      s_r[t][3] = src[3];
    }
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {
      const float4 lo = s_r[j][0];  // lox, loy, loz, rho
      const float4 hi = s_r[j][1];  // hix, hiy, hiz, Q00
      if (fz < lo.z || fz > hi.z) continue;                                      // warp-uniform
      if (lo.x > wx1 || hi.x < wx0 || lo.y > wy1 || hi.y < wy0) continue;         // warp-uniform
      const float4 of = s_r[j][2];  // offx, offy, offz, Q11
      const float4 q = s_r[j][3];   // Q22, Q01, Q02, Q12
      const float dx = fmaf(fx - lo.x, sp, -of.x);
      const float dz = fmaf(fz - lo.z, sp, -of.z);
      const float lx = fmaf(hi.w, dx, q.z * dz);          // Q00 dx + Q02 dz
      const float base_e = fmaf(dx, lx, q.x * dz * dz);   // Q00 dx^2 + Q02 dx dz + Q22 dz^2
      const float ly = fmaf(q.y, dx, q.w * dz);           // Q01 dx + Q12 dz
      const bool inx = fx >= lo.x && fx <= hi.x;
      {
        const float dy = fmaf(fy0 - lo.y, sp, -of.y);
        const float ex = ex2_approx(fmaf(dy, fmaf(of.w, dy, ly), base_e));
        if (inx && fy0 >= lo.y && fy0 <= hi.y) acc0 = fmaf(lo.w, ex, acc0);
      }
      {
        const float dy = fmaf(fy1 - lo.y, sp, -of.y);
        const float ex = ex2_approx(fmaf(dy, fmaf(of.w, dy, ly), base_e));
        if (inx && fy1 >= lo.y && fy1 <= hi.y) acc1 = fmaf(lo.w, ex, acc1);
      }
    }
  }
  const int wx = win.hi[0] - win.lo[0], wy = win.hi[1] - win.lo[1];
  if (x < win.hi[0] && z < win.hi[2]) {
    const int64_t zoff = static_cast<int64_t>(z - win.lo[2]) * wy;
    if (y0 < win.hi[1]) volume[(zoff + (y0 - win.lo[1])) * wx + (x - win.lo[0])] = acc0;
    if (y0 + 4 < win.hi[1]) volume[(zoff + (y0 + 4 - win.lo[1])) * wx + (x - win.lo[0])] = acc1;
  }
}

// Spatial walk order for the backward: key = 8^3 brick of the splat's (window-clipped) box
// corner, value = splat; sorted, consecutive warps then own nearby splats, so the grad
// volume is re-read from L2 instead of HBM (the walk order does not change any result:
// every splat's sums are owned by one warp).
__global__ void k_voxel_order_keys(const VoxelRec* __restrict__ rec, int64_t n, Window win, int nbx, int nby,
                                   uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const VoxelRec r = rec[i];
  const int x = max(static_cast<int>(r.lox), win.lo[0]) - win.lo[0];
  const int y = max(static_cast<int>(r.loy), win.lo[1]) - win.lo[1];
  const int z = max(static_cast<int>(r.loz), win.lo[2]) - win.lo[2];
  keys[i] = static_cast<uint32_t>(((z / kBrick) * nby + (y / kBrick)) * nbx + (x / kBrick));
  vals[i] = static_cast<uint32_t>(i);
}

// One warp per splat, grid-stride over the spatial walk order. Lanes walk the
// (window-clipped) box x-fastest in steps of 32 voxels. Moments of t = exp(-q/2) * w with
// world-unit offsets d: {t, t dx, t dy, t dz, t dx^2, t dy^2, t dz^2, t dx dy, t dx dz, t dy dz}.
__global__ void __launch_bounds__(256) k_voxel_bwd_pairs(const VoxelRec* __restrict__ rec,
                                                         const uint32_t* __restrict__ order,
                                                         int64_t n, Window win, float sp,
                                                         const float* __restrict__ grad,
                                                         float* __restrict__ mom) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int wx = win.hi[0] - win.lo[0], wy = win.hi[1] - win.lo[1];
  for (int64_t k = warp; k < n; k += n_warps) {
    const int64_t i = order ? static_cast<int64_t>(order[k]) : k;
    const VoxelRec r = rec[i];
    // grid-clipped box of the record, clipped again to the window for iteration
    const int x0 = max(static_cast<int>(r.lox), win.lo[0]), y0 = max(static_cast<int>(r.loy), win.lo[1]),
              z0 = max(static_cast<int>(r.loz), win.lo[2]);
    const int W = min(static_cast<int>(r.hix), win.hi[0] - 1) - x0 + 1,
              H = min(static_cast<int>(r.hiy), win.hi[1] - 1) - y0 + 1,
              D = min(static_cast<int>(r.hiz), win.hi[2] - 1) - z0 + 1;
    if (W <= 0 || H <= 0 || D <= 0) continue;  // moments were zero-filled
    // offsets are relative to the record's (grid-clipped) corner
    const float bx = static_cast<float>(x0) - r.lox, by = static_cast<float>(y0) - r.loy,
                bz = static_cast<float>(z0) - r.loz;
    // per-item base of the grad window at the box corner (32-bit offsets below)
    const float* __restrict__ g0 =
        grad + (static_cast<int64_t>(z0 - win.lo[2]) * wy + (y0 - win.lo[1])) * wx + (x0 - win.lo[0]);
    const uint32_t zstride = static_cast<uint32_t>(wy * wx);
    float m[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) m[k] = 0.f;
    // Lanes = box columns (blocks of <= 32) x row groups over the H*D (y, z) rows: dx is
    // lane-constant, so per voxel only {t, t dy, t dz, t dy^2, t dz^2, t dy dz} are
    // accumulated and folded with dx once per column block.
    for (int cb = 0; cb < W; cb += 32) {
      const int cw = min(32, W - cb);
      const float rc = rcp_approx(static_cast<float>(cw));
      const int G = static_cast<int>(32.5f * rc);  // floor(32 / cw), exact
      const int grp = static_cast<int>((static_cast<float>(lane) + 0.5f) * rc);
      const int col = lane - grp * cw;
      if (grp >= G) continue;
      const float dx = fmaf(bx + static_cast<float>(cb + col), sp, -r.offx);
      const float ax = r.Q00 * dx * dx, b1 = r.Q01 * dx, b2 = r.Q02 * dx;
      const float fG = static_cast<float>(G);
      const uint32_t ystride = static_cast<uint32_t>(G * wx);
      float t0 = 0.f, ty_ = 0.f, tz_ = 0.f, tyy = 0.f, tzz = 0.f, tyz = 0.f;
      for (int zz = 0; zz < D; ++zz) {
        const float dz = fmaf(bz + static_cast<float>(zz), sp, -r.offz);
        // per z-slice terms of the quadratic: e = dy (Q11 dy + Q12 dz + Q01 dx) + [dz (Q22 dz + Q02 dx) + Q00 dx^2]
        const float cy = fmaf(r.Q12, dz, b1);
        const float cz = fmaf(dz, fmaf(r.Q22, dz, b2), ax);
        uint32_t off = static_cast<uint32_t>(zz) * zstride + static_cast<uint32_t>(grp * wx + cb + col);
        float dy = fmaf(by + static_cast<float>(grp), sp, -r.offy);
        const float ddy = fG * sp;
        // rows grp, grp + G, ... < H of this slice; four grad loads in flight per step
        for (int yy = grp; yy < H; yy += 4 * G) {
          float w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) w[k] = (yy + k * G < H) ? __ldg(g0 + (off + k * ystride)) : 0.f;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float tt = ex2_approx(fmaf(dy, fmaf(r.Q11, dy, cy), cz)) * w[k];  // w = 0 past the box
            t0 += tt;
            const float ty = tt * dy, tz = tt * dz;
            ty_ += ty;
            tz_ += tz;
            tyy = fmaf(ty, dy, tyy);
            tzz = fmaf(tz, dz, tzz);
            tyz = fmaf(ty, dz, tyz);
            dy += ddy;
          }
          off += 4 * ystride;
        }
      }
      m[0] += t0;
      m[1] = fmaf(t0, dx, m[1]);
      m[2] += ty_;
      m[3] += tz_;
      m[4] = fmaf(t0 * dx, dx, m[4]);
      m[5] += tyy;
      m[6] += tzz;
      m[7] = fmaf(ty_, dx, m[7]);
      m[8] = fmaf(tz_, dx, m[8]);
      m[9] += tyz;
    }
#pragma unroll
    for (int k = 0; k < 10; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
    }
    if (lane < 10) {
      float v = m[0];
#pragma unroll
      for (int k = 1; k < 10; ++k)
        if (lane == k) v = m[k];
      mom[static_cast<int64_t>(lane) * n + i] = v;
    }
  }
}

inline unsigned blocks_for(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

}  // namespace

void launch_emit_brick_pairs(const VoxelRec* rec, const uint32_t* offsets, const uint32_t* counts,
                             int64_t n, const Window& win, int nbx, int nby, uint32_t* keys,
                             uint32_t* vals, cudaStream_t st) {
  if (n == 0) return;
  k_emit_brick_pairs<<<blocks_for(n, 256), 256, 0, st>>>(rec, offsets, counts, n, win, nbx, nby,
                                                         keys, vals);
  count_launch();
}

void launch_voxel_fwd(const VoxelRec* rec, const uint32_t* vals, const uint32_t* start,
                      const uint32_t* end, const Window& win, int nbx, int nby, int nbz,
                      float spacing, float* volume, cudaStream_t st) {
  const int64_t bricks = static_cast<int64_t>(nbx) * nby * nbz;
  if (bricks == 0) return;
  k_voxel_fwd<<<static_cast<unsigned>(bricks), 256, 0, st>>>(rec, vals, start, end, win, nbx, nby,
                                                             spacing, volume);
  count_launch();
}

void launch_voxel_order_keys(const VoxelRec* rec, int64_t n, const Window& win, int nbx, int nby,
                             uint32_t* keys, uint32_t* vals, cudaStream_t st) {
  if (n == 0) return;
  k_voxel_order_keys<<<blocks_for(n, 256), 256, 0, st>>>(rec, n, win, nbx, nby, keys, vals);
  count_launch();
}

void launch_voxel_bwd_pairs(const VoxelRec* rec, const uint32_t* order, int64_t n, const Window& win,
                            float spacing, const float* grad_volume, float* moments, cudaStream_t st) {
  if (n == 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 7) / 8;
  const unsigned blocks = static_cast<unsigned>(want < static_cast<int64_t>(sms) * 16 ? want : static_cast<int64_t>(sms) * 16);
  k_voxel_bwd_pairs<<<blocks, 256, 0, st>>>(rec, order, n, win, spacing, grad_volume, moments);
  count_launch();
}

}  // namespace gsct_dev
