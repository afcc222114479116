// Shared device helpers of the fp32 pair kernels (raster.cu, voxel.cu): MUFU exp2 / rcp,
// packed f32x2 arithmetic as inline PTX (never contracted by the compiler, so a value's
// rounding does not depend on where or in which unrolled step it is computed -- the
// voxel z-slab and raster duplicate/homogeneity bitwise properties rely on that) and the
// 32 x 32 warp bit-matrix transpose of the per-lane record filters.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace gsct_dev {

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

typedef unsigned long long f2_t;  // two packed fp32 values (lo, hi)
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t f2_bc(float x) { return f2_pack(x, x); }

// 32 x 32 bit-matrix transpose across a warp: on entry lane j holds row j (bit l = lane l
// is relevant to record j); on exit lane l holds column l (bit j = record j is relevant to
// lane l). Five xor-shuffle stages.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  const uint32_t M[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int s = 16 >> t;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? ((x & ~M[t]) | ((y >> s) & M[t])) : ((x & M[t]) | ((y << s) & ~M[t]));
  }
  return x;
}

}  // namespace gsct_dev
