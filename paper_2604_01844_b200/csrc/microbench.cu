// On-box throughput microbenchmarks: the roofline denominators for the pair kernels.
// MUFU ex2.approx.f32 (the one transcendental per splat-pixel / splat-voxel pair) and
// FP32 FFMA, each as 8 independent dependency chains per thread over a full device grid.
#include <cuda_runtime.h>

#include "gsct_internal.cuh"

namespace gsct_dev {

namespace {

__global__ void __launch_bounds__(256) k_ex2_bench(float* out, int iters) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = -1e-3f * static_cast<float>((threadIdx.x + k) & 63);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-a[k]));
      a[k] = y;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[0] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) k_ffma_bench(float* out, int iters, float b, float c) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1e-3f * static_cast<float>((threadIdx.x + k) & 63);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[0] = s;
}

}  // namespace

// Returns device ops/s (ex2 or FFMA instructions per second).
double run_microbench(int kind, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  cudaMalloc(&out, sizeof(float));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    if (kind == 0)
      k_ex2_bench<<<blocks, threads, 0, st>>>(out, iters);
    else
      k_ffma_bench<<<blocks, threads, 0, st>>>(out, iters, 0.999f, 1e-4f);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = static_cast<double>(blocks) * threads * iters * 8.0;
    if (rep > 0 && ms > 0.f) best = std::max(best, ops / (ms * 1e-3));
  }
  count_launch(4);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}

}  // namespace gsct_dev
