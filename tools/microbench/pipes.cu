// Pipe-throughput microbenchmarks on B200 (sm_100a): FFMA vs packed FFMA2, MUFU.EX2,
// mixes, and whether predicated-off lanes free MUFU cycles. Prints instr/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2u(float2 v){ return *reinterpret_cast<u64*>(&v);}
__device__ __forceinline__ float2 u2f(u64 v){ return *reinterpret_cast<float2*>(&v);}
__device__ __forceinline__ float ex2(float x){ float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;}
__device__ __forceinline__ void ffma2(u64& d, u64 a, u64 b){ asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b)); }
__device__ __forceinline__ void ffma1(float& d, float a, float b){ asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(d) : "f"(a), "f"(b)); }

template<int MODE>
__global__ void k(float* out, int iters, float a, float b, int pred_lanes){
  float x[8]; u64 y[8];
  for(int i=0;i<8;++i){ x[i]=threadIdx.x*1e-3f+i; y[i]=f2u(make_float2(x[i], x[i]+1)); }
  u64 A=f2u(make_float2(a,a)), B=f2u(make_float2(b,b));
  const bool on = (threadIdx.x & 31) < pred_lanes;
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<8;++i){
      if (MODE==0) ffma1(x[i], a, b);
      if (MODE==1) ffma2(y[i], A, B);
      if (MODE==2) x[i]=ex2(x[i]);
      if (MODE==3) { x[i]=ex2(x[i]); ffma2(y[i],A,B); ffma2(y[(i+1)&7],A,B); ffma2(y[(i+2)&7],A,B); ffma2(y[(i+3)&7],A,B);}  // 1 MUFU : 4 FFMA2
      if (MODE==4) { if (on) x[i]=ex2(x[i]); }
      if (MODE==5) { x[i]=ex2(x[i]); ffma1(x[(i+1)&7],a,b); ffma1(x[(i+2)&7],a,b); ffma1(x[(i+3)&7],a,b); ffma1(x[(i+4)&7],a,b);}  // 1 MUFU : 4 FFMA
      if (MODE==6) { asm volatile("add.f32x2 %0, %0, %1;" : "+l"(y[i]) : "l"(A)); }
      if (MODE==7) { asm volatile("add.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(a)); }
    }
  }
  float s=0; for(int i=0;i<8;++i){ float2 f=u2f(y[i]); s+=x[i]+f.x+f.y; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}

template<int MODE>
void run(const char* name, int per_iter_instr, int pred=32){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sms*8*1024*4);
  int iters=4096, threads=1024, blocks=sms*2;
  k<MODE><<<blocks,threads>>>(out, 16, 1.0001f, 1e-7f, pred);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks,threads>>>(out, iters, 1.0001f, 1e-7f, pred);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  double warp_instr = (double)blocks*threads/32*iters*8*per_iter_instr;
  double per_clk_sm = warp_instr / (ms*1e-3) / (clk*1e3) / sms;
  printf("%-28s %8.3f ms  %6.2f warp-instr/clk/SM (at max clock %d MHz)\n", name, ms, per_clk_sm, clk/1000);
  cudaFree(out);
}
int main(){
  run<0>("FFMA", 1); run<1>("FFMA2 (f32x2)", 1); run<7>("FADD", 1); run<6>("FADD2 (f32x2)",1);
  run<2>("MUFU.EX2", 1); run<4>("MUFU.EX2 16/32 lanes on", 1, 16); run<4>("MUFU.EX2 8/32 lanes on", 1, 8);
  run<3>("EX2 + 4 FFMA2", 5); run<5>("EX2 + 4 FFMA", 5);
  return 0;
}
