// Microbenchmark: issue throughput of scalar FFMA/FADD vs packed FFMA2/FADD2 and MUFU.RSQ
// on one B200 (all SMs, 8 independent chains per thread). Prints FP32 lane-ops per clock per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_pipes fp32_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float2 a) { return *reinterpret_cast<u64*>(&a); }
__device__ __forceinline__ float2 up(u64 a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c))); return up(d); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b))); return up(d); }

__global__ void k_ffma(float* out, int n, float b) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  float c = out[0];
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], c, b);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[1] = s;
}
__global__ void k_fadd(float* out, int n, float b) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  float c = out[0];
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] + c;
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[1] = s;
}
__global__ void k_ffma2(float* out, int n, float b) {
  float2 a[8]; for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 c = make_float2(out[0], out[0]), bb = make_float2(b, b);
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma2(a[i], c, bb);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 12345.f) out[1] = s;
}
__global__ void k_fadd2(float* out, int n, float b) {
  float2 a[8]; for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 c = make_float2(out[0], out[0]);
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = add2(a[i], c);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 12345.f) out[1] = s;
}
__global__ void k_rsq(float* out, int n, float b) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i + 1;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = rsqrtf(a[i]);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[1] = s;
}

template <class K>
void run(const char* name, K kern, float lanes_per_op) {
  float* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int n = 4096, threads = 512, blocks = sms * 4;
  kern<<<blocks, threads>>>(d, 16, 1.0f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kern<<<blocks, threads>>>(d, n, 1.0f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * n * 8 * lanes_per_op;  // lane-ops
  double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
  printf("%-8s %.3f ms  %.1f lane-ops/clk/SM (at %.0f MHz nominal)\n", name, ms, per_clk_sm, clk / 1e3);
  cudaFree(d);
}
int main() {
  run("FFMA", k_ffma, 1); run("FADD", k_fadd, 1); run("FFMA2", k_ffma2, 2); run("FADD2", k_fadd2, 2);
  run("MUFU.RSQ", k_rsq, 1);
  return 0;
}
