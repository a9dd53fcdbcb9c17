// Microbenchmark: SHFL and LDS throughput per SM (warp instructions per cycle) with W warps
// each issuing 8 independent chains. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfl_tput shfl_tput.cu
#include <cstdio>
__global__ void k_shfl(int iters, float* out, long long* cyc) {
  float v[8];
  for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __shfl_xor_sync(0xffffffffu, v[k], 1 + (k & 3));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  float s = 0; for (int k = 0; k < 8; ++k) s += v[k];
  out[threadIdx.x] = s;
}
__global__ void k_lds(int iters, float* out, long long* cyc) {
  __shared__ float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i;
  float v[8];
  for (int k = 0; k < 8; ++k) v[k] = 0;
  int idx = threadIdx.x & 31;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += sm[(idx + 32 * k + i) & 1023];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  float s = 0; for (int k = 0; k < 8; ++k) s += v[k];
  out[threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 4096 * 4);
  long long* cyc; cudaMalloc(&cyc, 8);
  long long h;
  const int iters = 1000;
  for (int w : {1, 2, 4, 8, 16}) {
    k_shfl<<<1, 32 * w>>>(iters, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("SHFL %2d warps: %.2f warp-instr/cycle/SM (%.1f cycles per chain step)\n", w, 8.0 * iters * w / h, (double)h / iters);
    k_lds<<<1, 32 * w>>>(iters, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS  %2d warps: %.2f warp-instr/cycle/SM\n", w, 8.0 * iters * w / h);
  }
  return 0;
}
