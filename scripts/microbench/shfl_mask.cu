// Does a per-8-lane-tile mask on __shfl_*_sync cost more than the full-warp mask when all
// 32 lanes are converged? (AL / IK tiles: 4 tiles per warp.) Prints ns per shuffle chain step.
#include <cstdio>
#include <cuda_runtime.h>
template <bool FULL>
__global__ void k(float* out, int n) {
  const int lane = threadIdx.x & 31;
  const unsigned mask = FULL ? 0xffffffffu : (0xFFu << (lane & ~7));
  float v = lane * 1.0f;
  for (int i = 0; i < n; ++i) {
    v += __shfl_up_sync(mask, v, 1, 8);
    v += __shfl_xor_sync(mask, v, 2, 8);
    v *= 0.5f;
  }
  if (v == 12345.f) out[0] = v;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  const int n = 100000;
  for (int full = 0; full < 2; ++full) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    if (full) k<true><<<1, 192>>>(d, 100); else k<false><<<1, 192>>>(d, 100);
    cudaEventRecord(a);
    if (full) k<true><<<1, 192>>>(d, n); else k<false><<<1, 192>>>(d, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s mask: %.2f ns per iteration (2 dependent shuffles + 3 flops)\n", full ? "full" : "tile", ms * 1e6 / n);
  }
  return 0;
}
