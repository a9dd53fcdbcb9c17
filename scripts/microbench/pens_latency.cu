// Microbenchmark: latency (cycles per call, one CTA) of the AL fixed-obstacle pass
// (al_tile.cuh pens_fixed_all_f2) for one sphere against 14 statics + 2 staged spheres,
// with 1 warp and with 6 warps resident (the C2 AL CTA shape).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -ftz=true
//        -prec-div=false -prec-sqrt=false -DSPASM_FTZ_FAST -I../../paper_2510_07674_b200/csrc -o pens_latency pens_latency.cu
#include <cstdio>
#include "al_tile.cuh"
using namespace spasm;

__global__ void k_pens(const TrajScene<float>* g_sc, int iters, int f0, int f1, float* out, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smem[];
  TrajScene<float>& sc = *reinterpret_cast<TrajScene<float>*>(smem);
  {
    const int4* src = reinterpret_cast<const int4*>(g_sc);
    int4* dst = reinterpret_cast<int4*>(smem);
    for (int i = threadIdx.x; i < (int)(sizeof(TrajScene<float>) / 16); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  float c[3] = {0.4f + 0.001f * threadIdx.x, -0.05f, 0.2f};
  float acc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float g[3] = {0.f, 0.f, 0.f};
    acc += pens_fixed_all_f2(sc, c, 0.055f, 0, (i & 1) != 0, g);
    c[0] += g[0] * 1e-6f;  // carry a dependency into the next call
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  out[threadIdx.x] = acc + c[0];
}

int main() {
  static TrajScene<float> h{};
  h.n_static = 14;
  for (int o = 0; o < 14; ++o) {
    h.st4[o][0] = 0.35f + 0.1f * (o % 2); h.st4[o][1] = -0.15f + 0.1f * ((o / 2) % 2); h.st4[o][2] = 0.05f + 0.1f * (o / 4);
    h.st4[o][3] = 0.05f;
  }
  for (int q = 0; q < 2; ++q) { h.staged4[q][0] = 0.3f; h.staged4[q][1] = -0.35f + 0.15f * q; h.staged4[q][2] = 0.1f; h.staged4[q][3] = 0.05f; }
  h.obs_np[0] = 8;  // 16 obstacles (14 statics + 2 staged) = 8 pairs = 2 groups
  for (int o = 0; o < 16; ++o)
    for (int k = 0; k < 4; ++k) h.obsp[0][o / 2][2 * k + (o & 1)] = o < 14 ? h.st4[o][k] : h.staged4[o - 14][k];
  TrajScene<float>* d; cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4096 * 4);
  long long* cyc; cudaMalloc(&cyc, 64 * 8);
  long long hc;
  cudaFuncSetAttribute(k_pens, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(h));
  for (int threads : {32, 192}) {
    k_pens<<<1, threads, sizeof(h)>>>(d, 1000, 0, 2, out, cyc); cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("pens_fixed_all_f2 (14 statics + 2 staged) %3d threads: %lld cycles/call\n", threads, hc);
  }
  return 0;
}
