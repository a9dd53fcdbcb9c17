// Microbenchmark: latency (cycles per call, one CTA) of the tile-cooperative FK (coop.cuh
// tile_fk) and of one damped-least-squares polish iteration's pieces, with 1 warp and with
// 6 warps resident (the C2 AL CTA shape). fp32, 7-DOF spatial chain with random axes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -ftz=true -prec-div=false -prec-sqrt=false -I../../paper_2510_07674_b200/csrc -o fk_latency fk_latency.cu
#include <cstdio>
#include "coop.cuh"
using namespace spasm;

__global__ void k_fk(const ChainDesc<float>* g_ch, int iters, float* out, long long* cyc) {
  __shared__ ChainDesc<float> ch;
  if (threadIdx.x == 0) ch = *g_ch;
  __syncthreads();
  const Tile tl = Tile::make_warp();
  LaneChain<float> lc;
  lc.load(ch, tl.j);
  float q = 0.1f * tl.j + 0.01f * (threadIdx.x >> 3);
  TileFrame<float> f;
  float acc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    tile_fk(tl, lc, q, f);
    q += f.ee[0] * 1e-3f;  // carry a dependency into the next call
    acc += f.Ree[4];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  out[threadIdx.x] = acc + q;
}

__global__ void k_dls(const ChainDesc<float>* g_ch, int iters, float* out, long long* cyc) {
  __shared__ ChainDesc<float> ch;
  if (threadIdx.x == 0) ch = *g_ch;
  __syncthreads();
  const Tile tl = Tile::make_warp();
  float col[5], e[5];
  for (int k = 0; k < 5; ++k) { col[k] = 0.1f * (k + 1) + 0.01f * tl.j; e[k] = 0.01f * k; }
  float acc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const float dq = tile_dls<float, 5>(tl, col, e, 1e-3f);
    col[0] += dq * 1e-3f;
    acc += dq;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  out[threadIdx.x] = acc;
}

__global__ void k_shfl(int iters, float* out, long long* cyc) {
  float v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_up_sync(0xffffffffu, v, 1, 8) + 1.f;
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  out[threadIdx.x] = v;
}

__global__ void k_lds(const float* g, int iters, float* out, long long* cyc) {
  __shared__ float s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (float)(i % 7);
  __syncthreads();
  int k = threadIdx.x & 7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) k = (int)s[k * 8 + (threadIdx.x & 7)];
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  out[threadIdx.x] = k;
}

__global__ void k_atan2_cmp(unsigned long long n, unsigned long long seed, unsigned long long* bad) {
  unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  unsigned long long nb = 0;
  for (; i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
    unsigned long long h = (i + seed) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    float y = __uint_as_float((unsigned)h), x = __uint_as_float((unsigned)(h >> 32));
    if (i & 1) { y = (float)((int)(h & 0xffff) - 32768) * 1e-4f; x = (float)((int)((h >> 16) & 0xffff) - 32768) * 1e-4f; }
    const float a = atan2f(y, x), b = atan2_nobranch(y, x);
    if (__float_as_uint(a) != __float_as_uint(b) && !(a != a && b != b)) ++nb;
  }
  atomicAdd(bad, nb);
}

int main2();
int main() {
  ChainDesc<float> h{};
  h.J = 7;
  for (int j = 0; j < 7; ++j) {
    h.axis[j][0] = (j % 3 == 0); h.axis[j][1] = (j % 3 == 1); h.axis[j][2] = (j % 3 == 2);
    h.offset[j][0] = 0.1f; h.offset[j][1] = 0.f; h.offset[j][2] = 0.2f;
    h.lo[j] = -3.f; h.hi[j] = 3.f;
  }
  for (int c = 0; c < 9; ++c) h.tool_R[c] = (c % 4 == 0);
  ChainDesc<float>* d; cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4096 * 4);
  long long* cyc; cudaMalloc(&cyc, 64 * 8);
  long long hc[1];
  for (int threads : {32, 192}) {
    k_fk<<<1, threads>>>(d, 1000, out, cyc); cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("tile_fk      %3d threads: %lld cycles/call\n", threads, hc[0]);
    k_dls<<<1, threads>>>(d, 1000, out, cyc); cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("tile_dls<5>  %3d threads: %lld cycles/call\n", threads, hc[0]);
    k_shfl<<<1, threads>>>(1000, out, cyc); cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("shfl+fadd    %3d threads: %lld cycles/iter\n", threads, hc[0]);
    k_lds<<<1, threads>>>(nullptr, 1000, out, cyc); cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("lds chain    %3d threads: %lld cycles/iter\n", threads, hc[0]);
  }
  {
    unsigned long long* bad; cudaMalloc(&bad, 8); cudaMemset(bad, 0, 8);
    k_atan2_cmp<<<1184, 256>>>(1ull << 28, 12345, bad);
    unsigned long long hb; cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    printf("atan2_nobranch vs atan2f: %llu mismatches in 2^28 inputs\n", hb);
  }
  return main2();
}

// variant: tile max through one REDUX.MAX on the (non-negative) float bit patterns
template <typename R, int NR>
__device__ __forceinline__ R tile_dls_redux(const Tile& tl, const R (&col)[NR], const R (&e)[NR], R damping) {
  R A[NR * NR];
#pragma unroll
  for (int a = 0; a < NR; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) {
      const R v = tl.sum(col[a] * col[b]);
      A[a * NR + b] = v + (a == b ? damping : R(0));
      A[b * NR + a] = A[a * NR + b];
    }
  R y[NR];
  chol_solve<R, NR>(A, e, y);
  R dq = R(0);
#pragma unroll
  for (int a = 0; a < NR; ++a) dq += col[a] * y[a];
  const R mx = __uint_as_float(__reduce_max_sync(tl.mask, __float_as_uint(fabsf(dq))));
  return dq * fminf(R(1), R(0.5) / fmaxf(mx, R(1e-12)));
}

__global__ void k_dls_redux(int iters, float* out, long long* cyc) {
  const Tile tl = Tile::make_warp();
  float col[5], e[5];
  for (int k = 0; k < 5; ++k) { col[k] = 0.1f * (k + 1) + 0.01f * tl.j; e[k] = 0.01f * k; }
  float acc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const float dq = tile_dls_redux<float, 5>(tl, col, e, 1e-3f);
    col[0] += dq * 1e-3f;
    acc += dq;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  out[threadIdx.x] = acc;
}

__global__ void k_redux_lat(int iters, float* out, long long* cyc) {
  unsigned v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __reduce_max_sync(0xffffffffu, v) + 1u;
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  out[threadIdx.x] = (float)v;
}

__global__ void k_polstep(const ChainDesc<float>* g_ch, int iters, float* out, long long* cyc) {
  __shared__ ChainDesc<float> ch;
  if (threadIdx.x == 0) ch = *g_ch;
  __syncthreads();
  const Tile tl = Tile::make_warp();
  PolishRun<float> run;
  float q = 0.3f + 0.05f * tl.j;
  const float tp[3] = {0.9f, 0.3f, 0.2f};
  run.begin(tl, ch, q);
  long long t0 = clock64();
  int n = 0;
  for (int i = 0; i < iters; ++i) {
    run.it = 0;  // keep iterating (no cap)
    run.step(tl, q, tp, 0.4f);
    ++n;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / n;
  out[threadIdx.x] = q;
}

int main2() {
  float* out; cudaMalloc(&out, 4096 * 4);
  long long* cyc; cudaMalloc(&cyc, 64 * 8);
  long long hc[1];
  {
    ChainDesc<float> h{};
    h.J = 7;
    for (int j = 0; j < 7; ++j) {
      h.axis[j][1] = (j % 2 == 1); h.axis[j][2] = (j % 2 == 0);
      h.offset[j][2] = 0.2f;
      h.lo[j] = -3.f; h.hi[j] = 3.f; h.full_circle[j] = 0;
    }
    for (int c = 0; c < 9; ++c) h.tool_R[c] = (c % 4 == 0);
    ChainDesc<float>* d; cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice);
    for (int threads : {32, 128, 704}) {
      k_polstep<<<1, threads>>>(d, 500, out, cyc); cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);
      printf("polish step (FK + DLS<5> + checks) %3d threads: %lld cycles/iter\n", threads, hc[0]);
    }
  }
  k_dls_redux<<<1, 32>>>(1000, out, cyc); cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("tile_dls<5> with REDUX max, 32 threads: %lld cycles/call\n", hc[0]);
  k_redux_lat<<<1, 32>>>(1000, out, cyc); cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("redux.max chain: %lld cycles/iter\n", hc[0]);
  return 0;
}
