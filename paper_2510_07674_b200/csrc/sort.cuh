// Stable device-wide LSD radix sort of (key, uint32 value) pairs, 8-bit digits.
//
// Replaces np.argsort(costs, kind="stable") in select_topk and in the final
// satisfying-particle ordering (reference particle_opt.py:195-200 and :363). Keys are
// order-preserving images of the IEEE costs (common.cuh order_key), values are row
// indices in ascending order, and every pass is stable, so ties resolve by index
// exactly like numpy's stable sort.
//
// Per pass: k_radix_hist (per-tile digit histogram, digit-major) -> k_radix_scan
// (exclusive scan over digit x tile) -> k_radix_scatter (stable in-tile ranking with
// __match_any_sync + per-warp digit counters, then scatter).
#pragma once
#include "common.cuh"

namespace spasm {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;  // per thread per tile
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kSortWarps = kSortThreads / 32;

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const K* __restrict__ keys, int64_t n, int shift,
                                                             unsigned int* __restrict__ hist, int nblocks,
                                                             unsigned int* __restrict__ totals) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const int64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(unsigned)((keys[i] >> shift) & 0xFF)], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
  // per-digit totals (integer atomics: order-independent, deterministic)
  if (h[threadIdx.x]) atomicAdd(&totals[threadIdx.x], h[threadIdx.x]);
}

// Block-wide (256 threads) exclusive scan; *total receives the block sum.
__device__ __forceinline__ unsigned int block_exclusive_scan256(unsigned int v, unsigned int* warp_sums,
                                                                unsigned int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const unsigned int w = lane < 8 ? warp_sums[lane] : 0u;
    unsigned int wi = w;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const unsigned int t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < 8) warp_sums[lane] = wi - w;  // exclusive warp offsets
    if (lane == 7) *total = wi;
  }
  __syncthreads();
  const unsigned int r = warp_sums[warp] + inc - v;
  __syncthreads();
  return r;
}

// Exclusive scan of the digit-major counters, one CTA per digit: the CTA for digit d starts
// from the total count of all smaller digits and scans its column of per-tile counts.
// (Replaces a single-CTA scan that took 120 us per pass at n = 1M.)
static __global__ void __launch_bounds__(256) k_radix_scan(unsigned int* __restrict__ hist, int nblocks,
                                                           const unsigned int* __restrict__ totals) {
  __shared__ unsigned int warp_sums[8];
  __shared__ unsigned int total;
  const int d = blockIdx.x;
  block_exclusive_scan256(threadIdx.x < d ? totals[threadIdx.x] : 0u, warp_sums, &total);
  unsigned int carry = total;  // count of all keys with a smaller digit
  unsigned int* col = hist + (int64_t)d * nblocks;
  for (int b = 0; b < nblocks; b += 256) {
    const int i = b + threadIdx.x;
    const unsigned int v = i < nblocks ? col[i] : 0u;
    const unsigned int ex = block_exclusive_scan256(v, warp_sums, &total);
    if (i < nblocks) col[i] = carry + ex;
    carry += total;
  }
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                                K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                                int64_t n, int shift,
                                                                const unsigned int* __restrict__ hist, int nblocks,
                                                                unsigned int* __restrict__ totals) {
  __shared__ unsigned int running[256];
  if (blockIdx.x == 0) totals[threadIdx.x] = 0;  // k_radix_scan has consumed them: reset for the next pass
  __shared__ unsigned int wcnt[kSortWarps][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  running[threadIdx.x] = hist[(int64_t)threadIdx.x * nblocks + blockIdx.x];
  for (int w = 0; w < kSortWarps; ++w) wcnt[w][threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int r = 0; r < kSortItems; ++r) {
    const int64_t i = base + r * kSortThreads + threadIdx.x;
    const bool valid = i < n;
    K key = valid ? kin[i] : K(0);
    uint32_t val = valid ? vin[i] : 0u;
    const unsigned digit = valid ? (unsigned)((key >> shift) & 0xFF) : 256u;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, digit);
    const unsigned rank = __popc(peers & lt_mask);
    const bool leader = rank == 0;
    if (valid && leader) wcnt[warp][digit] = __popc(peers);
    __syncthreads();
    {  // exclusive prefix over warps for digit = threadIdx.x, seeded by the running offset
      unsigned acc = running[threadIdx.x];
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const unsigned t = wcnt[w][threadIdx.x];
        wcnt[w][threadIdx.x] = acc;
        acc += t;
      }
      running[threadIdx.x] = acc;
    }
    __syncthreads();
    if (valid) {
      const unsigned pos = wcnt[warp][digit] + rank;
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
    for (int w = 0; w < kSortWarps; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
  }
}

// Small batches (n <= kSortCtaMax): every pass in ONE CTA of 1024 threads, chunks of 1024
// keys scattered in order (match_any ranks + per-warp digit offsets), so the sort stays
// stable and needs one launch instead of 3 per pass (the satisfying-particle ordering of
// particle_opt.py:363 runs on m <= 8k keys every restart; above 8k the multi-CTA passes win).
constexpr int kSortCtaMax = 8192;

template <typename K>
__global__ void __launch_bounds__(1024) k_radix_sort_cta(K* __restrict__ ka, uint32_t* __restrict__ va,
                                                         K* __restrict__ kb, uint32_t* __restrict__ vb, int n,
                                                         int key_bits) {
  __shared__ unsigned int run[256];
  __shared__ unsigned int wcnt[32][256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int shift = 0; shift < key_bits; shift += 8) {
    if (tid < 256) run[tid] = 0;
    for (int w = 0; w < 32; ++w)
      if (tid < 256) wcnt[w][tid] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += 1024) atomicAdd(&run[(unsigned)((ka[i] >> shift) & 0xFF)], 1u);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 256 digit counts (8 per lane)
      unsigned int c[8], tot = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        c[q] = run[lane * 8 + q];
        tot += c[q];
      }
      unsigned int inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += t;
      }
      unsigned int acc = inc - tot;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        run[lane * 8 + q] = acc;
        acc += c[q];
      }
    }
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
      const int i = base + tid;
      const bool valid = i < n;
      const K key = valid ? ka[i] : K(0);
      const uint32_t val = valid ? va[i] : 0u;
      const unsigned digit = valid ? (unsigned)((key >> shift) & 0xFF) : 256u;
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, digit);
      const unsigned rank = __popc(peers & lt_mask);
      if (valid && rank == 0) wcnt[warp][digit] = __popc(peers);
      __syncthreads();
      if (tid < 256) {
        unsigned int acc = run[tid];
        for (int w = 0; w < 32; ++w) {
          const unsigned int t = wcnt[w][tid];
          wcnt[w][tid] = acc;
          acc += t;
        }
        run[tid] = acc;
      }
      __syncthreads();
      if (valid) {
        const unsigned pos = wcnt[warp][digit] + rank;
        kb[pos] = key;
        vb[pos] = val;
      }
      __syncthreads();
      if (tid < 256)
        for (int w = 0; w < 32; ++w) wcnt[w][tid] = 0;
      __syncthreads();
    }
    K* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
}

// kernels radix_sort_pairs launches for n keys of key_bits bits
inline int radix_sort_launches(int64_t n, int key_bits) {
  if (n <= 1) return 0;
  return n <= kSortCtaMax ? 1 : 3 * (key_bits / 8);
}

// Host driver. Sorts (k0, v0) by key bits [0, key_bits) into (k1, v1) ping-pong
// buffers; returns through *result_in_1 whether the final data sits in k1/v1.
// hist must hold 256 * (ceil(n / kSortTile) + 1) counters: the last 256 are the per-digit
// totals of the current pass.
template <typename K>
inline cudaError_t radix_sort_pairs(K* k0, uint32_t* v0, K* k1, uint32_t* v1, int64_t n, int key_bits,
                                    unsigned int* hist, bool* result_in_1, cudaStream_t stream) {
  *result_in_1 = false;
  if (n <= 1) return cudaSuccess;
  if (n <= kSortCtaMax) {
    k_radix_sort_cta<K><<<1, 1024, 0, stream>>>(k0, v0, k1, v1, (int)n, key_bits);
    *result_in_1 = ((key_bits / 8) & 1) != 0;
    return cudaGetLastError();
  }
  const int nblocks = ceil_div(n, kSortTile);
  unsigned int* totals = hist + (int64_t)256 * nblocks;
  K* ka = k0; K* kb = k1; uint32_t* va = v0; uint32_t* vb = v1;
  bool in1 = false;
  cudaError_t e = cudaMemsetAsync(totals, 0, 256 * sizeof(unsigned int), stream);
  if (e != cudaSuccess) return e;
  for (int shift = 0; shift < key_bits; shift += 8) {
    k_radix_hist<K><<<nblocks, kSortThreads, 0, stream>>>(ka, n, shift, hist, nblocks, totals);
    k_radix_scan<<<256, 256, 0, stream>>>(hist, nblocks, totals);
    k_radix_scatter<K><<<nblocks, kSortThreads, 0, stream>>>(ka, va, kb, vb, n, shift, hist, nblocks, totals);
    std::swap(ka, kb);
    std::swap(va, vb);
    in1 = !in1;
  }
  *result_in_1 = in1;
  return cudaGetLastError();
}

}  // namespace spasm
