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
#include <cooperative_groups.h>

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

// Small batches (n <= kSortCtaMax = 1024): every pass in ONE CTA of 512 threads. Warp w
// owns the contiguous segment [w * 32 * ITEMS, (w + 1) * 32 * ITEMS); lane l holds its
// positions seg + i * 32 + l (i < ITEMS: coalesced loads, batch i = 32 consecutive keys).
// Per 8-bit digit pass:
//   1. per-warp digit counts cnt[w][d] (__match_any_sync peers; the batch's leader adds),
//   2. one exclusive scan over the counters in digit-major order (d, w): warp w's keys of
//      digit d land after every earlier warp's keys of digit d and every smaller digit,
//   3. each warp walks its batches again in order; the leader of a digit group takes its
//      base by a shared atomicAdd on cnt[w][d] (one warp's atomics on an address are
//      performed in issue order, so batch i precedes batch i+1) and broadcasts it; key i of
//      the group goes to base + its rank among the group,
// so every pass is stable and ties keep their index order (numpy's kind="stable"), with
// three CTA barriers per pass. One CTA's MATCH / atomic issue bounds it (2k / 4k / 8k keys:
// 24 / 34 / 50 us), so above 1k keys the cluster form below spreads the passes over SMs.
constexpr int kSortCtaThreads = 512;
constexpr int kSortCtaWarps = kSortCtaThreads / 32;
constexpr int kSortCtaMax = 2 * kSortCtaThreads;  // 1024 (above: k_radix_sort_cluster)
constexpr int kSortCntStride = 257;  // counter row stride: fewer bank conflicts in the digit-major scan

template <typename K, int ITEMS>
__global__ void __launch_bounds__(kSortCtaThreads) k_radix_sort_cta(K* ka, uint32_t* va, K* kb, uint32_t* vb, int n,
                                                                    int key_bits) {
  constexpr int NW = kSortCtaWarps, TPD = NW / 8;  // threads per digit in the scan (8 counters each)
  constexpr int G = ITEMS < 16 ? ITEMS : 16;       // keys per lane loaded together by the scatter walk
  __shared__ unsigned int cnt[NW * kSortCntStride];
  __shared__ unsigned int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int seg = warp * 32 * ITEMS + lane;
  unsigned int* const row = cnt + warp * kSortCntStride;
  for (int shift = 0; shift < key_bits; shift += 8) {
    // ka/va were written by this CTA in the previous pass (ordered by the barrier below):
    // plain loads, not the read-only path; the scatter walk re-reads the segment (L1 hits)
    // instead of holding it in registers across the scan, G keys per lane at a time
#pragma unroll
    for (int q = 0; q < 8; ++q) row[lane * 8 + q] = 0u;
    __syncwarp();
#pragma unroll
    for (int g0 = 0; g0 < ITEMS; g0 += ITEMS) {  // all the segment's loads together: one latency
      K key[ITEMS];
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) key[j] = seg + (g0 + j) * 32 < n ? ka[seg + (g0 + j) * 32] : K(0);
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const bool valid = seg + (g0 + j) * 32 < n;
        const unsigned d = valid ? (unsigned)((key[j] >> shift) & 0xFF) : 256u;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
        if (valid && (peers & lt_mask) == 0u) atomicAdd(&row[d], (unsigned)__popc(peers));
      }
    }
    __syncthreads();
    {  // exclusive scan over (digit, warp), digit-major: thread t owns digit t / TPD and 8 warps
      const int d = tid / TPD, w0 = (tid % TPD) * 8;
      unsigned int c[8], tot = 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = cnt[(w0 + j) * kSortCntStride + d];
        tot += c[j];
      }
      unsigned int inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += t;
      }
      if (lane == 31) wsum[warp] = inc;
      __syncthreads();
      if (warp == 0) {
        const unsigned int ws = lane < NW ? wsum[lane] : 0u;
        unsigned int wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned int t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
          if (lane >= o) wi += t;
        }
        if (lane < NW) wsum[lane] = wi - ws;
      }
      __syncthreads();
      unsigned int acc = wsum[warp] + inc - tot;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        cnt[(w0 + j) * kSortCntStride + d] = acc;
        acc += c[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int g0 = 0; g0 < ITEMS; g0 += G) {  // loads first (kb may alias ka for the compiler)
      K key[G];
      uint32_t val[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const bool valid = seg + (g0 + j) * 32 < n;
        key[j] = valid ? ka[seg + (g0 + j) * 32] : K(0);
        val[j] = valid ? va[seg + (g0 + j) * 32] : 0u;
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const bool valid = seg + (g0 + j) * 32 < n;
        const unsigned d = valid ? (unsigned)((key[j] >> shift) & 0xFF) : 256u;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
        const unsigned rank = (unsigned)__popc(peers & lt_mask);
        unsigned base = 0u;
        if (valid && rank == 0u) base = atomicAdd(&row[d], (unsigned)__popc(peers));
        base = __shfl_sync(0xFFFFFFFFu, base, __ffs(peers) - 1);
        if (valid) {
          kb[base + rank] = key[j];
          vb[base + rank] = val[j];
        }
      }
    }
    __syncthreads();  // the scattered pass is visible to every warp before the next pass loads it
    K* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
}

template <typename K>
inline void launch_sort_cta(K* k0, uint32_t* v0, K* k1, uint32_t* v1, int n, int key_bits, cudaStream_t stream) {
  constexpr int T = kSortCtaThreads;
  if (n <= T)
    k_radix_sort_cta<K, 1><<<1, T, 0, stream>>>(k0, v0, k1, v1, n, key_bits);
  else
    k_radix_sort_cta<K, 2><<<1, T, 0, stream>>>(k0, v0, k1, v1, n, key_bits);
}

// Mid-size batches (1024 < n <= kSortClusterMax): every pass in ONE launch of a thread-block
// cluster of C CTAs of 256 threads, CTA c owning the keys [c T, (c + 1) T), T = 256 ITEMS
// (ITEMS = 4 / 8 / 16 for n <= 8k / 16k / 64k; C <= 8, up to 16 through the non-portable
// cluster size). Per pass each CTA forms per-warp digit counts over warp-contiguous
// segments (as k_radix_sort_cta), its 256 threads (one per digit) sum them into the CTA's
// histogram and publish it; after a cluster barrier every CTA reads the C histograms through
// distributed shared memory, so digit d of CTA c starts at (keys of smaller digits anywhere)
// + (keys of digit d in CTAs < c), and each warp scatters with atomic bases. A fence and a
// second cluster barrier make the pass's global writes visible to the next pass's loads in
// the other CTAs (and keep every CTA's histogram alive while its peers read it). One launch
// replaces 12 (3 per pass) for the 16k-particle select of C2 / C4 and the 64k one of C3
// (particle_opt.py:195-200): 16k keys 35 us against 71 us (scripts/sort_timing.py, B200).
constexpr int kSortClThreads = 256;
constexpr int kSortClusterMax = 16 * kSortClThreads * 16;  // 65536

template <typename K, int ITEMS>
__global__ void __launch_bounds__(kSortClThreads) k_radix_sort_cluster(K* ka, uint32_t* va, K* kb, uint32_t* vb,
                                                                       int n, int key_bits) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int NW = kSortClThreads / 32;
  __shared__ unsigned int cnt[NW * kSortCntStride];
  __shared__ unsigned int hist[256];
  __shared__ unsigned int wsum[NW];
  const int C = (int)cl.num_blocks(), c = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int seg = c * kSortClThreads * ITEMS + warp * 32 * ITEMS + lane;
  unsigned int* const row = cnt + warp * kSortCntStride;
  for (int shift = 0; shift < key_bits; shift += 8) {
    K key[ITEMS];
    uint32_t val[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {  // written by the cluster in the previous pass: plain loads
      const int pos = seg + i * 32;
      key[i] = pos < n ? ka[pos] : K(0);
      val[i] = pos < n ? va[pos] : 0u;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) row[lane * 8 + q] = 0u;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool valid = seg + i * 32 < n;
      const unsigned d = valid ? (unsigned)((key[i] >> shift) & 0xFF) : 256u;
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
      if (valid && (peers & lt_mask) == 0u) atomicAdd(&row[d], (unsigned)__popc(peers));
    }
    __syncthreads();
    // thread d: the CTA's count of digit d, and each warp's exclusive prefix within the CTA
    unsigned int wpre[NW], h = 0u;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      wpre[w] = h;
      h += cnt[w * kSortCntStride + tid];
    }
    hist[tid] = h;
    cl.sync();  // every CTA's histogram of this pass is published
    unsigned int tot = 0u, pre = 0u;
    for (int r = 0; r < C; ++r) {
      const unsigned int v = cl.map_shared_rank(hist, r)[tid];
      tot += v;
      pre += r < c ? v : 0u;
    }
    // exclusive scan of the cluster-wide digit totals over the 256 digits
    unsigned int inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    unsigned int wbase = 0u;
#pragma unroll
    for (int w = 0; w < NW; ++w) wbase += w < warp ? wsum[w] : 0u;
    const unsigned int base = wbase + inc - tot + pre;
#pragma unroll
    for (int w = 0; w < NW; ++w) cnt[w * kSortCntStride + tid] = base + wpre[w];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool valid = seg + i * 32 < n;
      const unsigned d = valid ? (unsigned)((key[i] >> shift) & 0xFF) : 256u;
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
      const unsigned rank = (unsigned)__popc(peers & lt_mask);
      unsigned b = 0u;
      if (valid && rank == 0u) b = atomicAdd(&row[d], (unsigned)__popc(peers));
      b = __shfl_sync(0xFFFFFFFFu, b, __ffs(peers) - 1);
      if (valid) {
        kb[b + rank] = key[i];
        vb[b + rank] = val[i];
      }
    }
    __threadfence();  // this pass's scatter is visible cluster-wide before the next pass loads
    cl.sync();
    K* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
}

template <typename K, int ITEMS>
inline cudaError_t launch_sort_cluster_t(K* k0, uint32_t* v0, K* k1, uint32_t* v1, int n, int key_bits,
                                         cudaStream_t stream) {
  const unsigned C = (unsigned)((n + kSortClThreads * ITEMS - 1) / (kSortClThreads * ITEMS));
  if (C > 8) {  // 9-16 CTAs: B200 schedules clusters of up to 16 once the kernel opts in
    static const cudaError_t opt =
        cudaFuncSetAttribute(k_radix_sort_cluster<K, ITEMS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (opt != cudaSuccess) return opt;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kSortClThreads);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_radix_sort_cluster<K, ITEMS>, k0, v0, k1, v1, n, key_bits);
}

template <typename K>
inline cudaError_t launch_sort_cluster(K* k0, uint32_t* v0, K* k1, uint32_t* v1, int n, int key_bits,
                                       cudaStream_t stream) {
  if (n <= 8 * kSortClThreads * 4) return launch_sort_cluster_t<K, 4>(k0, v0, k1, v1, n, key_bits, stream);
  if (n <= 8 * kSortClThreads * 8) return launch_sort_cluster_t<K, 8>(k0, v0, k1, v1, n, key_bits, stream);
  return launch_sort_cluster_t<K, 16>(k0, v0, k1, v1, n, key_bits, stream);
}

// kernels radix_sort_pairs launches for n keys of key_bits bits
inline int radix_sort_launches(int64_t n, int key_bits) {
  if (n <= 1) return 0;
  return n <= kSortClusterMax ? 1 : 3 * (key_bits / 8);
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
    launch_sort_cta<K>(k0, v0, k1, v1, (int)n, key_bits, stream);
    *result_in_1 = ((key_bits / 8) & 1) != 0;
    return cudaGetLastError();
  }
  if (n <= kSortClusterMax) {
    *result_in_1 = ((key_bits / 8) & 1) != 0;
    return launch_sort_cluster<K>(k0, v0, k1, v1, (int)n, key_bits, stream);
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
