// fp32 stage-1 descent kernel for the tower scenes (C2 tower3c, C4 tower6r, tower4), the
// tower counterpart of stage1_tile.cuh: compile-time block count B, state in registers,
// LA = 4 lanes per particle. The cube-obstacle pairs (B x O, the bulk of the work) are split
// over the lanes (obstacle o on lane o % 4, table in shared memory) and shuffle-reduced;
// the stability, height and cube-pair terms are cheap and computed identically on every
// lane after the reduction. Semantics of TowerCostModel (tower.py:144-322) with fixed yaw,
// same as TowerEval<float, false> (stage1_models.cuh).
#pragma once
#include "stage1_tile.cuh"

namespace spasm {

template <int B, int LA>
struct TowerTile {
  static constexpr int D = 3 * B;

  // cube-obstacle pairs of this lane: pen = (radius + orad) - |c - o|
  template <bool WC, bool WG>
  static __device__ __forceinline__ float obstacles(const TowerTileScene& sc, const float* tab, bool Q, int lane,
                                                    const float (&x)[D], float (&g)[D]) {
    float cost = 0.f;
    if constexpr (WG) {
#pragma unroll
      for (int d = 0; d < D; ++d) g[d] = 0.f;
    }
    const int no = sc.n_obs;
    for (int o = lane; o < no; o += LA) {
      const float ox = tab[o], oy = tab[kMaxObstacles + o], oz = tab[2 * kMaxObstacles + o];
      const float rs = sc.radius + tab[3 * kMaxObstacles + o];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const float dx = x[3 * i] - ox, dy = x[3 * i + 1] - oy, dz = x[3 * i + 2] - oz;
        const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        const float inv = rsqrtf(fmaxf(d2, 1e-30f));
        const float pen = rs - d2 * inv;
        if constexpr (WC) {
          const float pc = fmaxf(pen, 0.f);
          cost = fmaf(sc.w_c, Q ? pc * pc : pc, cost);
        }
        if constexpr (WG) {
          // d cost / d c = -w s (c - o): linear s = 1/d, quadratic s = 2 pen / d (active pen > 0)
          const float s = pen > 0.f ? (Q ? 2.f * pen : 1.f) * inv : 0.f;
          g[3 * i] = fmaf(-sc.w_c * s, dx, g[3 * i]);
          g[3 * i + 1] = fmaf(-sc.w_c * s, dy, g[3 * i + 1]);
          g[3 * i + 2] = fmaf(-sc.w_c * s, dz, g[3 * i + 2]);
        }
      }
    }
    return cost;
  }

  // stability (suffix CoM vs footprint), heights and cube pairs; every lane
  template <bool WC, bool WG>
  static __device__ __forceinline__ void shared_terms(const TowerTileScene& sc, bool Q, const float (&x)[D],
                                                      float (&g)[D], float& cost) {
    float sx = 0.f, sy = 0.f, accx = 0.f, accy = 0.f;
    float sfx[B], sfy[B];  // suffix sums from the top (tower.py:208-210)
#pragma unroll
    for (int k = B - 1; k >= 0; --k) {
      sx = (k == B - 1) ? x[3 * k] : sx + x[3 * k];
      sy = (k == B - 1) ? x[3 * k + 1] : sy + x[3 * k + 1];
      sfx[k] = sx;
      sfy[k] = sy;
    }
#pragma unroll
    for (int i = 0; i + 1 < B; ++i) {
      const float cnt = (float)(B - 1 - i);
      const float relx = sfx[i + 1] / cnt - x[3 * i], rely = sfy[i + 1] / cnt - x[3 * i + 1];
      const float h = sc.half;
      const float dlx = relx - fminf(fmaxf(relx, -h), h), dly = rely - fminf(fmaxf(rely, -h), h);
      const float dist = sqrtf(dlx * dlx + dly * dly);
      if constexpr (WC) cost += Q ? sc.w_s * (dist * dist) : sc.w_s * dist;
      if constexpr (WG) {
        const float factor = sc.w_s * (Q ? 2.f * dist : (dist > 0.f ? 1.f : 0.f));
        const float gx = dist > 0.f ? factor * (dlx / dist) : 0.f, gy = dist > 0.f ? factor * (dly / dist) : 0.f;
        accx += gx / cnt;
        accy += gy / cnt;
        g[3 * (i + 1)] += accx;
        g[3 * (i + 1) + 1] += accy;
        g[3 * i] -= gx;
        g[3 * i + 1] -= gy;
      }
    }
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const float dz = x[3 * i + 2] - sc.target[i];
      if constexpr (WC) cost += Q ? sc.w_h * (dz * dz) : sc.w_h * fabsf(dz);
      if constexpr (WG) g[3 * i + 2] += sc.w_h * (Q ? 2.f * dz : (dz > 0.f ? 1.f : (dz < 0.f ? -1.f : 0.f)));
    }
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int j = i + 1; j < B; ++j) {
        const float dx = x[3 * i] - x[3 * j], dy = x[3 * i + 1] - x[3 * j + 1], dz = x[3 * i + 2] - x[3 * j + 2];
        const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        const float inv = rsqrtf(fmaxf(d2, 1e-30f));
        const float pen = sc.side - d2 * inv;
        if constexpr (WC) {
          const float pc = fmaxf(pen, 0.f);
          cost = fmaf(sc.w_c, Q ? pc * pc : pc, cost);
        }
        if constexpr (WG) {
          const float s = pen > 0.f ? -sc.w_c * (Q ? 2.f * pen : 1.f) * inv : 0.f;
          g[3 * i] = fmaf(s, dx, g[3 * i]);
          g[3 * i + 1] = fmaf(s, dy, g[3 * i + 1]);
          g[3 * i + 2] = fmaf(s, dz, g[3 * i + 2]);
          g[3 * j] = fmaf(-s, dx, g[3 * j]);
          g[3 * j + 1] = fmaf(-s, dy, g[3 * j + 1]);
          g[3 * j + 2] = fmaf(-s, dz, g[3 * j + 2]);
        }
      }
  }

  template <bool WC, bool WG>
  static __device__ __forceinline__ float eval(const TowerTileScene& sc, const float* tab, bool Q, int lane,
                                               const float (&x)[D], float (&g)[D]) {
    float cost = obstacles<WC, WG>(sc, tab, Q, lane, x, g);
    if constexpr (LA > 1) {
      if constexpr (WC) cost = lane_sum<LA>(cost);
      if constexpr (WG) {
#pragma unroll
        for (int d = 0; d < D; ++d) g[d] = lane_sum<LA>(g[d]);
      }
    }
    shared_terms<WC, WG>(sc, Q, x, g, cost);
    return cost;
  }
};

template <int B, int LA>
__global__ void __launch_bounds__(128) k_schedule_tower_tile(const __grid_constant__ TowerTileScene sc,
                                                             const float* __restrict__ src,
                                                             const uint32_t* __restrict__ rows, int64_t M, int k_lin,
                                                             int k_quad, double eta, double alpha,
                                                             float* __restrict__ out_values,
                                                             float* __restrict__ out_cost,
                                                             uint8_t* __restrict__ flagged,
                                                             unsigned int* __restrict__ flagged_count) {
  using T = TowerTile<B, LA>;
  constexpr int D = T::D;
  __shared__ float tab[4 * kMaxObstacles];
  for (int o = threadIdx.x; o < sc.n_obs; o += blockDim.x) {
    tab[o] = sc.ox[o];
    tab[kMaxObstacles + o] = sc.oy[o];
    tab[2 * kMaxObstacles + o] = sc.oz[o];
    tab[3 * kMaxObstacles + o] = sc.orad[o];
  }
  __syncthreads();
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(threadIdx.x % LA);
  const int64_t p = gtid / LA;
  const bool live = p < M;
  const int64_t row = live ? (rows ? (int64_t)rows[p] : p) : 0;
  float x[D], g[D];
#pragma unroll
  for (int d = 0; d < D; ++d) x[d] = live ? src[row * D + d] : sc.lower[d];
  bool bad = false;
  for (int k = 1; k <= k_lin + k_quad; ++k) {
    const bool quad = k > k_lin;
    // lr_schedule in float64 exactly as the reference, then cast (particle_opt.py:203-211)
    const float rate = quad ? (float)alpha : (float)(eta * (1.0 - (double)k / (double)k_lin));
    T::template eval<false, true>(sc, tab, quad, lane, x, g);
    tile_step<D>(sc, x, g, rate, bad);
  }
  const float fc = T::template eval<true, false>(sc, tab, true, lane, x, g);
  if (lane != 0 || !live) return;
#pragma unroll
  for (int d = 0; d < D; ++d) out_values[p * D + d] = x[d];
  out_cost[p] = fc;
  if (flagged) flagged[p] = bad ? 1 : 0;
  if (bad && flagged_count) atomicAdd(flagged_count, 1u);
}

}  // namespace spasm
