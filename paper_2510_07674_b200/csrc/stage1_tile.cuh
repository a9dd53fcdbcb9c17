// fp32 stage-1 descent kernel specialised for the tetris packing scenes (the C3/C5 hot
// loop): k_schedule_tile runs the whole K_lin + K_quad schedule (particle_opt.py:266-300)
// plus the final QUADRATIC cost with every table index known at compile time.
//
// Differences from the generic k_schedule (stage1_kernels.cuh), same semantics:
//   * the body count N is a template parameter, every pair loop is fully unrolled, the
//     particle state x and gradient g live in registers and every scene constant is a
//     constant-bank / uniform-register operand (no address arithmetic in the pair loop);
//   * V is the per-lane arithmetic type (float). Packing two particles per thread into
//     sm_100a FFMA2/FADD2 was tried and dropped: cicc -O3 needs > 15 min per unrolled
//     instantiation and ptxas then uses ~250 registers;
//   * LA > 1 splits one particle's a-spheres across LA lanes of a warp for small M;
//     partial gradients are combined with a butterfly __shfl_xor (north_star: warp-shuffle
//     reductions over spheres), the height term is added after the reduction, and every
//     lane applies the identical clamped step.
//   * pair math (fixed yaw, uniform sphere radius r, rsum = 2r):
//       linear:    s = [d2 < rsum^2] / d            (d2 = 0 -> zero gradient, the
//       quadratic: s = max(rsum / d - 1, 0) = pen/d  reference's coincident-centre rule)
//     with 1/d = rsqrt(max(d2, 1e-30)), d cost/d ca = -w s (ca - cb) (x2 in quadratic).
// Wall pairs use the cancellation-free form of pen_static_acc (stage1_models.cuh).
#pragma once
#include "stage1_models.cuh"

namespace spasm {

// ---- scalar / packed-pair arithmetic --------------------------------------------------
template <typename V> struct VX;

template <> struct VX<float> {
  static constexpr int P = 1;
  static __device__ __forceinline__ float add(float a, float b) { return a + b; }
  static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
  static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
  static __device__ __forceinline__ float fma(float a, float b, float c) { return fmaf(a, b, c); }
  static __device__ __forceinline__ float k(float s, float2) { return s; }
  static __device__ __forceinline__ float zero() { return 0.f; }
  static __device__ __forceinline__ float rsq(float d2) { return rsqrtf(fmaxf(d2, 1e-30f)); }
  static __device__ __forceinline__ float sel_lt(float a, float b, float v) { return a < b ? v : 0.f; }
  static __device__ __forceinline__ float sel_gt0(float a, float v) { return a > 0.f ? v : 0.f; }
  static __device__ __forceinline__ float relu(float a) { return fmaxf(a, 0.f); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdividef(a, b); }
  static __device__ __forceinline__ float shfl_xor(float a, int m) { return __shfl_xor_sync(0xffffffffu, a, m); }
  static __device__ __forceinline__ float get(float a, int) { return a; }
  static __device__ __forceinline__ void set(float& a, int, float v) { a = v; }
};

// ---- the tile model ---------------------------------------------------------------------
template <int N, int LA, typename V>
struct TetrisTile {
  using O = VX<V>;
  static constexpr int D = 3 * N;
  static constexpr int SA = kTileSpb / LA;  // a-spheres of each body handled by one lane

  // lane-specific local offsets of the lane's a-spheres (LA > 1 only)
  struct Lane {
    V ax[N][SA], ay[N][SA], az[N][SA];
  };

  static __device__ __forceinline__ void init_lane(const TetrisTileScene& sc, int lane, Lane& L) {
    if constexpr (LA > 1) {
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int k = 0; k < SA; ++k) {
          const int a = i * kTileSpb + lane * SA + k;
          L.ax[i][k] = O::k(sc.lx[a], sc.lx2[a]);
          L.ay[i][k] = O::k(sc.ly[a], sc.ly2[a]);
          L.az[i][k] = O::k(sc.lz[a], sc.lz2[a]);
        }
    }
  }

  // Partial (lane) cost and/or gradient of the pair terms; the caller reduces across the
  // LA lanes and adds the height term. Q: quadratic mode.
  template <bool WC, bool WG, bool Q>
  static __device__ __forceinline__ V pairs(const TetrisTileScene& sc, const Lane& L, const V (&x)[D], V (&g)[D]) {
    V cost = O::zero();
    if constexpr (WG) {
#pragma unroll
      for (int d = 0; d < D; ++d) g[d] = O::zero();
    }
    const V rs = O::k(sc.rs, sc.rs_2), rs2 = O::k(sc.rs2, sc.rs2_2);
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int k = 0; k < SA; ++k) {
        const int a = i * kTileSpb + k;  // LA == 1 only
        const V lax = LA > 1 ? L.ax[i][k] : O::k(sc.lx[a], sc.lx2[a]);
        const V lay = LA > 1 ? L.ay[i][k] : O::k(sc.ly[a], sc.ly2[a]);
        const V laz = LA > 1 ? L.az[i][k] : O::k(sc.lz[a], sc.lz2[a]);
        const V wax = O::add(x[3 * i], lax), way = O::add(x[3 * i + 1], lay), waz = O::add(x[3 * i + 2], laz);
        // ---- body-body pairs (i < j), _interactions.py:46-60, 135-178
#pragma unroll
        for (int j = i + 1; j < N; ++j) {
          const V tx = O::sub(wax, x[3 * j]), ty = O::sub(way, x[3 * j + 1]), tz = O::sub(waz, x[3 * j + 2]);
          V gx = O::zero(), gy = O::zero(), gz = O::zero(), cp = O::zero();
#pragma unroll
          for (int sb = 0; sb < kTileSpb; ++sb) {
            const int b = j * kTileSpb + sb;
            const V dx = O::sub(tx, O::k(sc.lx[b], sc.lx2[b]));
            const V dy = O::sub(ty, O::k(sc.ly[b], sc.ly2[b]));
            const V dz = O::sub(tz, O::k(sc.lz[b], sc.lz2[b]));
            const V d2 = O::fma(dz, dz, O::fma(dy, dy, O::mul(dx, dx)));
            const V inv = O::rsq(d2);
            if constexpr (WC) {
              const V pc = O::relu(O::sub(rs, O::mul(d2, inv)));
              cp = Q ? O::fma(pc, pc, cp) : O::add(cp, pc);
            }
            if constexpr (WG) {
              const V s = Q ? O::relu(O::fma(rs, inv, O::k(-1.f, make_float2(-1.f, -1.f)))) : O::sel_lt(d2, rs2, inv);
              gx = O::fma(s, dx, gx);
              gy = O::fma(s, dy, gy);
              gz = O::fma(s, dz, gz);
            }
          }
          if constexpr (WC) cost = O::fma(O::k(sc.w_bb, make_float2(sc.w_bb, sc.w_bb)), cp, cost);
          if constexpr (WG) {
            const float w = Q ? -2.f * sc.w_bb : -sc.w_bb;
            const V wv = O::k(w, make_float2(w, w));
            const V nw = O::k(-w, make_float2(-w, -w));
            g[3 * i] = O::fma(wv, gx, g[3 * i]);
            g[3 * i + 1] = O::fma(wv, gy, g[3 * i + 1]);
            g[3 * i + 2] = O::fma(wv, gz, g[3 * i + 2]);
            g[3 * j] = O::fma(nw, gx, g[3 * j]);
            g[3 * j + 1] = O::fma(nw, gy, g[3 * j + 1]);
            g[3 * j + 2] = O::fma(nw, gz, g[3 * j + 2]);
          }
        }
        // ---- sphere vs wall (cancellation-free form), _interactions.py:62-73
#pragma unroll
        for (int st = 0; st < kTileWalls; ++st) {
          const V vx = O::sub(wax, O::k(sc.ax[st], sc.ax2[st]));
          const V vy = O::sub(way, O::k(sc.ay[st], sc.ay2[st]));
          const V vz = O::sub(waz, O::k(sc.az[st], sc.az2[st]));
          const V vn = O::fma(vz, O::k(sc.nz[st], sc.nz2[st]),
                              O::fma(vy, O::k(sc.ny[st], sc.ny2[st]), O::mul(vx, O::k(sc.nx[st], sc.nx2[st]))));
          const V vv = O::fma(vz, vz, O::fma(vy, vy, O::mul(vx, vx)));
          const V q = O::fma(vn, O::k(sc.two_wr[st], sc.twr2[st]), vv);  // d^2 - R^2
          const V d2 = O::add(q, O::k(sc.wr2[st], sc.wrsq2[st]));
          const V inv = O::rsq(d2);
          const V dpr = O::fma(d2, inv, O::k(sc.wr[st], sc.wr_2[st]));  // d + R
          const V pen = O::sub(O::k(sc.r, sc.r_2), O::div(q, dpr));
          if constexpr (WC) {
            const V pc = O::relu(pen);
            cost = Q ? O::fma(O::k(sc.w_bs, make_float2(sc.w_bs, sc.w_bs)), O::mul(pc, pc), cost)
                     : O::fma(O::k(sc.w_bs, make_float2(sc.w_bs, sc.w_bs)), pc, cost);
          }
          if constexpr (WG) {
            const float w = Q ? -2.f * sc.w_bs : -sc.w_bs;
            const V s = O::sel_gt0(pen, Q ? O::mul(O::mul(O::k(w, make_float2(w, w)), pen), inv)
                                          : O::mul(O::k(w, make_float2(w, w)), inv));
            // diff = c - s = v + R n
            g[3 * i] = O::fma(s, O::add(vx, O::k(sc.wrn_x[st], sc.wrnx2[st])), g[3 * i]);
            g[3 * i + 1] = O::fma(s, O::add(vy, O::k(sc.wrn_y[st], sc.wrny2[st])), g[3 * i + 1]);
            g[3 * i + 2] = O::fma(s, O::add(vz, O::k(sc.wrn_z[st], sc.wrnz2[st])), g[3 * i + 2]);
          }
        }
      }
    }
    return cost;
  }

  // Height term (tetris.py:226-238; sign(0) == 0), identical on every lane.
  template <bool WC, bool WG, bool Q>
  static __device__ __forceinline__ void height(const TetrisTileScene& sc, const V (&x)[D], V (&g)[D], V& cost) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int c = 0; c < O::P; ++c) {
        const float dz = O::get(x[3 * i + 2], c) - sc.z_star;
        if constexpr (WC) O::set(cost, c, O::get(cost, c) + (Q ? sc.w_h * (dz * dz) : sc.w_h * fabsf(dz)));
        if constexpr (WG)
          O::set(g[3 * i + 2], c,
                 O::get(g[3 * i + 2], c) +
                     (Q ? sc.w_h * (2.f * dz) : sc.w_h * (dz > 0.f ? 1.f : (dz < 0.f ? -1.f : 0.f))));
      }
    }
  }
};

template <int LA, typename V>
__device__ __forceinline__ V lane_sum(V v) {
  if constexpr (LA >= 2) v = VX<V>::add(v, VX<V>::shfl_xor(v, 1));
  if constexpr (LA >= 4) v = VX<V>::add(v, VX<V>::shfl_xor(v, 2));
  return v;
}

// Full cost/gradient of the particle(s) on every lane of the group.
template <class T, int LA, typename V, bool WC, bool WG, bool Q>
__device__ __forceinline__ V tile_eval(const TetrisTileScene& sc, const typename T::Lane& L, const V (&x)[T::D],
                                      V (&g)[T::D]) {
  V cost = T::template pairs<WC, WG, Q>(sc, L, x, g);
  if constexpr (LA > 1) {
    if constexpr (WC) cost = lane_sum<LA>(cost);
    if constexpr (WG) {
#pragma unroll
      for (int d = 0; d < T::D; ++d) g[d] = lane_sum<LA>(g[d]);
    }
  }
  T::template height<WC, WG, Q>(sc, x, g, cost);
  return cost;
}

// One clamped step per particle component with the NaN freeze (particle_opt.py:214-228).
template <int D, typename V>
__device__ __forceinline__ void tile_step(const TetrisTileScene& sc, V (&x)[D], const V (&g)[D], float rate,
                                          bool (&bad)[VX<V>::P]) {
  using O = VX<V>;
#pragma unroll
  for (int c = 0; c < O::P; ++c) {
    bool b = false;
#pragma unroll
    for (int d = 0; d < D; ++d) b |= !isfinite(O::get(g[d], c));
    bad[c] |= b;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      float v = O::get(x[d], c);
      if (!b) v = v - rate * O::get(g[d], c);
      v = fminf(fmaxf(v, sc.lower[d]), sc.upper[d]);
      O::set(x[d], c, v);
    }
  }
}

template <int N, int LA, typename V>
__global__ void __launch_bounds__(128) k_schedule_tile(const __grid_constant__ TetrisTileScene sc,
                                                       const float* __restrict__ src, const uint32_t* __restrict__ rows,
                                                       int64_t M, int k_lin, int k_quad, double eta, double alpha,
                                                       float* __restrict__ out_values, float* __restrict__ out_cost,
                                                       uint8_t* __restrict__ flagged,
                                                       unsigned int* __restrict__ flagged_count) {
  using T = TetrisTile<N, LA, V>;
  using O = VX<V>;
  constexpr int D = T::D, P = O::P;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(threadIdx.x % LA);
  const int64_t p0 = (gtid / LA) * P;  // first particle of this lane group
  V x[D], g[D];
#pragma unroll
  for (int c = 0; c < P; ++c) {
    const int64_t p = p0 + c;
    const bool live = p < M;
    const int64_t row = live ? (rows ? (int64_t)rows[p] : p) : 0;
#pragma unroll
    for (int d = 0; d < D; ++d) O::set(x[d], c, live ? src[row * D + d] : sc.lower[d]);
  }
  typename T::Lane L;
  T::init_lane(sc, lane, L);
  bool bad[P];
#pragma unroll
  for (int c = 0; c < P; ++c) bad[c] = false;
  for (int k = 1; k <= k_lin; ++k) {
    // lr_schedule in float64 exactly as the reference, then cast (particle_opt.py:203-211)
    const float rate = (float)(eta * (1.0 - (double)k / (double)k_lin));
    tile_eval<T, LA, V, false, true, false>(sc, L, x, g);
    tile_step<D, V>(sc, x, g, rate, bad);
  }
  for (int k = 0; k < k_quad; ++k) {
    tile_eval<T, LA, V, false, true, true>(sc, L, x, g);
    tile_step<D, V>(sc, x, g, (float)alpha, bad);
  }
  const V fc = tile_eval<T, LA, V, true, false, true>(sc, L, x, g);
  if (lane != 0) return;
#pragma unroll
  for (int c = 0; c < P; ++c) {
    const int64_t p = p0 + c;
    if (p >= M) break;
#pragma unroll
    for (int d = 0; d < D; ++d) out_values[p * D + d] = O::get(x[d], c);
    out_cost[p] = O::get(fc, c);
    if (flagged) flagged[p] = bad[c] ? 1 : 0;
    if (bad[c] && flagged_count) atomicAdd(flagged_count, 1u);
  }
}

}  // namespace spasm
