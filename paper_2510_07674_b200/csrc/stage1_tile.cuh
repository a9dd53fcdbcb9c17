// fp32 stage-1 descent kernel specialised for the tetris packing scenes (the C1/C3/C5 hot
// loop): k_schedule_tile runs the whole K_lin + K_quad schedule (particle_opt.py:266-300)
// plus the final QUADRATIC cost with every table index known at compile time.
//
// Differences from the generic k_schedule (stage1_kernels.cuh), same semantics:
//   * the body count N is a template parameter, every pair loop is fully unrolled, the
//     particle state x and gradient g live in registers and every scene constant is a
//     constant-bank operand (no address arithmetic in the pair loops);
//   * LA lanes of a warp share one particle: lane l owns a-sphere l*SA..l*SA+SA-1 of every
//     body (vs all spheres of the later bodies and the walls). Partial gradients are
//     combined with a butterfly __shfl_xor (north_star: warp-shuffle reductions over
//     spheres), the height term is added after the reduction, and every lane applies the
//     identical clamped step. LA = 4 measured fastest for every batch size;
//   * sphere pairs (fixed yaw, uniform sphere radius r, rsum = 2r), two b-spheres per
//     sm_100a FADD2/FMUL2/FFMA2 instruction (the scalar halves of a packed register pair
//     are plain registers, so the per-pair MUFU.RSQ and selects need no unpacking):
//       t = rsum / d - 1 = pen / d, active iff t > 0;  linear s = 1/d,  quadratic s = t
//     with 1/d = rsqrt(d2 + 1e-30) (coincident centres: dx = 0 -> zero gradient, the
//     reference's rule) and d cost/d ca = -w s (ca - cb) (x2 in quadratic);
//   * walls: the four box walls of box_wall_spheres (tetris.py:54-70, normals +x, -x, +y,
//     -y, verified on the host) in the cancellation-free form of pen_static_acc with the
//     axis-aligned normal folded in: q = |v|^2 + 2R v.n = d^2 - R^2, pen = r - q / (d + R).
//     (A branch skipping walls with q above the penetration bound was measured slower:
//     divergence plus 204 registers.)
//   * packing two particles per thread into sm_100a FFMA2/FADD2 was tried and dropped:
//     cicc -O3 needs > 15 min per unrolled instantiation and ptxas then uses ~250
//     registers.
#pragma once
#include "f32x2.cuh"
#include "stage1_kernels.cuh"

namespace spasm {

template <int N, int LA>
struct TetrisTile {
  static constexpr int D = 3 * N;
  static constexpr int SA = kTileSpb / LA;  // a-spheres of each body handled by one lane

  // Local offsets of the lane's a-spheres: constant-bank operands when LA == 1, else read
  // from a shared-memory copy of the sphere table (lane-dependent index, no registers held).
  struct Lane {
    const float* tab;  // shared [3][N * kTileSpb]
    int base;          // lane * SA
  };

  static __device__ __forceinline__ float off(const TetrisTileScene& sc, const Lane& L, int c, int i, int k) {
    if constexpr (LA > 1) {
      return L.tab[c * N * kTileSpb + i * kTileSpb + L.base + k];
    } else {
      const int a = i * kTileSpb + k;
      return c == 0 ? sc.lx[a] : (c == 1 ? sc.ly[a] : sc.lz[a]);
    }
  }

  // Gradient of the two walls along one axis (+axis, -axis) as one packed pair: VA = the
  // sphere's coordinate minus the two tangent points, PERP = squared off-axis part of v,
  // VO / VZ = the other horizontal / the vertical component (duplicated). Accumulates
  // into packed per-sphere accumulators GA (axis), GO (other), GZ.
  static __device__ __forceinline__ void wall_pair_grad(const TetrisTileScene& sc, unsigned qmask, F2 VA, F2 PERP,
                                                        F2 VO, F2 VZ, F2& GA, F2& GO, F2& GZ) {
    const F2 QQ = f2_fma(VA, F2{sc.two_wr_pm}, f2_fma(VA, VA, PERP));  // d^2 - R^2
    const F2 D2 = f2_add(QQ, F2{sc.wr2_d});                           // ~R^2 > 0
    float d2a, d2b, qa, qb;
    f2_split(D2, d2a, d2b);
    f2_split(QQ, qa, qb);
    const F2 INV = f2_make(rsqrtf(d2a), rsqrtf(d2b));
    float da, db;
    f2_split(f2_fma(D2, INV, F2{sc.wr_d}), da, db);  // d + R
    const F2 PEN = f2_sub(F2{sc.r_d}, f2_make(__fdividef(qa, da), __fdividef(qb, db)));
    float pa, pb;
    f2_split(PEN, pa, pb);
    // linear: -w / d; quadratic: -2 w pen / d  (k = -2w, factor 0.5 or pen)
    float sa, sb;
    f2_split(f2_mul(f2_mul(f2_make(pick(qmask, pa, 0.5f), pick(qmask, pb, 0.5f)), INV), F2{sc.k_bs_d}), sa, sb);
    const F2 S = f2_make(pa > 0.f ? sa : 0.f, pb > 0.f ? sb : 0.f);
    GA = f2_fma(S, f2_add(VA, F2{sc.wr_pm}), GA);  // diff = c - s = v + R n
    GO = f2_fma(S, VO, GO);
    GZ = f2_fma(S, VZ, GZ);
  }

  // Cost of the two walls along one axis as one packed pair: w * pen+ (or pen+^2).
  static __device__ __forceinline__ float wall_pair_cost(const TetrisTileScene& sc, bool Q, F2 VA, F2 PERP) {
    const F2 QQ = f2_fma(VA, F2{sc.two_wr_pm}, f2_fma(VA, VA, PERP));  // d^2 - R^2
    const F2 D2 = f2_add(QQ, F2{sc.wr2_d});
    float d2a, d2b, qa, qb;
    f2_split(D2, d2a, d2b);
    f2_split(QQ, qa, qb);
    float da, db;
    f2_split(f2_fma(D2, f2_make(rsqrtf(d2a), rsqrtf(d2b)), F2{sc.wr_d}), da, db);  // d + R
    const float pa = fmaxf(sc.r - __fdividef(qa, da), 0.f), pb = fmaxf(sc.r - __fdividef(qb, db), 0.f);
    return sc.w_bs * (Q ? fmaf(pa, pa, pb * pb) : pa + pb);
  }

  // Partial (lane) cost and/or gradient of the pair terms; the caller reduces across the
  // LA lanes and adds the height term. Q: quadratic mode, a runtime (warp-uniform) flag so
  // the linear and quadratic phases share one copy of the unrolled code (the two-copy
  // form stalled 42 % of issue slots on instruction-cache misses at N = 8).
  template <bool WC, bool WG>
  static __device__ __forceinline__ float pairs(const TetrisTileScene& sc, const Lane& L, bool Q, const float (&x)[D],
                                                float (&g)[D]) {
    float cost = 0.f;
    const unsigned qmask = Q ? 0xFFFFFFFFu : 0u;
    if constexpr (WG) {
#pragma unroll
      for (int d = 0; d < D; ++d) g[d] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int k = 0; k < SA; ++k) {
        const float wax = x[3 * i] + off(sc, L, 0, i, k);
        const float way = x[3 * i + 1] + off(sc, L, 1, i, k);
        const float waz = x[3 * i + 2] + off(sc, L, 2, i, k);
        // ---- body-body pairs (i < j), _interactions.py:46-60, 135-178
#pragma unroll
        for (int j = 0; j < N; ++j) {  // constant trip count: always fully unrolled
          if (j <= i) continue;
          const float tx = wax - x[3 * j], ty = way - x[3 * j + 1], tz = waz - x[3 * j + 2];
          float gx = 0.f, gy = 0.f, gz = 0.f, cp = 0.f;
          if constexpr (WC) {  // packed like the gradient path: pen = rsum - d
            const F2 TX = f2_dup(tx), TY = f2_dup(ty), TZ = f2_dup(tz);
            F2 CP = f2_dup(0.f);
#pragma unroll
            for (int h = 0; h < kTileSpb; h += 2) {
              const int b2 = (j * kTileSpb + h) / 2;
              const F2 DX = f2_sub(TX, F2{sc.px[b2]}), DY = f2_sub(TY, F2{sc.py[b2]}), DZ = f2_sub(TZ, F2{sc.pz[b2]});
              const F2 D2 = f2_fma(DZ, DZ, f2_fma(DY, DY, f2_fma(DX, DX, F2{sc.tiny_d})));
              float d2a, d2b;
              f2_split(D2, d2a, d2b);
              float pa, pb;
              f2_split(f2_sub(F2{sc.rs_d}, f2_mul(D2, f2_make(rsqrtf(d2a), rsqrtf(d2b)))), pa, pb);
              const F2 PC = f2_make(fmaxf(pa, 0.f), fmaxf(pb, 0.f));
              CP = Q ? f2_fma(PC, PC, CP) : f2_add(CP, PC);
            }
            float l, r;
            f2_split(CP, l, r);
            cp = l + r;
          }
          if constexpr (WG) {
            // two b-spheres per packed op; the uniform Q picks the mode's scale
            const F2 TX = f2_dup(tx), TY = f2_dup(ty), TZ = f2_dup(tz);
            F2 GX = f2_dup(0.f), GY = GX, GZ = GX;
#pragma unroll
            for (int h = 0; h < kTileSpb; h += 2) {
              const int b2 = (j * kTileSpb + h) / 2;
              const F2 DX = f2_sub(TX, F2{sc.px[b2]}), DY = f2_sub(TY, F2{sc.py[b2]}), DZ = f2_sub(TZ, F2{sc.pz[b2]});
              // d2 + 1e-30: keeps 1/d finite at coincident centres (zero gradient there)
              // without a clamp instruction; 1e-30 is far below any fp32 pair distance^2
              const F2 D2 = f2_fma(DZ, DZ, f2_fma(DY, DY, f2_fma(DX, DX, F2{sc.tiny_d})));
              float d2a, d2b;
              f2_split(D2, d2a, d2b);
              const F2 INV = f2_make(rsqrtf(d2a), rsqrtf(d2b));
              // t = rsum/d - 1 = pen/d; active iff t > 0. quadratic s = t, linear s = 1/d
              float ta, tb, ia, ib;
              f2_split(f2_fma(F2{sc.rs_d}, INV, F2{sc.m1_d}), ta, tb);
              f2_split(INV, ia, ib);
              const F2 S = f2_make(ta > 0.f ? pick(qmask, ta, ia) : 0.f, tb > 0.f ? pick(qmask, tb, ib) : 0.f);
              GX = f2_fma(S, DX, GX);
              GY = f2_fma(S, DY, GY);
              GZ = f2_fma(S, DZ, GZ);
            }
            float l, r;
            f2_split(GX, l, r);
            gx = l + r;
            f2_split(GY, l, r);
            gy = l + r;
            f2_split(GZ, l, r);
            gz = l + r;
          }
          if constexpr (WC) cost = fmaf(sc.w_bb, cp, cost);
          if constexpr (WG) {
            const float w = Q ? -2.f * sc.w_bb : -sc.w_bb;
            g[3 * i] = fmaf(w, gx, g[3 * i]);
            g[3 * i + 1] = fmaf(w, gy, g[3 * i + 1]);
            g[3 * i + 2] = fmaf(w, gz, g[3 * i + 2]);
            g[3 * j] = fmaf(-w, gx, g[3 * j]);
            g[3 * j + 1] = fmaf(-w, gy, g[3 * j + 1]);
            g[3 * j + 2] = fmaf(-w, gz, g[3 * j + 2]);
          }
        }
        // ---- sphere vs the four walls (+x, -x, +y, -y), _interactions.py:62-73
        const float vz = waz - sc.wall_az;
        const float vyx = way - sc.wall_ay_x;  // off-axis component of the x walls
        const float vxy = wax - sc.wall_ax_y;  // ... and of the y walls
        const float px = fmaf(vyx, vyx, vz * vz), py = fmaf(vxy, vxy, vz * vz);
        float gx = 0.f, gy = 0.f, gz = 0.f;
        if constexpr (WC) {
          cost += wall_pair_cost(sc, Q, f2_sub(f2_dup(wax), F2{sc.wa_x}), f2_dup(px)) +
                  wall_pair_cost(sc, Q, f2_sub(f2_dup(way), F2{sc.wa_y}), f2_dup(py));
        }
        if constexpr (WG) {
          F2 GX = f2_dup(0.f), GY = GX, GZ = GX;
          const F2 VZ = f2_dup(vz);
          wall_pair_grad(sc, qmask, f2_sub(f2_dup(wax), F2{sc.wa_x}), f2_dup(px), f2_dup(vyx), VZ, GX, GY, GZ);
          wall_pair_grad(sc, qmask, f2_sub(f2_dup(way), F2{sc.wa_y}), f2_dup(py), f2_dup(vxy), VZ, GY, GX, GZ);
          float l, r;
          f2_split(GX, l, r);
          gx = l + r;
          f2_split(GY, l, r);
          gy = l + r;
          f2_split(GZ, l, r);
          gz = l + r;
        }
        if constexpr (WG) {
          g[3 * i] += gx;
          g[3 * i + 1] += gy;
          g[3 * i + 2] += gz;
        }
      }
    }
    return cost;
  }

  // Height term (tetris.py:226-238; sign(0) == 0), identical on every lane.
  template <bool WC, bool WG>
  static __device__ __forceinline__ void height(const TetrisTileScene& sc, bool Q, const float (&x)[D], float (&g)[D],
                                                float& cost) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const float dz = x[3 * i + 2] - sc.z_star;
      if constexpr (WC) cost += Q ? sc.w_h * (dz * dz) : sc.w_h * fabsf(dz);
      if constexpr (WG) g[3 * i + 2] += Q ? sc.w_h * (2.f * dz) : sc.w_h * (dz > 0.f ? 1.f : (dz < 0.f ? -1.f : 0.f));
    }
  }
};

template <int LA>
__device__ __forceinline__ float lane_sum(float v) {
  if constexpr (LA >= 2) v += __shfl_xor_sync(0xffffffffu, v, 1);
  if constexpr (LA >= 4) v += __shfl_xor_sync(0xffffffffu, v, 2);
  if constexpr (LA >= 8) v += __shfl_xor_sync(0xffffffffu, v, 4);
  return v;
}

// Full cost/gradient of the particle on every lane of the group.
template <class T, int LA, bool WC, bool WG>
__device__ __forceinline__ float tile_eval(const TetrisTileScene& sc, const typename T::Lane& L, bool Q,
                                           const float (&x)[T::D], float (&g)[T::D]) {
  float cost = T::template pairs<WC, WG>(sc, L, Q, x, g);
  if constexpr (LA > 1) {
    if constexpr (WC) cost = lane_sum<LA>(cost);
    if constexpr (WG) {
#pragma unroll
      for (int d = 0; d < T::D; ++d) g[d] = lane_sum<LA>(g[d]);
    }
  }
  T::template height<WC, WG>(sc, Q, x, g, cost);
  return cost;
}

// One clamped step with the NaN freeze (particle_opt.py:214-228).
template <int D, class SC>
__device__ __forceinline__ void tile_step(const SC& sc, float (&x)[D], const float (&g)[D], float rate, bool& bad) {
  bool b = false;
#pragma unroll
  for (int d = 0; d < D; ++d) b |= !isfinite(g[d]);
  bad |= b;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    float v = x[d];
    if (!b) v = v - rate * g[d];
    x[d] = fminf(fmaxf(v, sc.lower[d]), sc.upper[d]);
  }
}

template <int N, int LA>
__global__ void __launch_bounds__(128, 4) k_schedule_tile(const __grid_constant__ TetrisTileScene sc,
                                                       const float* __restrict__ src, const uint32_t* __restrict__ rows,
                                                       int64_t M, int k_lin, int k_quad, double eta, double alpha,
                                                       float* __restrict__ out_values, float* __restrict__ out_cost,
                                                       uint8_t* __restrict__ flagged,
                                                       unsigned int* __restrict__ flagged_count) {
  using T = TetrisTile<N, LA>;
  constexpr int D = T::D;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(threadIdx.x % LA);
  const int64_t p = gtid / LA;
  const bool live = p < M;  // dead lanes still run (full-warp shuffles) on a valid row
  const int64_t row = live ? (rows ? (int64_t)rows[p] : p) : 0;
  float x[D], g[D];
#pragma unroll
  for (int d = 0; d < D; ++d) x[d] = live ? src[row * D + d] : sc.lower[d];
  __shared__ float tab[3 * N * kTileSpb];
  for (int e = threadIdx.x; e < N * kTileSpb; e += blockDim.x) {
    tab[e] = sc.lx[e];
    tab[N * kTileSpb + e] = sc.ly[e];
    tab[2 * N * kTileSpb + e] = sc.lz[e];
  }
  __syncthreads();
  const typename T::Lane L{tab, lane * T::SA};
  bool bad = false;
  // K_lin linear steps then K_quad quadratic steps, one loop over the shared eval code
  for (int k = 1; k <= k_lin + k_quad; ++k) {
    const bool quad = k > k_lin;
    // lr_schedule in float64 exactly as the reference, then cast (particle_opt.py:203-211)
    const float rate = quad ? (float)alpha : (float)(eta * (1.0 - (double)k / (double)k_lin));
    tile_eval<T, LA, false, true>(sc, L, quad, x, g);
    tile_step<D>(sc, x, g, rate, bad);
  }
  const float fc = tile_eval<T, LA, true, false>(sc, L, true, x, g);
  if (lane != 0 || !live) return;
#pragma unroll
  for (int d = 0; d < D; ++d) out_values[p * D + d] = x[d];
  out_cost[p] = fc;
  if (flagged) flagged[p] = bad ? 1 : 0;
  if (bad && flagged_count) atomicAdd(flagged_count, 1u);
}

// LINEAR cost + ranking key of freshly sampled rows (particle_opt.py:326-330), LA lanes per
// row like the schedule; the rows come from k_sample (stage1_kernels.cuh).
template <int N, int LA>
__global__ void __launch_bounds__(128) k_keys_tile(const __grid_constant__ TetrisTileScene sc,
                                                   const float* __restrict__ values, int64_t row_offset, int64_t rows_n,
                                                   uint32_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  using T = TetrisTile<N, LA>;
  constexpr int D = T::D;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(threadIdx.x % LA);
  const int64_t p = gtid / LA;
  const bool live = p < rows_n;
  __shared__ float tab[3 * N * kTileSpb];
  for (int e = threadIdx.x; e < N * kTileSpb; e += blockDim.x) {
    tab[e] = sc.lx[e];
    tab[N * kTileSpb + e] = sc.ly[e];
    tab[2 * N * kTileSpb + e] = sc.lz[e];
  }
  __syncthreads();
  float x[D], g[D];
#pragma unroll
  for (int d = 0; d < D; ++d) x[d] = live ? values[p * D + d] : sc.lower[d];
  const typename T::Lane L{tab, lane * T::SA};
  const float c = tile_eval<T, LA, true, false>(sc, L, false, x, g);
  if (lane != 0 || !live) return;
  keys[p] = order_key(c);
  idx[p] = (uint32_t)(row_offset + p);
}

}  // namespace spasm
