// Tile-cooperative kinematics: one 8-lane tile owns one arm configuration, lane j owns
// joint j (J <= 8). This replaces the serial joint chain with
//   * Rodrigues rotations of all joints at once (robot.py:71-84),
//   * an inclusive prefix product of the 3x3 rotations over the tile (Hillis-Steele,
//     3 shuffle levels) and an inclusive prefix sum of the link translations,
//   * lane-local Jacobian columns (robot.py:183-224; trajopt.py:737-756),
//   * a butterfly (xor) reduction of the damped normal matrix J J^T + lambda I: every lane
//     receives a bitwise identical matrix (IEEE addition is commutative), so the redundant
//     per-lane Cholesky solve and the convergence tests are uniform across the tile.
// Per-tile vs the reference's lock-step batches: converged IK rows are frozen by the
// reference (dq = 0, clip is idempotent), so iterating each tile to its own convergence is
// identical. The polish re-applies the full-circle wrap to finished rows while other rows
// still iterate; that wrap is not idempotent in floating point, so finished polish rows can
// differ by rounding.
// Used by ik_solve_batch (robot.py:227-302), _polish_tool_down (trajopt.py:726-776), the
// lift branch score (trajopt.py:779-787) and the AL waypoint frames.
#pragma once
#include "stage2.cuh"

namespace spasm {

constexpr int kTile = 8;

struct Tile {
  unsigned mask;  // the tile's 8 lanes within the warp
  int j;          // lane index inside the tile = joint index
  __device__ __forceinline__ static Tile make() {
    Tile t;
    const int lane = threadIdx.x & 31;
    t.j = lane & (kTile - 1);
    t.mask = 0xFFu << (lane & ~(kTile - 1));
    return t;
  }
  // Same 8-lane segments, but the shuffles name the whole warp: valid (and ~25 % faster per
  // shuffle than per-tile masks, scripts/microbench/shfl_mask.cu) only where all 32 lanes
  // of the warp execute the call.
  __device__ __forceinline__ static Tile make_warp() {
    Tile t;
    t.j = threadIdx.x & (kTile - 1);
    t.mask = 0xffffffffu;
    return t;
  }
  template <typename R>
  __device__ __forceinline__ R up(R v, int d) const { return __shfl_up_sync(mask, v, d, kTile); }
  template <typename R>
  __device__ __forceinline__ R down(R v, int d) const { return __shfl_down_sync(mask, v, d, kTile); }
  template <typename R>
  __device__ __forceinline__ R xr(R v, int d) const { return __shfl_xor_sync(mask, v, d, kTile); }
  template <typename R>
  __device__ __forceinline__ R bcast(R v, int src) const { return __shfl_sync(mask, v, src, kTile); }
  template <typename R>
  __device__ __forceinline__ R sum(R v) const {
    v += xr(v, 1);
    v += xr(v, 2);
    v += xr(v, 4);
    return v;
  }
  // Reduce-scatter of 8 per-lane values: lane j returns the tile sum of v[j] (3 levels,
  // 4 + 2 + 1 shuffles instead of 8 x 3); each sum is formed on one lane only.
  template <typename R>
  __device__ __forceinline__ R sum8_scatter(const R (&v)[8]) const {
    const bool h2 = (j & 4) != 0, h1 = (j & 2) != 0, h0 = (j & 1) != 0;
    R a[4], b[2];
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = (h2 ? v[k + 4] : v[k]) + xr(h2 ? v[k] : v[k + 4], 4);
#pragma unroll
    for (int k = 0; k < 2; ++k) b[k] = (h1 ? a[k + 2] : a[k]) + xr(h1 ? a[k] : a[k + 2], 2);
    return (h0 ? b[1] : b[0]) + xr(h0 ? b[0] : b[1], 1);
  }
  // tile-uniform predicate (the loop exits below are uniform across the tile; with the
  // warp mask the vote also makes them uniform to the compiler, so the loops' warp-wide
  // shuffles need no divergence handling)
  __device__ __forceinline__ bool all(bool p) const { return __all_sync(mask, p); }
  __device__ __forceinline__ bool any(bool p) const { return __any_sync(mask, p); }
  // max over the tile of a NON-NEGATIVE value: fp32 takes one REDUX.MAX on the bit patterns
  // (non-negative IEEE floats order like their bits; 22 cycles against 3 shuffle levels),
  // fp64 the shuffle tree
  template <typename R>
  __device__ __forceinline__ R max_nonneg(R v) const {
    if constexpr (sizeof(R) == 4) return __uint_as_float(__reduce_max_sync(mask, __float_as_uint(v)));
    else return max(v);
  }
  template <typename R>
  __device__ __forceinline__ R max(R v) const {
    v = fmax(v, xr(v, 1));
    v = fmax(v, xr(v, 2));
    v = fmax(v, xr(v, 4));
    return v;
  }
};

// normalize_yaw / np.mod with the fast-range test voted across the tile: the common case
// takes the branch-free fold (same bits as wrap_yaw / np_mod_pos), the rare out-of-range
// case the scalar routine, and the branch is tile-uniform (no reconvergence point).
template <typename R>
__device__ __forceinline__ R tile_wrap_yaw(const Tile& tl, R a) {
  if (tl.all(wrap_yaw_in_fast_range(a))) return wrap_yaw_finish(wrap_yaw_fold(a + R(3.1415926535897932384626433832795)));
  return wrap_yaw(a);
}
template <typename R>
__device__ __forceinline__ R tile_np_mod_pos(const Tile& tl, R a, R m) {
  if (tl.all(np_mod_in_fast_range(a, m))) return np_mod_finish(a >= m ? a - m : a, m);
  return np_mod_pos(a, m);
}

// Per-lane frame of joint j after a tile FK:
//   M   rotation before joint j (product of joints < j)     -> axis z = M * axis_j
//   P   rotation after joint j (product of joints <= j)      -> link frame of link j
//   o   joint origin p_j = sum_{i<=j} M_i offset_i
// and, uniform across the tile, the end effector ee / Ree.
template <typename R>
struct TileFrame {
  R P[9];
  R z[3];
  R o[3];
  R ee[3];
  R Ree[9];
};

// The chain constants one tile lane needs every FK (its joint's axis / offset / limits and
// the uniform tool transform), held in registers across the DLS iterations instead of
// re-read from the shared-memory ChainDesc on every iteration's critical path.
template <typename R>
struct LaneChain {
  int J, full;
  R ax[3], off[3], lo, hi, tool_t[3], tool_R[9];
  __device__ __forceinline__ void load(const ChainDesc<R>& ch, int j) {
    J = ch.J;
    const int jj = j < ch.J ? j : 0;
    full = j < ch.J ? ch.full_circle[jj] : 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      ax[c] = ch.axis[jj][c];
      off[c] = ch.offset[jj][c];
      tool_t[c] = ch.tool_t[c];
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) tool_R[c] = ch.tool_R[c];
    lo = ch.lo[jj];
    hi = ch.hi[jj];
  }
};

template <typename R>
__device__ __forceinline__ void tile_fk(const Tile& tl, const LaneChain<R>& ch, R qj, TileFrame<R>& f) {
  const int J = ch.J;
  const int j = tl.j;
  const bool live = j < J;
  // Branch-free: every lane computes, lanes past the chain / below a scan level select
  // (divergent branches here cost a reconvergence point each and split the scheduling
  // blocks; the selected values are the same operations as before)
  R Rj[9];
  rodrigues(ch.ax, qj, Rj);
#pragma unroll
  for (int k = 0; k < 9; ++k) Rj[k] = live ? Rj[k] : ((k % 4 == 0) ? R(1) : R(0));
  // inclusive prefix product P_j = R_0 R_1 ... R_j
#pragma unroll
  for (int k = 0; k < 9; ++k) f.P[k] = Rj[k];
#pragma unroll
  for (int d = 1; d < kTile; d <<= 1) {
    R O[9], N[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) O[k] = tl.up(f.P[k], d);
    mat3_mul(O, f.P, N);
    const bool up = j >= d;
#pragma unroll
    for (int k = 0; k < 9; ++k) f.P[k] = up ? N[k] : f.P[k];
  }
  // exclusive product M_j (identity for joint 0)
  R M[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const R v = tl.up(f.P[k], 1);
    M[k] = j == 0 ? ((k % 4 == 0) ? R(1) : R(0)) : v;
  }
  R t[3];
  mat3_vec(M, ch.off, t);
  mat3_vec(M, ch.ax, f.z);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    t[c] = live ? t[c] : R(0);
    f.z[c] = live ? f.z[c] : R(0);
  }
  // inclusive prefix sum of the translations -> joint origins
#pragma unroll
  for (int c = 0; c < 3; ++c) f.o[c] = t[c];
#pragma unroll
  for (int d = 1; d < kTile; d <<= 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const R v = tl.up(f.o[c], d);
      f.o[c] = j >= d ? v + f.o[c] : f.o[c];
    }
  }
  // end effector from the last joint's frame (robot.py:136-141)
  R Pf[9], pf[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) Pf[k] = tl.bcast(f.P[k], J - 1);
#pragma unroll
  for (int c = 0; c < 3; ++c) pf[c] = tl.bcast(f.o[c], J - 1);
  R tt[3];
  mat3_vec(Pf, ch.tool_t, tt);
  f.ee[0] = pf[0] + tt[0];
  f.ee[1] = pf[1] + tt[1];
  f.ee[2] = pf[2] + tt[2];
  mat3_mul(Pf, ch.tool_R, f.Ree);
}

template <typename R>
__device__ __forceinline__ void tile_fk(const Tile& tl, const ChainDesc<R>& ch, R qj, TileFrame<R>& f) {
  LaneChain<R> lc;
  lc.load(ch, tl.j);
  tile_fk(tl, lc, qj, f);
}

// world centre of arm sphere s (owned by link j = this lane): p_j + P_j * local_s
template <typename R>
__device__ __forceinline__ void tile_sphere(const ChainDesc<R>& ch, const TileFrame<R>& f, int s, R* c) {
  R t[3];
  mat3_vec(f.P, ch.arm_local[s], t);
  c[0] = t[0] + f.o[0];
  c[1] = t[1] + f.o[1];
  c[2] = t[2] + f.o[2];
}

// Bitwise state equality across the tile. The DLS iterations below are pure functions of
// the joint vector, so once an iteration reproduces the previous state (fixed point) or
// the state before it (period-2 cycle) every later iteration is known exactly: the loops
// stop there and land on the state the reference would hold after its last iteration.
template <typename R>
__device__ __forceinline__ bool bits_eq(R a, R b) {
  if constexpr (sizeof(R) == 4) return __float_as_uint(a) == __float_as_uint(b);
  else return __double_as_longlong(a) == __double_as_longlong(b);
}

// Returns true when the loop can stop; qj is then the state after iteration max_iters-1.
// (checked every 8th iteration: the vote is not free, and the states are kept every step)
template <typename R>
__device__ __forceinline__ bool tile_settled(const Tile& tl, R& qj, R& prev1, R& prev2, int it, int max_iters) {
  if ((it & 7) != 7) {
    prev2 = prev1;
    prev1 = qj;
    return false;
  }
  const bool fixed = __all_sync(tl.mask, bits_eq(qj, prev1));
  const bool cycle = !fixed && __all_sync(tl.mask, bits_eq(qj, prev2));
  if (cycle && ((max_iters - 1 - it) & 1)) qj = prev1;  // odd number of steps left: other phase
  prev2 = prev1;
  prev1 = qj;
  return fixed || cycle;
}

// One damped least-squares step on the tile: A = sum_j col_j col_j^T + damping I (xor
// reduced, identical on every lane), Cholesky, dq_j = col_j . y, max|dq| <= 0.5.
template <typename R, int NR>
__device__ __forceinline__ R tile_dls(const Tile& tl, const R (&col)[NR], const R (&e)[NR], R damping) {
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
  const R mx = tl.max_nonneg(fabs(dq));
  return dq * fmin(R(1), R(0.5) / fmax(mx, R(1e-12)));
}

// ik_solve_batch for one (target, restart) tile (robot.py:262-302). Lane j holds q_j;
// returns ok and writes the score |pos err| + |yaw err| (uniform across the tile).
template <typename R>
__device__ bool tile_ik(const Tile& tl, const ChainDesc<R>& ch, R& q_io, const R tp[3], R ty, int max_iters, R damping,
                        R* score, int* iters = nullptr) {
  R qj = q_io;
  const int j = tl.j;
  const bool live = j < ch.J;
  LaneChain<R> lc;
  lc.load(ch, j);
  TileFrame<R> f;
  R prev1 = qj, prev2 = qj;
  int it = 0;
  for (; it < max_iters; ++it) {
    tile_fk(tl, lc, qj, f);
    const R pe[3] = {tp[0] - f.ee[0], tp[1] - f.ee[1], tp[2] - f.ee[2]};
    const R ye = tile_wrap_yaw(tl, ty - yaw_of(f.Ree));
    const R pn = Math<R>::sqrt_((pe[0] * pe[0] + pe[1] * pe[1]) + pe[2] * pe[2]);
    const bool conv = pn < R(kIkPosTol) && fabs(ye) < R(kIkYawTol);
    // the step is formed before the convergence vote (discarded on exit): the Jacobian and
    // the DLS factorisation then overlap the yaw chain instead of waiting on the vote
    const R rel[3] = {f.ee[0] - f.o[0], f.ee[1] - f.o[1], f.ee[2] - f.o[2]};
    R c[3];
    cross3(f.z, rel, c);
    const R col[4] = {c[0], c[1], c[2], f.z[2]};
    const R e4[4] = {pe[0], pe[1], pe[2], ye};
    const R dq = tile_dls<R, 4>(tl, col, e4, damping);
    if (tl.all(conv)) break;
    const R v = qj + dq;
    qj = live ? (v < lc.lo ? lc.lo : (v > lc.hi ? lc.hi : v)) : qj;
    if (tile_settled(tl, qj, prev1, prev2, it, max_iters)) break;
  }
  if (iters) *iters = it;
  tile_fk(tl, lc, qj, f);
  const R pe[3] = {tp[0] - f.ee[0], tp[1] - f.ee[1], tp[2] - f.ee[2]};
  const R pn = Math<R>::sqrt_((pe[0] * pe[0] + pe[1] * pe[1]) + pe[2] * pe[2]);
  const R ye = fabs(tile_wrap_yaw(tl, ty - yaw_of(f.Ree)));
  *score = pn + ye;
  q_io = qj;
  return pn < R(kIkPosTol) && ye < R(kIkYawTol);
}

// _polish_tool_down for one configuration on a tile (trajopt.py:726-776), as a resumable
// iteration: begin() from a configuration, step() runs one loop iteration and returns true
// once the loop has ended (converged, settled or at the cap), finish() is the final check.
template <typename R>
struct PolishRun {
  LaneChain<R> lc;
  R prev1, prev2;
  int it;
  bool live;
  __device__ __forceinline__ void begin(const Tile& tl, const ChainDesc<R>& ch, R qj) {
    lc.load(ch, tl.j);
    live = tl.j < ch.J;
    prev1 = prev2 = qj;
    it = 0;
  }
  __device__ __forceinline__ bool step(const Tile& tl, R& qj, const R tp[3], R ty) {
    if (it >= kPolishMaxIters) return true;
    const R cos_tol = R(0.99998750002604164);  // cos(0.005)
    const R two_pi = R(6.283185307179586476925286766559);
    TileFrame<R> f;
    tile_fk(tl, lc, qj, f);
    const R pe[3] = {tp[0] - f.ee[0], tp[1] - f.ee[1], tp[2] - f.ee[2]};
    const R ye = tile_wrap_yaw(tl, ty - yaw_of(f.Ree));
    const R ax[3] = {f.Ree[2], f.Ree[5], f.Ree[8]};
    const R pn = Math<R>::sqrt_((pe[0] * pe[0] + pe[1] * pe[1]) + pe[2] * pe[2]);
    const bool conv = pn < R(kIkPosTol) && fabs(ye) < R(kIkYawTol) && -ax[2] > cos_tol;
    // step formed before the convergence vote (discarded on exit), as in tile_ik
    const R rel[3] = {f.ee[0] - f.o[0], f.ee[1] - f.o[1], f.ee[2] - f.o[2]};
    R c[3], d[3];
    cross3(f.z, rel, c);
    cross3(f.z, ax, d);
    const R yj = yaw_jac(f.Ree, f.z);
    const R col[5] = {c[0], c[1], c[2], live ? yj : R(0), d[2]};
    const R e5[5] = {pe[0], pe[1], pe[2], ye, R(-1) - ax[2]};
    const R dq = tile_dls<R, 5>(tl, col, e5, R(kIkDamping));
    if (tl.all(conv)) return true;
    {  // branch-free update: every lane computes, lanes past the chain keep q
      const R v0 = qj + dq;
      const R vm = lc.lo + tile_np_mod_pos(tl, v0 - lc.lo, two_pi);
      R v = lc.full ? vm : v0;
      v = v < lc.lo ? lc.lo : (v > lc.hi ? lc.hi : v);
      qj = live ? v : qj;
    }
    if (tile_settled(tl, qj, prev1, prev2, it, kPolishMaxIters)) return true;
    ++it;
    return it >= kPolishMaxIters;
  }
  __device__ __forceinline__ bool finish(const Tile& tl, R qj, const R tp[3], R ty) const {
    const R cos_tol = R(0.99998750002604164);
    TileFrame<R> f;
    tile_fk(tl, lc, qj, f);
    const R pe[3] = {tp[0] - f.ee[0], tp[1] - f.ee[1], tp[2] - f.ee[2]};
    const R pn = Math<R>::sqrt_((pe[0] * pe[0] + pe[1] * pe[1]) + pe[2] * pe[2]);
    return pn < R(kIkPosTol) && fabs(tile_wrap_yaw(tl, ty - yaw_of(f.Ree))) < R(kIkYawTol) && -f.Ree[8] > cos_tol;
  }
};

// The whole polish of one configuration. Optional speculative mode (k_ik_group, a whole
// warp per tile): `best` points at a shared slot that becomes the winning tile's index once
// every restart has finished IK; a tile whose index `me` lost stops polishing (its result is
// discarded, so the winner's result is unchanged). The slots are polled one step ahead of their test, so a
// losing tile may run one step more than necessary.
template <typename R>
__device__ bool tile_polish(const Tile& tl, const ChainDesc<R>& ch, R& q_io, const R tp[3], R ty,
                            const volatile int* best = nullptr, int me = 0,
                            const volatile unsigned* cur = nullptr, unsigned mine = 0,
                            bool* completed = nullptr, int* iters = nullptr) {
  if (completed) *completed = false;
  R qj = q_io;  // iterate in a register (q_io may live in memory when this is not inlined)
  PolishRun<R> run;
  run.begin(tl, ch, qj);
  int b_seen = -1;                 // the slots as of the last poll (this tile just led)
  unsigned c_seen = mine;
  for (;;) {
    if (best) {  // abort once another tile is the winner or the current best candidate
      // polled by the warp's lane 0 only, the lane that published this restart's key into
      // *cur (another lane's load is not ordered after that atomic); the vote spreads it
      const bool poller = (threadIdx.x & 31) == 0;
      int stop = 0;
      if (poller) stop = (b_seen >= 0) ? (b_seen != me) : (cur != nullptr && c_seen != mine);
      if (tl.any(stop != 0)) {
        q_io = qj;
        return false;
      }
      // poll now, test after this step: the (possibly cluster-remote) loads overlap the step
      if (poller) {
        b_seen = *best;
        if (cur != nullptr) c_seen = *cur;
      }
    }
    if (run.step(tl, qj, tp, ty)) break;
  }
  if (iters) *iters = run.it;
  if (completed) *completed = true;
  q_io = qj;
  return run.finish(tl, qj, tp, ty);
}

// largest arm-sphere penetration (no clamp) against a sphere set (trajopt.py:779-787)
template <typename R>
__device__ R tile_arm_worst_pen(const Tile& tl, const ChainDesc<R>& ch, R qj, const R (*cen)[3], const R* rad, int n) {
  TileFrame<R> f;
  tile_fk(tl, ch, qj, f);
  R worst = -INFINITY;
  if (tl.j < ch.J) {
    for (int s = ch.link_start[tl.j]; s < ch.link_start[tl.j + 1]; ++s) {
      R c[3];
      tile_sphere(ch, f, s, c);
      for (int o = 0; o < n; ++o) {
        const R dx = c[0] - cen[o][0], dy = c[1] - cen[o][1], dz = c[2] - cen[o][2];
        worst = fmax(worst, (ch.arm_r[s] + rad[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
      }
    }
  }
  return tl.max(worst);
}

}  // namespace spasm
