// Stage-2 kernels: the trajectory half of the SPaSM pipeline on sm_100a.
//
//   k_al_eval      _evaluate forward/backward (trajopt.py:416-653) -> trajectory_cost,
//                  al_value_and_gradient (trajopt.py:664-723)
//   k_validate     validate (trajopt.py:1071-1153)
//   k_solve_al     the whole augmented-Lagrangian solve (trajopt.py:936-1063) as ONE
//                  persistent launch: every CTA owns one trajectory particle and runs its
//                  inner steps, pick retraction, re-evaluation, validation and multiplier
//                  updates with the particle resident in shared memory.
//   k_ik_group     ik_solve_batch (robot.py:227-302): one warp per (draw, target), one lane
//                  per seeded restart, first-minimum selection by warp shuffles; optional
//                  tool-down polish (trajopt.py:726-776) and arm/static branch score
//                  (trajopt.py:779-787) on the winning lane (lift_placements draws).
//   k_lift_combine lift_placements' draw selection, particle survival and endpoint
//                  assembly (trajopt.py:844-876), stream-compacted on the device.
//   k_init_traj    init_trajectories (trajopt.py:892-923) with the bit-exact PCG64 stream.
//
// CTA mapping of the AL kernels: one thread per waypoint w = (segment b, step t) of the
// particle (W = B*T threads, rounded to warps) plus one auxiliary warp for per-segment
// work (placed-block poses, final-waypoint Jacobians, the free-yaw placement twin cost,
// reductions of the placed-block gradient partials). Per-waypoint arrays live in shared
// memory column-major ([field][w]) so every thread touches its own bank column. All
// reductions run in a fixed order (no atomics): results are deterministic per seed.
#pragma once
#include <cooperative_groups.h>

#include "al_tile.cuh"
#include "coop.cuh"
#include "seedseq.cuh"
#include "stage2.cuh"

namespace spasm {

// Diagnostic counters of k_ik_group (spasm_ik_profile), summed over CTAs while enabled:
// [0] CTAs, [1] cycles to the last restart's IK, [2] cycles to the end, [3] max IK
// iterations, [4] winner IK iterations, [5] winner polish iterations (post-IK part),
// [6] winners polished speculatively to completion, [7] restarts' IK iterations (sum); maxima
// over CTAs: [8] cycles to the last restart's IK, [9] cycles to the end, [10] winner polish
// iterations, [11] IK iterations
static __device__ unsigned long long g_ik_prof[12];
static __device__ int g_ik_prof_on;

// orders this thread's earlier shared-memory writes (own CTA or a cluster peer's) before its
// later ones as seen from any CTA of the cluster
__device__ __forceinline__ void cluster_fence() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }

// ---------------------------------------------------------------------------------------
// IK / lifting
// ---------------------------------------------------------------------------------------
struct IkOut {
  void* sol;          // [G][J] R
  uint8_t* ik_ok;     // [G]
  uint8_t* pol_ok;    // [G] (polish requested)
  void* score;        // [G] R
  void* pen;          // [G] R (branch score; 0 without statics)
};

// grasp target of group g = (draw a, target t): staged targets first (sc.pick_*),
// then placements rows[p][b] (trajopt.py:831-833; robot.py:325-334)
template <typename R>
__device__ __forceinline__ void lift_target(const TrajScene<R>& sc, const double* rows, int D, int t, R tp[3],
                                            R* ty) {
  const int B = sc.B;
  if (t < B) {
    tp[0] = sc.pick_pos[t][0];
    tp[1] = sc.pick_pos[t][1];
    tp[2] = sc.pick_pos[t][2];
    *ty = sc.pick_yaw[t];
    return;
  }
  const int p = (t - B) / B, b = (t - B) - p * B;
  const int per = sc.free_rows ? 4 : 3;
  const double* r = rows + (int64_t)p * D + b * per;
  const double yaw = sc.free_rows ? (double)wrap_yaw<double>(r[3]) : 0.0;
  const double c = cos(yaw), s = sin(yaw);
  const double ox = (double)sc.grasp_off[0], oy = (double)sc.grasp_off[1], oz = (double)sc.grasp_off[2];
  tp[0] = (R)(r[0] + c * ox - s * oy);
  tp[1] = (R)(r[1] + s * ox + c * oy);
  tp[2] = (R)(r[2] + oz);
  *ty = (R)wrap_yaw<double>(yaw + (double)sc.grasp_yaw);
}

// one thread-block cluster of CS CTAs per (draw, target) group (CS = 1: a plain CTA); the
// group's seeded restarts are dealt out rpc per CTA, one 8-lane tile per restart, each tile in
// its own warp (lanes 8-31 idle) so that restarts in different phases (IK vs speculative
// polish) never share a warp and serialise on divergence. Splitting a group over a cluster
// spreads its warps over several SMs: an IK iteration issues ~110 warp-wide SHFLs and an SM
// issues one per cycle (profiles/r02_microbench_shfl_lds_throughput.txt), so 16 restart
// warps on one SM wait on each other's shuffles. The group's selection slots (keys, scores,
// flags, the finished count, the speculation key and the winner) live in the shared memory
// of the cluster's rank-0 CTA and are reached through distributed shared memory.
// MAXT = the block-size bound: 512 (<= 16 restarts per CTA) lets ptxas use 128 registers (the
// per-iteration FK/DLS state spills under the 64-register cap of 1024-thread blocks).
template <typename R, int MAXT>
__global__ void __launch_bounds__(MAXT) k_ik_group(const TrajScene<R>* __restrict__ g_scene, int n_targets, int n_draws,
                                                  uint64_t seed, uint64_t draw_stride, int restarts, int max_iters,
                                                  double damping, const double* __restrict__ tpos_in,
                                                  const double* __restrict__ tyaw_in, const double* __restrict__ rows,
                                                  int D, int polish, int score_statics, IkOut out,
                                                  const int32_t* __restrict__ n_rows, int rpc) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  const int grp = blockIdx.x / CS;
  // device row count (stage-1 result read in place): groups of absent rows exit at once
  // (uniform over the cluster: every CTA of it serves the same group)
  if (n_rows && (int)(grp % n_targets) >= g_scene->B + *n_rows * g_scene->B) return;
  __shared__ ChainDesc<R> ch_s;
  __shared__ R s_key[32], s_score[32];
  __shared__ int s_ok[32];
  __shared__ int s_best, s_done;
  __shared__ unsigned int s_cur;  // best fp32-image key among finished restarts (speculation)
  __shared__ int s_its[32];
  const bool prof = g_ik_prof_on != 0;
  const long long t_start = prof ? clock64() : 0;
  if (threadIdx.x == 0 && crank == 0) {
    s_best = -1;
    s_done = 0;
    s_cur = ~0u;
  }
  const TrajScene<R>& sc = *g_scene;
  {
    const int4* src = reinterpret_cast<const int4*>(&sc.ch);
    int4* dst = reinterpret_cast<int4*>(&ch_s);
    for (int i = threadIdx.x; i < (int)(sizeof(ChainDesc<R>) / sizeof(int4)); i += blockDim.x) dst[i] = src[i];
  }
  cl.sync();  // rank 0's slots are initialised before any CTA of the cluster touches them
  // the group's slots in rank 0 (generic pointers into distributed shared memory)
  volatile R* const key_p = cl.map_shared_rank(s_key, 0);
  volatile R* const score_p = cl.map_shared_rank(s_score, 0);
  volatile int* const ok_p = cl.map_shared_rank(s_ok, 0);
  volatile int* const its_p = cl.map_shared_rank(s_its, 0);
  int* const best_p = cl.map_shared_rank(&s_best, 0);
  int* const done_p = cl.map_shared_rank(&s_done, 0);
  unsigned int* const cur_p = cl.map_shared_rank(&s_cur, 0);
  const ChainDesc<R>& ch = ch_s;
  const int a = grp / n_targets, t = grp - a * n_targets;
  const int J = ch.J;
  // every lane of a restart's warp runs the tile (4 identical replicas of the 8-lane tile),
  // so its shuffles can name the whole warp (Tile::make_warp); lanes 0-7 write results
  const Tile tl = Tile::make_warp();
  const int tile = crank * rpc + (int)(threadIdx.x >> 5);
  const bool tile_lane = (threadIdx.x & 31) < kTile;
  const bool lane0 = (threadIdx.x & 31) == 0;
  R tp[3], ty;
  if (tpos_in) {
    tp[0] = (R)tpos_in[3 * t];
    tp[1] = (R)tpos_in[3 * t + 1];
    tp[2] = (R)tpos_in[3 * t + 2];
    ty = (R)tyaw_in[t];
  } else {
    lift_target<R>(sc, rows, D, t, tp, &ty);
  }
  R qj = R(0);
  int spec_its = 0;
  bool pol_spec = true, spec_done = false;
  R ik_q = R(0);
  // warp-uniform role predicates from votes (uniform to the compiler: the warp-wide tile
  // shuffles inside need no divergence handling)
  if (__all_sync(0xffffffffu, tile < restarts)) {
    if (tl.j < J) {
      // seeds[t] = uniform(lower, upper, (restarts, dof)) of SeedSequence(seed, (t,)) (robot.py:255-257)
      Pcg64 g;
      g.init(seedseq_pcg64_dev(seed + (uint64_t)a * draw_stride, (uint64_t)t));
      g.advance((uint64_t)tile * J + tl.j);
      const double lo = ch.lo64[tl.j], hi = ch.hi64[tl.j];
      qj = (R)__dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), g.next_double()));  // no FMA: numpy's rounding
    }
    R score;
    int its = 0;
    const bool ok = tile_ik<R>(tl, ch, qj, tp, ty, max_iters, R(damping), &score, &its);
    if (prof && lane0) its_p[tile] = its;
    const R key = (ok ? R(0) : R(1e6)) + score;
    // speculation order: the fp32 image of the key; the exact winner is s_best below
    // A 32-bit slot: a 64-bit atomicMin on a cluster peer's shared memory did not behave as
    // one (about 1 in 12 winners then saw a larger key replace its own and dropped its
    // speculative polish; scripts/ik_cluster_sweep.py), 32-bit shared atomics are native. A
    // restart whose key ties the leader's does not lead (strict <); the exact first-minimum
    // winner is still s_best, and a winner that did not polish speculatively polishes after.
    const unsigned mine = order_key((float)key);
    int last = 0, lead = 0;
    if (lane0) {
      key_p[tile] = key;
      score_p[tile] = score;
      ok_p[tile] = ok;
      cluster_fence();
      lead = atomicMin(cur_p, mine) > mine;
      last = atomicAdd(done_p, 1) == restarts - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    lead = __shfl_sync(0xffffffffu, lead, 0);
    if (last && lane0) {  // the last restart to finish picks the first minimum (np.argmin)
      cluster_fence();
      int b = 0;
      for (int r = 1; r < restarts; ++r)
        if (key_p[r] < key_p[b]) b = r;
      *((volatile int*)best_p) = b;
      if (prof) {
        atomicAdd(&g_ik_prof[1], (unsigned long long)(clock64() - t_start));
        atomicMax(&g_ik_prof[8], (unsigned long long)(clock64() - t_start));
        int mx = 0;
        unsigned long long sum = 0;
        for (int r = 0; r < restarts; ++r) {
          mx = max(mx, its_p[r]);
          sum += its_p[r];
        }
        atomicAdd(&g_ik_prof[3], (unsigned long long)mx);
        atomicMax(&g_ik_prof[11], (unsigned long long)mx);
        atomicAdd(&g_ik_prof[4], (unsigned long long)its_p[b]);
        atomicAdd(&g_ik_prof[7], sum);
      }
    }
    // speculative polish (lift path): the best restart finished so far starts polishing
    // its IK result at once and stops if a better one finishes or another tile wins, so
    // the winner's polish usually overlaps the slower restarts' IK iterations
    ik_q = qj;
    if (polish && __all_sync(0xffffffffu, lead != 0))
      pol_spec = tile_polish<R>(tl, ch, qj, tp, ty, best_p, tile, cur_p, mine, &spec_done, &spec_its);
  }
  cl.sync();  // every restart has finished IK and the winner is known
  const int best = *((volatile int*)best_p);
  int best_ok = 0;
  R best_score = R(0);
  if (tile == best) {
    best_ok = ok_p[best];
    best_score = score_p[best];
  }
  cl.sync();  // rank 0's slots are not read past this point (its CTA may exit)
  if (!__all_sync(0xffffffffu, tile == best)) return;  // the whole winner warp stays: its polish shuffles warp-wide
  bool pol = true;
  R pen = R(0);
  if (polish) {
    int pits = 0;
    if (!spec_done) {  // the winner was not (fully) polished speculatively: polish it now
      qj = ik_q;
      pol_spec = tile_polish<R>(tl, ch, qj, tp, ty, nullptr, 0, nullptr, 0, nullptr, &pits);
    }
    if (prof && lane0) {
      atomicAdd(&g_ik_prof[5], (unsigned long long)(pits + (spec_done ? spec_its : 0)));
      atomicMax(&g_ik_prof[10], (unsigned long long)(pits + (spec_done ? spec_its : 0)));
      if (spec_done) atomicAdd(&g_ik_prof[6], 1ull);
    }
    pol = pol_spec;
    if (score_statics && sc.n_static > 0) pen = tile_arm_worst_pen<R>(tl, ch, qj, sc.st_c, sc.st_r, sc.n_static);
  }
  if (prof && lane0) {
    atomicAdd(&g_ik_prof[0], 1ull);
    atomicAdd(&g_ik_prof[2], (unsigned long long)(clock64() - t_start));
    atomicMax(&g_ik_prof[9], (unsigned long long)(clock64() - t_start));
  }
  if (!tile_lane) return;
  if (tl.j < J) reinterpret_cast<R*>(out.sol)[(int64_t)grp * J + tl.j] = qj;
  if (tl.j == 0) {
    out.ik_ok[grp] = (uint8_t)best_ok;
    if (out.pol_ok) out.pol_ok[grp] = (uint8_t)pol;
    reinterpret_cast<R*>(out.score)[grp] = best_score;
    if (out.pen) reinterpret_cast<R*>(out.pen)[grp] = pen;
  }
}

// polish a batch of configurations (the _polish_tool_down API), one tile per row
template <typename R>
__global__ void k_polish(const TrajScene<R>* __restrict__ g_scene, int n, R* __restrict__ Q,
                         const double* __restrict__ tpos, const double* __restrict__ tyaw, uint8_t* __restrict__ ok) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  if (i >= n) return;  // whole tiles exit together
  const ChainDesc<R>& ch = g_scene->ch;
  const Tile tl = Tile::make();
  const int J = ch.J;
  R qj = tl.j < J ? Q[(int64_t)i * J + tl.j] : R(0);
  const R tp[3] = {(R)tpos[3 * i], (R)tpos[3 * i + 1], (R)tpos[3 * i + 2]};
  const bool r = tile_polish<R>(tl, ch, qj, tp, (R)tyaw[i]);
  if (tl.j == 0) ok[i] = (uint8_t)r;
  if (tl.j < J) Q[(int64_t)i * J + tl.j] = qj;
}

// lift_placements tail (trajopt.py:844-876): per target, replay the draws in order keeping
// the least-penetrating successful one; per particle, survive iff every placement lifted;
// stream-compact the survivors and assemble (pick, place) endpoints. One CTA.
// status[0] = first unreachable staged pose (-1 none), status[1] = kept count.
template <typename R>
__global__ void __launch_bounds__(1024) k_lift_combine(const R* __restrict__ sol, const uint8_t* __restrict__ ik_ok,
                                                       const uint8_t* __restrict__ pol_ok, const R* __restrict__ pen,
                                                       int stride_targets, int n_draws, int J, int B, int P,
                                                       R* __restrict__ best, uint8_t* __restrict__ okt,
                                                       int32_t* __restrict__ kept, R* __restrict__ endpoints,
                                                       int32_t* __restrict__ status, const int32_t* __restrict__ n_rows) {
  __shared__ int s_scan[1024];
  // with a device row count only its first rows exist (their groups were the only ones run)
  int n_targets = stride_targets;
  if (n_rows) {
    P = min(P, (int)*n_rows);
    n_targets = B + P * B;
  }
  __shared__ int s_carry;
  __shared__ int s_pickfail;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_carry = 0;
    s_pickfail = 0x7fffffff;
  }
  __syncthreads();
  for (int t = tid; t < n_targets; t += blockDim.x) {
    bool ok = false;
    R bp = R(INFINITY);
    int bi = -1;
    for (int a = 0; a < n_draws; ++a) {
      const int g = a * stride_targets + t;
      const bool dok = ik_ok[g] && pol_ok[g];
      const R pv = pen[g];
      if (dok && (!ok || pv < bp)) {
        bi = g;
        bp = pv;
      }
      ok = ok || dok;
    }
    okt[t] = (uint8_t)ok;
    for (int j = 0; j < J; ++j) best[(int64_t)t * J + j] = bi >= 0 ? sol[(int64_t)bi * J + j] : R(0);
    if (t < B && !ok) atomicMin(&s_pickfail, t);
  }
  __syncthreads();
  // survivors, in particle order
  for (int base = 0; base < P; base += blockDim.x) {
    const int p = base + tid;
    int keep = 0;
    if (p < P) {
      keep = 1;
      for (int b = 0; b < B; ++b) keep &= okt[B + p * B + b];
    }
    s_scan[tid] = keep;
    __syncthreads();
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {
      const int v = tid >= off ? s_scan[tid - off] : 0;
      __syncthreads();
      s_scan[tid] += v;
      __syncthreads();
    }
    if (keep) kept[s_carry + s_scan[tid] - 1] = p;
    __syncthreads();
    if (tid == 0) s_carry += s_scan[blockDim.x - 1];
    __syncthreads();
  }
  const int nk = s_carry;
  for (int i = tid; i < nk * B * 2 * J; i += blockDim.x) {
    const int j = i % J;
    const int e = (i / J) % 2;
    const int b = (i / (2 * J)) % B;
    const int k = i / (2 * J * B);
    const int t = e == 0 ? b : B + kept[k] * B + b;
    endpoints[i] = best[(int64_t)t * J + j];
  }
  if (tid == 0) {
    status[0] = s_pickfail == 0x7fffffff ? -1 : s_pickfail;
    status[1] = nk;
  }
}

// init_trajectories (trajopt.py:892-923): nodes = endpoints + K uniform waypoints from the
// trajectory stream (C-order draw index ((p*B + b)*K + k)*J + j), k_interp even steps per leg.
template <typename R>
__global__ void k_init_traj(const TrajScene<R>* __restrict__ g_scene, const R* __restrict__ endpoints, int P,
                            const int32_t* __restrict__ n_active, int B, int K, int n_interp, Pcg64State st,
                            R* __restrict__ out) {
  const ChainDesc<R>& ch = g_scene->ch;
  const int J = ch.J;
  const int T = n_interp * (K + 1) + 1;
  const int64_t total = (int64_t)P * B * T * J;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int j = (int)(i % J);
  const int t = (int)((i / J) % T);
  const int b = (int)((i / ((int64_t)J * T)) % B);
  const int64_t p = i / ((int64_t)J * T * B);
  if (n_active && p >= *n_active) return;
  auto node = [&](int k) -> double {
    if (k == 0) return (double)endpoints[(((p * B + b) * 2 + 0) * J) + j];
    if (k == K + 1) return (double)endpoints[(((p * B + b) * 2 + 1) * J) + j];
    Pcg64 g;
    g.init(st);
    g.advance((uint64_t)(((p * B + b) * K + (k - 1)) * J + j));
    const double lo = ch.lo64[j], hi = ch.hi64[j];
    return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), g.next_double()));  // no FMA: numpy's rounding
  };
  double v;
  if (t == T - 1) {
    v = node(K + 1);
  } else {
    const int leg = t / n_interp, s = t - leg * n_interp;
    const double a = node(leg), d = node(leg + 1) - a;
    v = a + d * ((double)s / (double)n_interp);
  }
  out[i] = (R)v;
}

// forward kinematics of a batch (robot.fk_batch): ee (n,3), rot (n,9), origins/axes (n,J,3)
template <typename R>
__global__ void k_fk(const TrajScene<R>* __restrict__ g_scene, const R* __restrict__ Q, int n, R* __restrict__ ee,
                     R* __restrict__ rot, R* __restrict__ org, R* __restrict__ axs, R* __restrict__ yawjac) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const ChainDesc<R>& ch = g_scene->ch;
  const int J = ch.J;
  R o[kMaxJ][3], z[kMaxJ][3], e[3], Rm[9];
  fk_frames<R>(ch, Q + (int64_t)i * J, o, z, e, Rm);
  for (int c = 0; c < 3; ++c) ee[3 * (int64_t)i + c] = e[c];
  for (int c = 0; c < 9; ++c) rot[9 * (int64_t)i + c] = Rm[c];
  for (int j = 0; j < J; ++j)
    for (int c = 0; c < 3; ++c) {
      if (org) org[((int64_t)i * J + j) * 3 + c] = o[j][c];
      if (axs) axs[((int64_t)i * J + j) * 3 + c] = z[j][c];
    }
  if (yawjac)
    for (int j = 0; j < J; ++j) yawjac[(int64_t)i * J + j] = yaw_jac(Rm, z[j]);
}

}  // namespace spasm
