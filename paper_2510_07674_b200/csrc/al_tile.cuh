// The augmented-Lagrangian engine of stage 2, one CTA per trajectory particle.
//
// Thread mapping: one 8-lane tile per waypoint w = (segment b, step t), lane j = joint j
// (W = B*T tiles), plus one auxiliary warp for per-segment work. One inner step is two
// CTA-wide barriers; the phases between them overlap:
//
//   A  aux:   tile FK of the B final waypoints (4 tiles per warp), placed block poses
//             (trajopt.py:448-472) -> arrive at named barrier kBarPlaced; then the
//             free-yaw placement twin's cost + gradient (trajopt.py:281-302, 531-539).
//      tiles: P1 tile FK of the waypoint (coop.cuh), arm-sphere centres of link j on lane
//             j, held-block spheres round-robin over lanes; sync kBarPlaced (only the
//             placed poses cross warps); P2 path-length leg, start terms, penetrations vs
//             the segment's fixed obstacles (statics + later staged blocks); P3 penetrations
//             vs earlier placed blocks, their placed-pose partials (tile reduced),
//             Jacobian-transpose products: lane k gets
//             z_k . (sum_{link>=k} a x g - o_k x sum_{link>=k} g) from a suffix scan.
//   -- __syncthreads --
//   B  every tile lane forms the totals, constraint vector and multiplier scales itself
//      (same operands, same order: identical bits on every lane); the final-waypoint tiles
//      sum their segment's placed-pose partials; lane k assembles dL/dq_k (path length,
//      arm, held, placement chain through the final-waypoint Jacobian and exact yaw
//      Jacobian, start alignment) and either stores it or applies the clamped descent
//      step in place.
//   -- __syncthreads --
//
// Reductions run in a fixed order (xor trees, ordered loops; no atomics): deterministic.
// Reference: trajopt.py:396-653 (value + gradient), 936-1063 (solve), 1071-1153 (validate).
#pragma once
#include "coop.cuh"
#include "f32x2.cuh"
#include "stage1_models.cuh"
#include "twin_warp.cuh"

namespace spasm {

// ---- placement twin (the free-yaw copy of the stage-1 model, trajopt.py:281-302) ------
template <typename R>
struct NoTwin {
  int dim;
};
template <typename R, int KIND> struct TwinSceneOf { using type = NoTwin<R>; };
template <typename R> struct TwinSceneOf<R, 1> { using type = TetrisScene<R>; };
template <typename R> struct TwinSceneOf<R, 2> { using type = TowerScene<R>; };

constexpr int kMaxAlThreads = 512;  // 60 waypoint tiles + the aux warp; <= 128 registers
constexpr int kXS = 8;  // row stride of x / g / unit in shared memory ([w][joint])
constexpr int kAlItems = 3;  // sphere items per tile lane (arm + held spheres of a waypoint <= 24)

struct AlLayout {
  int W, NW, NA, nthreads, nwarps, J, B, T, S, SB, NB;  // NA: aux warps (2 when B > 4 fits)
  int scene, twin, x, g, unit, ee, rot, armw, ga, hp, gh, pg, pl, pyaw, seg, rows, gpose, scr, pgsum, red, scal, flags;
  int total;
};

template <typename R>
__host__ __device__ inline AlLayout al_layout(int B, int T, int J, int S, int SB, int NB) {
  AlLayout L;
  L.W = B * T;
  L.NW = (L.W * kTile + 31) / 32 * 32;
  // B > 4 placed poses take two rounds of the aux warp's 4 FK tiles; a second aux warp runs
  // blocks 4-7 in parallel when the block size allows
  L.NA = (B > 4 && L.NW + 64 <= kMaxAlThreads) ? 2 : 1;
  L.nthreads = L.NW + 32 * L.NA;
  L.nwarps = L.nthreads / 32;
  L.J = J;
  L.B = B;
  L.T = T;
  L.S = S;
  L.SB = SB;
  L.NB = NB;
  const int W = L.W;
  const int r = (int)sizeof(R);
  int off = 0;
  auto take = [&off](int bytes) {
    const int o = off;
    off += (bytes + 15) & ~15;
    return o;
  };
  L.scene = take((int)sizeof(TrajScene<R>));
  // the placement twin's tables: the aux warp's lanes index them with different obstacle /
  // sphere numbers, which a kernel-parameter (constant bank) copy serialises per address
  L.twin = take((int)(sizeof(TetrisScene<R>) > sizeof(TowerScene<R>) ? sizeof(TetrisScene<R>) : sizeof(TowerScene<R>)));
  L.x = take(W * kXS * r);
  L.g = take(W * kXS * r);
  L.unit = take(W * kXS * r);
  L.ee = take(3 * W * r);
  L.rot = take(9 * W * r);
  L.armw = take(3 * (S > 0 ? S : 1) * W * r);
  L.ga = take(3 * (S > 0 ? S : 1) * W * r);
  L.hp = take(3 * (SB > 0 ? SB : 1) * W * r);
  L.gh = take(3 * (SB > 0 ? SB : 1) * W * r);
  L.pg = take(8 * B * W * r);
  L.pl = take(4 * (NB > 0 ? NB : 1) * r);  // placed block spheres (x, y, z, radius)
  L.pyaw = take(2 * (NB > 0 ? NB : 1) * r);  // d(placed sphere xy)/d(block yaw)
  L.seg = take(3 * B * r);  // psi | cp | sp
  L.rows = take(4 * B * r);
  L.gpose = take(4 * B * r);
  L.scr = take(twin_warp_scratch(B > 0 ? B : 1) * r);  // warp twin: per-lane gradient slots (twin_warp.cuh)
  L.pgsum = take(8 * B * r);
  L.red = take(4 * L.nwarps * r);
  L.scal = take(32 * r);
  L.flags = take(16 * 4);
  L.total = off;
  return L;
}

// scal[] slots
enum : int {
  kObj = 0, kCarm, kCblk, kCplace, kLag, kCons0, kCons1, kCons2, kSc0, kSc1, kSc2, kLam0, kLam1, kLam2, kMu, kPrev,
  kWorst, kLr
};

// Optional phase timer (diagnostic, spasm_al_profile): thread 0 accumulates clock64()
// deltas between consecutive marks; off unless enabled (one predicated branch per mark).
static __device__ unsigned long long g_al_prof[12];
static __device__ unsigned long long g_al_arrive[2][8];  // [tile thread 0 | aux lane 0][phase]
static __device__ unsigned long long g_al_warp[32][8];    // [warp (lane 0)][phase]: own work per warp
static __device__ unsigned long long g_al_polish[4];      // pick polish: iterations, calls, at the cap, max
static __device__ int g_al_prof_on;
struct AlProf {
  bool on = false;
  long long t = 0;
  __device__ __forceinline__ void start() {
    on = g_al_prof_on != 0;
    if (on) t = clock64();
  }
  // before a phase-ending barrier: how long this thread's own work in the phase took
  __device__ __forceinline__ void arrive(int k, int aux_tid) {
    if (on && (threadIdx.x & 31) == 0) {
      const unsigned long long d = (unsigned long long)(clock64() - t);
      atomicAdd(&g_al_warp[threadIdx.x >> 5][k], d);
      if (threadIdx.x == 0 || threadIdx.x == aux_tid) atomicAdd(&g_al_arrive[threadIdx.x == 0 ? 0 : 1][k], d);
    }
  }
  // after the barrier: phase time (slowest warp) as seen by thread 0
  __device__ __forceinline__ void mark(int k) {
    if (on) {
      const long long n = clock64();
      if (threadIdx.x == 0) atomicAdd(&g_al_prof[k], (unsigned long long)(n - t));
      t = n;
    }
  }
};

// named barrier 2: the aux warp arrives once the placed poses are written, the tile warps
// sync on it before their first read of them (every warp converged at the call)
constexpr int kBarPlaced = 2;
__device__ __forceinline__ void bar_placed_arrive(int count) {
  asm volatile("bar.arrive 2, %0;" ::"r"(count) : "memory");
}
__device__ __forceinline__ void bar_placed_sync(int count) { asm volatile("bar.sync 2, %0;" ::"r"(count) : "memory"); }
// named barrier 1 between the two aux warps (NA = 2): the second arrives after its placed
// poses, the first syncs before the placement twin reads all of them
__device__ __forceinline__ void bar_aux_arrive() { asm volatile("bar.arrive 1, 64;" ::: "memory"); }
__device__ __forceinline__ void bar_aux_sync() { asm volatile("bar.sync 1, 64;" ::: "memory"); }


template <typename R>
struct AlCtx {
  AlProf prof;
  AlLayout L;
  TrajScene<R>* sc;
  R *x, *g, *unit, *ee, *rot, *armw, *ga, *hp, *gh, *pg, *pl, *pyaw, *psi, *cp, *sp, *rows, *gpose, *scr, *pgsum, *red, *scal;
  int* flags;
  // this thread's waypoint geometry, fixed for the launch: formed once (geom) instead of
  // re-derived (an integer division, dependent shared-memory loads) at every inner step
  int g_b, g_t, g_h0, g_nh, g_f0, g_f1, g_slo, g_shi;
  bool g_manip, g_interior;

  // after the scene is resident in shared memory (al_load)
  __device__ void geom(int T) {
    const int tid = threadIdx.x;
    const int w = tid >> 3, j = tid & 7;
    const bool is_wp = tid < L.NW && w < L.W;
    g_manip = sc->manip != 0;
    g_b = is_wp ? w / T : 0;
    g_t = is_wp ? w - g_b * T : 0;
    g_interior = g_manip && g_t >= 1 && g_t <= T - 2;
    g_h0 = g_manip ? sc->blk_start[g_b] : 0;
    g_nh = g_manip ? sc->blk_start[g_b + 1] - g_h0 : 0;
    g_f0 = g_manip ? sc->blk_start[g_b + 1] : 0;
    g_f1 = g_manip ? sc->n_blk : 0;
    g_slo = j < L.J ? sc->ch.link_start[j] : 0;
    g_shi = j < L.J ? sc->ch.link_start[j + 1] : 0;
  }

  __device__ void bind(unsigned char* base, const AlLayout& l) {
    L = l;
    sc = reinterpret_cast<TrajScene<R>*>(base + L.scene);
    x = reinterpret_cast<R*>(base + L.x);
    g = reinterpret_cast<R*>(base + L.g);
    unit = reinterpret_cast<R*>(base + L.unit);
    ee = reinterpret_cast<R*>(base + L.ee);
    rot = reinterpret_cast<R*>(base + L.rot);
    armw = reinterpret_cast<R*>(base + L.armw);
    ga = reinterpret_cast<R*>(base + L.ga);
    hp = reinterpret_cast<R*>(base + L.hp);
    gh = reinterpret_cast<R*>(base + L.gh);
    pg = reinterpret_cast<R*>(base + L.pg);
    pl = reinterpret_cast<R*>(base + L.pl);
    pyaw = reinterpret_cast<R*>(base + L.pyaw);
    psi = reinterpret_cast<R*>(base + L.seg);
    cp = psi + L.B;
    sp = cp + L.B;
    rows = reinterpret_cast<R*>(base + L.rows);
    gpose = reinterpret_cast<R*>(base + L.gpose);
    scr = reinterpret_cast<R*>(base + L.scr);
    pgsum = reinterpret_cast<R*>(base + L.pgsum);
    red = reinterpret_cast<R*>(base + L.red);
    scal = reinterpret_cast<R*>(base + L.scal);
    flags = reinterpret_cast<int*>(base + L.flags);
  }
};

// penetration of one sphere pair; returns the (linear or squared) value and, when active,
// the unscaled slope (d value / d ca = -slope * (ca - cb)) (trajopt.py:396-413)
template <typename R>
__device__ __forceinline__ R pen_term(R dx, R dy, R dz, R rsum, bool quad, R* slope) {
  if constexpr (sizeof(R) == 4) {
    // fp32: one MUFU.RSQ for both d and 1/d (d2 = 0 -> d = NaN -> inactive, zero slope)
    const R d2 = (dx * dx + dy * dy) + dz * dz;
    const R inv = rsqrtf(d2);
    const R d = d2 * inv;
    R pen = rsum - d;
    const bool live = pen > R(0);
    pen = live ? pen : R(0);
    *slope = live ? (quad ? R(2) * pen * inv : inv) : R(0);
    return quad ? pen * pen : pen;
  } else {
    const R d = Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz);
    R pen = rsum - d;
    pen = pen > R(0) ? pen : R(0);
    const bool live = pen > R(0) && d > R(0);
    *slope = live ? (quad ? R(2) * pen / d : R(1) / d) : R(0);
    return quad ? pen * pen : pen;
  }
}

// fp32: the same, two obstacles per packed FADD2 / FMUL2 / FFMA2 (one MUFU.RSQ per
// obstacle); an odd tail is paired with a dummy at the sphere centre (d2 = 0: inactive).
struct PenAcc2 {
  F2 v, gx, gy, gz;
};
__device__ __forceinline__ PenAcc2 pen_two(PenAcc2 a, F2 cx, F2 cy, F2 cz, float r, bool quad, float ax, float ay,
                                           float az, float ar, float bx, float by, float bz, float br) {
  const F2 dx = f2_sub(cx, f2_make(ax, bx)), dy = f2_sub(cy, f2_make(ay, by)), dz = f2_sub(cz, f2_make(az, bz));
  const F2 d2 = f2_fma(dz, dz, f2_fma(dy, dy, f2_mul(dx, dx)));
  float d2a, d2b;
  f2_split(d2, d2a, d2b);
  const float ia = rsqrtf(d2a), ib = rsqrtf(d2b);
  const F2 pen = f2_sub(f2_make(r + ar, r + br), f2_mul(d2, f2_make(ia, ib)));
  float pa, pb;
  f2_split(pen, pa, pb);
  const bool la = pa > 0.f, lb = pb > 0.f;  // NaN (d2 = 0) -> inactive
  pa = la ? pa : 0.f;
  pb = lb ? pb : 0.f;
  const float sa = la ? (quad ? 2.f * pa * ia : ia) : 0.f, sb = lb ? (quad ? 2.f * pb * ib : ib) : 0.f;
  const F2 P = f2_make(pa, pb), SL = f2_make(-sa, -sb);
  a.v = quad ? f2_fma(P, P, a.v) : f2_add(a.v, P);
  a.gx = f2_fma(SL, dx, a.gx);
  a.gy = f2_fma(SL, dy, a.gy);
  a.gz = f2_fma(SL, dz, a.gz);
  return a;
}

// pen_two with the obstacle pair already packed (PX = (ax, bx), ...)
__device__ __forceinline__ PenAcc2 pen_two_packed(PenAcc2 a, F2 cx, F2 cy, F2 cz, float r, bool quad, F2 PX, F2 PY,
                                                  F2 PZ, float ar, float br) {
  const F2 dx = f2_sub(cx, PX), dy = f2_sub(cy, PY), dz = f2_sub(cz, PZ);
  const F2 d2 = f2_fma(dz, dz, f2_fma(dy, dy, f2_mul(dx, dx)));
  float d2a, d2b;
  f2_split(d2, d2a, d2b);
  const float ia = rsqrtf(d2a), ib = rsqrtf(d2b);
  const F2 pen = f2_sub(f2_make(r + ar, r + br), f2_mul(d2, f2_make(ia, ib)));
  float pa, pb;
  f2_split(pen, pa, pb);
  const bool la = pa > 0.f, lb = pb > 0.f;
  pa = la ? pa : 0.f;
  pb = lb ? pb : 0.f;
  const float sa = la ? (quad ? 2.f * pa * ia : ia) : 0.f, sb = lb ? (quad ? 2.f * pb * ib : ib) : 0.f;
  const F2 P = f2_make(pa, pb), SL = f2_make(-sa, -sb);
  a.v = quad ? f2_fma(P, P, a.v) : f2_add(a.v, P);
  a.gx = f2_fma(SL, dx, a.gx);
  a.gy = f2_fma(SL, dy, a.gy);
  a.gz = f2_fma(SL, dz, a.gz);
  return a;
}

// fp32: the segment's packed obstacle list (TrajScene::obsp), kObsGroup independent pair
// chains per iteration (the loop branch stops chains overlapping across iterations)
__device__ __forceinline__ float pens_fixed_all_f2(const TrajScene<float>& sc, const float* c, float r, int b,
                                                   bool quad, float* g) {
  const F2 cx = f2_dup(c[0]), cy = f2_dup(c[1]), cz = f2_dup(c[2]);
  PenAcc2 a;
  a.v = a.gx = a.gy = a.gz = f2_dup(0.f);
  const ulonglong2* sp = reinterpret_cast<const ulonglong2*>(sc.obsp[b]);
  const int np = sc.obs_np[b];
  for (int p0 = 0; p0 < np; p0 += kObsGroup) {
#pragma unroll
    for (int u = 0; u < kObsGroup; ++u) {
      const ulonglong2 XY = sp[2 * (p0 + u)], ZR = sp[2 * (p0 + u) + 1];
      float ra, rb;
      f2_split(F2{ZR.y}, ra, rb);
      a = pen_two_packed(a, cx, cy, cz, r, quad, F2{XY.x}, F2{XY.y}, F2{ZR.x}, ra, rb);
    }
  }
  float v0, v1, x0, x1, y0, y1, z0, z1;
  f2_split(a.v, v0, v1);
  f2_split(a.gx, x0, x1);
  f2_split(a.gy, y0, y1);
  f2_split(a.gz, z0, z1);
  g[0] += x0 + x1;
  g[1] += y0 + y1;
  g[2] += z0 + z1;
  return v0 + v1;
}

// One sphere against every fixed obstacle (statics, then staged spheres [f0, f1)), on one
// lane: returns the summed value and adds the unscaled gradient to g.
template <typename R>
__device__ __forceinline__ R pens_fixed_all(const TrajScene<R>& sc, const R* c, R r, int b, int f0, int f1, bool quad,
                                            R* g) {
  if constexpr (sizeof(R) == 4) return pens_fixed_all_f2(sc, c, r, b, quad, g);
  const R cx = c[0], cy = c[1], cz = c[2];
  R v = R(0), gx = R(0), gy = R(0), gz = R(0);
#pragma unroll 4
  for (int o = 0; o < sc.n_static; ++o) {
    const R dx = cx - sc.st_c[o][0], dy = cy - sc.st_c[o][1], dz = cz - sc.st_c[o][2];
    R sl;
    v += pen_term(dx, dy, dz, r + sc.st_r[o], quad, &sl);
    gx -= sl * dx;
    gy -= sl * dy;
    gz -= sl * dz;
  }
#pragma unroll 2
  for (int o = f0; o < f1; ++o) {
    const R dx = cx - sc.staged[o][0], dy = cy - sc.staged[o][1], dz = cz - sc.staged[o][2];
    R sl;
    v += pen_term(dx, dy, dz, r + sc.br[o], quad, &sl);
    gx -= sl * dx;
    gy -= sl * dy;
    gz -= sl * dz;
  }
  g[0] += gx;
  g[1] += gy;
  g[2] += gz;
  return v;
}

// One sphere (c, radius rr) against the placed spheres [q0, q1) of one block: adds the
// penetration sum to v, the position slope sum to (ax, ay, az) and the yaw slope to aw
// (trajopt.py:601-635; pyaw = d(sphere xy)/d(block yaw)). (A packed f32x2 form, two placed
// spheres per instruction as in the fixed-obstacle pass, measured slower: blocks have 1-4
// spheres, so the pair loop rarely runs and its reductions and registers cost more.)
template <typename R>
__device__ __forceinline__ void placed_pass(const R* pl, const R* pyaw, R cx, R cy, R cz, R rr, int q0,
                                            int q1, bool quad, R& v, R& ax, R& ay, R& az, R& aw) {
  for (int q = q0; q < q1; ++q) {
    R px, py, pz, pr, wx, wy;
    if constexpr (sizeof(R) == 4) {  // one LDS.128 + one LDS.64 per placed sphere
      const float4 P = reinterpret_cast<const float4*>(pl)[q];
      const float2 Y = reinterpret_cast<const float2*>(pyaw)[q];
      px = P.x, py = P.y, pz = P.z, pr = P.w, wx = Y.x, wy = Y.y;
    } else {
      px = pl[4 * q], py = pl[4 * q + 1], pz = pl[4 * q + 2], pr = pl[4 * q + 3];
      wx = pyaw[2 * q], wy = pyaw[2 * q + 1];
    }
    const R dx = cx - px, dy = cy - py, dz = cz - pz;
    R sl;
    v += pen_term(dx, dy, dz, rr + pr, quad, &sl);
    const R fx = sl * dx, fy = sl * dy, fz = sl * dz;
    ax += fx;
    ay += fy;
    az += fz;
    aw += fx * wx + fy * wy;
  }
}

// Per-step state a waypoint tile carries across the phases (registers).
template <typename R>
struct WpState {
  R z[3], o[3], ee[3], Ree[9];
  R garm, gblk;       // unscaled joint gradients of the arm / held penetration sums
  R d0[3], fac, dy0;  // start-alignment terms (t == 0)
};

// ---------------------------------------------------------------------------------------
// al_eval: evaluate the AL objective, constraints and (want_grad) gradient of the CTA's
// particle. With lr > 0 the clamped descent step (trajopt.py:993-1002) is applied to x in
// place; otherwise (want_grad) the gradient is left in g[w*8 + k]. Ends with a barrier.
// ---------------------------------------------------------------------------------------
template <typename R, int KIND, int SPB>
__device__ __forceinline__ void al_eval(AlCtx<R>& C, const typename TwinSceneOf<R, KIND>::type& tw, const AlParams& prm, bool quad,
                        bool pquad, bool want_grad, R lr) {
  const TrajScene<R>& sc = *C.sc;
  const ChainDesc<R>& ch = sc.ch;
  const int tid = threadIdx.x;
  // sizes from the kernel-parameter layout (uniform to the compiler; equal to the scene's)
  const int W = C.L.W, J = C.L.J, T = prm.T, B = C.L.B, S = C.L.S, SBn = C.L.SB;
  const bool manip = C.g_manip;
  const bool is_aux = tid >= C.L.NW;
  const int lane = tid & 31;
  const int w = tid >> 3;
  const bool is_wp = !is_aux && w < W;
  const Tile tl = Tile::make();
  const Tile tlw = Tile::make_warp();  // for the calls every lane of the warp reaches
  const int j = tl.j;
  const int b = C.g_b, t = C.g_t;
  const bool interior = C.g_interior;
  const int h0 = C.g_h0, nh = C.g_nh, f0 = C.g_f0, f1 = C.g_f1;
  const R w_start = R(prm.w_start);
  const int bar_count = C.L.NW + 32 * C.L.NA;
  WpState<R> st;
  R obj_w = R(0), carm = R(0), cblk = R(0);

  // warp-role predicates from a warp vote: uniform by construction, so ptxas can branch on
  // them without divergence handling and the warp-wide shuffles inside stay plain SHFLs
  const bool aux_warp = __all_sync(0xffffffffu, is_aux);
  if (aux_warp) {
    // ================= phase A, aux warp ==================================================
    if (manip) {
      // placed poses from the final waypoints: the aux warp runs the B final-waypoint FKs
      // itself (4 tiles of 8 lanes, uniform trip count) so no tile waits for another warp's
      // FK; identical frames to the waypoint tiles' (same code, same operands)
      const int sub = lane >> 3;
      const int aux_id = (tid - C.L.NW) >> 5;  // second aux warp (NA = 2): blocks 4-7
      for (int base = 4 * aux_id; base < B; base += 4 * C.L.NA) {
        const int bb = base + sub;
        const bool act = bb < B;
        const int wf = (act ? bb : 0) * T + T - 1;
        const R qj = j < J ? C.x[wf * kXS + j] : R(0);
        TileFrame<R> f;
        tile_fk(tlw, ch, qj, f);
        if (act) {
          const R ps = yaw_of(f.Ree) - sc.grasp_yaw;
          R s, c;
          Math<R>::sincos_(ps, &s, &c);
          if (j == 0) {
            const R ox = sc.grasp_off[0], oy = sc.grasp_off[1];
            C.psi[bb] = ps;
            C.cp[bb] = c;
            C.sp[bb] = s;
            C.rows[4 * bb + 0] = f.ee[0] - (c * ox - s * oy);
            C.rows[4 * bb + 1] = f.ee[1] - (s * ox + c * oy);
            C.rows[4 * bb + 2] = f.ee[2] - sc.grasp_off[2];
            C.rows[4 * bb + 3] = ps;
          }
          for (int q = sc.blk_start[bb] + j; q < sc.blk_start[bb + 1]; q += kTile) {
            const R ux = sc.bu[q][0], uy = sc.bu[q][1], uz = sc.bu[q][2];
            C.pl[4 * q + 0] = f.ee[0] + c * ux - s * uy;
            C.pl[4 * q + 1] = f.ee[1] + s * ux + c * uy;
            C.pl[4 * q + 2] = f.ee[2] + uz;
            C.pl[4 * q + 3] = sc.br[q];
            // d(block sphere q)/d(placed yaw) (trajopt.py:601-635), once per step here
            // instead of in every (item, sphere) pair of the placed-block pass
            C.pyaw[2 * q + 0] = -s * ux - c * uy;
            C.pyaw[2 * q + 1] = c * ux - s * uy;
          }
        }
      }
      __syncwarp();
      if (C.L.NA == 2) {  // the twin below reads every block's pose: meet the second aux warp
        if (aux_id == 1) bar_aux_arrive();
        else bar_aux_sync();
      }
      bar_placed_arrive(bar_count);
      if (aux_id == 1) goto aux_done;  // the second aux warp only places blocks 4-7
      if (C.prof.on && lane == 0) atomicAdd(&g_al_arrive[1][5], (unsigned long long)(clock64() - C.prof.t));
      R cpl = twin_warp<R, KIND, SPB>(tw, C.rows, C.gpose, C.scr, lane, want_grad, pquad);
      if (C.prof.on && lane == 0) atomicAdd(&g_al_arrive[1][6], (unsigned long long)(clock64() - C.prof.t));
      if (sc.anchor) {  // yaw anchor (trajopt.py:531-539): lane bb takes segment bb, warp-summed
        R av = R(0);
        for (int bb = lane; bb < B; bb += 32) {
          const R wp = wrap_yaw(C.psi[bb]);
          av += pquad ? wp * wp : fabs(wp);
          if (want_grad) C.gpose[4 * bb + 3] += pquad ? R(2) * wp : (wp > R(0) ? R(1) : (wp < R(0) ? R(-1) : R(0)));
        }
        cpl += warp_sum_fixed(av);
      }
      if (lane == 0) C.scal[kCplace] = cpl;
    }
  aux_done:;
  } else {
    // ================= phase A, waypoint tiles ============================================
    // ---- P1: tile FK, sphere centres
    const int wq = is_wp ? w : 0;  // padding tiles mirror waypoint 0 (no writes)
    const R qj = j < J ? C.x[wq * kXS + j] : R(0);
    {
      TileFrame<R> f;
      tile_fk(tlw, ch, qj, f);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        st.z[c] = f.z[c];
        st.o[c] = f.o[c];
        st.ee[c] = f.ee[c];
      }
#pragma unroll
      for (int c = 0; c < 9; ++c) st.Ree[c] = f.Ree[c];
      if (is_wp) {
        if (j == 0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) C.ee[w * 3 + c] = f.ee[c];
#pragma unroll
          for (int c = 0; c < 9; ++c) C.rot[w * 9 + c] = f.Ree[c];
        }
        if (j < J)
          for (int s = C.g_slo; s < C.g_shi; ++s) tile_sphere(ch, f, s, C.armw + (w * S + s) * 3);
        if (interior) {  // held block = Ree @ FLIP @ u + ee (trajopt.py:441-447)
          for (int s = j; s < nh; s += kTile) {
            const R ux = sc.bu[h0 + s][0], uy = sc.bu[h0 + s][1], uz = sc.bu[h0 + s][2];
            R* h = C.hp + (w * SBn + s) * 3;
            h[0] = ((f.Ree[0] * ux - f.Ree[1] * uy) - f.Ree[2] * uz) + f.ee[0];
            h[1] = ((f.Ree[3] * ux - f.Ree[4] * uy) - f.Ree[5] * uz) + f.ee[1];
            h[2] = ((f.Ree[6] * ux - f.Ree[7] * uy) - f.Ree[8] * uz) + f.ee[2];
          }
        }
      }
    }
    C.prof.arrive(0, C.L.NW);
    // the placed poses (aux warp) are the only cross-warp input of P2/P3; the sync also
    // orders this warp's own P1 writes (held spheres are read by other lanes below)
    if (manip) bar_placed_sync(bar_count);
    else __syncwarp();
    C.prof.mark(0);

    // ---- P2: leg, start terms, fixed obstacles
    // path length (trajopt.py:474-476): tile sum of the leg's squared components
    R dv = R(0);
    if (is_wp && t < T - 1 && j < J) dv = C.x[(wq + 1) * kXS + j] - qj;
    const R s2 = tlw.sum(dv * dv);
    if (is_wp && t < T - 1) {
      const R ln = Math<R>::sqrt_(s2);
      if (j == 0) obj_w += ln;
      C.unit[w * kXS + j] = (ln > R(1e-12) && j < J) ? dv / ln : R(0);
    }
    // start alignment (trajopt.py:477-494), uniform across the tile
    if (is_wp && manip && t == 0) {
      st.d0[0] = st.ee[0] - sc.pick_pos[b][0];
      st.d0[1] = st.ee[1] - sc.pick_pos[b][1];
      st.d0[2] = st.ee[2] - sc.pick_pos[b][2];
      R cosd = -st.Ree[8];
      cosd = cosd < R(-1) ? R(-1) : (cosd > R(1) ? R(1) : cosd);
      const R th = Math<R>::acos_(cosd);
      st.dy0 = wrap_yaw(yaw_of(st.Ree) - sc.pick_yaw[b]);
      const R sth = Math<R>::sqrt_(fmax(R(1) - cosd * cosd, R(0)));
      st.fac = sth > R(1e-8) ? R(-2) * th / fmax(sth, R(1e-8)) : (cosd > R(0) ? R(-2) : R(0));
      if (j == 0)
        obj_w += w_start * ((((st.d0[0] * st.d0[0] + st.d0[1] * st.d0[1]) + st.d0[2] * st.d0[2]) + th * th) +
                            st.dy0 * st.dy0);
    }
    C.prof.arrive(5, C.L.NW);  // sub-mark: leg + start terms done
    // Sphere-major: the tile's 8 lanes take the waypoint's spheres (arm spheres, then the
    // held-block spheres) round-robin, each against the whole fixed list, so a sphere's
    // gradient stays lane-local (no tile sums) and the values join the warp sums below.
    if (is_wp) {
      const int n_items = S + (interior ? nh : 0);
      for (int it = j; it < n_items; it += kTile) {
        const bool arm = it < S;
        const int s = arm ? it : it - S;
        const R* c = arm ? C.armw + (w * S + s) * 3 : C.hp + (w * SBn + s) * 3;
        R gg[3] = {R(0), R(0), R(0)};
        const R v = pens_fixed_all(sc, c, arm ? ch.arm_r[s] : sc.br[h0 + s], b, f0, f1, quad, gg);
        R* go = arm ? C.ga + (w * S + s) * 3 : C.gh + (w * SBn + s) * 3;
        go[0] = gg[0];
        go[1] = gg[1];
        go[2] = gg[2];
        if (arm) carm += v;
        else cblk += v;
      }
    }
    C.prof.arrive(1, C.L.NW);
    __syncwarp();  // P3 reads the sphere gradients other lanes of the tile wrote
    C.prof.mark(1);

    // ---- P3: placed blocks, placed-pose partials, J^T products
    st.garm = R(0);
    st.gblk = R(0);
    if (manip && B > 1) {
      // Sphere-major like P2: the lane's items (arm spheres, then held-block spheres; item
      // it = j + 8k) against the placed spheres of every earlier block. The items' gradients
      // accumulate in registers and join their P2 slots (written by this same lane) once at
      // the end; the per-block placed-pose partials are tile reduce-scattered per block.
      // Uniform trip count over the warp (blocks jb < B - 1; segment b uses jb < b) so the
      // reduce-scatter can use the warp-mask shuffles.
      const int n_items = is_wp ? S + (interior ? nh : 0) : 0;
      R gi[kAlItems][3];
#pragma unroll
      for (int k = 0; k < kAlItems; ++k) gi[k][0] = gi[k][1] = gi[k][2] = R(0);
      for (int jb = 0; jb + 1 < B; ++jb) {
        const bool act = is_wp && jb < b;
        // a warp whose tiles all sit in segments <= jb has nothing here (its reduce-scatter
        // would sum zeros it does not store): skip the block, warp-uniformly
        if (!__any_sync(0xffffffffu, act)) continue;
        R A[4] = {R(0), R(0), R(0), R(0)}, H[4] = {R(0), R(0), R(0), R(0)};
        if (act) {
          const int q0 = sc.blk_start[jb], q1 = sc.blk_start[jb + 1];
#pragma unroll
          for (int k = 0; k < kAlItems; ++k) {
            const int it = j + kTile * k;
            if (it >= n_items) break;
            const bool arm = it < S;
            const int si = arm ? it : it - S;
            const R* c = arm ? C.armw + (w * S + si) * 3 : C.hp + (w * SBn + si) * 3;
            const R cx = c[0], cy = c[1], cz = c[2];
            const R rr = arm ? ch.arm_r[si] : sc.br[h0 + si];
            R v = R(0), ax = R(0), ay = R(0), az = R(0), aw = R(0);
            placed_pass(C.pl, C.pyaw, cx, cy, cz, rr, q0, q1, quad, v, ax, ay, az, aw);
            gi[k][0] -= ax;
            gi[k][1] -= ay;
            gi[k][2] -= az;
            if (arm) {
              A[0] += ax;
              A[1] += ay;
              A[2] += az;
              A[3] += aw;
              carm += v;
            } else {
              H[0] += ax;
              H[1] += ay;
              H[2] += az;
              H[3] += aw;
              cblk += v;
            }
          }
        }
        if (want_grad) {  // tile reduce-scatter: lane j stores [class j/4][block jb][G xyz | G yaw][j%4]
          const R v8[8] = {A[0], A[1], A[2], A[3], H[0], H[1], H[2], H[3]};
          const R r = tlw.sum8_scatter(v8);
          if (act) C.pg[((w * 2 + (j >> 2)) * B + jb) * 4 + (j & 3)] = r;
        }
      }
      if (want_grad) {
#pragma unroll
        for (int k = 0; k < kAlItems; ++k) {
          const int it = j + kTile * k;
          if (it >= n_items) break;
          R* go = it < S ? C.ga + (w * S + it) * 3 : C.gh + (w * SBn + it - S) * 3;
          go[0] += gi[k][0];
          go[1] += gi[k][1];
          go[2] += gi[k][2];
        }
      }
    }
    __syncwarp();  // the J^T products below read sphere gradients other lanes of the tile own
    if (want_grad) {
      // arm: suffix sums over links >= k of (g, a x g), lane k = joint k (trajopt.py:586-590)
      // the link's first sphere by selects (no divergent branch: every lane of the warp runs
      // it), further spheres of multi-sphere links in the loop
      R G[3], Mv[3];
      const int wq = is_wp ? w : 0;
      {
        const bool ok = is_wp && C.g_slo < C.g_shi;
        const int s0 = ok ? C.g_slo : 0;
        const R* a = C.armw + (wq * S + s0) * 3;
        const R* gg = C.ga + (wq * S + s0) * 3;
        R m[3];
        cross3(a, gg, m);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          G[c] = ok ? R(0) + gg[c] : R(0);
          Mv[c] = ok ? R(0) + m[c] : R(0);
        }
      }
      for (int s = C.g_slo + 1; s < C.g_shi; ++s) {
        const R* a = C.armw + (w * S + s) * 3;
        const R* gg = C.ga + (w * S + s) * 3;
        R m[3];
        cross3(a, gg, m);
        G[0] += gg[0];
        G[1] += gg[1];
        G[2] += gg[2];
        Mv[0] += m[0];
        Mv[1] += m[1];
        Mv[2] += m[2];
      }
#pragma unroll
      for (int d = 1; d < kTile; d <<= 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const R gv = tlw.down(G[c], d), mv = tlw.down(Mv[c], d);
          const bool in = j + d < kTile;
          G[c] = in ? G[c] + gv : G[c];
          Mv[c] = in ? Mv[c] + mv : Mv[c];
        }
      }
      R og[3];
      cross3(st.o, G, og);
      st.garm = (st.z[0] * (Mv[0] - og[0]) + st.z[1] * (Mv[1] - og[1])) + st.z[2] * (Mv[2] - og[2]);
      // held block: every joint moves it (trajopt.py:592-599)
      R Gh[3], Mh[3];
      {  // the lane's first held sphere by selects, more (blocks of > 8 spheres) in the loop
        const bool ok = interior && is_wp && j < nh;
        const int s0 = ok ? j : 0;
        const R* a = C.hp + (wq * SBn + s0) * 3;
        const R* gg = C.gh + (wq * SBn + s0) * 3;
        R m[3];
        cross3(a, gg, m);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          Gh[c] = ok ? R(0) + gg[c] : R(0);
          Mh[c] = ok ? R(0) + m[c] : R(0);
        }
      }
      if (interior && is_wp) {
        for (int s = j + kTile; s < nh; s += kTile) {
          const R* a = C.hp + (w * SBn + s) * 3;
          const R* gg = C.gh + (w * SBn + s) * 3;
          R m[3];
          cross3(a, gg, m);
          Gh[0] += gg[0];
          Gh[1] += gg[1];
          Gh[2] += gg[2];
          Mh[0] += m[0];
          Mh[1] += m[1];
          Mh[2] += m[2];
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        Gh[c] = tlw.sum(Gh[c]);
        Mh[c] = tlw.sum(Mh[c]);
      }
      cross3(st.o, Gh, og);
      st.gblk = (st.z[0] * (Mh[0] - og[0]) + st.z[1] * (Mh[1] - og[1])) + st.z[2] * (Mh[2] - og[2]);
    }
    // warp partial sums of the scalars (fixed xor-tree order)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      obj_w += __shfl_xor_sync(0xffffffffu, obj_w, off);
      carm += __shfl_xor_sync(0xffffffffu, carm, off);
      cblk += __shfl_xor_sync(0xffffffffu, cblk, off);
    }
    if (lane == 0) {
      C.red[4 * (tid >> 5) + 0] = obj_w;
      C.red[4 * (tid >> 5) + 1] = carm;
      C.red[4 * (tid >> 5) + 2] = cblk;
    }
    C.prof.arrive(2, C.L.NW);
  }
  __syncthreads();
  C.prof.mark(2);

  // ================= phase B ==============================================================
  // totals, constraint vector and multiplier scales (trajopt.py:541-548): formed by thread
  // 0 for the records and, redundantly, by every lane that assembles a gradient (same
  // operands in the same order: bitwise identical), so no further barrier is needed
  const bool grad_lane = want_grad && is_wp && j < J;
  R s_pl = R(0), s_arm = R(0), s_blk = R(0);
  if (tid == 0 || grad_lane) {
    R o = R(0), ca = R(0), cb = R(0);
#pragma unroll 4
    for (int wi = 0; wi < C.L.NW / 32; ++wi) {
      o += C.red[4 * wi];
      ca += C.red[4 * wi + 1];
      cb += C.red[4 * wi + 2];
    }
    const R cpl = manip ? C.scal[kCplace] : R(0);
    const R c0 = R(prm.w_place) * cpl, c1 = R(prm.w_arm) * ca, c2 = R(prm.w_block) * cb;
    const R mu = C.scal[kMu];
    const R l0 = C.scal[kLam0], l1 = C.scal[kLam1], l2 = C.scal[kLam2];
    s_pl = (l0 + mu * c0) * R(prm.w_place);
    s_arm = (l1 + mu * c1) * R(prm.w_arm);
    s_blk = (l2 + mu * c2) * R(prm.w_block);
    if (tid == 0) {
      C.scal[kObj] = o;
      C.scal[kCarm] = ca;
      C.scal[kCblk] = cb;
      C.scal[kCons0] = c0;
      C.scal[kCons1] = c1;
      C.scal[kCons2] = c2;
      C.scal[kLag] = o + ((l0 * c0 + l1 * c1) + l2 * c2) + R(0.5) * mu * ((c0 * c0 + c1 * c1) + c2 * c2);
      C.scal[kSc0] = s_pl;
      C.scal[kSc1] = s_arm;
      C.scal[kSc2] = s_blk;
    }
  }
  // placed-block partials of segment b summed over the later segments' waypoints, in
  // waypoint order, by its final-waypoint tile: lane j forms item j ([class j/4][xyz|yaw])
  if (want_grad && manip && is_wp && t == T - 1) {
    const int cls = j >> 2, i = j & 3;
    R s0 = R(0), s1 = R(0);  // two interleaved partial sums (fixed order)
    int wv = (b + 1) * T;
    for (; wv + 1 < W; wv += 2) {
      s0 += C.pg[((wv * 2 + cls) * B + b) * 4 + i];
      s1 += C.pg[(((wv + 1) * 2 + cls) * B + b) * 4 + i];
    }
    if (wv < W) s0 += C.pg[((wv * 2 + cls) * B + b) * 4 + i];
    C.pgsum[(cls * B + b) * 4 + i] = s0 + s1;
    __syncwarp(tl.mask);
  }

  C.prof.arrive(7, C.L.NW);  // sub-mark: totals + placed partial sums done
  // gradient assembly (lane k = joint k) + optional update
  if (grad_lane) {
    R gq = R(0);
    if (t < T - 1) gq -= C.unit[w * kXS + j];
    if (t >= 1) gq += C.unit[(w - 1) * kXS + j];
    gq += s_arm * st.garm;
    gq += s_blk * st.gblk;
    if (manip && t == T - 1) {  // placement chain (trajopt.py:601-635)
      const R ox = sc.grasp_off[0], oy = sc.grasp_off[1];
      const R c = C.cp[b], s = C.sp[b];
      const R dox = s * ox + c * oy, doy = -c * ox + s * oy;
      const R gp0 = s_pl * C.gpose[4 * b], gp1 = s_pl * C.gpose[4 * b + 1], gp2 = s_pl * C.gpose[4 * b + 2],
              gp3 = s_pl * C.gpose[4 * b + 3];
      const R gyp = (gp0 * dox + gp1 * doy) + gp3;
      const R Gx = s_arm * C.pgsum[(0 * B + b) * 4 + 0] + s_blk * C.pgsum[(1 * B + b) * 4 + 0];
      const R Gy = s_arm * C.pgsum[(0 * B + b) * 4 + 1] + s_blk * C.pgsum[(1 * B + b) * 4 + 1];
      const R Gz = s_arm * C.pgsum[(0 * B + b) * 4 + 2] + s_blk * C.pgsum[(1 * B + b) * 4 + 2];
      const R Gw = s_arm * C.pgsum[(0 * B + b) * 4 + 3] + s_blk * C.pgsum[(1 * B + b) * 4 + 3];
      const R rel[3] = {st.ee[0] - st.o[0], st.ee[1] - st.o[1], st.ee[2] - st.o[2]};
      R jl[3];
      cross3(st.z, rel, jl);
      gq += ((Gx + gp0) * jl[0] + (Gy + gp1) * jl[1]) + (Gz + gp2) * jl[2];
      gq += (Gw + gyp) * yaw_jac(st.Ree, st.z);
    }
    if (manip && t == 0) {  // start alignment (trajopt.py:637-651)
      const R ax0[3] = {st.Ree[2], st.Ree[5], st.Ree[8]};
      const R rel[3] = {st.ee[0] - st.o[0], st.ee[1] - st.o[1], st.ee[2] - st.o[2]};
      R jl[3], dc[3];
      cross3(st.z, rel, jl);
      cross3(st.z, ax0, dc);
      gq += w_start * R(2) * ((st.d0[0] * jl[0] + st.d0[1] * jl[1]) + st.d0[2] * jl[2]);
      gq += w_start * st.fac * (-dc[2]);
      gq += w_start * R(2) * st.dy0 * yaw_jac(st.Ree, st.z);
    }
    if (lr > R(0)) {  // x <- clip(x - clip(lr g, +-0.1), lower, upper) (trajopt.py:997-1002)
      R stp = lr * gq;
      stp = stp < R(-0.1) ? R(-0.1) : (stp > R(0.1) ? R(0.1) : stp);
      R v = C.x[w * kXS + j] - stp;
      v = v < ch.lo[j] ? ch.lo[j] : (v > ch.hi[j] ? ch.hi[j] : v);
      if (!manip) {
        if (w == 0) v = sc.start[j];
        if (w == T - 1) v = sc.goal[j];
      }
      C.x[w * kXS + j] = v;
    } else {
      C.g[w * kXS + j] = gq;
    }
  }
  C.prof.arrive(4, C.L.NW);
  __syncthreads();
  C.prof.mark(4);
}

// ---------------------------------------------------------------------------------------
// validation of the CTA's particle (trajopt.py:1071-1153). Requires ee/rot/armw/hp of the
// current x (a preceding al_eval). Leaves the max violation in scal[kWorst].
// ---------------------------------------------------------------------------------------
template <typename R, int KIND, int SPB>
__device__ __forceinline__ void al_validate(AlCtx<R>& C, const typename TwinSceneOf<R, KIND>::type& tw, const AlParams& prm) {
  const TrajScene<R>& sc = *C.sc;
  const ChainDesc<R>& ch = sc.ch;
  const int tid = threadIdx.x;
  // sizes from the kernel-parameter layout (uniform to the compiler; equal to the scene's)
  const int W = C.L.W, J = C.L.J, T = prm.T, B = C.L.B, S = C.L.S, SBn = C.L.SB;
  const bool manip = sc.manip != 0;
  const bool is_aux = tid >= C.L.NW && tid < C.L.NW + 32;  // the first aux warp (a second one idles)
  const int lane = tid & 31;
  const int w = tid >> 3;
  const bool is_wp = tid < C.L.NW && w < W;
  const int j = tid & 7;
  const int b = is_wp ? w / T : 0;
  const int t = is_wp ? w - b * T : 0;
  // placed blocks from the final waypoints: inverse_grasp of the wrapped EE pose
  if (is_aux && manip && lane < B) {
    const int bb = lane, wf = bb * T + T - 1;
    const R* Rf = C.rot + wf * 9;
    const R* ef = C.ee + wf * 3;
    const R yaw = wrap_yaw(wrap_yaw(yaw_of(Rf)) - sc.grasp_yaw);
    R s, c;
    Math<R>::sincos_(yaw, &s, &c);
    const R ox = sc.grasp_off[0], oy = sc.grasp_off[1], oz = sc.grasp_off[2];
    const R px = ef[0] - (c * ox - s * oy), py = ef[1] - (s * ox + c * oy), pz = ef[2] - oz;
    C.rows[4 * bb + 0] = px;
    C.rows[4 * bb + 1] = py;
    C.rows[4 * bb + 2] = pz;
    C.rows[4 * bb + 3] = yaw;
    for (int q = sc.blk_start[bb]; q < sc.blk_start[bb + 1]; ++q) {
      const R lx = sc.bu[q][0] + ox, ly = sc.bu[q][1] + oy, lz = sc.bu[q][2] + oz;
      C.pl[4 * q + 0] = (lx * c - ly * s) + px;
      C.pl[4 * q + 1] = (lx * s + ly * c) + py;
      C.pl[4 * q + 2] = lz + pz;
      C.pl[4 * q + 3] = sc.br[q];
    }
  }
  __syncthreads();
  R worst = R(0);
  if (is_aux && manip) {
    R place = twin_warp<R, KIND, SPB>(tw, C.rows, nullptr, C.scr, lane, false, false);
    if (lane == 0) {
      if (sc.anchor)
        for (int bb = 0; bb < B; ++bb) place += fabs(wrap_yaw(C.rows[4 * bb + 3]));
      worst = fmax(worst, place);
    }
  } else if (is_aux && lane == 0) {
    {
      for (int k = 0; k < J; ++k) {
        worst = fmax(worst, fabs(C.x[0 * kXS + k] - sc.start[k]));
        worst = fmax(worst, fabs(C.x[(T - 1) * kXS + k] - sc.goal[k]));
      }
    }
  } else if (is_wp) {
    if (j < J) {
      const R q = C.x[w * kXS + j];
      worst = fmax(worst, fmax(q - ch.hi[j], ch.lo[j] - q));
    }
    const int f0 = manip ? sc.blk_start[b + 1] : 0, f1 = manip ? sc.n_blk : 0;
    const int p_end = manip ? sc.blk_start[b] : 0;  // placed spheres of blocks j < b
    const bool any_obs = (sc.n_static + (f1 - f0) + p_end) > 0;
    if (any_obs) {
      auto check = [&](const R* c, R r) {
        for (int o = 0; o < sc.n_static; ++o) {
          const R dx = c[0] - sc.st_c[o][0], dy = c[1] - sc.st_c[o][1], dz = c[2] - sc.st_c[o][2];
          worst = fmax(worst, (r + sc.st_r[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
        }
        for (int o = f0; o < f1; ++o) {
          const R dx = c[0] - sc.staged[o][0], dy = c[1] - sc.staged[o][1], dz = c[2] - sc.staged[o][2];
          worst = fmax(worst, (r + sc.br[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
        }
        for (int o = 0; o < p_end; ++o) {
          const R dx = c[0] - C.pl[4 * o], dy = c[1] - C.pl[4 * o + 1], dz = c[2] - C.pl[4 * o + 2];
          worst = fmax(worst, (r + sc.br[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
        }
      };
      if (j < J)
        for (int s = ch.link_start[j]; s < ch.link_start[j + 1]; ++s) check(C.armw + (w * S + s) * 3, ch.arm_r[s]);
      if (manip && t >= 1 && t <= T - 2) {
        const int h0 = sc.blk_start[b], nh = sc.blk_start[b + 1] - h0;
        for (int s = j; s < nh; s += kTile) check(C.hp + (w * SBn + s) * 3, sc.br[h0 + s]);
      }
    }
    if (manip && t == 0 && j == 0) {
      const R* Rm = C.rot + w * 9;
      const R dx = C.ee[w * 3] - sc.pick_pos[b][0], dy = C.ee[w * 3 + 1] - sc.pick_pos[b][1],
              dz = C.ee[w * 3 + 2] - sc.pick_pos[b][2];
      worst = fmax(worst, Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
      worst = fmax(worst, fabs(wrap_yaw(wrap_yaw(yaw_of(Rm)) - sc.pick_yaw[b])));
      R cd = -Rm[8];
      cd = cd < R(-1) ? R(-1) : (cd > R(1) ? R(1) : cd);
      worst = fmax(worst, Math<R>::acos_(cd));
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, off));
  if (lane == 0) C.red[4 * (tid >> 5) + 3] = worst;
  __syncthreads();
  if (tid == 0) {
    R wv = R(0);
    for (int wi = 0; wi < C.L.nwarps; ++wi) wv = fmax(wv, C.red[4 * wi + 3]);
    C.scal[kWorst] = wv;
  }
  __syncthreads();
}

// load the trajectory scene + particle p into shared memory (x rows [w][8])
template <typename R>
__device__ void al_load(AlCtx<R>& C, const TrajScene<R>* g_scene, const R* values, int64_t p) {
  const int tid = threadIdx.x;
  {
    const int4* src = reinterpret_cast<const int4*>(g_scene);
    int4* dst = reinterpret_cast<int4*>(C.sc);
    const int n = (int)(sizeof(TrajScene<R>) / sizeof(int4));
    for (int i = tid; i < n; i += blockDim.x) dst[i] = src[i];
  }
  const int W = C.L.W, J = C.L.J;
  const R* v = values + p * (int64_t)W * J;
  for (int i = tid; i < W * kXS; i += blockDim.x) {
    const int w = i / kXS, k = i - w * kXS;
    C.x[i] = k < J ? v[w * J + k] : R(0);
  }
  if (tid < 32) C.scal[tid] = R(0);
  __syncthreads();
}

// copy the kernel-parameter twin scene into shared memory (see AlLayout::twin)
template <typename TW>
__device__ const TW& twin_smem(unsigned char* smem, const AlLayout& L, const TW& tw) {
  TW* dst = reinterpret_cast<TW*>(smem + L.twin);
  const int* src = reinterpret_cast<const int*>(&tw);
  int* d = reinterpret_cast<int*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(TW) / sizeof(int)); i += blockDim.x) d[i] = src[i];
  __syncthreads();
  return *dst;
}

template <typename R>
__device__ void al_store_x(const AlCtx<R>& C, R* dst) {
  const int W = C.L.W, J = C.L.J;
  for (int i = threadIdx.x; i < W * J; i += blockDim.x) {
    const int w = i / J, k = i - w * J;
    dst[i] = C.x[w * kXS + k];
  }
}

// ---------------------------------------------------------------------------------------
// k_al_eval: trajectory_cost / al_value_and_gradient for a batch (CTA per particle)
// ---------------------------------------------------------------------------------------
template <typename R, int KIND, int SPB>
__global__ void __launch_bounds__(kMaxAlThreads) k_al_eval(const TrajScene<R>* __restrict__ g_scene,
                                                           const typename TwinSceneOf<R, KIND>::type tw, AlLayout L,
                                                           AlParams prm, const R* __restrict__ values,
                                                           const R* __restrict__ lam, const R* __restrict__ mu,
                                                           int mode, int place_mode, int want_grad,
                                                           R* __restrict__ obj, R* __restrict__ cons,
                                                           R* __restrict__ lag, R* __restrict__ grad) {
  extern __shared__ __align__(16) unsigned char smem[];
  AlCtx<R> C;
  C.bind(smem, L);
  const int64_t p = blockIdx.x;
  al_load(C, g_scene, values, p);
  const auto& tws = twin_smem(smem, L, tw);
  C.geom(prm.T);
  if (threadIdx.x == 0) {
    C.scal[kLam0] = lam ? lam[3 * p] : R(0);
    C.scal[kLam1] = lam ? lam[3 * p + 1] : R(0);
    C.scal[kLam2] = lam ? lam[3 * p + 2] : R(0);
    C.scal[kMu] = mu ? mu[p] : R(0);
  }
  __syncthreads();
  al_eval<R, KIND, SPB>(C, tws, prm, mode == 1, place_mode == 1, want_grad != 0, R(0));
  if (threadIdx.x == 0) {
    if (obj) obj[p] = C.scal[kObj];
    if (cons) {
      cons[3 * p] = C.scal[kCons0];
      cons[3 * p + 1] = C.scal[kCons1];
      cons[3 * p + 2] = C.scal[kCons2];
    }
    if (lag) lag[p] = C.scal[kLag];
  }
  if (want_grad && grad) {
    const int W = L.W, J = L.J;
    R* gout = grad + p * (int64_t)W * J;
    for (int i = threadIdx.x; i < W * J; i += blockDim.x) {
      const int w = i / J, k = i - w * J;
      gout[i] = C.g[w * kXS + k];
    }
  }
}

// k_validate: validate() for a batch of trajectories (CTA per trajectory)
template <typename R, int KIND, int SPB>
__global__ void __launch_bounds__(kMaxAlThreads) k_validate(const TrajScene<R>* __restrict__ g_scene,
                                                            const typename TwinSceneOf<R, KIND>::type tw, AlLayout L,
                                                            AlParams prm, const R* __restrict__ values,
                                                            uint8_t* __restrict__ feasible,
                                                            R* __restrict__ violation) {
  extern __shared__ __align__(16) unsigned char smem[];
  AlCtx<R> C;
  C.bind(smem, L);
  const int64_t p = blockIdx.x;
  al_load(C, g_scene, values, p);
  const auto& tws = twin_smem(smem, L, tw);
  C.geom(prm.T);
  al_eval<R, KIND, SPB>(C, tws, prm, false, false, false, R(0));  // FK tables for the current x
  al_validate<R, KIND, SPB>(C, tws, prm);
  if (threadIdx.x == 0) {
    const R wv = C.scal[kWorst];
    violation[p] = wv;
    feasible[p] = (uint8_t)(wv < R(prm.eps));
  }
}

// ---------------------------------------------------------------------------------------
// k_solve_al: solve_al (trajopt.py:936-1063), one CTA per trajectory particle.
//
// Particles only interact through "stop at the first outer iteration in which ANY
// particle validates". Each CTA publishes its first feasible outer with atomicMin on
// *kstar and stops as soon as a lower-indexed outer has produced a feasible particle
// (it has then recorded every outer <= kstar). Per-outer records and the snapshot at
// the particle's first feasible outer make the final choice (lowest objective among
// the particles feasible at kstar, first index on ties) independent of CTA timing.
// ---------------------------------------------------------------------------------------
struct AlRecords {
  void *mu, *lam, *cons, *upd, *obj, *viol;  // [outer][P] (x3 for lam/cons/upd), dtype R
  uint8_t* feas;                             // [outer][P]
  int32_t* first_feas;                       // [P] first feasible outer or -1
  int32_t* n_outers;                         // [P] outers completed
  int* kstar;                                // global min feasible outer (INT_MAX = none yet)
  void* best_x;                              // [P][B][T][J] snapshot at first feasible outer
  const int32_t* n_active;                   // device count of live particles (nullptr = gridDim.x)
};

// MAXT: the block-size bound. 256 (C2-sized particles, <= 28 waypoints) lets ptxas keep the
// whole tower engine in up to 255 registers; 512 caps it at 128 (launch_solve_al picks).
template <typename R, int KIND, int SPB, int MAXT = kMaxAlThreads>
__global__ void __launch_bounds__(MAXT, 1) k_solve_al(const TrajScene<R>* __restrict__ g_scene,
                                                            const typename TwinSceneOf<R, KIND>::type tw, AlLayout L,
                                                            AlParams prm, const R* __restrict__ values, int P,
                                                            AlRecords rec) {
  extern __shared__ __align__(16) unsigned char smem[];
  AlCtx<R> C;
  C.bind(smem, L);
  const int p = blockIdx.x;
  if (rec.n_active && p >= *rec.n_active) return;
  al_load(C, g_scene, values, p);
  const auto& tws = twin_smem(smem, L, tw);
  C.geom(prm.T);
  const TrajScene<R>& sc = *C.sc;
  const ChainDesc<R>& ch = sc.ch;
  const int tid = threadIdx.x;
  const int W = L.W, J = ch.J, T = prm.T;
  const bool manip = sc.manip != 0;
  R* r_mu = reinterpret_cast<R*>(rec.mu);
  R* r_lam = reinterpret_cast<R*>(rec.lam);
  R* r_cons = reinterpret_cast<R*>(rec.cons);
  R* r_upd = reinterpret_cast<R*>(rec.upd);
  R* r_obj = reinterpret_cast<R*>(rec.obj);
  R* r_viol = reinterpret_cast<R*>(rec.viol);
  if (tid == 0) {
    C.scal[kMu] = R(prm.mu0);
    C.scal[kPrev] = R(INFINITY);
    C.flags[0] = 0;
  }
  __syncthreads();
  C.prof.start();
  const R denom = R(prm.inner_steps - 1 > 1 ? prm.inner_steps - 1 : 1);
  int first = -1, done = 0;
  for (int outer = 0; outer < prm.outer_iters; ++outer) {
    if (tid == 0) C.flags[0] = (outer > *((volatile int*)rec.kstar)) ? 1 : 0;
    __syncthreads();
    if (C.flags[0]) break;
    for (int k = 0; k < prm.inner_steps; ++k) {
      const R lr = R(prm.lr_init) + (R(prm.lr_final) - R(prm.lr_init)) * (R(k) / denom);
      al_eval<R, KIND, SPB>(C, tws, prm, false, prm.place_mode == 1, true, lr);
    }
    // retract pick waypoints to the exact grasp (trajopt.py:1004-1007), lane j = joint j.
    // With at least B tile warps, warp bb polishes segment bb as 4 identical 8-lane replicas
    // (warp-mask shuffles, replicas exit together); else one tile per segment.
    if (manip && L.NW / 32 >= L.B) {
      if (__all_sync(0xffffffffu, (tid >> 5) < L.B)) {  // warp-uniform (vote): plain shuffles inside
        const Tile tlw = Tile::make_warp();
        const int bb = tid >> 5;
        const int w0 = bb * T;
        R qj = tlw.j < J ? C.x[w0 * kXS + tlw.j] : R(0);
        int its = 0;
        tile_polish<R>(tlw, ch, qj, sc.pick_pos[bb], sc.pick_yaw[bb], nullptr, 0, nullptr, 0, nullptr, &its);
        if (C.prof.on && (tid & 31) == 0) {
          atomicAdd(&g_al_polish[0], (unsigned long long)its);
          atomicAdd(&g_al_polish[1], 1ull);
          if (its >= kPolishMaxIters) atomicAdd(&g_al_polish[2], 1ull);
          atomicMax(&g_al_polish[3], (unsigned long long)its);
        }
        __syncwarp();  // the replica lanes' reads of x above precede lanes 0-7's writes
        if ((tid & 31) < kTile && tlw.j < J) C.x[w0 * kXS + tlw.j] = qj;
      }
    } else if (manip && (tid >> 3) < L.B) {
      const Tile tl = Tile::make();
      const int bb = tid >> 3;
      const int w0 = bb * T;
      R qj = tl.j < J ? C.x[w0 * kXS + tl.j] : R(0);
      tile_polish<R>(tl, ch, qj, sc.pick_pos[bb], sc.pick_yaw[bb]);
      if (tl.j < J) C.x[w0 * kXS + tl.j] = qj;
    }
    __syncthreads();
    C.prof.mark(8);  // pick-waypoint polish (+ the last inner step's tail)
    al_eval<R, KIND, SPB>(C, tws, prm, false, prm.place_mode == 1, false, R(0));
    al_validate<R, KIND, SPB>(C, tws, prm);
    C.prof.mark(9);  // re-evaluation + validate (eval marks fold into 0-4)
    if (tid == 0) {
      const int64_t o = (int64_t)outer * P + p;
      const R mu = C.scal[kMu];
      const R c0 = C.scal[kCons0], c1 = C.scal[kCons1], c2 = C.scal[kCons2];
      const R l0 = C.scal[kLam0], l1 = C.scal[kLam1], l2 = C.scal[kLam2];
      const R u0 = l0 + mu * c0, u1 = l1 + mu * c1, u2 = l2 + mu * c2;
      const R worst = C.scal[kWorst];
      const bool feas = worst < R(prm.eps);
      r_mu[o] = mu;
      r_lam[3 * o] = l0;
      r_lam[3 * o + 1] = l1;
      r_lam[3 * o + 2] = l2;
      r_cons[3 * o] = c0;
      r_cons[3 * o + 1] = c1;
      r_cons[3 * o + 2] = c2;
      r_upd[3 * o] = u0;
      r_upd[3 * o + 1] = u1;
      r_upd[3 * o + 2] = u2;
      r_obj[o] = C.scal[kObj];
      r_viol[o] = worst;
      rec.feas[o] = (uint8_t)feas;
      C.flags[1] = feas ? 1 : 0;
      if (feas) {
        atomicMin(rec.kstar, outer);
      } else {
        // lam <- lam + mu c; mu *= beta where max c > prev / 10 (trajopt.py:1051-1054)
        C.scal[kLam0] = u0;
        C.scal[kLam1] = u1;
        C.scal[kLam2] = u2;
        const R v = fmax(fmax(c0, c1), c2);
        if (v > C.scal[kPrev] / R(10)) C.scal[kMu] = mu * R(prm.beta);
        C.scal[kPrev] = v;
      }
    }
    __syncthreads();
    done = outer + 1;
    if (C.flags[1]) {
      first = outer;
      al_store_x(C, reinterpret_cast<R*>(rec.best_x) + (int64_t)p * W * J);
      break;
    }
  }
  if (tid == 0) {
    rec.first_feas[p] = first;
    rec.n_outers[p] = done;
  }
}

}  // namespace spasm
