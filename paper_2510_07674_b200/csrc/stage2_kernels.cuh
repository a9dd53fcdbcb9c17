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
#include "seedseq.cuh"
#include "stage1_models.cuh"
#include "stage2.cuh"

namespace spasm {

// ---- placement twin (the free-yaw copy of the stage-1 model, trajopt.py:281-302) ------
template <typename R>
struct NoTwin {
  int dim;
};
template <typename R, int KIND> struct TwinSceneOf { using type = NoTwin<R>; };
template <typename R> struct TwinSceneOf<R, 1> { using type = TetrisScene<R>; };
template <typename R> struct TwinSceneOf<R, 2> { using type = TowerScene<R>; };

template <typename R, int KIND, int SPB, bool WG, bool Q>
__device__ __forceinline__ R twin_run_t(const typename TwinSceneOf<R, KIND>::type& ts, const R* rows, R* grad,
                                        R* scr) {
  if constexpr (KIND == 1) {
    return TetrisEval<R, SPB, true>::template run<true, WG, Q>(ts, rows, grad, scr, 1);
  } else if constexpr (KIND == 2) {
    return TowerEval<R, true>::template run<true, WG, Q>(ts, rows, grad, scr, 1);
  } else {
    return R(0);
  }
}

template <typename R, int KIND, int SPB>
__device__ __forceinline__ R twin_run(const typename TwinSceneOf<R, KIND>::type& ts, const R* rows, R* grad, R* scr,
                                      bool want_grad, bool quad) {
  if (want_grad) {
    return quad ? twin_run_t<R, KIND, SPB, true, true>(ts, rows, grad, scr)
                : twin_run_t<R, KIND, SPB, true, false>(ts, rows, grad, scr);
  }
  return quad ? twin_run_t<R, KIND, SPB, false, true>(ts, rows, grad, scr)
              : twin_run_t<R, KIND, SPB, false, false>(ts, rows, grad, scr);
}

// ---- shared-memory layout of one AL CTA -----------------------------------------------
constexpr int kMaxAlThreads = 320;  // W <= 288 waypoints per particle + the aux warp
struct AlLayout {
  int W, NW, nthreads, nwarps, J, B, T, S, SB;
  // offsets in bytes from the dynamic smem base
  int scene, x, g, unit, ee, rot, org, axs, armw, ga, hp, gh, pg, pl, seg, rows, gpose, scr, jlf, yjf, pgsum, red,
      scal, flags;
  int total;
};

template <typename R>
__host__ __device__ inline AlLayout al_layout(int B, int T, int J, int S, int SB, int NB) {
  AlLayout L;
  L.W = B * T;
  L.NW = (L.W + 31) / 32 * 32;
  L.nthreads = L.NW + 32;
  L.nwarps = L.nthreads / 32;
  L.J = J;
  L.B = B;
  L.T = T;
  L.S = S;
  L.SB = SB;
  const int W = L.W;
  int off = 0;
  auto take = [&off](int bytes) {
    const int o = off;
    off += (bytes + 15) & ~15;
    return o;
  };
  const int r = (int)sizeof(R);
  L.scene = take((int)sizeof(TrajScene<R>));
  L.x = take(J * W * r);
  L.g = take(J * W * r);
  L.unit = take(J * W * r);
  L.ee = take(3 * W * r);
  L.rot = take(9 * W * r);
  L.org = take(3 * J * W * r);
  L.axs = take(3 * J * W * r);
  L.armw = take(3 * (S > 0 ? S : 1) * W * r);
  L.ga = take(3 * (S > 0 ? S : 1) * W * r);
  L.hp = take(3 * (SB > 0 ? SB : 1) * W * r);
  L.gh = take(3 * (SB > 0 ? SB : 1) * W * r);
  L.pg = take(8 * B * W * r);
  L.pl = take(3 * (NB > 0 ? NB : 1) * r);
  L.seg = take(3 * B * r);      // psi | cp | sp
  L.rows = take(4 * B * r);
  L.gpose = take(4 * B * r);
  L.scr = take((2 * B + 2) * r);
  L.jlf = take(3 * J * B * r);
  L.yjf = take(J * B * r);
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
  kWorst, kUpd0, kUpd1, kUpd2
};

template <typename R>
struct AlCtx {
  AlLayout L;
  TrajScene<R>* sc;
  R *x, *g, *unit, *ee, *rot, *org, *axs, *armw, *ga, *hp, *gh, *pg, *pl, *psi, *cp, *sp, *rows, *gpose, *scr, *jlf,
      *yjf, *pgsum, *red, *scal;
  int* flags;

  __device__ void bind(unsigned char* base, const AlLayout& l) {
    L = l;
    sc = reinterpret_cast<TrajScene<R>*>(base + L.scene);
    x = reinterpret_cast<R*>(base + L.x);
    g = reinterpret_cast<R*>(base + L.g);
    unit = reinterpret_cast<R*>(base + L.unit);
    ee = reinterpret_cast<R*>(base + L.ee);
    rot = reinterpret_cast<R*>(base + L.rot);
    org = reinterpret_cast<R*>(base + L.org);
    axs = reinterpret_cast<R*>(base + L.axs);
    armw = reinterpret_cast<R*>(base + L.armw);
    ga = reinterpret_cast<R*>(base + L.ga);
    hp = reinterpret_cast<R*>(base + L.hp);
    gh = reinterpret_cast<R*>(base + L.gh);
    pg = reinterpret_cast<R*>(base + L.pg);
    pl = reinterpret_cast<R*>(base + L.pl);
    psi = reinterpret_cast<R*>(base + L.seg);
    cp = psi + L.B;
    sp = cp + L.B;
    rows = reinterpret_cast<R*>(base + L.rows);
    gpose = reinterpret_cast<R*>(base + L.gpose);
    scr = reinterpret_cast<R*>(base + L.scr);
    jlf = reinterpret_cast<R*>(base + L.jlf);
    yjf = reinterpret_cast<R*>(base + L.yjf);
    pgsum = reinterpret_cast<R*>(base + L.pgsum);
    red = reinterpret_cast<R*>(base + L.red);
    scal = reinterpret_cast<R*>(base + L.scal);
    flags = reinterpret_cast<int*>(base + L.flags);
  }
};

// penetration of one sphere pair; returns the (linear or squared) value and, when active,
// the unscaled gradient slope (d value / d ca = -slope * (ca - cb)) (trajopt.py:396-413)
template <typename R>
__device__ __forceinline__ R pen_term(R dx, R dy, R dz, R rsum, bool quad, R* slope) {
  const R d = Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz);
  R pen = rsum - d;
  pen = pen > R(0) ? pen : R(0);
  const bool live = pen > R(0) && d > R(0);
  *slope = live ? (quad ? R(2) * pen / d : R(1) / d) : R(0);
  return quad ? pen * pen : pen;
}

// ---------------------------------------------------------------------------------------
// al_eval: one evaluation of the AL objective / constraints (and gradient) for the CTA's
// particle held in ctx.x. On return (after a barrier): scal[kObj..kSc2] hold obj, the
// constraint parts and the multiplier scales; with want_grad, ctx.g holds dL/dx.
// ---------------------------------------------------------------------------------------
template <typename R, int KIND, int SPB>
__device__ void al_eval(AlCtx<R>& C, const typename TwinSceneOf<R, KIND>::type& tw, const AlParams& prm, bool quad,
                        bool pquad, bool want_grad) {
  const TrajScene<R>& sc = *C.sc;
  const ChainDesc<R>& ch = sc.ch;
  const int tid = threadIdx.x;
  const int W = C.L.W, J = ch.J, T = prm.T, B = sc.B, S = ch.S;
  const bool manip = sc.manip != 0;
  const bool is_wp = tid < W;
  const int lane = tid & 31;
  const bool is_aux = tid >= C.L.NW;
  const int b = is_wp ? tid / T : 0;
  const int t = is_wp ? tid - b * T : 0;
  const R w_start = R(prm.w_start);

  // ---------------- P1: forward kinematics of every waypoint -------------------------
  R obj_w = R(0), carm = R(0), cblk = R(0);
  R ee[3] = {R(0), R(0), R(0)}, Rm[9];
  if (is_wp) {
    fk_eval<R>(ch, C.x + tid, W, C.org + tid, C.axs + tid, S ? C.armw + tid : nullptr, W, ee, Rm);
#pragma unroll
    for (int i = 0; i < 3; ++i) C.ee[i * W + tid] = ee[i];
#pragma unroll
    for (int i = 0; i < 9; ++i) C.rot[i * W + tid] = Rm[i];
    // path length (trajopt.py:474-476)
    if (t < T - 1) {
      R dv[kMaxJ];
      R s2 = R(0);
      for (int k = 0; k < J; ++k) {
        dv[k] = C.x[k * W + tid + 1] - C.x[k * W + tid];
        s2 += dv[k] * dv[k];
      }
      const R ln = Math<R>::sqrt_(s2);
      obj_w += ln;
      for (int k = 0; k < J; ++k) C.unit[k * W + tid] = ln > R(1e-12) ? dv[k] / ln : R(0);
    }
    // start alignment (trajopt.py:477-494)
    if (manip && t == 0) {
      const R d0x = ee[0] - sc.pick_pos[b][0], d0y = ee[1] - sc.pick_pos[b][1], d0z = ee[2] - sc.pick_pos[b][2];
      R cosd = -Rm[8];
      cosd = cosd < R(-1) ? R(-1) : (cosd > R(1) ? R(1) : cosd);
      const R th = Math<R>::acos_(cosd);
      const R dy0 = wrap_yaw(yaw_of(Rm) - sc.pick_yaw[b]);
      obj_w += w_start * ((((d0x * d0x + d0y * d0y) + d0z * d0z) + th * th) + dy0 * dy0);
    }
  }
  __syncthreads();

  // ---------------- P2: aux = placed poses; waypoints = fixed-obstacle penetrations -----
  if (is_aux) {
    if (manip && lane < B) {
      const int bb = lane;
      const int wf = bb * T + T - 1;
      R Rf[9], ef[3];
#pragma unroll
      for (int i = 0; i < 9; ++i) Rf[i] = C.rot[i * W + wf];
#pragma unroll
      for (int i = 0; i < 3; ++i) ef[i] = C.ee[i * W + wf];
      const R ps = yaw_of(Rf) - sc.grasp_yaw;
      R s, c;
      Math<R>::sincos_(ps, &s, &c);
      C.psi[bb] = ps;
      C.cp[bb] = c;
      C.sp[bb] = s;
      const R ox = sc.grasp_off[0], oy = sc.grasp_off[1], oz = sc.grasp_off[2];
      C.rows[4 * bb + 0] = ef[0] - (c * ox - s * oy);
      C.rows[4 * bb + 1] = ef[1] - (s * ox + c * oy);
      C.rows[4 * bb + 2] = ef[2] - oz;
      C.rows[4 * bb + 3] = ps;
      for (int q = sc.blk_start[bb]; q < sc.blk_start[bb + 1]; ++q) {
        const R ux = sc.bu[q][0], uy = sc.bu[q][1], uz = sc.bu[q][2];
        C.pl[3 * q + 0] = ef[0] + c * ux - s * uy;
        C.pl[3 * q + 1] = ef[1] + s * ux + c * uy;
        C.pl[3 * q + 2] = ef[2] + uz;
      }
      if (want_grad) {
        for (int k = 0; k < J; ++k) {
          const R z[3] = {C.axs[(3 * k) * W + wf], C.axs[(3 * k + 1) * W + wf], C.axs[(3 * k + 2) * W + wf]};
          const R rel[3] = {ef[0] - C.org[(3 * k) * W + wf], ef[1] - C.org[(3 * k + 1) * W + wf],
                            ef[2] - C.org[(3 * k + 2) * W + wf]};
          R cr[3];
          cross3(z, rel, cr);
          C.jlf[(bb * J + k) * 3 + 0] = cr[0];
          C.jlf[(bb * J + k) * 3 + 1] = cr[1];
          C.jlf[(bb * J + k) * 3 + 2] = cr[2];
          C.yjf[bb * J + k] = yaw_jac(Rf, z);
        }
      }
    }
  } else if (is_wp) {
    // arm spheres vs the segment's fixed obstacles: statics + still-staged later blocks
    const int f_blk0 = manip ? sc.blk_start[b + 1] : 0, f_blk1 = manip ? sc.n_blk : 0;
    for (int s = 0; s < S; ++s) {
      const R ax = C.armw[(3 * s) * W + tid], ay = C.armw[(3 * s + 1) * W + tid], az = C.armw[(3 * s + 2) * W + tid];
      const R rs = ch.arm_r[s];
      R gx = R(0), gy = R(0), gz = R(0);
      for (int o = 0; o < sc.n_static; ++o) {
        const R dx = ax - sc.st_c[o][0], dy = ay - sc.st_c[o][1], dz = az - sc.st_c[o][2];
        R sl;
        carm += pen_term(dx, dy, dz, rs + sc.st_r[o], quad, &sl);
        gx -= sl * dx;
        gy -= sl * dy;
        gz -= sl * dz;
      }
      for (int o = f_blk0; o < f_blk1; ++o) {
        const R dx = ax - sc.staged[o][0], dy = ay - sc.staged[o][1], dz = az - sc.staged[o][2];
        R sl;
        carm += pen_term(dx, dy, dz, rs + sc.br[o], quad, &sl);
        gx -= sl * dx;
        gy -= sl * dy;
        gz -= sl * dz;
      }
      C.ga[(3 * s) * W + tid] = gx;
      C.ga[(3 * s + 1) * W + tid] = gy;
      C.ga[(3 * s + 2) * W + tid] = gz;
    }
    // held block on interior waypoints (trajopt.py:441-447, 516-529)
    if (manip && t >= 1 && t <= T - 2) {
      const int h0 = sc.blk_start[b], nh = sc.blk_start[b + 1] - h0;
      for (int s = 0; s < nh; ++s) {
        const R ux = sc.bu[h0 + s][0], uy = sc.bu[h0 + s][1], uz = sc.bu[h0 + s][2];
        // rot @ FLIP: columns 1 and 2 negated
        const R hx = ((Rm[0] * ux - Rm[1] * uy) - Rm[2] * uz) + ee[0];
        const R hy = ((Rm[3] * ux - Rm[4] * uy) - Rm[5] * uz) + ee[1];
        const R hz = ((Rm[6] * ux - Rm[7] * uy) - Rm[8] * uz) + ee[2];
        C.hp[(3 * s) * W + tid] = hx;
        C.hp[(3 * s + 1) * W + tid] = hy;
        C.hp[(3 * s + 2) * W + tid] = hz;
        const R rh = sc.br[h0 + s];
        R gx = R(0), gy = R(0), gz = R(0);
        for (int o = 0; o < sc.n_static; ++o) {
          const R dx = hx - sc.st_c[o][0], dy = hy - sc.st_c[o][1], dz = hz - sc.st_c[o][2];
          R sl;
          cblk += pen_term(dx, dy, dz, rh + sc.st_r[o], quad, &sl);
          gx -= sl * dx;
          gy -= sl * dy;
          gz -= sl * dz;
        }
        for (int o = f_blk0; o < f_blk1; ++o) {
          const R dx = hx - sc.staged[o][0], dy = hy - sc.staged[o][1], dz = hz - sc.staged[o][2];
          R sl;
          cblk += pen_term(dx, dy, dz, rh + sc.br[o], quad, &sl);
          gx -= sl * dx;
          gy -= sl * dy;
          gz -= sl * dz;
        }
        C.gh[(3 * s) * W + tid] = gx;
        C.gh[(3 * s + 1) * W + tid] = gy;
        C.gh[(3 * s + 2) * W + tid] = gz;
      }
    }
  }
  __syncthreads();

  // ---------------- P3: aux = placement twin; waypoints = placed-block penetrations -----
  R garm[kMaxJ], gblk[kMaxJ];
#pragma unroll
  for (int k = 0; k < kMaxJ; ++k) {
    garm[k] = R(0);
    gblk[k] = R(0);
  }
  if (is_aux) {
    if (manip && lane == 0) {
      R cpl = twin_run<R, KIND, SPB>(tw, C.rows, C.gpose, C.scr, want_grad, pquad);
      if (sc.anchor) {
        for (int bb = 0; bb < B; ++bb) {
          const R wp = wrap_yaw(C.psi[bb]);
          cpl += pquad ? wp * wp : fabs(wp);
          if (want_grad) C.gpose[4 * bb + 3] += pquad ? R(2) * wp : (wp > R(0) ? R(1) : (wp < R(0) ? R(-1) : R(0)));
        }
      }
      C.scal[kCplace] = cpl;
    }
  } else if (is_wp) {
    if (manip) {
      for (int j = 0; j < b; ++j) {
        const R cj = C.cp[j], sj = C.sp[j];
        R A0 = R(0), A1 = R(0), A2 = R(0), A3 = R(0), H0 = R(0), H1 = R(0), H2 = R(0), H3 = R(0);
        for (int q = sc.blk_start[j]; q < sc.blk_start[j + 1]; ++q) {
          const R px = C.pl[3 * q], py = C.pl[3 * q + 1], pz = C.pl[3 * q + 2], rq = sc.br[q];
          const R drx = -sj * sc.bu[q][0] - cj * sc.bu[q][1];
          const R dry = cj * sc.bu[q][0] - sj * sc.bu[q][1];
          R Gx = R(0), Gy = R(0), Gz = R(0);
          for (int s = 0; s < S; ++s) {
            const R dx = C.armw[(3 * s) * W + tid] - px, dy = C.armw[(3 * s + 1) * W + tid] - py,
                    dz = C.armw[(3 * s + 2) * W + tid] - pz;
            R sl;
            carm += pen_term(dx, dy, dz, ch.arm_r[s] + rq, quad, &sl);
            if (want_grad && sl != R(0)) {
              C.ga[(3 * s) * W + tid] -= sl * dx;
              C.ga[(3 * s + 1) * W + tid] -= sl * dy;
              C.ga[(3 * s + 2) * W + tid] -= sl * dz;
              Gx += sl * dx;
              Gy += sl * dy;
              Gz += sl * dz;
            }
          }
          A0 += Gx;
          A1 += Gy;
          A2 += Gz;
          A3 += Gx * drx + Gy * dry;
          if (t >= 1 && t <= T - 2) {
            R Hx = R(0), Hy = R(0), Hz = R(0);
            const int h0 = sc.blk_start[b], nh = sc.blk_start[b + 1] - h0;
            for (int s = 0; s < nh; ++s) {
              const R dx = C.hp[(3 * s) * W + tid] - px, dy = C.hp[(3 * s + 1) * W + tid] - py,
                      dz = C.hp[(3 * s + 2) * W + tid] - pz;
              R sl;
              cblk += pen_term(dx, dy, dz, sc.br[h0 + s] + rq, quad, &sl);
              if (want_grad && sl != R(0)) {
                C.gh[(3 * s) * W + tid] -= sl * dx;
                C.gh[(3 * s + 1) * W + tid] -= sl * dy;
                C.gh[(3 * s + 2) * W + tid] -= sl * dz;
                Hx += sl * dx;
                Hy += sl * dy;
                Hz += sl * dz;
              }
            }
            H0 += Hx;
            H1 += Hy;
            H2 += Hz;
            H3 += Hx * drx + Hy * dry;
          }
        }
        if (want_grad) {  // placed-block partials of this waypoint: [class][block j][G xyz | G yaw]
          C.pg[((0 * B + j) * 4 + 0) * W + tid] = A0;
          C.pg[((0 * B + j) * 4 + 1) * W + tid] = A1;
          C.pg[((0 * B + j) * 4 + 2) * W + tid] = A2;
          C.pg[((0 * B + j) * 4 + 3) * W + tid] = A3;
          C.pg[((1 * B + j) * 4 + 0) * W + tid] = H0;
          C.pg[((1 * B + j) * 4 + 1) * W + tid] = H1;
          C.pg[((1 * B + j) * 4 + 2) * W + tid] = H2;
          C.pg[((1 * B + j) * 4 + 3) * W + tid] = H3;
        }
      }
    }
    if (want_grad) {
      // arm: grad_k = z_k . (sum_{link(s)>=k} a_s x g_s - o_k x sum g_s)   (trajopt.py:586-590)
      R Gs[3] = {R(0), R(0), R(0)}, Ms[3] = {R(0), R(0), R(0)};
      for (int k = J - 1; k >= 0; --k) {
        for (int s = ch.link_start[k]; s < ch.link_start[k + 1]; ++s) {
          const R a[3] = {C.armw[(3 * s) * W + tid], C.armw[(3 * s + 1) * W + tid], C.armw[(3 * s + 2) * W + tid]};
          const R gg[3] = {C.ga[(3 * s) * W + tid], C.ga[(3 * s + 1) * W + tid], C.ga[(3 * s + 2) * W + tid]};
          R m[3];
          cross3(a, gg, m);
          Gs[0] += gg[0];
          Gs[1] += gg[1];
          Gs[2] += gg[2];
          Ms[0] += m[0];
          Ms[1] += m[1];
          Ms[2] += m[2];
        }
        const R o[3] = {C.org[(3 * k) * W + tid], C.org[(3 * k + 1) * W + tid], C.org[(3 * k + 2) * W + tid]};
        const R z[3] = {C.axs[(3 * k) * W + tid], C.axs[(3 * k + 1) * W + tid], C.axs[(3 * k + 2) * W + tid]};
        R og[3];
        cross3(o, Gs, og);
        const R v = (z[0] * (Ms[0] - og[0]) + z[1] * (Ms[1] - og[1])) + z[2] * (Ms[2] - og[2]);
#pragma unroll
        for (int kk = 0; kk < kMaxJ; ++kk)
          if (kk == k) garm[kk] = v;
      }
      // held block: every joint moves it (trajopt.py:592-599)
      if (manip && t >= 1 && t <= T - 2) {
        R Gh[3] = {R(0), R(0), R(0)}, Mh[3] = {R(0), R(0), R(0)};
        const int nh = sc.blk_start[b + 1] - sc.blk_start[b];
        for (int s = 0; s < nh; ++s) {
          const R a[3] = {C.hp[(3 * s) * W + tid], C.hp[(3 * s + 1) * W + tid], C.hp[(3 * s + 2) * W + tid]};
          const R gg[3] = {C.gh[(3 * s) * W + tid], C.gh[(3 * s + 1) * W + tid], C.gh[(3 * s + 2) * W + tid]};
          R m[3];
          cross3(a, gg, m);
          Gh[0] += gg[0];
          Gh[1] += gg[1];
          Gh[2] += gg[2];
          Mh[0] += m[0];
          Mh[1] += m[1];
          Mh[2] += m[2];
        }
#pragma unroll
        for (int k = 0; k < kMaxJ; ++k) {
          if (k >= J) break;
          const R o[3] = {C.org[(3 * k) * W + tid], C.org[(3 * k + 1) * W + tid], C.org[(3 * k + 2) * W + tid]};
          const R z[3] = {C.axs[(3 * k) * W + tid], C.axs[(3 * k + 1) * W + tid], C.axs[(3 * k + 2) * W + tid]};
          R og[3];
          cross3(o, Gh, og);
          gblk[k] = (z[0] * (Mh[0] - og[0]) + z[1] * (Mh[1] - og[1])) + z[2] * (Mh[2] - og[2]);
        }
      }
    }
  }
  // warp partial sums of the scalars (fixed xor-tree order)
  if (!is_aux) {
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
  }
  __syncthreads();

  // ---------------- P4: totals, multiplier scales; aux reduces placed partials ----------
  if (tid == 0) {
    R o = R(0), ca = R(0), cb = R(0);
    for (int wi = 0; wi < C.L.NW / 32; ++wi) {
      o += C.red[4 * wi];
      ca += C.red[4 * wi + 1];
      cb += C.red[4 * wi + 2];
    }
    const R cpl = manip ? C.scal[kCplace] : R(0);
    const R c0 = R(prm.w_place) * cpl, c1 = R(prm.w_arm) * ca, c2 = R(prm.w_block) * cb;
    const R mu = C.scal[kMu];
    const R l0 = C.scal[kLam0], l1 = C.scal[kLam1], l2 = C.scal[kLam2];
    C.scal[kObj] = o;
    C.scal[kCarm] = ca;
    C.scal[kCblk] = cb;
    C.scal[kCons0] = c0;
    C.scal[kCons1] = c1;
    C.scal[kCons2] = c2;
    C.scal[kLag] = o + ((l0 * c0 + l1 * c1) + l2 * c2) + R(0.5) * mu * ((c0 * c0 + c1 * c1) + c2 * c2);
    C.scal[kSc0] = (l0 + mu * c0) * R(prm.w_place);
    C.scal[kSc1] = (l1 + mu * c1) * R(prm.w_arm);
    C.scal[kSc2] = (l2 + mu * c2) * R(prm.w_block);
  }
  if (want_grad && manip && is_aux) {
    for (int it = lane; it < 8 * B; it += 32) {
      R s = R(0);
      const int j = (it / 4) % B;
      // only waypoints of later segments contribute to block j
      for (int w = (j + 1) * T; w < W; ++w) s += C.pg[it * W + w];
      C.pgsum[it] = s;
    }
  }
  __syncthreads();

  // ---------------- P5: gradient assembly ------------------------------------------------
  if (want_grad && is_wp) {
    const R s_pl = C.scal[kSc0], s_arm = C.scal[kSc1], s_blk = C.scal[kSc2];
    R gq[kMaxJ];
#pragma unroll
    for (int k = 0; k < kMaxJ; ++k) {
      if (k >= J) break;
      R v = R(0);
      if (t < T - 1) v -= C.unit[k * W + tid];
      if (t >= 1) v += C.unit[k * W + tid - 1];
      v += s_arm * garm[k];
      v += s_blk * gblk[k];
      gq[k] = v;
    }
    if (manip && t == T - 1) {
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
#pragma unroll
      for (int k = 0; k < kMaxJ; ++k) {
        if (k >= J) break;
        const R* jl = C.jlf + (b * J + k) * 3;
        gq[k] += ((Gx + gp0) * jl[0] + (Gy + gp1) * jl[1]) + (Gz + gp2) * jl[2];
        gq[k] += (Gw + gyp) * C.yjf[b * J + k];
      }
    }
    if (manip && t == 0) {
      const R d0[3] = {ee[0] - sc.pick_pos[b][0], ee[1] - sc.pick_pos[b][1], ee[2] - sc.pick_pos[b][2]};
      const R ax0[3] = {Rm[2], Rm[5], Rm[8]};
      R cosd = -Rm[8];
      cosd = cosd < R(-1) ? R(-1) : (cosd > R(1) ? R(1) : cosd);
      const R th = Math<R>::acos_(cosd);
      const R dy0 = wrap_yaw(yaw_of(Rm) - sc.pick_yaw[b]);
      const R sth = Math<R>::sqrt_(fmax(R(1) - cosd * cosd, R(0)));
      const R fac = sth > R(1e-8) ? R(-2) * th / fmax(sth, R(1e-8)) : (cosd > R(0) ? R(-2) : R(0));
#pragma unroll
      for (int k = 0; k < kMaxJ; ++k) {
        if (k >= J) break;
        const R z[3] = {C.axs[(3 * k) * W + tid], C.axs[(3 * k + 1) * W + tid], C.axs[(3 * k + 2) * W + tid]};
        const R rel[3] = {ee[0] - C.org[(3 * k) * W + tid], ee[1] - C.org[(3 * k + 1) * W + tid],
                          ee[2] - C.org[(3 * k + 2) * W + tid]};
        R jl[3], dc[3];
        cross3(z, rel, jl);
        cross3(z, ax0, dc);
        gq[k] += w_start * R(2) * ((d0[0] * jl[0] + d0[1] * jl[1]) + d0[2] * jl[2]);
        gq[k] += w_start * fac * (-dc[2]);
        gq[k] += w_start * R(2) * dy0 * yaw_jac(Rm, z);
      }
    }
    for (int k = 0; k < J; ++k) C.g[k * W + tid] = gq[k];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
// validation of the CTA's particle (trajopt.py:1071-1153). Requires ctx.ee/rot/armw of the
// current x (computed by a preceding al_eval). Leaves the max violation in scal[kWorst].
// ---------------------------------------------------------------------------------------
template <typename R, int KIND, int SPB>
__device__ void al_validate(AlCtx<R>& C, const typename TwinSceneOf<R, KIND>::type& tw, const AlParams& prm) {
  const TrajScene<R>& sc = *C.sc;
  const ChainDesc<R>& ch = sc.ch;
  const int tid = threadIdx.x;
  const int W = C.L.W, J = ch.J, T = prm.T, B = sc.B, S = ch.S;
  const bool manip = sc.manip != 0;
  const bool is_wp = tid < W;
  const int lane = tid & 31;
  const bool is_aux = tid >= C.L.NW;
  const int b = is_wp ? tid / T : 0;
  const int t = is_wp ? tid - b * T : 0;
  // placed blocks from the final waypoints: inverse_grasp of the wrapped EE pose
  if (is_aux && manip && lane < B) {
    const int bb = lane, wf = bb * T + T - 1;
    R Rf[9], ef[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) Rf[i] = C.rot[i * W + wf];
#pragma unroll
    for (int i = 0; i < 3; ++i) ef[i] = C.ee[i * W + wf];
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
      C.pl[3 * q + 0] = (lx * c - ly * s) + px;
      C.pl[3 * q + 1] = (lx * s + ly * c) + py;
      C.pl[3 * q + 2] = lz + pz;
    }
  }
  __syncthreads();
  R worst = R(0);
  if (is_aux && lane == 0) {
    if (manip) {
      R place = twin_run<R, KIND, SPB>(tw, C.rows, nullptr, C.scr, false, false);
      if (sc.anchor)
        for (int bb = 0; bb < B; ++bb) place += fabs(wrap_yaw(C.rows[4 * bb + 3]));
      worst = fmax(worst, place);
    } else {
      for (int k = 0; k < J; ++k) {
        worst = fmax(worst, fabs(C.x[k * W + 0] - sc.start[k]));
        worst = fmax(worst, fabs(C.x[k * W + T - 1] - sc.goal[k]));
      }
    }
  } else if (is_wp) {
    for (int k = 0; k < J; ++k) {
      const R q = C.x[k * W + tid];
      worst = fmax(worst, fmax(q - ch.hi[k], ch.lo[k] - q));
    }
    const int f_blk0 = manip ? sc.blk_start[b + 1] : 0, f_blk1 = manip ? sc.n_blk : 0;
    const int p_end = manip ? sc.blk_start[b] : 0;  // placed spheres of blocks j < b
    const bool any_obs = (sc.n_static + (f_blk1 - f_blk0) + p_end) > 0;
    if (any_obs) {
      for (int s = 0; s < S; ++s) {
        const R ax = C.armw[(3 * s) * W + tid], ay = C.armw[(3 * s + 1) * W + tid], az = C.armw[(3 * s + 2) * W + tid];
        const R rs = ch.arm_r[s];
        for (int o = 0; o < sc.n_static; ++o) {
          const R dx = ax - sc.st_c[o][0], dy = ay - sc.st_c[o][1], dz = az - sc.st_c[o][2];
          worst = fmax(worst, (rs + sc.st_r[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
        }
        for (int o = f_blk0; o < f_blk1; ++o) {
          const R dx = ax - sc.staged[o][0], dy = ay - sc.staged[o][1], dz = az - sc.staged[o][2];
          worst = fmax(worst, (rs + sc.br[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
        }
        for (int o = 0; o < p_end; ++o) {
          const R dx = ax - C.pl[3 * o], dy = ay - C.pl[3 * o + 1], dz = az - C.pl[3 * o + 2];
          worst = fmax(worst, (rs + sc.br[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
        }
      }
      if (manip && t >= 1 && t <= T - 2) {
        R Rm[9], ee[3];
#pragma unroll
        for (int i = 0; i < 9; ++i) Rm[i] = C.rot[i * W + tid];
#pragma unroll
        for (int i = 0; i < 3; ++i) ee[i] = C.ee[i * W + tid];
        for (int q = sc.blk_start[b]; q < sc.blk_start[b + 1]; ++q) {
          const R ux = sc.bu[q][0], uy = sc.bu[q][1], uz = sc.bu[q][2];
          const R hx = ((Rm[0] * ux - Rm[1] * uy) - Rm[2] * uz) + ee[0];
          const R hy = ((Rm[3] * ux - Rm[4] * uy) - Rm[5] * uz) + ee[1];
          const R hz = ((Rm[6] * ux - Rm[7] * uy) - Rm[8] * uz) + ee[2];
          const R rh = sc.br[q];
          for (int o = 0; o < sc.n_static; ++o) {
            const R dx = hx - sc.st_c[o][0], dy = hy - sc.st_c[o][1], dz = hz - sc.st_c[o][2];
            worst = fmax(worst, (rh + sc.st_r[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
          }
          for (int o = f_blk0; o < f_blk1; ++o) {
            const R dx = hx - sc.staged[o][0], dy = hy - sc.staged[o][1], dz = hz - sc.staged[o][2];
            worst = fmax(worst, (rh + sc.br[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
          }
          for (int o = 0; o < p_end; ++o) {
            const R dx = hx - C.pl[3 * o], dy = hy - C.pl[3 * o + 1], dz = hz - C.pl[3 * o + 2];
            worst = fmax(worst, (rh + sc.br[o]) - Math<R>::sqrt_((dx * dx + dy * dy) + dz * dz));
          }
        }
      }
    }
    if (manip && t == 0) {
      R Rm[9];
#pragma unroll
      for (int i = 0; i < 9; ++i) Rm[i] = C.rot[i * W + tid];
      const R dx = C.ee[tid] - sc.pick_pos[b][0], dy = C.ee[W + tid] - sc.pick_pos[b][1],
              dz = C.ee[2 * W + tid] - sc.pick_pos[b][2];
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
    R w = R(0);
    for (int wi = 0; wi < C.L.nwarps; ++wi) w = fmax(w, C.red[4 * wi + 3]);
    C.scal[kWorst] = w;
  }
  __syncthreads();
}

// load the trajectory scene + particle p into shared memory (x in [k][w] columns)
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
  for (int i = tid; i < W * J; i += blockDim.x) {
    const int w = i / J, k = i - w * J;
    C.x[k * W + w] = v[i];
  }
  if (tid < 32) C.scal[tid] = R(0);
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
// k_al_eval: trajectory_cost / al_value_and_gradient for a batch (CTA per particle)
// ---------------------------------------------------------------------------------------
template <typename R, int KIND, int SPB>
__global__ void __launch_bounds__(kMaxAlThreads) k_al_eval(const TrajScene<R>* __restrict__ g_scene,
                                                  const typename TwinSceneOf<R, KIND>::type tw, AlLayout L,
                                                  AlParams prm, const R* __restrict__ values,
                                                  const R* __restrict__ lam, const R* __restrict__ mu, int mode,
                                                  int place_mode, int want_grad, R* __restrict__ obj,
                                                  R* __restrict__ cons, R* __restrict__ lag, R* __restrict__ grad) {
  extern __shared__ __align__(16) unsigned char smem[];
  AlCtx<R> C;
  C.bind(smem, L);
  const int64_t p = blockIdx.x;
  al_load(C, g_scene, values, p);
  if (threadIdx.x == 0) {
    C.scal[kLam0] = lam ? lam[3 * p] : R(0);
    C.scal[kLam1] = lam ? lam[3 * p + 1] : R(0);
    C.scal[kLam2] = lam ? lam[3 * p + 2] : R(0);
    C.scal[kMu] = mu ? mu[p] : R(0);
  }
  __syncthreads();
  al_eval<R, KIND, SPB>(C, tw, prm, mode == 1, place_mode == 1, want_grad != 0);
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
      gout[i] = C.g[k * W + w];
    }
  }
}

// k_validate: validate() for a batch of trajectories (CTA per trajectory)
template <typename R, int KIND, int SPB>
__global__ void __launch_bounds__(kMaxAlThreads) k_validate(const TrajScene<R>* __restrict__ g_scene,
                                                   const typename TwinSceneOf<R, KIND>::type tw, AlLayout L,
                                                   AlParams prm, const R* __restrict__ values,
                                                   uint8_t* __restrict__ feasible, R* __restrict__ violation) {
  extern __shared__ __align__(16) unsigned char smem[];
  AlCtx<R> C;
  C.bind(smem, L);
  const int64_t p = blockIdx.x;
  al_load(C, g_scene, values, p);
  al_eval<R, KIND, SPB>(C, tw, prm, false, false, false);  // FK tables for the current x
  al_validate<R, KIND, SPB>(C, tw, prm);
  if (threadIdx.x == 0) {
    const R w = C.scal[kWorst];
    violation[p] = w;
    feasible[p] = (uint8_t)(w < R(prm.eps));
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

template <typename R, int KIND, int SPB>
__global__ void __launch_bounds__(kMaxAlThreads) k_solve_al(const TrajScene<R>* __restrict__ g_scene,
                                                   const typename TwinSceneOf<R, KIND>::type tw, AlLayout L,
                                                   AlParams prm, const R* __restrict__ values, int P,
                                                   AlRecords rec) {
  extern __shared__ __align__(16) unsigned char smem[];
  AlCtx<R> C;
  C.bind(smem, L);
  const int p = blockIdx.x;
  if (rec.n_active && p >= *rec.n_active) return;
  al_load(C, g_scene, values, p);
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
  const R denom = R(prm.inner_steps - 1 > 1 ? prm.inner_steps - 1 : 1);
  int first = -1, done = 0;
  for (int outer = 0; outer < prm.outer_iters; ++outer) {
    if (tid == 0) C.flags[0] = (outer > *((volatile int*)rec.kstar)) ? 1 : 0;
    __syncthreads();
    if (C.flags[0]) break;
    for (int k = 0; k < prm.inner_steps; ++k) {
      const R lr = R(prm.lr_init) + (R(prm.lr_final) - R(prm.lr_init)) * (R(k) / denom);
      al_eval<R, KIND, SPB>(C, tw, prm, false, prm.place_mode == 1, true);
      if (tid < W) {
        for (int j = 0; j < J; ++j) {
          R st = lr * C.g[j * W + tid];
          st = st < R(-0.1) ? R(-0.1) : (st > R(0.1) ? R(0.1) : st);
          R v = C.x[j * W + tid] - st;
          v = v < ch.lo[j] ? ch.lo[j] : (v > ch.hi[j] ? ch.hi[j] : v);
          C.x[j * W + tid] = v;
        }
        if (!manip) {  // pinned endpoints (trajopt.py:1000-1002)
          if (tid == 0)
            for (int j = 0; j < J; ++j) C.x[j * W] = sc.start[j];
          if (tid == T - 1)
            for (int j = 0; j < J; ++j) C.x[j * W + T - 1] = sc.goal[j];
        }
      }
      __syncthreads();
    }
    // retract pick waypoints to the exact grasp (trajopt.py:1004-1007)
    if (manip && tid < sc.B) {
      R q[kMaxJ];
      const int w0 = tid * T;
      for (int j = 0; j < J; ++j) q[j] = C.x[j * W + w0];
      polish_thread<R>(ch, q, sc.pick_pos[tid], sc.pick_yaw[tid]);
      for (int j = 0; j < J; ++j) C.x[j * W + w0] = q[j];
    }
    __syncthreads();
    al_eval<R, KIND, SPB>(C, tw, prm, false, prm.place_mode == 1, false);
    al_validate<R, KIND, SPB>(C, tw, prm);
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
      R* bx = reinterpret_cast<R*>(rec.best_x) + (int64_t)p * W * J;
      for (int i = tid; i < W * J; i += blockDim.x) {
        const int w = i / J, k = i - w * J;
        bx[i] = C.x[k * W + w];
      }
      break;
    }
  }
  if (tid == 0) {
    rec.first_feas[p] = first;
    rec.n_outers[p] = done;
  }
}

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

// one warp per (draw, target) group; lane = restart
template <typename R>
__global__ void __launch_bounds__(128) k_ik_group(const TrajScene<R>* __restrict__ g_scene, int n_targets, int n_draws,
                                                  uint64_t seed, uint64_t draw_stride, int restarts, int max_iters,
                                                  double damping, const double* __restrict__ tpos_in,
                                                  const double* __restrict__ tyaw_in, const double* __restrict__ rows,
                                                  int D, int polish, int score_statics, IkOut out) {
  __shared__ ChainDesc<R> ch_s;
  const TrajScene<R>& sc = *g_scene;
  {
    const int4* src = reinterpret_cast<const int4*>(&sc.ch);
    int4* dst = reinterpret_cast<int4*>(&ch_s);
    for (int i = threadIdx.x; i < (int)(sizeof(ChainDesc<R>) / sizeof(int4)); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const ChainDesc<R>& ch = ch_s;
  const int lane = threadIdx.x & 31;
  const int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (grp >= n_targets * n_draws) return;
  const int a = grp / n_targets, t = grp - a * n_targets;
  const int J = ch.J;
  R tp[3], ty;
  if (tpos_in) {
    tp[0] = (R)tpos_in[3 * t];
    tp[1] = (R)tpos_in[3 * t + 1];
    tp[2] = (R)tpos_in[3 * t + 2];
    ty = (R)tyaw_in[t];
  } else {
    lift_target<R>(sc, rows, D, t, tp, &ty);
  }
  R q[kMaxJ];
  R key = R(INFINITY), score = R(0);
  bool ok = false;
  if (lane < restarts) {
    Pcg64 g;
    g.init(seedseq_pcg64_dev(seed + (uint64_t)a * draw_stride, (uint64_t)t));
    g.advance((uint64_t)lane * J);
    for (int j = 0; j < J; ++j) {
      const double lo = ch.lo64[j], hi = ch.hi64[j];
      q[j] = (R)(lo + (hi - lo) * g.next_double());
    }
    ok = ik_thread<R>(ch, q, tp, ty, max_iters, R(damping), &score);
    key = (ok ? R(0) : R(1e6)) + score;
  }
  // first minimum over restarts (np.argmin)
  R bk = key;
  int bl = lane;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const R ok2 = __shfl_xor_sync(0xffffffffu, bk, off);
    const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
    if (ok2 < bk || (ok2 == bk && ol < bl)) {
      bk = ok2;
      bl = ol;
    }
  }
  if (lane != bl) return;
  R* sol = reinterpret_cast<R*>(out.sol) + (int64_t)grp * J;
  bool pol = true;
  R pen = R(0);
  if (polish) {
    pol = polish_thread<R>(ch, q, tp, ty);
    if (score_statics && sc.n_static > 0) pen = arm_worst_pen<R>(ch, q, sc.st_c, sc.st_r, sc.n_static);
  }
  for (int j = 0; j < J; ++j) sol[j] = q[j];
  out.ik_ok[grp] = (uint8_t)ok;
  if (out.pol_ok) out.pol_ok[grp] = (uint8_t)pol;
  reinterpret_cast<R*>(out.score)[grp] = score;
  if (out.pen) reinterpret_cast<R*>(out.pen)[grp] = pen;
}

// polish a batch of configurations (the _polish_tool_down API), thread per row
template <typename R>
__global__ void k_polish(const TrajScene<R>* __restrict__ g_scene, int n, R* __restrict__ Q,
                         const double* __restrict__ tpos, const double* __restrict__ tyaw, uint8_t* __restrict__ ok) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const ChainDesc<R>& ch = g_scene->ch;
  const int J = ch.J;
  R q[kMaxJ];
  for (int j = 0; j < J; ++j) q[j] = Q[(int64_t)i * J + j];
  const R tp[3] = {(R)tpos[3 * i], (R)tpos[3 * i + 1], (R)tpos[3 * i + 2]};
  ok[i] = (uint8_t)polish_thread<R>(ch, q, tp, (R)tyaw[i]);
  for (int j = 0; j < J; ++j) Q[(int64_t)i * J + j] = q[j];
}

// lift_placements tail (trajopt.py:844-876): per target, replay the draws in order keeping
// the least-penetrating successful one; per particle, survive iff every placement lifted;
// stream-compact the survivors and assemble (pick, place) endpoints. One CTA.
// status[0] = first unreachable staged pose (-1 none), status[1] = kept count.
template <typename R>
__global__ void __launch_bounds__(1024) k_lift_combine(const R* __restrict__ sol, const uint8_t* __restrict__ ik_ok,
                                                       const uint8_t* __restrict__ pol_ok, const R* __restrict__ pen,
                                                       int n_targets, int n_draws, int J, int B, int P,
                                                       R* __restrict__ best, uint8_t* __restrict__ okt,
                                                       int32_t* __restrict__ kept, R* __restrict__ endpoints,
                                                       int32_t* __restrict__ status) {
  __shared__ int s_scan[1024];
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
      const int g = a * n_targets + t;
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
    return lo + (hi - lo) * g.next_double();
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
