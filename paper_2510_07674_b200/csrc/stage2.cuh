// Stage-2 (trajectory) device tables and per-thread kinematics routines.
//
//   ChainDesc   KinematicChain + flattened link-sphere table     (robot.py:29-68, trajopt.py:311-321)
//   TrajScene   _Geometry of one problem                           (trajopt.py:235-367)
//   fk_eval     forward kinematics: translate, then rotate about the body axis
//               (robot.py:71-84, 120-180)
//   yaw_jac     exact d(tool yaw)/dq                               (robot.py:194-224)
//   chol_solve  SPD solve for the 4x4 / 5x5 damped least-squares systems (robot.py:283,
//               trajopt.py:759; numpy uses LU, both are exact to rounding for SPD A)
//   (the IK / polish iterations themselves are tile-cooperative: coop.cuh)
#pragma once
#include "rng.cuh"
#include "scene.cuh"

namespace spasm {

constexpr int kMaxJ = 8;          // joints
constexpr int kMaxArmS = 16;      // arm spheres
constexpr int kMaxSeg = 8;        // segments (= blocks)
constexpr int kMaxBlkS = 64;      // block spheres over all blocks
constexpr int kMaxStat2 = 128;    // static obstacle spheres
constexpr int kIkRestarts = 16;   // ik_solve_batch default restarts (robot.py:230)
constexpr double kIkPosTol = 1e-4, kIkYawTol = 1e-3, kIkDamping = 1e-3;  // robot.py:22-24
constexpr int kPolishMaxIters = 1000;                                     // trajopt.py:100
constexpr int kObsGroup = 4;                                               // obstacle pairs per pass iteration
constexpr int kObsPairs = ((128 + 64) / 2 + kObsGroup - 1) / kObsGroup * kObsGroup;  // statics + staged, padded

template <typename R>
struct alignas(16) ChainDesc {
  int J;                          // dof
  int S;                          // arm spheres, sorted by link
  int link_start[kMaxJ + 1];      // arm sphere range per link
  int full_circle[kMaxJ];         // (upper - lower) >= 2 pi - 1e-9 (trajopt.py:736)
  R axis[kMaxJ][3];
  R offset[kMaxJ][3];
  R lo[kMaxJ], hi[kMaxJ];
  double lo64[kMaxJ], hi64[kMaxJ];  // float64 limits for the bit-exact seed draws
  R tool_t[3];
  R tool_R[9];
  R arm_local[kMaxArmS][3];
  R arm_r[kMaxArmS];
};

template <typename R>
struct alignas(16) TrajScene {
  ChainDesc<R> ch;
  int manip;                      // manipulation (1) or point-to-point motion (0)
  int B;                          // segments
  int anchor;                     // fixed-yaw problem: pull placed yaws to 0
  int n_static;
  int n_blk;                      // block spheres in total
  int free_rows;                  // stage-1 placement rows carry yaw (x,y,z,yaw) per block
  int blk_start[kMaxSeg + 1];     // block sphere ranges (skeleton order)
  R grasp_off[3];
  R grasp_yaw;
  R bu[kMaxBlkS][3];              // block sphere centre relative to the grasp point (u = local - offset)
  R br[kMaxBlkS];
  R staged[kMaxBlkS][3];          // block spheres at their staged (initial) poses
  R st_c[kMaxStat2][3];
  R st_r[kMaxStat2];
  // packed copies (x, y, z, radius) of st_c / st_r and staged / br for the fp32 hot loops:
  // one 16-byte shared-memory load per obstacle instead of four
  alignas(16) R st4[kMaxStat2][4];
  alignas(16) R staged4[kMaxBlkS][4];
  // fp32 fixed-obstacle lists per segment b (the statics, then the staged spheres of blocks
  // > b), two by two in packed-pair order (x0 x1 y0 y1 z0 z1 r0 r1) so two 16-byte loads
  // give the f32x2 operands of a pair, padded with far dummies (inactive) to whole groups of
  // kObsGroup pairs: the pass then runs kObsGroup independent pair chains per iteration
  alignas(16) R obsp[sizeof(R) == 4 ? kMaxSeg : 1][kObsPairs][8];
  int obs_np[kMaxSeg];            // pairs in obsp[b], a multiple of kObsGroup
  R pick_pos[kMaxSeg][3];         // grasp targets over the staged poses
  R pick_yaw[kMaxSeg];
  double pick_pos64[kMaxSeg][3];
  double pick_yaw64[kMaxSeg];
  R start[kMaxJ], goal[kMaxJ];    // motion endpoints
};

// TrajOptConfig (trajopt.py:118-177) + solve_al knobs, POD for the kernels
struct AlParams {
  double w_start, w_arm, w_block, w_place;
  double mu0, beta, lr_init, lr_final, eps;
  int outer_iters, inner_steps;
  int place_mode;                 // placement-term mode inside solve_al (variant B: LINEAR)
  int T;                          // waypoints per segment
};

// ---------------------------------------------------------------------------
template <typename R>
__host__ __device__ __forceinline__ void mat3_mul(const R* a, const R* b, R* c) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) c[3 * i + k] = (a[3 * i] * b[k] + a[3 * i + 1] * b[3 + k]) + a[3 * i + 2] * b[6 + k];
}

template <typename R>
__host__ __device__ __forceinline__ void mat3_vec(const R* a, const R* v, R* out) {
#pragma unroll
  for (int i = 0; i < 3; ++i) out[i] = (a[3 * i] * v[0] + a[3 * i + 1] * v[1]) + a[3 * i + 2] * v[2];
}

template <typename R>
__device__ __forceinline__ void rodrigues(const R* ax, R q, R* M) {
  R s, c;
  Math<R>::sincos_(q, &s, &c);
  const R oc = R(1) - c;
  const R K[9] = {R(0), -ax[2], ax[1], ax[2], R(0), -ax[0], -ax[1], ax[0], R(0)};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) M[3 * i + k] = (c * (i == k ? R(1) : R(0)) + s * K[3 * i + k]) + oc * (ax[i] * ax[k]);
}

// Full FK of one configuration q[j * qs]. Optional outputs (nullptr = skip), all with
// element stride `os`: joint origins/axes (J x 3) and arm sphere centres (S x 3).
// Returns end-effector position and rotation in registers.
template <typename R>
__device__ __forceinline__ void fk_eval(const ChainDesc<R>& ch, const R* q, int qs, R* org, R* axs, R* armw, int os,
                                        R ee[3], R Ree[9]) {
  R p[3] = {R(0), R(0), R(0)};
  R M[9] = {R(1), R(0), R(0), R(0), R(1), R(0), R(0), R(0), R(1)};
  for (int j = 0; j < ch.J; ++j) {
    R t[3];
    mat3_vec(M, ch.offset[j], t);
    p[0] += t[0];
    p[1] += t[1];
    p[2] += t[2];
    if (axs) {
      mat3_vec(M, ch.axis[j], t);
      axs[(3 * j) * os] = t[0];
      axs[(3 * j + 1) * os] = t[1];
      axs[(3 * j + 2) * os] = t[2];
    }
    if (org) {
      org[(3 * j) * os] = p[0];
      org[(3 * j + 1) * os] = p[1];
      org[(3 * j + 2) * os] = p[2];
    }
    R Rj[9], N[9];
    rodrigues(ch.axis[j], q[j * qs], Rj);
    mat3_mul(M, Rj, N);
#pragma unroll
    for (int k = 0; k < 9; ++k) M[k] = N[k];
    if (armw) {
      for (int s = ch.link_start[j]; s < ch.link_start[j + 1]; ++s) {
        mat3_vec(M, ch.arm_local[s], t);
        armw[(3 * s) * os] = t[0] + p[0];
        armw[(3 * s + 1) * os] = t[1] + p[1];
        armw[(3 * s + 2) * os] = t[2] + p[2];
      }
    }
  }
  R t[3];
  mat3_vec(M, ch.tool_t, t);
  ee[0] = p[0] + t[0];
  ee[1] = p[1] + t[1];
  ee[2] = p[2] + t[2];
  mat3_mul(M, ch.tool_R, Ree);
}

template <typename R>
__device__ __forceinline__ R yaw_of(const R* Rm) {
  return Math<R>::atan2_(Rm[3], Rm[0]);
}

// normalize_yaw pieces: x = a + pi in (-2m, 2m) (m = 2 pi; every yaw difference here) is
// the fast range, where fmod(x, m) is x, x - m or x + m, each exact (Sterbenz), so the fold
// gives fmod's bits without its loop (fmod(-m, m) = -0 vs +0 here: both fail the w < 0
// test of the finish, same result)
template <typename R>
__device__ __forceinline__ bool wrap_yaw_in_fast_range(R a) {
  const R two_pi = R(6.283185307179586476925286766559);
  const R x = a + R(3.1415926535897932384626433832795);
  return x > -R(2) * two_pi && x < R(2) * two_pi;
}
template <typename R>
__device__ __forceinline__ R wrap_yaw_fold(R x) {
  const R two_pi = R(6.283185307179586476925286766559);
  return x >= two_pi ? x - two_pi : (x <= -two_pi ? x + two_pi : x);
}
template <typename R>
__device__ __forceinline__ R wrap_yaw_finish(R w) {
  const R two_pi = R(6.283185307179586476925286766559);
  const R pi = R(3.1415926535897932384626433832795);
  w = w < R(0) ? w + two_pi : w;
  w -= pi;
  return w <= -pi ? w + two_pi : w;
}

// normalize_yaw: wrap into (-pi, pi] (geometry.py:31-38; numpy remainder semantics)
template <typename R>
__device__ __forceinline__ R wrap_yaw(R a) {
  const R two_pi = R(6.283185307179586476925286766559);
  const R pi = R(3.1415926535897932384626433832795);
  const R x = a + pi;
  R w = wrap_yaw_in_fast_range(a) ? wrap_yaw_fold(x) : fmod(x, two_pi);
  return wrap_yaw_finish(w);
}

// np.mod(a, m) for m > 0 (npy_divmod: result carries the divisor's sign)
// a in [-m, 2m) (a clamped joint plus a step <= 0.5 rad) is the fast range: fmod is a - m
// or a, and a - m is exact there (Sterbenz), so the fold gives fmod's bits without its loop
template <typename R>
__device__ __forceinline__ bool np_mod_in_fast_range(R a, R m) {
  return a >= -m && a < R(2) * m;
}
template <typename R>
__device__ __forceinline__ R np_mod_finish(R r, R m) {
  return r != R(0) ? (r < R(0) ? r + m : r) : R(0);
}
template <typename R>
__device__ __forceinline__ R np_mod_pos(R a, R m) {
  const R r = np_mod_in_fast_range(a, m) ? (a >= m ? a - m : a) : fmod(a, m);
  return np_mod_finish(r, m);
}

// d yaw / d q_j from dR/dq_j = [z_j]x R; 0 near gimbal (den < 1e-12)
template <typename R>
__device__ __forceinline__ R yaw_jac(const R* Rm, const R* z) {
  const R r00 = Rm[0], r10 = Rm[3], r20 = Rm[6];
  const R den = r00 * r00 + r10 * r10;
  // dcol0 = z x col0
  const R dx = z[1] * r20 - z[2] * r10;
  const R dy = z[2] * r00 - z[0] * r20;
  const R v = (r00 * dy - r10 * dx) / den;
  return den < R(1e-12) ? R(0) : v;  // a select: no branch in the DLS loops
}

template <typename R>
__device__ __forceinline__ void cross3(const R* a, const R* b, R* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

// Solve (A) y = e for SPD A (N x N, row-major) by Cholesky in registers.
template <typename R, int N>
__device__ __forceinline__ void chol_solve(R* A, const R* e, R* y) {
  if constexpr (sizeof(R) == 4) {
    // fp32 (perf path): one MUFU.RSQ per pivot, multiplications instead of divisions
    R inv[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R d = A[j * N + j];
#pragma unroll
      for (int k = 0; k < j; ++k) d -= A[j * N + k] * A[j * N + k];
      inv[j] = rsqrtf(d);
#pragma unroll
      for (int i = j + 1; i < N; ++i) {
        R s = A[i * N + j];
#pragma unroll
        for (int k = 0; k < j; ++k) s -= A[i * N + k] * A[j * N + k];
        A[i * N + j] = s * inv[j];
      }
    }
    R z[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = e[i];
#pragma unroll
      for (int k = 0; k < i; ++k) s -= A[i * N + k] * z[k];
      z[i] = s * inv[i];
    }
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
      R s = z[i];
#pragma unroll
      for (int k = i + 1; k < N; ++k) s -= A[k * N + i] * y[k];
      y[i] = s * inv[i];
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R d = A[j * N + j];
#pragma unroll
      for (int k = 0; k < j; ++k) d -= A[j * N + k] * A[j * N + k];
      d = Math<R>::sqrt_(d);
      A[j * N + j] = d;
#pragma unroll
      for (int i = j + 1; i < N; ++i) {
        R s = A[i * N + j];
#pragma unroll
        for (int k = 0; k < j; ++k) s -= A[i * N + k] * A[j * N + k];
        A[i * N + j] = s / d;
      }
    }
    R z[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = e[i];
#pragma unroll
      for (int k = 0; k < i; ++k) s -= A[i * N + k] * z[k];
      z[i] = s / A[i * N + i];
    }
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
      R s = z[i];
#pragma unroll
      for (int k = i + 1; k < N; ++k) s -= A[k * N + i] * y[k];
      y[i] = s / A[i * N + i];
    }
  }
}

// FK returning origins/axes in registers (J <= kMaxJ), for the IK / polish lanes
template <typename R>
__device__ __forceinline__ void fk_frames(const ChainDesc<R>& ch, const R* q, R (&org)[kMaxJ][3], R (&axs)[kMaxJ][3],
                                          R ee[3], R Ree[9]) {
  fk_eval<R>(ch, q, 1, &org[0][0], &axs[0][0], nullptr, 1, ee, Ree);
}

}  // namespace spasm
