// Host-side launchers for the stage-2 kernels, templated on R and instantiated once per
// precision (stage2_f32.cu / stage2_f64.cu).
#pragma once
#include "stage2_kernels.cuh"
#include "traj.hpp"

namespace spasm {
int ik_cluster_option();  // spasm_set_option("ik_cluster") (capi.cu)
}

namespace spasm {

// Calls f(std::integral_constant<int, KIND>{}, twin scene) for the handle's twin family.
template <typename R, class F>
inline int dispatch_twin(const Traj& tr, F&& f) {
  switch (tr.kind) {
    case kTwinTetris:
      return f(std::integral_constant<int, 1>{}, tr.twin->tetris<R>());
    case kTwinTower:
      return f(std::integral_constant<int, 2>{}, tr.twin->tower<R>());
    default:
      return f(std::integral_constant<int, 0>{}, NoTwin<R>{0});
  }
}

template <typename R>
inline int al_layout_for(const Traj& tr, int T, AlLayout* L) {
  *L = al_layout<R>(tr.B, T, tr.J, tr.S, tr.SB, tr.NB);
  SPASM_REQUIRE(T >= 2, "segments need at least two waypoints");
  SPASM_REQUIRE(L->nthreads <= kMaxAlThreads, "too many waypoints per particle (B*T must be <= 60)");
  SPASM_REQUIRE(tr.S + tr.SB <= kTile * kAlItems, "arm spheres + spheres of one block must be <= 24");
  SPASM_REQUIRE(L->total <= 227 * 1024, "trajectory particle does not fit in shared memory");
  return SPASM_OK;
}

template <typename R>
int launch_al_eval(const Traj& tr, const AlParams& prm, const R* values, int64_t P, const R* lam, const R* mu,
                   int mode, int pmode, int want_grad, R* obj, R* cons, R* lag, R* grad, cudaStream_t s) {
  if (P <= 0) return SPASM_OK;
  AlLayout L;
  int st = al_layout_for<R>(tr, prm.T, &L);
  if (st) return st;
  return dispatch_twin<R>(tr, [&](auto kind, const auto& tw) -> int {
    constexpr int K = decltype(kind)::value;
    auto kern = k_al_eval<R, K, 0>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
    kern<<<(unsigned)P, L.nthreads, L.total, s>>>(tr.dev<R>(), tw, L, prm, values, lam, mu, mode, pmode, want_grad,
                                                   obj, cons, lag, grad);
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  });
}

template <typename R>
int launch_validate(const Traj& tr, const AlParams& prm, const R* values, int64_t P, uint8_t* feas, R* viol,
                    cudaStream_t s) {
  if (P <= 0) return SPASM_OK;
  AlLayout L;
  int st = al_layout_for<R>(tr, prm.T, &L);
  if (st) return st;
  return dispatch_twin<R>(tr, [&](auto kind, const auto& tw) -> int {
    constexpr int K = decltype(kind)::value;
    auto kern = k_validate<R, K, 0>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
    kern<<<(unsigned)P, L.nthreads, L.total, s>>>(tr.dev<R>(), tw, L, prm, values, feas, viol);
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  });
}

// final selection of solve_al (trajopt.py:1042-1057): kstar = first outer with a
// feasible particle; among those particles the lowest objective (first index on ties);
// on failure the least violation over every recorded outer. One CTA.
template <typename R>
__global__ void __launch_bounds__(256) k_al_finalize(AlRecords rec, int P, int O, int WJ,
                                                     const int32_t* __restrict__ lift_status, R* __restrict__ best_out,
                                                     AlResultBlock* __restrict__ res) {
  __shared__ double s_v[256];
  __shared__ int s_i[256];
  __shared__ int s_best;
  const int tid = threadIdx.x;
  const int n_act = rec.n_active ? *rec.n_active : P;
  const int kstar = *rec.kstar;
  const R* obj = reinterpret_cast<const R*>(rec.obj);
  const R* viol = reinterpret_cast<const R*>(rec.viol);
  double bv = INFINITY;
  int bi = 0x7fffffff;
  const bool ok = kstar < O;
  for (int p = tid; p < n_act; p += blockDim.x) {
    if (ok) {
      if (rec.first_feas[p] == kstar) {
        const double v = (double)obj[(int64_t)kstar * P + p];
        if (v < bv || (v == bv && p < bi)) {
          bv = v;
          bi = p;
        }
      }
    } else {
      for (int o = 0; o < rec.n_outers[p]; ++o) bv = fmin(bv, (double)viol[(int64_t)o * P + p]);
    }
  }
  s_v[tid] = bv;
  s_i[tid] = bi;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (tid < off) {
      const double v2 = s_v[tid + off];
      const int i2 = s_i[tid + off];
      if (v2 < s_v[tid] || (v2 == s_v[tid] && i2 < s_i[tid])) {
        s_v[tid] = v2;
        s_i[tid] = i2;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    AlResultBlock r;
    r.n_active = n_act;
    r.lift_pick_fail = lift_status ? lift_status[0] : -1;
    r.kstar = ok ? kstar : -1;
    r.best_p = ok ? s_i[0] : -1;
    r.n_outers = ok ? kstar + 1 : O;
    r.objective = ok ? s_v[0] : INFINITY;
    r.least_violation = ok ? 0.0 : s_v[0];
    r.status = (r.lift_pick_fail >= 0 || n_act == 0) ? SPASM_LIFT_FAILURE : (ok ? SPASM_OK : SPASM_AL_FAILURE);
    *res = r;
    s_best = r.best_p;
  }
  __syncthreads();
  if (s_best >= 0 && best_out) {
    const R* bx = reinterpret_cast<const R*>(rec.best_x) + (int64_t)s_best * WJ;
    for (int i = tid; i < WJ; i += blockDim.x) best_out[i] = bx[i];
  }
}

template <typename R>
int launch_solve_al(const Traj& tr, const AlParams& prm, const R* values, int64_t P, AlRecords rec,
                    const int32_t* lift_status, R* best_out, AlResultBlock* res_dev, cudaStream_t s) {
  AlLayout L;
  int st = al_layout_for<R>(tr, prm.T, &L);
  if (st) return st;
  SPASM_CUDA_TRY(cudaMemsetAsync(rec.kstar, 0x7f, sizeof(int), s));
  if (P > 0) {
    st = dispatch_twin<R>(tr, [&](auto kind, const auto& tw) -> int {
      constexpr int K = decltype(kind)::value;
      auto kern = k_solve_al<R, K, 0>;
      if constexpr (sizeof(R) == 4) {
        if (L.nthreads <= 256) kern = k_solve_al<R, K, 0, 256>;  // room for more registers per thread
      }
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
      kern<<<(unsigned)P, L.nthreads, L.total, s>>>(tr.dev<R>(), tw, L, prm, values, (int)P, rec);
      SPASM_CHECK_LAUNCH();
      return SPASM_OK;
    });
    if (st) return st;
  }
  k_al_finalize<R><<<1, 256, 0, s>>>(rec, (int)P, prm.outer_iters, L.W * L.J, lift_status, best_out, res_dev);
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

template <typename R>
int launch_ik(const Traj& tr, int n_targets, int n_draws, uint64_t seed, uint64_t stride, int restarts, int max_iters,
              double damping, const double* tpos, const double* tyaw, const double* rows, int D, int polish,
              int score_statics, IkOut out, cudaStream_t s, const int32_t* n_rows) {
  if (n_targets <= 0) return SPASM_OK;
  SPASM_REQUIRE(restarts >= 1 && restarts <= 32, "restarts must be in [1, 32]");
  const int64_t groups = (int64_t)n_targets * n_draws;
  // cluster size: spread each group's restart warps over CS CTAs (k_ik_group) so that the
  // busiest SM carries the fewest restart warps, assuming the CTAs spread evenly over the
  // SMs (CS in {1, 2, 4, 8}, the largest on ties: more SMs share the same worst load)
  int cs = 1;
  int64_t best_load = INT64_MAX;
  for (int c = 1; c <= 8; c *= 2) {
    const int rpc = (restarts + c - 1) / c;
    if (c > restarts || groups * c > (int64_t)1 << 30) break;
    const int64_t load = ((groups * c + kNumSMs - 1) / kNumSMs) * rpc;
    if (load <= best_load) {
      best_load = load;
      cs = c;
    }
  }
  if (ik_cluster_option() > 0) cs = ik_cluster_option() < restarts ? ik_cluster_option() : restarts;
  const int rpc = (restarts + cs - 1) / cs;
  const int bs = rpc * 32;  // one warp per restart tile
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(groups * cs));
  cfg.blockDim = dim3((unsigned)bs);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // the 512-thread bound (128 registers) whenever a CTA holds at most 16 restarts and the
  // CTAs fit the register file side by side; else the 1024-thread bound (64 registers)
  const bool narrow = bs <= 512 && (bs <= 256 || groups * cs <= kNumSMs);
  if (narrow)
    SPASM_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_ik_group<R, 512>, tr.dev<R>(), n_targets, n_draws, seed, stride, restarts,
                                      max_iters, damping, tpos, tyaw, rows, D, polish, score_statics, out, n_rows, rpc));
  else
    SPASM_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_ik_group<R, 1024>, tr.dev<R>(), n_targets, n_draws, seed, stride, restarts,
                                      max_iters, damping, tpos, tyaw, rows, D, polish, score_statics, out, n_rows, rpc));
  return SPASM_OK;
}

template <typename R>
int launch_polish(const Traj& tr, R* Q, const double* tpos, const double* tyaw, int64_t n, uint8_t* ok,
                  cudaStream_t s) {
  if (n <= 0) return SPASM_OK;
  k_polish<R><<<ceil_div(n * kTile, 64), 64, 0, s>>>(tr.dev<R>(), (int)n, Q, tpos, tyaw, ok);
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

template <typename R>
int launch_lift_combine(const R* sol, const uint8_t* ik_ok, const uint8_t* pol_ok, const R* pen, int n_targets,
                        int n_draws, int J, int B, int P, R* best, uint8_t* okt, int32_t* kept, R* endpoints,
                        int32_t* status, cudaStream_t s, const int32_t* n_rows) {
  k_lift_combine<R><<<1, 1024, 0, s>>>(sol, ik_ok, pol_ok, pen, n_targets, n_draws, J, B, P, best, okt, kept,
                                       endpoints, status, n_rows);
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

template <typename R>
int launch_init_traj(const Traj& tr, const R* endpoints, int64_t P, int B, const int32_t* n_active, int K, int n_interp,
                     const Pcg64State& st, R* out, cudaStream_t s) {
  const int T = n_interp * (K + 1) + 1;
  const int64_t total = P * B * T * tr.J;
  if (total <= 0) return SPASM_OK;
  k_init_traj<R><<<ceil_div(total, 256), 256, 0, s>>>(tr.dev<R>(), endpoints, (int)P, n_active, B, K, n_interp, st,
                                                      out);
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

template <typename R>
int launch_fk(const Traj& tr, const R* Q, int64_t n, R* ee, R* rot, R* org, R* axs, R* yj, cudaStream_t s) {
  if (n <= 0) return SPASM_OK;
  k_fk<R><<<ceil_div(n, 128), 128, 0, s>>>(tr.dev<R>(), Q, (int)n, ee, rot, org, axs, yj);
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

}  // namespace spasm
