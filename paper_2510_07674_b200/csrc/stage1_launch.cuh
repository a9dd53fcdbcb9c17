// Host-side launchers for the stage-1 kernels, templated on R and instantiated once
// per precision (stage1_f32.cu / stage1_f64.cu) so each precision gets its own
// compiler flags (fp64 is built with -fmad=false to keep numpy's rounding per op).
#pragma once
#include <type_traits>
#include "model.hpp"
#include "sort.cuh"
#include "stage1_kernels.cuh"

namespace spasm {

// Device-resident restart inputs for the sampler kernels while a stage-1 restart is being
// captured as a CUDA graph (capi.cu); nullptr otherwise.
const RestartParams* restart_override();

// Stage-1 tile-kernel switch (spasm_set_option("stage1_tile", v)): -1 auto, 0 generic
// kernel only, 1..4 force a tile variant (stage1tile_f32.cu).
int stage1_tile_mode();
int tower_lanes_option();
// fp32 tetris tile schedule (stage1tile_f32.cu); returns -1 when not applicable.
int launch_schedule_tile(const Model& m, const float* src, const uint32_t* rows, int64_t M, int k_lin, int k_quad,
                         double eta, double alpha, float* out_values, float* out_cost, uint8_t* flagged,
                         unsigned int* flagged_count, cudaStream_t s);

// fp32 tower tile schedule (stage1towertile_f32.cu); returns -1 when not applicable.
int launch_schedule_tower_tile(const Model& m, const float* src, const uint32_t* rows, int64_t M, int k_lin,
                               int k_quad, double eta, double alpha, float* out_values, float* out_cost,
                               uint8_t* flagged, unsigned int* flagged_count, cudaStream_t s);

// fp32 tetris tile sample + evaluate (stage1tile_f32.cu); returns -1 when not applicable.
int launch_sample_eval_tile(const Model& m, const Pcg64State& st, int64_t row_offset, int64_t rows_n,
                            const double* warm, int64_t n_warm, int use_philox, uint64_t seed, uint32_t restart,
                            float* values, uint32_t* keys, uint32_t* idx, cudaStream_t s);

inline int pick_block(int64_t P, size_t per_thread_bytes) {
  int bs = 128;
  if (P < (int64_t)kNumSMs * 128 * 2) bs = 64;
  if (P < (int64_t)kNumSMs * 64 * 2) bs = 32;
  while (bs > 32 && per_thread_bytes * bs > 200 * 1024) bs >>= 1;
  return bs;
}

template <typename Kern>
inline void allow_big_smem(Kern kernel) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

// Calls f(E{}, scene) with the compile-time specialisation matching the model.
template <typename R, class F>
inline int dispatch_model(const Model& m, F&& f) {
  if (m.kind == ModelKind::Tetris) {
    const TetrisScene<R>& sc = m.tetris<R>();
    if (sc.free_yaw) {
      switch (sc.spb) {
        case 1: return f(TetrisEval<R, 1, true>{}, sc);
        case 2: return f(TetrisEval<R, 2, true>{}, sc);
        case 4: return f(TetrisEval<R, 4, true>{}, sc);
        default: return f(TetrisEval<R, 0, true>{}, sc);
      }
    }
    switch (sc.spb) {
      case 1: return f(TetrisEval<R, 1, false>{}, sc);
      case 2: return f(TetrisEval<R, 2, false>{}, sc);
      case 4: return f(TetrisEval<R, 4, false>{}, sc);
      default: return f(TetrisEval<R, 0, false>{}, sc);
    }
  }
  const TowerScene<R>& sc = m.tower<R>();
  if (sc.free_yaw) return f(TowerEval<R, true>{}, sc);
  return f(TowerEval<R, false>{}, sc);
}

template <typename R>
int launch_evaluate(const Model& m, const R* values, int64_t P, int quad, R* costs, cudaStream_t s) {
  if (P <= 0) return SPASM_OK;
  return dispatch_model<R>(m, [&](auto e, const auto& sc) -> int {
    using E = decltype(e);
    const size_t per = (size_t)(sc.dim + E::scratch_per_thread(sc)) * sizeof(R);
    const int bs = pick_block(P, per);
    const size_t smem = per * bs;
    if (quad) {
      allow_big_smem(k_evaluate<E, R, true>);
      k_evaluate<E, R, true><<<ceil_div(P, bs), bs, smem, s>>>(sc, values, P, costs);
    } else {
      allow_big_smem(k_evaluate<E, R, false>);
      k_evaluate<E, R, false><<<ceil_div(P, bs), bs, smem, s>>>(sc, values, P, costs);
    }
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  });
}

template <typename R>
int launch_gradient(const Model& m, const R* values, int64_t P, int quad, R* grad, cudaStream_t s) {
  if (P <= 0) return SPASM_OK;
  return dispatch_model<R>(m, [&](auto e, const auto& sc) -> int {
    using E = decltype(e);
    const size_t per = (size_t)(2 * sc.dim + E::scratch_per_thread(sc)) * sizeof(R);
    const int bs = pick_block(P, per);
    const size_t smem = per * bs;
    if (quad) {
      allow_big_smem(k_gradient<E, R, true>);
      k_gradient<E, R, true><<<ceil_div(P, bs), bs, smem, s>>>(sc, values, P, grad);
    } else {
      allow_big_smem(k_gradient<E, R, false>);
      k_gradient<E, R, false><<<ceil_div(P, bs), bs, smem, s>>>(sc, values, P, grad);
    }
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  });
}

template <typename R>
int launch_sample_eval(const Model& m, const Pcg64State& st, int64_t row_offset, int64_t N, const double* warm,
                       int64_t n_warm, int use_philox, uint64_t seed, uint32_t restart, R* values,
                       typename KeyOf<R>::type* keys, uint32_t* idx, cudaStream_t s) {
  if (N <= 0) return SPASM_OK;
  if constexpr (std::is_same<R, float>::value) {
    const int r = launch_sample_eval_tile(m, st, row_offset, N, warm, n_warm, use_philox, seed, restart, values, keys,
                                          idx, s);
    if (r != -1) return r;
  }
  return dispatch_model<R>(m, [&](auto e, const auto& sc) -> int {
    using E = decltype(e);
    const size_t per = (size_t)(sc.dim + E::scratch_per_thread(sc)) * sizeof(R);
    const int bs = pick_block(N, per);
    allow_big_smem(k_sample_eval<E, R>);
    k_sample_eval<E, R><<<ceil_div(N, bs), bs, per * bs, s>>>(sc, m.bounds, st, row_offset, N, warm, n_warm,
                                                            use_philox, seed, restart, values, keys, idx,
                                                            restart_override());
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  });
}

template <typename R>
int launch_schedule(const Model& m, const R* src, const uint32_t* rows, int64_t M, int k_lin, int k_quad,
                    double eta, double alpha, double eps, R* out_values, R* out_cost, uint8_t* flagged,
                    unsigned int* flagged_count, R* trace_cost, uint8_t* trace_sat, int n_traced,
                    const StepRule& rule, cudaStream_t s) {
  if (M <= 0) return SPASM_OK;
  if constexpr (std::is_same<R, float>::value) {
    if (trace_cost == nullptr && rule.is_reference()) {
      int r = launch_schedule_tile(m, src, rows, M, k_lin, k_quad, eta, alpha, out_values, out_cost, flagged,
                                   flagged_count, s);
      if (r != -1) return r;
      r = launch_schedule_tower_tile(m, src, rows, M, k_lin, k_quad, eta, alpha, out_values, out_cost, flagged,
                                     flagged_count, s);
      if (r != -1) return r;
    }
  }
  return dispatch_model<R>(m, [&](auto e, const auto& sc) -> int {
    using E = decltype(e);
    const size_t per = (size_t)((rule.adam ? 4 : 2) * sc.dim + E::scratch_per_thread(sc)) * sizeof(R);
    const int bs = pick_block(M, per);
    const size_t smem = per * bs;
    if (trace_cost != nullptr && n_traced > 0) {
      allow_big_smem(k_schedule<E, R, true>);
      k_schedule<E, R, true><<<ceil_div(M, bs), bs, smem, s>>>(sc, src, rows, M, k_lin, k_quad, eta, alpha, eps,
                                                               out_values, out_cost, flagged, flagged_count,
                                                               trace_cost, trace_sat, n_traced, rule);
    } else {
      allow_big_smem(k_schedule<E, R, false>);
      k_schedule<E, R, false><<<ceil_div(M, bs), bs, smem, s>>>(sc, src, rows, M, k_lin, k_quad, eta, alpha, eps,
                                                                out_values, out_cost, flagged, flagged_count,
                                                                nullptr, nullptr, 0, rule);
    }
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  });
}

template <typename R>
int launch_sample(const Bounds64& bd, int D, const Pcg64State& st, int64_t row_offset, const uint32_t* rows, int64_t N,
                  const double* warm, int64_t n_warm, int use_philox, uint64_t seed, uint32_t restart, R* values,
                  cudaStream_t s) {
  if (N <= 0) return SPASM_OK;
  const size_t per = (size_t)D * sizeof(R);
  const int bs = pick_block(N, per);
  allow_big_smem(k_sample<R>);
  k_sample<R><<<ceil_div(N, bs), bs, per * bs, s>>>(bd, st, row_offset, rows, N, D, warm, n_warm, use_philox, seed,
                                                    restart, values, restart_override());
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

template <typename R>
int launch_step(R* values, const R* grad, int64_t P, int D, R rate, const R* lower, const R* upper, uint8_t* flagged,
                cudaStream_t s) {
  if (P <= 0) return SPASM_OK;
  k_step<R><<<ceil_div(P, 128), 128, 0, s>>>(values, grad, P, D, rate, lower, upper, flagged);
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

template <typename R>
int launch_sort(typename KeyOf<R>::type* k0, uint32_t* v0, typename KeyOf<R>::type* k1, uint32_t* v1, int64_t n,
                unsigned int* hist, bool* in1, cudaStream_t s) {
  cudaError_t e = radix_sort_pairs<typename KeyOf<R>::type>(k0, v0, k1, v1, n, 8 * (int)sizeof(R), hist, in1, s);
  if (e != cudaSuccess) {
    set_last_error(std::string("radix sort: ") + cudaGetErrorString(e));
    return SPASM_ERR_CUDA;
  }
  return SPASM_OK;
}

// Build ordering keys for the satisfying-particle extraction: rows whose cost is not
// below eps get the maximal key so they sort last; counts the satisfying rows.
template <typename R>
__global__ void k_sat_keys(const R* __restrict__ cost, int64_t M, double eps, typename KeyOf<R>::type* __restrict__ keys,
                           uint32_t* __restrict__ vals, unsigned int* __restrict__ n_sat) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= M) return;
  const R c = cost[p];
  const bool sat = (double)c < eps;
  keys[p] = sat ? order_key(c) : (typename KeyOf<R>::type)(~(typename KeyOf<R>::type)0);
  vals[p] = (uint32_t)p;
  if (sat) atomicAdd(n_sat, 1u);
}

template <typename R>
int launch_sat_keys(const R* cost, int64_t M, double eps, typename KeyOf<R>::type* keys, uint32_t* vals,
                    unsigned int* n_sat, cudaStream_t s) {
  if (M <= 0) return SPASM_OK;
  k_sat_keys<R><<<ceil_div(M, 256), 256, 0, s>>>(cost, M, eps, keys, vals, n_sat);
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

}  // namespace spasm
