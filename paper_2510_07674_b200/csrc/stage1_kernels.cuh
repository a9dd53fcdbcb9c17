// Stage-1 kernels (templated on the cost model E and the arithmetic type R).
//
//   k_evaluate     CostModel.evaluate         (particle_opt.py:52-53)
//   k_gradient     CostModel.gradient         (particle_opt.py:55-56)
//   k_sample_eval  restart_stream + sample_uniform + inject_warm_start + LINEAR evaluate
//                  + ranking keys             (particle_opt.py:176-192, 250-263, 330)
//   k_schedule     run_descent_schedule: K_lin linear steps with the decaying rate, K_quad
//                  quadratic steps, NaN freeze, clamp, then the final QUADRATIC cost,
//                  all in one launch with the particle resident in shared memory
//                  (particle_opt.py:203-228, 266-300, 359)
//   k_step         _step_values for cost models that supply their own gradient
//                  (particle_opt.py:214-228)
//   k_sample       sample_uniform without a fused cost (generic cost models)
#pragma once
#include "rng.cuh"
#include "stage1_models.cuh"

namespace spasm {

template <typename R>
__device__ __forceinline__ R* particle_smem(int tid) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return reinterpret_cast<R*>(smem_raw) + tid;
}

// Cooperative, coalesced load of bs particle rows into the column-major smem tile.
template <typename R, typename Src>
__device__ __forceinline__ void load_rows(R* tile, const Src* __restrict__ src, const uint32_t* __restrict__ rows,
                                          int64_t p0, int64_t P, int D, int bs) {
  const int64_t n = (int64_t)min((int64_t)bs, P - p0) * D;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int r = (int)(e / D), d = (int)(e % D);
    const int64_t row = rows ? (int64_t)rows[p0 + r] : p0 + r;
    tile[d * bs + r] = (R)src[row * D + d];
  }
}

template <typename R>
__device__ __forceinline__ void store_rows(R* __restrict__ dst, const R* tile, int64_t p0, int64_t P, int D, int bs) {
  const int64_t n = (int64_t)min((int64_t)bs, P - p0) * D;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int r = (int)(e / D), d = (int)(e % D);
    dst[(p0 + r) * D + d] = tile[d * bs + r];
  }
}

// ---------------------------------------------------------------------------
template <class E, typename R, bool Q>
__global__ void k_evaluate(const typename E::Scene sc, const R* __restrict__ values, int64_t P, R* __restrict__ costs) {
  const int bs = blockDim.x;
  const int D = sc.dim;
  R* base = particle_smem<R>(0);
  const int64_t p0 = (int64_t)blockIdx.x * bs;
  load_rows<R, R>(base, values, nullptr, p0, P, D, bs);
  __syncthreads();
  const int64_t p = p0 + threadIdx.x;
  if (p >= P) return;
  R* x = base + threadIdx.x;
  R* scr = base + (int64_t)D * bs + threadIdx.x;
  const R c = E::template run<true, false, Q>(sc, x, nullptr, scr, bs);
  costs[p] = c;
}

template <class E, typename R, bool Q>
__global__ void k_gradient(const typename E::Scene sc, const R* __restrict__ values, int64_t P, R* __restrict__ grad) {
  const int bs = blockDim.x;
  const int D = sc.dim;
  R* base = particle_smem<R>(0);
  const int64_t p0 = (int64_t)blockIdx.x * bs;
  load_rows<R, R>(base, values, nullptr, p0, P, D, bs);
  __syncthreads();
  const int64_t p = p0 + threadIdx.x;
  if (p < P) {
    R* x = base + threadIdx.x;
    R* g = base + (int64_t)D * bs + threadIdx.x;
    R* scr = base + (int64_t)2 * D * bs + threadIdx.x;
    E::template run<false, true, Q>(sc, x, g, scr, bs);
  }
  __syncthreads();
  store_rows<R>(grad, base + (int64_t)D * bs, p0, P, D, bs);
}

// ---------------------------------------------------------------------------
// Sampling: numpy Generator.uniform(lower, upper, size=(N, D)) == lower + (upper-lower)*u
// with u = next_double() drawn in C order from one PCG64 stream per restart. Row i
// jumps ahead by (row_offset + i) * D outputs, so any contiguous shard of rows (one GPU
// of G) reproduces exactly the rows of the single centralized draw.
__device__ __forceinline__ double uniform_draw(double lo, double hi, double u) {
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
}

template <typename R>
__device__ __forceinline__ void sample_row(R* x, int bs, const Pcg64State& st, int64_t grow, int D, const Bounds64& bd,
                                           const double* __restrict__ warm, int64_t n_warm, int use_philox,
                                           uint64_t philox_seed, uint32_t restart) {
  if (grow < n_warm) {
    // inject_warm_start: clamp(seed) into bounds (particle_opt.py:250-263)
    for (int d = 0; d < D; ++d) {
      double v = warm[grow * D + d];
      v = v < bd.lo[d] ? bd.lo[d] : (v > bd.hi[d] ? bd.hi[d] : v);
      x[d * bs] = (R)v;
    }
    return;
  }
  if (!use_philox) {
    Pcg64 rng;
    rng.init(st);
    rng.advance((uint64_t)grow * (uint64_t)D);
    for (int d = 0; d < D; ++d) x[d * bs] = (R)uniform_draw(bd.lo[d], bd.hi[d], rng.next_double());
  } else {
    // perf-mode sampler: Philox4x32-10, counter = (row lo, row hi, restart, word block)
    const uint2 key = make_uint2((uint32_t)philox_seed, (uint32_t)(philox_seed >> 32));
    for (int d0 = 0; d0 < D; d0 += 4) {
      const uint4 r = Philox4x32::gen(make_uint4((uint32_t)grow, (uint32_t)(grow >> 32), restart, (uint32_t)(d0 >> 2)), key);
      const uint32_t w[4] = {r.x, r.y, r.z, r.w};
      for (int k = 0; k < 4 && d0 + k < D; ++k) {
        const int d = d0 + k;
        const double u = (double)(w[k] >> 8) * (1.0 / 16777216.0);
        x[d * bs] = (R)uniform_draw(bd.lo[d], bd.hi[d], u);
      }
    }
  }
}

template <class E, typename R>
__global__ void k_sample_eval(const typename E::Scene sc, const Bounds64 bd, Pcg64State st, int64_t row_offset,
                              int64_t N, const double* __restrict__ warm, int64_t n_warm, int use_philox,
                              uint64_t philox_seed, uint32_t restart, R* __restrict__ values,
                              typename KeyOf<R>::type* __restrict__ keys, uint32_t* __restrict__ idx,
                              const RestartParams* __restrict__ rp) {
  if (rp) {  // graph launch: restart inputs from device memory
    st = rp->st;
    philox_seed = rp->seed;
    restart = rp->restart;
  }
  const int bs = blockDim.x;
  const int D = sc.dim;
  R* base = particle_smem<R>(0);
  const int64_t p0 = (int64_t)blockIdx.x * bs;
  const int64_t p = p0 + threadIdx.x;
  R* x = base + threadIdx.x;
  if (p < N) sample_row<R>(x, bs, st, row_offset + p, D, bd, warm, n_warm, use_philox, philox_seed, restart);
  __syncthreads();
  store_rows<R>(values, base, p0, N, D, bs);
  if (p >= N) return;
  R* scr = base + (int64_t)D * bs + threadIdx.x;
  const R c = E::template run<true, false, false>(sc, x, nullptr, scr, bs);
  keys[p] = order_key(c);
  idx[p] = (uint32_t)(row_offset + p);
}

// rows (optional): draw the listed global rows instead of [row_offset, row_offset+N), so a
// rank can re-create any row of the centralized draw (the sharded top-M, shard.cu).
template <typename R>
__global__ void k_sample(const Bounds64 bd, Pcg64State st, int64_t row_offset, const uint32_t* __restrict__ rows,
                         int64_t N, int D, const double* __restrict__ warm, int64_t n_warm, int use_philox,
                         uint64_t philox_seed, uint32_t restart, R* __restrict__ values,
                         const RestartParams* __restrict__ rp) {
  if (rp) {  // graph launch: restart inputs from device memory
    st = rp->st;
    philox_seed = rp->seed;
    restart = rp->restart;
  }
  const int bs = blockDim.x;
  R* base = particle_smem<R>(0);
  const int64_t p0 = (int64_t)blockIdx.x * bs;
  const int64_t p = p0 + threadIdx.x;
  if (p < N) {
    const int64_t grow = rows ? (int64_t)rows[p] : row_offset + p;
    sample_row<R>(base + threadIdx.x, bs, st, grow, D, bd, warm, n_warm, use_philox, philox_seed, restart);
  }
  __syncthreads();
  store_rows<R>(values, base, p0, N, D, bs);
}

// ---------------------------------------------------------------------------
// One clamped step x <- clip(x - rate * g); a row with any non-finite gradient
// component is frozen (g := 0) and flagged (particle_opt.py:221-228).
template <typename R>
__device__ __forceinline__ bool apply_step(R* x, R* g, int D, int bs, R rate, const R* lower, const R* upper) {
  bool bad = false;
  for (int d = 0; d < D; ++d) bad |= !Math<R>::finite(g[d * bs]);
  for (int d = 0; d < D; ++d) {
    R v = x[d * bs];
    if (!bad) v = v - rate * g[d * bs];
    v = v < lower[d] ? lower[d] : (v > upper[d] ? upper[d] : v);
    x[d * bs] = v;
  }
  return bad;
}

template <typename R>
__global__ void k_step(R* __restrict__ values, const R* __restrict__ grad, int64_t P, int D, R rate,
                       const R* __restrict__ lower, const R* __restrict__ upper, uint8_t* __restrict__ flagged) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  bool bad = false;
  for (int d = 0; d < D; ++d) bad |= !Math<R>::finite(grad[p * D + d]);
  for (int d = 0; d < D; ++d) {
    R v = values[p * D + d];
    if (!bad) v = v - rate * grad[p * D + d];
    v = v < lower[d] ? lower[d] : (v > upper[d] ? upper[d] : v);
    values[p * D + d] = v;
  }
  if (bad && flagged) flagged[p] = 1;
}

// ---------------------------------------------------------------------------
// Fused descent schedule. rows (optional) gathers the top-M selection from the
// sampled batch so the selected rows never round-trip through a separate copy.
// Trace (optional): per step, the active-mode cost and quadratic satisfaction of the
// first n_traced particles (particle_opt.py:286-297).
// Perf-mode update (StepRule, scene.cuh): Adam and/or annealed Philox noise. am/av hold the
// Adam moments (column layout like x); t is the 1-based step count, p the batch row.
template <typename R>
__device__ __forceinline__ bool apply_step_rule(R* x, R* g, R* am, R* av, int D, int bs, R rate, const R* lower,
                                                const R* upper, const StepRule& rule, int t, int64_t p, R sigma) {
  bool bad = false;
  for (int d = 0; d < D; ++d) bad |= !Math<R>::finite(g[d * bs]);
  const R c1 = R(1) - (R)pow((double)rule.b1, (double)t), c2 = R(1) - (R)pow((double)rule.b2, (double)t);
  const uint2 key = make_uint2((uint32_t)rule.seed, (uint32_t)(rule.seed >> 32));
  R z[2] = {R(0), R(0)};
  for (int d = 0; d < D; ++d) {
    R v = x[d * bs];
    if (!bad) {
      R u = g[d * bs];
      if (rule.adam) {
        const R m = R(rule.b1) * am[d * bs] + (R(1) - R(rule.b1)) * u;
        const R s2 = R(rule.b2) * av[d * bs] + (R(1) - R(rule.b2)) * u * u;
        am[d * bs] = m;
        av[d * bs] = s2;
        u = (m / c1) / (Math<R>::sqrt_(s2 / c2) + R(rule.eps));
      }
      v = v - rate * u;
      if (sigma > R(0)) {
        if ((d & 1) == 0) {  // Box-Muller pair per two dimensions
          const uint4 r4 = Philox4x32::gen(
              make_uint4((uint32_t)p, (uint32_t)(p >> 32) ^ ((uint32_t)t << 8), rule.restart, 0x80000000u | (uint32_t)d),
              key);
          const double u1 = ((double)(r4.x >> 8) + 0.5) * (1.0 / 16777216.0);
          const double u2 = (double)(r4.y >> 8) * (1.0 / 16777216.0);
          const double rad = sqrt(-2.0 * log(u1));
          z[0] = (R)(rad * cos(6.283185307179586 * u2));
          z[1] = (R)(rad * sin(6.283185307179586 * u2));
        }
        v = v + sigma * (upper[d] - lower[d]) * z[d & 1];
      }
    }
    v = v < lower[d] ? lower[d] : (v > upper[d] ? upper[d] : v);
    x[d * bs] = v;
  }
  return bad;
}

template <class E, typename R, bool TRACE>
__global__ void k_schedule(const typename E::Scene sc, const R* __restrict__ src, const uint32_t* __restrict__ rows,
                           int64_t M, int k_lin, int k_quad, double eta, double alpha, double eps,
                           R* __restrict__ out_values, R* __restrict__ out_cost, uint8_t* __restrict__ flagged,
                           unsigned int* __restrict__ flagged_count, R* __restrict__ trace_cost,
                           uint8_t* __restrict__ trace_sat, int n_traced, const StepRule rule) {
  const int bs = blockDim.x;
  const int D = sc.dim;
  R* base = particle_smem<R>(0);
  const int64_t p0 = (int64_t)blockIdx.x * bs;
  load_rows<R, R>(base, src, rows, p0, M, D, bs);
  __syncthreads();
  const int64_t p = p0 + threadIdx.x;
  if (p < M) {
    R* x = base + threadIdx.x;
    R* g = base + (int64_t)D * bs + threadIdx.x;
    R* scr = base + (int64_t)2 * D * bs + threadIdx.x;
    const bool ref = rule.is_reference();
    R* am = base + (int64_t)(2 * D + E::scratch_per_thread(sc)) * bs + threadIdx.x;  // Adam moments (perf mode)
    R* av = am + (int64_t)D * bs;
    if (rule.adam)
      for (int d = 0; d < D; ++d) am[d * bs] = av[d * bs] = R(0);
    bool bad = false;
    int step = 0;
    for (int k = 1; k <= k_lin; ++k) {
      // lr_schedule in float64 exactly as the reference, then cast (particle_opt.py:203-211)
      const R rate = (R)(eta * (1.0 - (double)k / (double)k_lin));
      E::template run<false, true, false>(sc, x, g, scr, bs);
      if (ref)
        bad |= apply_step<R>(x, g, D, bs, rate, sc.lower, sc.upper);
      else
        bad |= apply_step_rule<R>(x, g, am, av, D, bs, rate, sc.lower, sc.upper, rule, step + 1, p,
                                  R(rule.noise) * R(1.0 - (double)k / (double)k_lin));
      if constexpr (TRACE) {
        if (p < n_traced) {
          const R cl = E::template run<true, false, false>(sc, x, nullptr, scr, bs);
          const R cq = E::template run<true, false, true>(sc, x, nullptr, scr, bs);
          trace_cost[(int64_t)step * n_traced + p] = cl;
          trace_sat[(int64_t)step * n_traced + p] = (double)cq < eps;
        }
      }
      ++step;
    }
    for (int k = 0; k < k_quad; ++k) {
      E::template run<false, true, true>(sc, x, g, scr, bs);
      if (ref)
        bad |= apply_step<R>(x, g, D, bs, (R)alpha, sc.lower, sc.upper);
      else
        bad |= apply_step_rule<R>(x, g, am, av, D, bs, (R)alpha, sc.lower, sc.upper, rule, step + 1, p, R(0));
      if constexpr (TRACE) {
        if (p < n_traced) {
          const R cq = E::template run<true, false, true>(sc, x, nullptr, scr, bs);
          trace_cost[(int64_t)step * n_traced + p] = cq;
          trace_sat[(int64_t)step * n_traced + p] = (double)cq < eps;
        }
      }
      ++step;
    }
    const R fc = E::template run<true, false, true>(sc, x, nullptr, scr, bs);
    out_cost[p] = fc;
    if (flagged) flagged[p] = bad ? 1 : 0;
    if (bad && flagged_count) atomicAdd(flagged_count, 1u);
  }
  __syncthreads();
  store_rows<R>(out_values, base, p0, M, D, bs);
}

}  // namespace spasm
