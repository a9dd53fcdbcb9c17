// Sharded stage-1 restart (multi-GPU): the device halves of one restart of
// particle_opt.solve (reference particle_opt.py:325-384) when the N sampled rows are split
// into contiguous per-rank ranges. Between the halves the host exchanges the local elite
// runs (one all-gather of m records per rank over NCCL); after the second half it
// exchanges the rank's satisfying candidates (one all-gather of p_return records).
//
// Exactness: row i of the restart's centralized draw is a pure function of (seed, restart,
// i) (PCG64 jump-ahead, k_sample), every rank sorts (order_key(cost), global row) pairs,
// and the merge ranks each record against every other run by binary search on the same
// lexicographic key. The merged order is therefore exactly np.argsort(costs,
// kind="stable")[:m] of the single centralized batch (particle_opt.py:195-200), for any
// world size, and each rank re-draws the rows of its slice of that order instead of
// receiving their values.
#include <algorithm>
#include <cstring>

#include "../../include/spasm.h"
#include "launchers.hpp"
#include "scene.cuh"

namespace spasm {

StepRule step_rule(const spasm_solve_config& cfg, int restart);  // capi.cu

static size_t shard_align(size_t x) { return (x + 255) & ~(size_t)255; }

struct ShardLayout {
  size_t values, keys0, keys1, idx0, idx1, hist, top, opt_in, opt_values, opt_cost, flagged, counters, sk0, sk1, sv0,
      sv1, chosen, recheck, total;
};

template <typename R>
static ShardLayout shard_layout(int D, const spasm_solve_config& cfg, int64_t n_local, int64_t m_local) {
  using K = typename KeyOf<R>::type;
  ShardLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = shard_align(off + std::max<size_t>(bytes, 1));
    return o;
  };
  const int64_t nl = std::max<int64_t>(n_local, 1), ml = std::max<int64_t>(m_local, 1);
  const int64_t tiles = (std::max(nl, ml) + 2047) / 2048 + 1;
  L.values = take((size_t)nl * D * sizeof(R));
  L.keys0 = take((size_t)nl * sizeof(K));
  L.keys1 = take((size_t)nl * sizeof(K));
  L.idx0 = take((size_t)nl * 4);
  L.idx1 = take((size_t)nl * 4);
  L.hist = take((size_t)tiles * 256 * 4);
  L.top = take((size_t)cfg.m * 4);
  L.opt_in = take((size_t)ml * D * sizeof(R));
  L.opt_values = take((size_t)ml * D * sizeof(R));
  L.opt_cost = take((size_t)ml * sizeof(R));
  L.flagged = take((size_t)ml);
  L.counters = take(64);
  L.sk0 = take((size_t)ml * sizeof(K));
  L.sk1 = take((size_t)ml * sizeof(K));
  L.sv0 = take((size_t)ml * 4);
  L.sv1 = take((size_t)ml * 4);
  L.chosen = take((size_t)cfg.p_return * D * sizeof(R));
  L.recheck = take((size_t)cfg.p_return * sizeof(R));
  L.total = off;
  return L;
}

// Local elite run: the first min(m, n) sorted (key, row) pairs widened to u64 records,
// padded with all-ones records (which sort after every real record).
template <typename K>
__global__ void k_elite_records(const K* __restrict__ keys, const uint32_t* __restrict__ rows, int64_t n, int64_t m,
                                ulonglong2* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  ulonglong2 r;
  if (j < n) {
    r.x = (unsigned long long)keys[j];
    r.y = (unsigned long long)rows[j];
  } else {
    r.x = ~0ull;
    r.y = ~0ull;
  }
  out[j] = r;
}

__device__ __forceinline__ bool rec_less(const ulonglong2& a, const ulonglong2& b) {
  return a.x < b.x || (a.x == b.x && a.y < b.y);
}

// Merge G sorted runs of m records into the global first m rows. A record's global rank
// is its position in its own run plus, for every other run, the number of records that
// precede it there (lower bound). Real records are distinct (global rows are unique), so
// ranks of real records are a permutation; padding ranks behind >= m real records.
// Runs hold run_len records each (m for the all-gather protocol; the largest per-rank
// contribution for the top-m select protocol, whose runs together hold exactly m records).
__global__ void k_merge_runs(const ulonglong2* __restrict__ runs, int G, int64_t run_len, int64_t m,
                             uint32_t* __restrict__ top) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)G * run_len) return;
  const int g = (int)(i / run_len);
  const int64_t j = i - (int64_t)g * run_len;
  const ulonglong2 rec = runs[i];
  if (rec.y == ~0ull) return;
  int64_t rank = j;
  for (int h = 0; h < G && rank < m; ++h) {
    if (h == g) continue;
    const ulonglong2* run = runs + (int64_t)h * run_len;
    int64_t lo = 0, hi = run_len;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (rec_less(run[mid], rec)) lo = mid + 1;
      else hi = mid;
    }
    rank += lo;
  }
  if (rank < m) top[rank] = (uint32_t)rec.y;
}

// Candidate block (float64): [n_sat, flagged, k, then p_return records of
// (global position in the top-m order, global row, quadratic cost, re-check cost, values[D])].
template <typename R>
__global__ void k_shard_candidates(const uint32_t* __restrict__ order, const unsigned int* __restrict__ counters,
                                   int p_return, const R* __restrict__ opt_values, const R* __restrict__ opt_cost,
                                   const uint32_t* __restrict__ rows, int64_t pos_lo, int D, R* __restrict__ chosen,
                                   double* __restrict__ cand) {
  const int c = blockIdx.x;
  const int k = min((int)counters[0], p_return);
  if (c == 0 && threadIdx.x == 0) {
    cand[0] = (double)counters[0];
    cand[1] = (double)counters[1];
    cand[2] = (double)k;
  }
  double* rec = cand + 3 + (int64_t)c * (4 + D);
  const uint32_t q = c < k ? order[c] : 0u;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const R v = c < k ? opt_values[(int64_t)q * D + d] : (R)0;
    chosen[(int64_t)c * D + d] = v;
    rec[4 + d] = (double)v;
  }
  if (threadIdx.x == 0) {
    rec[0] = c < k ? (double)(pos_lo + q) : -1.0;
    rec[1] = c < k ? (double)rows[q] : -1.0;
    rec[2] = c < k ? (double)opt_cost[q] : 0.0;
  }
}

template <typename R>
__global__ void k_cand_recheck(const R* __restrict__ recheck, int p_return, int D, double* __restrict__ cand) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < p_return) cand[3 + (int64_t)c * (4 + D) + 3] = (double)recheck[c];
}

template <typename R>
static int shard_select_impl(const Model& m, const spasm_solve_config& cfg, int restart, int64_t row_lo,
                             int64_t n_local, const double* warm, int64_t n_warm, void* ws, int64_t ws_bytes,
                             uint64_t* elite, int32_t* launches, cudaStream_t s) {
  using K = typename KeyOf<R>::type;
  const ShardLayout L = shard_layout<R>(m.dim, cfg, n_local, 1);
  SPASM_REQUIRE(ws != nullptr && (size_t)ws_bytes >= L.total, "shard workspace too small");
  char* base = static_cast<char*>(ws);
  R* values = reinterpret_cast<R*>(base + L.values);
  K* k0 = reinterpret_cast<K*>(base + L.keys0);
  K* k1 = reinterpret_cast<K*>(base + L.keys1);
  uint32_t* i0 = reinterpret_cast<uint32_t*>(base + L.idx0);
  uint32_t* i1 = reinterpret_cast<uint32_t*>(base + L.idx1);
  unsigned int* hist = reinterpret_cast<unsigned int*>(base + L.hist);
  const Pcg64State st = restart_state(cfg.seed, (uint64_t)restart);
  int r = launch_sample_eval<R>(m, st, row_lo, n_local, warm, n_warm, cfg.sampler, cfg.seed, (uint32_t)restart, values,
                                k0, i0, s);
  if (r) return r;
  bool in1 = false;
  if ((r = launch_sort<R>(k0, i0, k1, i1, n_local, hist, &in1, s))) return r;
  if (elite) {  // all-gather protocol: the local elite run (the top-m select protocol reads the sorted keys in place)
    k_elite_records<K><<<ceil_div(cfg.m, 256), 256, 0, s>>>(in1 ? k1 : k0, in1 ? i1 : i0, n_local, cfg.m,
                                                            reinterpret_cast<ulonglong2*>(elite));
    SPASM_CHECK_LAUNCH();
  }
  if (launches) {
    const int sample = (sizeof(R) == 4 && m.tile_ok && stage1_tile_mode() != 0) ? 2 : 1;
    *launches = (n_local > 0 ? sample : 0) + radix_sort_launches(n_local, 8 * (int)sizeof(R)) + (elite ? 1 : 0);
  }
  return SPASM_OK;
}

template <typename R>
static int shard_descend_impl(const Model& m, const spasm_solve_config& cfg, int restart, const uint64_t* elite_all,
                              int world, int64_t run_len, int64_t pos_lo, int64_t pos_hi, const double* warm, int64_t n_warm, void* ws,
                              int64_t ws_bytes, double* cand, int32_t* launches, cudaStream_t s) {
  using K = typename KeyOf<R>::type;
  const int D = m.dim;
  const int64_t ml = pos_hi - pos_lo;
  const ShardLayout L = shard_layout<R>(D, cfg, 1, ml);
  SPASM_REQUIRE(ws != nullptr && (size_t)ws_bytes >= L.total, "shard workspace too small");
  char* base = static_cast<char*>(ws);
  uint32_t* top = reinterpret_cast<uint32_t*>(base + L.top);
  R* opt_in = reinterpret_cast<R*>(base + L.opt_in);
  R* opt_values = reinterpret_cast<R*>(base + L.opt_values);
  R* opt_cost = reinterpret_cast<R*>(base + L.opt_cost);
  uint8_t* flagged = reinterpret_cast<uint8_t*>(base + L.flagged);
  unsigned int* counters = reinterpret_cast<unsigned int*>(base + L.counters);
  K* sk0 = reinterpret_cast<K*>(base + L.sk0);
  K* sk1 = reinterpret_cast<K*>(base + L.sk1);
  uint32_t* sv0 = reinterpret_cast<uint32_t*>(base + L.sv0);
  uint32_t* sv1 = reinterpret_cast<uint32_t*>(base + L.sv1);
  unsigned int* hist = reinterpret_cast<unsigned int*>(base + L.hist);
  R* chosen = reinterpret_cast<R*>(base + L.chosen);
  R* recheck = reinterpret_cast<R*>(base + L.recheck);

  const int64_t gm = (int64_t)world * run_len;
  k_merge_runs<<<ceil_div(gm, 256), 256, 0, s>>>(reinterpret_cast<const ulonglong2*>(elite_all), world, run_len,
                                                 cfg.m, top);
  SPASM_CHECK_LAUNCH();
  const Pcg64State st = restart_state(cfg.seed, (uint64_t)restart);
  int r = launch_sample<R>(m.bounds, D, st, 0, top + pos_lo, ml, warm, n_warm, cfg.sampler, cfg.seed,
                           (uint32_t)restart, opt_in, s);
  if (r) return r;
  SPASM_CUDA_TRY(cudaMemsetAsync(counters, 0, 64, s));
  if ((r = launch_schedule<R>(m, opt_in, nullptr, ml, cfg.k_lin, cfg.k_quad, cfg.eta_init, cfg.alpha, cfg.epsilon,
                              opt_values, opt_cost, flagged, counters + 1, nullptr, nullptr, 0,
                              step_rule(cfg, restart), s)))
    return r;
  if ((r = launch_sat_keys<R>(opt_cost, ml, cfg.epsilon, sk0, sv0, counters, s))) return r;
  bool in1 = false;
  if ((r = launch_sort<R>(sk0, sv0, sk1, sv1, ml, hist, &in1, s))) return r;
  k_shard_candidates<R><<<cfg.p_return, 32, 0, s>>>(in1 ? sv1 : sv0, counters, cfg.p_return, opt_values, opt_cost,
                                                    top + pos_lo, pos_lo, D, chosen, cand);
  SPASM_CHECK_LAUNCH();
  // independent soundness re-check of the rank's candidates (particle_opt.py:366)
  if ((r = launch_evaluate<R>(m, chosen, cfg.p_return, 1, recheck, s))) return r;
  k_cand_recheck<R><<<ceil_div(cfg.p_return, 128), 128, 0, s>>>(recheck, cfg.p_return, D, cand);
  SPASM_CHECK_LAUNCH();
  if (launches) {
    const int ps = radix_sort_launches(ml, 8 * (int)sizeof(R));
    *launches = 1 + (ml > 0 ? 3 : 0) + (ml > 1 ? ps : 0) + 3;
  }
  return SPASM_OK;
}

// ---- exact distributed top-m selection (the select protocol) -----------------------------
// Instead of gathering every rank's m best records, the ranks agree on the key K* of the
// global m-th record by an MSB-first radix select: per 8-bit digit, every rank counts its
// (already sorted) keys under the current prefix per digit value (binary searches), the
// 256 counts are summed across ranks (one small all-reduce), and the digit holding the m-th
// record extends the prefix. After key_bits/8 digits the prefix is K* and `remaining` is
// how many K*-keyed records the top m takes. Ties at K* go to the lowest global rows, i.e.
// to the lower ranks first (contiguous row shards), which the host allots from the
// per-rank (less, ties) counts. Each rank then contributes its first less_r + t_r sorted
// records -- m records in total across the ranks -- and the descend merge ranks only those.
struct TopmState {
  unsigned long long prefix;  // chosen key bits above the current digit
  long long remaining;        // 1-based rank of the m-th record inside the prefix class
  int pass, key_bits;
};

template <typename K>
__device__ __forceinline__ int64_t lower_bound_key(const K* a, int64_t n, K v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <typename K>
__device__ __forceinline__ int64_t upper_bound_key(const K* a, int64_t n, K v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <typename K>
__global__ void k_topm_hist(const K* __restrict__ keys, int64_t n, const TopmState* __restrict__ st,
                            long long* __restrict__ hist) {
  const int d = threadIdx.x;
  if (d >= 256) return;
  const int shift = st->key_bits - 8 * (st->pass + 1);
  const K lo = (K)st->prefix | ((K)d << shift);
  const K span = shift == 0 ? (K)0 : (K)((((K)1) << shift) - 1);
  hist[d] = (long long)(upper_bound_key(keys, n, (K)(lo | span)) - lower_bound_key(keys, n, lo));
}

__global__ void k_topm_pick(TopmState* __restrict__ st, const long long* __restrict__ hist) {
  if (threadIdx.x != 0) return;
  const int shift = st->key_bits - 8 * (st->pass + 1);
  long long rem = st->remaining;
  int d = 0;
  for (; d < 255; ++d) {
    if (rem <= hist[d]) break;
    rem -= hist[d];
  }
  st->prefix |= (unsigned long long)d << shift;
  st->remaining = rem;
  st->pass += 1;
}

template <typename K>
__global__ void k_topm_local(const K* __restrict__ keys, int64_t n, const TopmState* __restrict__ st,
                             long long* __restrict__ out) {
  if (threadIdx.x != 0) return;
  const K ks = (K)st->prefix;
  const int64_t less = lower_bound_key(keys, n, ks);
  out[0] = less;
  out[1] = upper_bound_key(keys, n, ks) - less;
  out[2] = st->remaining;  // K*-keyed records the global top m takes
}

template <typename K>
__global__ void k_topm_contrib(const K* __restrict__ keys, const uint32_t* __restrict__ rows, int64_t take,
                               int64_t cap, ulonglong2* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cap) return;
  ulonglong2 r;
  r.x = j < take ? (unsigned long long)keys[j] : ~0ull;
  r.y = j < take ? (unsigned long long)rows[j] : ~0ull;
  out[j] = r;
}

int validate_cfg(const spasm_solve_config* cfg);  // capi.cu: the single-GPU solve's checks

// the single-GPU validator plus the shard path's own row bound (row 0xFFFFFFFF is the
// padding sentinel of the elite runs)
static int validate_shard_cfg(const spasm_model* model, const spasm_solve_config* cfg) {
  SPASM_REQUIRE(model != nullptr, "null model");
  const int r = validate_cfg(cfg);
  if (r) return r;
  SPASM_REQUIRE(cfg->n < (int64_t)0xFFFFFFFF, "n exceeds 2^32 - 1 rows");
  return SPASM_OK;
}

}  // namespace spasm

using namespace spasm;

struct spasm_model : public spasm::Model {};

extern "C" {

int64_t spasm_shard_workspace_bytes(const spasm_model* model, int dtype, const spasm_solve_config* cfg,
                                    int64_t n_local, int64_t m_local) {
  if (!model || !cfg || n_local < 0 || m_local < 0) return -1;
  if (dtype == SPASM_F64) return (int64_t)shard_layout<double>(model->dim, *cfg, n_local, m_local).total;
  return (int64_t)shard_layout<float>(model->dim, *cfg, n_local, m_local).total;
}

int spasm_shard_select(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int restart, int64_t row_lo,
                       int64_t n_local, const double* warm_dev, int64_t n_warm, void* workspace,
                       int64_t workspace_bytes, uint64_t* elite, int32_t* launches, void* stream) {
  int r = validate_shard_cfg(model, cfg);
  if (r) return r;
  SPASM_REQUIRE(restart >= 0, "restart must be >= 0");
  SPASM_REQUIRE(row_lo >= 0 && n_local >= 0 && row_lo + n_local <= cfg->n, "row range outside [0, n)");
  SPASM_DTYPE_SWITCH(dtype, return shard_select_impl<R>(*model, *cfg, restart, row_lo, n_local, warm_dev, n_warm,
                                                        workspace, workspace_bytes, elite, launches,
                                                        as_stream(stream)););
}

int spasm_shard_descend(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int restart,
                        const uint64_t* elite_all, int world, int64_t run_len, int64_t pos_lo, int64_t pos_hi,
                        const double* warm_dev, int64_t n_warm, void* workspace, int64_t workspace_bytes,
                        double* candidates, int32_t* launches, void* stream) {
  int r = validate_shard_cfg(model, cfg);
  if (r) return r;
  SPASM_REQUIRE(restart >= 0, "restart must be >= 0");
  SPASM_REQUIRE(world >= 1, "world must be >= 1");
  SPASM_REQUIRE(run_len >= 1 && run_len <= cfg->m, "run length outside [1, m]");
  SPASM_REQUIRE(0 <= pos_lo && pos_lo <= pos_hi && pos_hi <= cfg->m, "position range outside [0, m]");
  SPASM_REQUIRE(elite_all != nullptr && candidates != nullptr, "null buffer");
  SPASM_DTYPE_SWITCH(dtype, return shard_descend_impl<R>(*model, *cfg, restart, elite_all, world, run_len, pos_lo,
                                                         pos_hi, warm_dev, n_warm, workspace, workspace_bytes,
                                                         candidates, launches, as_stream(stream)););
}

int64_t spasm_shard_topm_state_bytes(void) { return (int64_t)sizeof(TopmState); }

int spasm_shard_topm_init(int dtype, int64_t m, void* state, void* stream) {
  SPASM_REQUIRE(state != nullptr && m >= 1, "bad top-m state");
  SPASM_REQUIRE(dtype == SPASM_F32 || dtype == SPASM_F64, "dtype must be SPASM_F32 or SPASM_F64");
  TopmState h{0ull, (long long)m, 0, dtype == SPASM_F64 ? 64 : 32};
  // pageable source: staged by the driver before the call returns
  SPASM_CUDA_TRY(cudaMemcpyAsync(state, &h, sizeof(h), cudaMemcpyHostToDevice, as_stream(stream)));
  return SPASM_OK;
}

int spasm_shard_topm_hist(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int64_t n_local,
                          void* workspace, const void* state, int64_t* hist, void* stream) {
  int r = validate_shard_cfg(model, cfg);
  if (r) return r;
  SPASM_REQUIRE(workspace && state && hist, "null buffer");
  SPASM_DTYPE_SWITCH(dtype, {
    using K = typename KeyOf<R>::type;
    const ShardLayout L = shard_layout<R>(model->dim, *cfg, n_local, 1);
    const K* keys = reinterpret_cast<const K*>(static_cast<const char*>(workspace) + L.keys0);  // sorted (4 / 8 passes)
    k_topm_hist<K><<<1, 256, 0, as_stream(stream)>>>(keys, n_local, static_cast<const TopmState*>(state),
                                                     reinterpret_cast<long long*>(hist));
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  });
}

int spasm_shard_topm_pick(void* state, const int64_t* hist_sum, void* stream) {
  SPASM_REQUIRE(state && hist_sum, "null buffer");
  k_topm_pick<<<1, 32, 0, as_stream(stream)>>>(static_cast<TopmState*>(state),
                                              reinterpret_cast<const long long*>(hist_sum));
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

int spasm_shard_topm_local(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int64_t n_local,
                           void* workspace, const void* state, int64_t* counts, void* stream) {
  int r = validate_shard_cfg(model, cfg);
  if (r) return r;
  SPASM_REQUIRE(workspace && state && counts, "null buffer");
  SPASM_DTYPE_SWITCH(dtype, {
    using K = typename KeyOf<R>::type;
    const ShardLayout L = shard_layout<R>(model->dim, *cfg, n_local, 1);
    const K* keys = reinterpret_cast<const K*>(static_cast<const char*>(workspace) + L.keys0);
    k_topm_local<K><<<1, 32, 0, as_stream(stream)>>>(keys, n_local, static_cast<const TopmState*>(state),
                                                    reinterpret_cast<long long*>(counts));
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  });
}

int spasm_shard_topm_contrib(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int64_t n_local,
                             void* workspace, int64_t take, int64_t cap, uint64_t* records, void* stream) {
  int r = validate_shard_cfg(model, cfg);
  if (r) return r;
  SPASM_REQUIRE(workspace && records, "null buffer");
  SPASM_REQUIRE(0 <= take && take <= cap && take <= n_local && cap >= 1, "bad contribution size");
  SPASM_DTYPE_SWITCH(dtype, {
    using K = typename KeyOf<R>::type;
    const ShardLayout L = shard_layout<R>(model->dim, *cfg, n_local, 1);
    const char* base = static_cast<const char*>(workspace);
    k_topm_contrib<K><<<ceil_div(cap, 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const K*>(base + L.keys0), reinterpret_cast<const uint32_t*>(base + L.idx0), take, cap,
        reinterpret_cast<ulonglong2*>(records));
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  });
}

}  // extern "C"
