// extern "C" boundary of libspasm.so (declared in include/spasm.h).
//
// Also hosts the native stage-1 restart loop (spasm_solve), the C++ equivalent of
// particle_opt.solve (reference particle_opt.py:303-400): per restart it launches
// sample+evaluate, the stable top-M sort, the fused descent schedule, the satisfying
// ordering and the re-check, then reads back one small result block.
#include <algorithm>
#include <cuda_runtime.h>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/spasm.h"
#include "model.hpp"
#include "rng.cuh"
#include "seedseq.cuh"
#include "scene.cuh"
#include "launchers.hpp"

namespace spasm {

// Process-wide cache of the pinned result-staging buffers. Models are often short-lived (the
// C4 replanning loop builds one per tick): cudaMallocHost / cudaFreeHost per model cost
// milliseconds of driver time with a long tail, so released buffers are kept for reuse.
// A buffer is released only after its model's last solve has read its results.
namespace {
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;
size_t g_pin_bytes = 0;                        // bytes held by the free list
constexpr size_t kPinCacheMax = 32;            // entries
constexpr size_t kPinCacheBytes = 64u << 20;   // and bytes (spasm_trim releases everything)
}  // namespace

cudaError_t pinned_get(void** p, size_t bytes, size_t* got) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_free.lower_bound(bytes);
    if (it != g_pin_free.end() && it->first <= 4 * bytes + 65536) {
      *p = it->second;
      *got = it->first;
      g_pin_bytes -= it->first;
      g_pin_free.erase(it);
      return cudaSuccess;
    }
  }
  const cudaError_t e = cudaMallocHost(p, bytes);
  *got = e == cudaSuccess ? bytes : 0;
  return e;
}

void pinned_put(void* p, size_t bytes) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (g_pin_free.size() < kPinCacheMax && g_pin_bytes + bytes <= kPinCacheBytes) {
      g_pin_free.emplace(bytes, p);
      g_pin_bytes += bytes;
      return;
    }
  }
  cudaFreeHost(p);
}

// release every cached pinned buffer (spasm_trim)
void pinned_trim() {
  std::multimap<size_t, void*> drop;
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    drop.swap(g_pin_free);
    g_pin_bytes = 0;
  }
  for (auto& kv : drop) cudaFreeHost(kv.second);
}

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

static int g_stage1_tile = -1;  // spasm_set_option("stage1_tile", ...)
int stage1_tile_mode() { return g_stage1_tile; }
static int g_tower_lanes = 0;  // spasm_set_option("tower_lanes", ...): 0 auto, 1/2/4/8 lanes per particle
int tower_lanes_option() { return g_tower_lanes; }
static int g_ik_cluster = 0;  // spasm_set_option("ik_cluster", ...): 0 auto, 1/2/4/8 CTAs per lift group
int ik_cluster_option() { return g_ik_cluster; }
static int g_graphs = 1;       // spasm_set_option("graphs", ...): CUDA-graph the stage-1 restart
static thread_local const RestartParams* g_restart_override = nullptr;
const RestartParams* restart_override() { return g_restart_override; }


// ---- small helper kernels for the solve loop --------------------------------------
template <typename R>
__global__ void k_gather_chosen(const uint32_t* __restrict__ order, const unsigned int* __restrict__ n_sat, int p_return,
                                const R* __restrict__ opt_values, const R* __restrict__ opt_cost,
                                const uint32_t* __restrict__ top_idx, int D, R* __restrict__ chosen_vals,
                                double* __restrict__ out_vals, double* __restrict__ out_cost,
                                int32_t* __restrict__ out_idx) {
  const int c = blockIdx.x;
  const int k = min((int)*n_sat, p_return);
  if (c >= p_return) return;
  const uint32_t pos = c < k ? order[c] : 0u;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const R v = opt_values[(int64_t)pos * D + d];
    chosen_vals[(int64_t)c * D + d] = v;
    out_vals[(int64_t)c * D + d] = (double)v;
  }
  if (threadIdx.x == 0) {
    out_cost[c] = (double)opt_cost[pos];
    out_idx[c] = c < k ? (int32_t)top_idx[pos] : -1;
  }
}

template <typename R>
__global__ void k_copy_recheck(const R* __restrict__ c, int n, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (double)c[i];
}

__global__ void k_trace_ids(const uint32_t* __restrict__ top, int n, int32_t* __restrict__ ids) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = (int32_t)top[i];
}

// ---- workspace layout -------------------------------------------------------------
struct ResLayout;
static size_t res_layout_bytes(int D, int p);

struct SolveLayout {
  size_t values, keys0, keys1, idx0, idx1, hist, opt_values, opt_cost, flagged, counters, skeys0, skeys1, svals0,
      svals1, chosen_vals, recheck, warm, res, total;
  size_t res_bytes;
  int64_t n, m;
  int D, p;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

template <typename R>
static SolveLayout make_layout(int D, const spasm_solve_config& cfg, int64_t n_warm) {
  using K = typename KeyOf<R>::type;
  SolveLayout L;
  L.n = cfg.n;
  L.m = cfg.m;
  L.D = D;
  L.p = cfg.p_return;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  const int64_t tiles = (std::max(cfg.n, cfg.m) + 2047) / 2048 + 1;
  L.values = take((size_t)cfg.n * D * sizeof(R));
  L.keys0 = take((size_t)cfg.n * sizeof(K));
  L.keys1 = take((size_t)cfg.n * sizeof(K));
  L.idx0 = take((size_t)cfg.n * 4);
  L.idx1 = take((size_t)cfg.n * 4);
  L.hist = take((size_t)tiles * 256 * 4);
  L.opt_values = take((size_t)cfg.m * D * sizeof(R));
  L.opt_cost = take((size_t)cfg.m * sizeof(R));
  L.flagged = take((size_t)cfg.m);
  L.counters = take(64);
  L.skeys0 = take((size_t)cfg.m * sizeof(K));
  L.skeys1 = take((size_t)cfg.m * sizeof(K));
  L.svals0 = take((size_t)cfg.m * 4);
  L.svals1 = take((size_t)cfg.m * 4);
  L.chosen_vals = take((size_t)cfg.p_return * D * sizeof(R));
  L.recheck = take((size_t)cfg.p_return * sizeof(R));
  L.warm = take((size_t)std::max<int64_t>(n_warm, 1) * D * 8);
  // result block (res_layout): counters | out_* (last restart) | final_* (compacted)
  L.res_bytes = res_layout_bytes(D, cfg.p_return);
  L.res = take(L.res_bytes);
  L.total = off;
  return L;
}

int validate_cfg(const spasm_solve_config* cfg) {
  SPASM_REQUIRE(cfg != nullptr, "null solve config");
  SPASM_REQUIRE(cfg->m >= 1 && cfg->m <= cfg->n, "need 1 <= m <= n");
  SPASM_REQUIRE(cfg->n <= (int64_t)0xFFFFFFFF, "n exceeds 2^32 rows");
  SPASM_REQUIRE(cfg->k_lin >= 0 && cfg->k_quad >= 0, "step counts must be nonnegative");
  SPASM_REQUIRE(cfg->eta_init > 0 && cfg->alpha > 0, "learning rates must be positive");
  SPASM_REQUIRE(cfg->epsilon > 0, "epsilon must be positive");
  SPASM_REQUIRE(cfg->p_return >= 1, "p_return must be >= 1");
  SPASM_REQUIRE(cfg->max_restarts >= 1, "max_restarts must be >= 1");
  SPASM_REQUIRE(cfg->n_traced >= 0 && cfg->n_traced <= cfg->m, "n_traced must be in [0, m]");
  SPASM_REQUIRE(cfg->update == 0 || cfg->update == 1, "update must be 0 (gradient step) or 1 (Adam)");
  SPASM_REQUIRE(cfg->noise_sigma >= 0.f, "noise_sigma must be >= 0");
  if (cfg->update == 1)
    SPASM_REQUIRE(cfg->adam_beta1 >= 0.f && cfg->adam_beta1 < 1.f && cfg->adam_beta2 >= 0.f && cfg->adam_beta2 < 1.f &&
                      cfg->adam_eps > 0.f,
                  "Adam needs 0 <= beta1, beta2 < 1 and eps > 0");
  return SPASM_OK;
}

StepRule step_rule(const spasm_solve_config& cfg, int restart) {
  StepRule r;
  r.adam = cfg.update;
  r.b1 = cfg.adam_beta1;
  r.b2 = cfg.adam_beta2;
  r.eps = cfg.adam_eps;
  r.noise = cfg.noise_sigma;
  r.seed = cfg.seed;
  r.restart = (uint32_t)restart;
  return r;
}

// ---- the restart loop on the device (CUDA graph with a conditional WHILE node) ------------
// The result block in the workspace (copied to pinned host memory once, at the end):
//   counters  [0] n_sat  [1] flagged (both reset per restart)
//             [8] last restart run  [9] stopped  [10] flagged total  [11] n_final  [12] success
//   out_*     the last restart's first p_return satisfying rows (stable cost order), their
//             costs, re-check costs and batch indices (k_gather_chosen / k_copy_recheck)
//   final_*   the rows that passed the re-check, compacted (particle_opt.py:366 chosen =
//             chosen[satisfaction]); device consumers (stage-2 lifting) read these in place
struct ResLayout {
  size_t vals, cost, recheck, idx, fvals, fcost, fidx, bytes;
};
static ResLayout res_layout(int D, int p) {
  ResLayout r;
  size_t o = 64;
  r.vals = o;
  o += (size_t)p * D * 8;
  r.cost = o;
  o += (size_t)p * 8;
  r.recheck = o;
  o += (size_t)p * 8;
  r.idx = o;
  o += (size_t)p * 4;
  o = (o + 7) & ~(size_t)7;
  r.fvals = o;
  o += (size_t)p * D * 8;
  r.fcost = o;
  o += (size_t)p * 8;
  r.fidx = o;
  o += (size_t)p * 4;
  r.bytes = (o + 63) & ~(size_t)63;
  return r;
}

static size_t res_layout_bytes(int D, int p) { return res_layout(D, p).bytes; }

// chosen = chosen[recheck < eps], compacted (one thread; p_return is small)
__device__ void compact_chosen(char* res, const ResLayout RL, int p, int D, double eps) {
  unsigned int* c = reinterpret_cast<unsigned int*>(res);
  const int k = min((int)c[0], p);
  const double* v = reinterpret_cast<const double*>(res + RL.vals);
  const double* co = reinterpret_cast<const double*>(res + RL.cost);
  const double* re = reinterpret_cast<const double*>(res + RL.recheck);
  const int32_t* ix = reinterpret_cast<const int32_t*>(res + RL.idx);
  double* fv = reinterpret_cast<double*>(res + RL.fvals);
  double* fc = reinterpret_cast<double*>(res + RL.fcost);
  int32_t* fi = reinterpret_cast<int32_t*>(res + RL.fidx);
  int w = 0;
  for (int i = 0; i < k; ++i) {
    if (!(re[i] < eps)) continue;
    for (int d = 0; d < D; ++d) fv[(int64_t)w * D + d] = v[(int64_t)i * D + d];
    fc[w] = co[i];
    fi[w] = ix[i];
    ++w;
  }
  c[11] = (unsigned)w;
  c[12] = w > 0 ? 1u : 0u;
}

__global__ void k_finalize(char* res, ResLayout RL, int p, int D, double eps) {
  if (threadIdx.x == 0 && blockIdx.x == 0) compact_chosen(res, RL, p, D, eps);
}

// restart r's PCG64 state = SeedSequence(entropy=seed, spawn_key=(r,)) (particle_opt.py:176-178)
__global__ void k_restart_begin(RestartParams* rp) {
  if (threadIdx.x == 0 && blockIdx.x == 0) rp->st = seedseq_pcg64_dev(rp->seed, rp->restart);
}

// end of one restart: accumulate the flag count; stop at the first restart with any
// satisfying particle (particle_opt.py:360-376) or after max_restarts (:325, :385-400)
__global__ void k_restart_end(cudaGraphConditionalHandle h, RestartParams* rp, char* res, ResLayout RL, int p, int D,
                              double eps, int max_restarts) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned int* c = reinterpret_cast<unsigned int*>(res);
  c[10] += c[1];
  const unsigned int r = rp->restart;
  c[8] = r;
  const bool sat = c[0] > 0;
  const bool stop = sat || (int)r + 1 >= max_restarts;
  if (sat) compact_chosen(res, RL, p, D, eps);
  c[9] = stop ? 1u : 0u;
  if (!stop) rp->restart = r + 1;
  cudaGraphSetConditional(h, stop ? 0u : 1u);
}

// the timing events of a pending solve
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

template <typename R>
static int restart_launch_count(const Model& m, const spasm_solve_config& cfg, bool tr) {
  // sample_eval [+ tile keys], 2 sorts (3 kernels per 8-bit pass), schedule, [trace ids],
  // sat keys, gather, re-check evaluate, re-check copy
  const int bits = 8 * (int)sizeof(R);
  const int sample = (sizeof(R) == 4 && m.tile_ok && stage1_tile_mode() != 0) ? 2 : 1;
  return sample + radix_sort_launches(cfg.n, bits) + 1 + (tr ? 1 : 0) + 1 + radix_sort_launches(cfg.m, bits) + 3;
}

// Starts a solve. Graph path (reference step rule, no trace, a repeated shape): ONE graph
// launch runs every restart on the device -- no host round trip until solve_collect.
// Otherwise the restarts run from the host (one sync per restart) and the result is parsed
// here. Either way solve_collect returns it.
template <typename R>
static int solve_launch(Model& m, const spasm_solve_config& cfg, const double* warm_host, int64_t n_warm, void* ws,
                        int64_t ws_bytes, R* trace_cost, uint8_t* trace_sat, int32_t* trace_ids, cudaStream_t s) {
  using K = typename KeyOf<R>::type;
  const int D = m.dim;
  SolveLayout L = make_layout<R>(D, cfg, n_warm);
  SPASM_REQUIRE(ws != nullptr && (size_t)ws_bytes >= L.total, "solve workspace too small");
  SPASM_REQUIRE(n_warm >= 0 && n_warm <= cfg.n, "more warm seeds than particles");
  const ResLayout RL = res_layout(D, cfg.p_return);
  char* base = static_cast<char*>(ws);
  R* values = reinterpret_cast<R*>(base + L.values);
  K* keys0 = reinterpret_cast<K*>(base + L.keys0);
  K* keys1 = reinterpret_cast<K*>(base + L.keys1);
  uint32_t* idx0 = reinterpret_cast<uint32_t*>(base + L.idx0);
  uint32_t* idx1 = reinterpret_cast<uint32_t*>(base + L.idx1);
  unsigned int* hist = reinterpret_cast<unsigned int*>(base + L.hist);
  R* opt_values = reinterpret_cast<R*>(base + L.opt_values);
  R* opt_cost = reinterpret_cast<R*>(base + L.opt_cost);
  uint8_t* flagged = reinterpret_cast<uint8_t*>(base + L.flagged);
  K* sk0 = reinterpret_cast<K*>(base + L.skeys0);
  K* sk1 = reinterpret_cast<K*>(base + L.skeys1);
  uint32_t* sv0 = reinterpret_cast<uint32_t*>(base + L.svals0);
  uint32_t* sv1 = reinterpret_cast<uint32_t*>(base + L.svals1);
  R* chosen_vals = reinterpret_cast<R*>(base + L.chosen_vals);
  R* recheck = reinterpret_cast<R*>(base + L.recheck);
  double* warm_dev = reinterpret_cast<double*>(base + L.warm);
  char* res = base + L.res;
  unsigned int* counters = reinterpret_cast<unsigned int*>(res);
  double* out_vals = reinterpret_cast<double*>(res + RL.vals);
  double* out_cost = reinterpret_cast<double*>(res + RL.cost);
  double* out_recheck = reinterpret_cast<double*>(res + RL.recheck);
  int32_t* out_idx = reinterpret_cast<int32_t*>(res + RL.idx);

  if (m.pinned_bytes < L.res_bytes) {
    pinned_put(m.pinned, m.pinned_bytes);
    m.pinned = nullptr;
    m.pinned_bytes = 0;
    SPASM_CUDA_TRY(pinned_get(&m.pinned, L.res_bytes, &m.pinned_bytes));
  }
  char* host = static_cast<char*>(m.pinned);
  SolvePending& P = m.pend;
  P = SolvePending{};
  P.dtype_size = (int)sizeof(R);
  P.cfg = cfg;
  P.res_bytes = L.res_bytes;
  P.res_dev = res;
  P.ws = ws;
  P.n_warm = n_warm;

  if (n_warm > 0)
    SPASM_CUDA_TRY(cudaMemcpyAsync(warm_dev, warm_host, (size_t)n_warm * D * 8, cudaMemcpyHostToDevice, s));
  if (!m.ev0) SPASM_CUDA_TRY(cudaEventCreate(&m.ev0));
  if (!m.ev1) SPASM_CUDA_TRY(cudaEventCreate(&m.ev1));
  SPASM_CUDA_TRY(cudaEventRecord(m.ev0, s));

  const bool tr = trace_cost != nullptr && cfg.n_traced > 0;
  const int per_restart_launches = restart_launch_count<R>(m, cfg, tr && trace_ids);

  // One restart's device work on stream ss (no host copy: the result block stays on the device).
  auto body = [&](int restart, const Pcg64State& st, cudaStream_t ss) -> int {
    int r = launch_sample_eval<R>(m, st, 0, cfg.n, n_warm ? warm_dev : nullptr, n_warm, cfg.sampler, cfg.seed,
                                  (uint32_t)restart, values, keys0, idx0, ss);
    if (r) return r;
    bool in1 = false;
    if ((r = launch_sort<R>(keys0, idx0, keys1, idx1, cfg.n, hist, &in1, ss))) return r;
    const uint32_t* top = in1 ? idx1 : idx0;
    SPASM_CUDA_TRY(cudaMemsetAsync(res, 0, 16, ss));  // per-restart counters; the loop state persists
    if ((r = launch_schedule<R>(m, values, top, cfg.m, cfg.k_lin, cfg.k_quad, cfg.eta_init, cfg.alpha, cfg.epsilon,
                                opt_values, opt_cost, flagged, counters + 1, tr ? trace_cost : nullptr,
                                tr ? trace_sat : nullptr, tr ? cfg.n_traced : 0, step_rule(cfg, restart), ss)))
      return r;
    if (tr && trace_ids) {
      k_trace_ids<<<ceil_div(cfg.n_traced, 256), 256, 0, ss>>>(top, cfg.n_traced, trace_ids);
      SPASM_CHECK_LAUNCH();
    }
    if ((r = launch_sat_keys<R>(opt_cost, cfg.m, cfg.epsilon, sk0, sv0, counters, ss))) return r;
    bool sin1 = false;
    if ((r = launch_sort<R>(sk0, sv0, sk1, sv1, cfg.m, hist, &sin1, ss))) return r;
    const uint32_t* order = sin1 ? sv1 : sv0;
    k_gather_chosen<R><<<cfg.p_return, 32, 0, ss>>>(order, counters, cfg.p_return, opt_values, opt_cost, top, D,
                                                    chosen_vals, out_vals, out_cost, out_idx);
    SPASM_CHECK_LAUNCH();
    // independent soundness re-check: fresh QUADRATIC evaluation of the chosen rows
    if ((r = launch_evaluate<R>(m, chosen_vals, cfg.p_return, 1, recheck, ss))) return r;
    k_copy_recheck<R><<<ceil_div(cfg.p_return, 128), 128, 0, ss>>>(recheck, cfg.p_return, out_recheck);
    SPASM_CHECK_LAUNCH();
    return SPASM_OK;
  };

  // graph of the whole restart loop (reference GD step, no trace): built once per (model,
  // workspace, config) and relaunched for every later solve with the same shapes:
  //   memset(loop state) -> H2D(seed) -> WHILE { k_restart_begin, restart body, k_restart_end }
  //   -> D2H(result block)
  bool use_graph = g_graphs && !tr && step_rule(cfg, 0).is_reference();
  if (use_graph) {
    Model::GraphKeyPod key;
    std::memset(&key, 0, sizeof(key));
    key.ws = ws;
    key.host = host;
    key.dtype = (int)sizeof(R);
    key.n = cfg.n;
    key.m = cfg.m;
    key.k_lin = cfg.k_lin;
    key.k_quad = cfg.k_quad;
    key.eta = cfg.eta_init;
    key.alpha = cfg.alpha;
    key.eps = cfg.epsilon;
    key.p_return = cfg.p_return;
    key.max_restarts = cfg.max_restarts;
    key.sampler = cfg.sampler;
    key.n_warm = n_warm;
    key.tile = stage1_tile_mode();
    key.tower_lanes = tower_lanes_option();
    const bool cached = m.gexec && std::memcmp(&key, &m.gkey, sizeof(key)) == 0;
    // capture only from the second solve with the same shapes: a model solved once (e.g. a
    // replanning tick's fresh model) never pays for a capture it would not reuse
    const bool repeat = std::memcmp(&key, &m.gkey_seen, sizeof(key)) == 0;
    m.gkey_seen = key;
    if (!cached && !repeat) use_graph = false;
  }
  if (use_graph) {
    const Model::GraphKeyPod& key = m.gkey_seen;
    if (!m.gexec || std::memcmp(&key, &m.gkey, sizeof(key)) != 0) {
      if (m.gexec) cudaGraphExecDestroy(m.gexec);
      m.gexec = nullptr;
      if (!m.cap) SPASM_CUDA_TRY(cudaStreamCreateWithFlags(&m.cap, cudaStreamNonBlocking));
      if (!m.rp_dev) SPASM_CUDA_TRY(cudaMalloc(&m.rp_dev, sizeof(RestartParams)));
      if (!m.rp_host) SPASM_CUDA_TRY(cudaMallocHost(&m.rp_host, sizeof(RestartParams)));
      cudaGraph_t g = nullptr;
      SPASM_CUDA_TRY(cudaGraphCreate(&g, 0));
      struct GraphGuard {
        cudaGraph_t g;
        ~GraphGuard() {
          if (g) cudaGraphDestroy(g);
        }
      } guard{g};
      cudaGraphConditionalHandle h;
      SPASM_CUDA_TRY(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
      cudaGraphNode_t n_set, n_rp, n_loop, n_out;
      cudaMemsetParams ms{};
      ms.dst = res;
      ms.value = 0;
      ms.elementSize = 4;
      ms.width = 16;  // the 64-byte counter block
      ms.height = 1;
      SPASM_CUDA_TRY(cudaGraphAddMemsetNode(&n_set, g, nullptr, 0, &ms));
      SPASM_CUDA_TRY(cudaGraphAddMemcpyNode1D(&n_rp, g, &n_set, 1, m.rp_dev, m.rp_host, sizeof(RestartParams),
                                              cudaMemcpyHostToDevice));
      cudaGraphNodeParams wp{};
      wp.type = cudaGraphNodeTypeConditional;
      wp.conditional.handle = h;
      wp.conditional.type = cudaGraphCondTypeWhile;
      wp.conditional.size = 1;
      SPASM_CUDA_TRY(cudaGraphAddNode(&n_loop, g, &n_rp, 1, &wp));
      cudaGraph_t loop_body = wp.conditional.phGraph_out[0];
      SPASM_CUDA_TRY(cudaStreamBeginCaptureToGraph(m.cap, loop_body, nullptr, nullptr, 0,
                                                   cudaStreamCaptureModeThreadLocal));
      k_restart_begin<<<1, 1, 0, m.cap>>>(m.rp_dev);
      g_restart_override = m.rp_dev;
      int r = body(0, restart_state(cfg.seed, 0), m.cap);
      g_restart_override = nullptr;
      if (!r) {
        k_restart_end<<<1, 32, 0, m.cap>>>(h, m.rp_dev, res, RL, cfg.p_return, D, cfg.epsilon, cfg.max_restarts);
        if (cudaGetLastError() != cudaSuccess) r = SPASM_ERR_CUDA;
      }
      cudaGraph_t captured = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(m.cap, &captured);
      if (r) {
        if (r == SPASM_ERR_CUDA) set_last_error("restart-loop capture: kernel launch failed");
        return r;
      }
      SPASM_CUDA_TRY(ec);
      SPASM_CUDA_TRY(cudaGraphAddMemcpyNode1D(&n_out, g, &n_loop, 1, host, res, L.res_bytes, cudaMemcpyDeviceToHost));
      SPASM_CUDA_TRY(cudaGraphInstantiate(&m.gexec, g, 0));
      m.gkey = key;
    }
    m.rp_host->seed = cfg.seed;
    m.rp_host->restart = 0;
    SPASM_CUDA_TRY(cudaGraphLaunch(m.gexec, s));
    SPASM_CUDA_TRY(cudaEventRecord(m.ev1, s));
    P.graph = true;
    P.per_restart_launches = per_restart_launches + 2;  // + k_restart_begin / k_restart_end
    P.active = true;
    return SPASM_OK;
  }

  // host-driven restarts: one sync per restart to read n_sat (particle_opt.py:325-376)
  SPASM_CUDA_TRY(cudaMemsetAsync(res, 0, 64, s));
  const int per_restart = cfg.k_lin + cfg.k_quad;
  const double* h_vals = reinterpret_cast<const double*>(host + RL.vals);
  const double* h_cost = reinterpret_cast<const double*>(host + RL.cost);
  const double* h_re = reinterpret_cast<const double*>(host + RL.recheck);
  const int32_t* h_idx = reinterpret_cast<const int32_t*>(host + RL.idx);
  spasm_solve_report& rep = P.rep;
  std::memset(&rep, 0, sizeof(rep));
  P.rc = SPASM_NO_SOLUTION;
  P.rows.clear();
  int total_steps = 0, total_flagged = 0, launches = 0;
  for (int restart = 0; restart < cfg.max_restarts; ++restart) {
    const int r = body(restart, restart_state(cfg.seed, (uint64_t)restart), s);
    if (r) return r;
    SPASM_CUDA_TRY(cudaMemcpyAsync(host, res, L.res_bytes, cudaMemcpyDeviceToHost, s));
    SPASM_CUDA_TRY(cudaStreamSynchronize(s));
    const unsigned int* hc = reinterpret_cast<const unsigned int*>(host);
    total_steps += per_restart;
    launches += per_restart_launches;
    total_flagged += (int)hc[1];
    const int n_sat = (int)hc[0];
    if (n_sat > 0) {
      const int k = std::min(n_sat, (int)cfg.p_return);
      for (int c = 0; c < k; ++c) {
        if (!(h_re[c] < cfg.epsilon)) continue;  // chosen = chosen[recheck]
        P.rows.insert(P.rows.end(), h_vals + (size_t)c * D, h_vals + (size_t)(c + 1) * D);
        P.costs.push_back(h_cost[c]);
        P.idx.push_back(h_idx[c]);
      }
      const int w = (int)P.costs.size();
      rep.success = w > 0;
      rep.restarts = restart;
      rep.n_satisfying = n_sat;
      rep.n_chosen = w;
      P.rc = w > 0 ? SPASM_OK : SPASM_NO_SOLUTION;
      // the compacted rows for device consumers (stage-2 lifting), as the graph path leaves them
      k_finalize<<<1, 1, 0, s>>>(res, RL, cfg.p_return, D, cfg.epsilon);
      SPASM_CHECK_LAUNCH();
      launches += 1;
      break;
    }
    rep.restarts = cfg.max_restarts;
  }
  rep.steps = total_steps;
  rep.launches = launches;
  rep.flagged = total_flagged;
  SPASM_CUDA_TRY(cudaEventRecord(m.ev1, s));
  P.graph = false;
  P.active = true;
  return SPASM_OK;
}

// Waits for a launched solve (the only host sync of the graph path) and fills the outputs.
static int solve_collect(Model& m, double* particles, double* costs, int64_t* indices, spasm_solve_report* rep) {
  SolvePending& P = m.pend;
  SPASM_REQUIRE(P.active, "no launched solve to collect");
  P.active = false;
  const int D = m.dim;
  const spasm_solve_config& cfg = P.cfg;
  SPASM_CUDA_TRY(cudaEventSynchronize(m.ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, m.ev0, m.ev1);
  if (!P.graph) {
    *rep = P.rep;
    rep->device_ms = ms;
    const int w = (int)P.costs.size();
    if (w > 0) std::memcpy(particles, P.rows.data(), (size_t)w * D * 8);
    for (int c = 0; c < w; ++c) {
      costs[c] = P.costs[c];
      indices[c] = P.idx[c];
    }
    return P.rc;
  }
  const ResLayout RL = res_layout(D, cfg.p_return);
  const char* host = static_cast<const char*>(m.pinned);
  const unsigned int* hc = reinterpret_cast<const unsigned int*>(host);
  std::memset(rep, 0, sizeof(*rep));
  const int last = (int)hc[8];
  const int n_sat = (int)hc[0];
  const int runs = n_sat > 0 ? last + 1 : cfg.max_restarts;
  rep->steps = runs * (cfg.k_lin + cfg.k_quad);
  rep->launches = runs * P.per_restart_launches;
  rep->flagged = (int)hc[10];
  rep->device_ms = ms;
  if (n_sat == 0) {
    rep->restarts = cfg.max_restarts;
    return SPASM_NO_SOLUTION;
  }
  const int w = (int)hc[11];
  std::memcpy(particles, host + RL.fvals, (size_t)w * D * 8);
  std::memcpy(costs, host + RL.fcost, (size_t)w * 8);
  const int32_t* fi = reinterpret_cast<const int32_t*>(host + RL.fidx);
  for (int c = 0; c < w; ++c) indices[c] = fi[c];
  rep->success = w > 0;
  rep->restarts = last;
  rep->n_satisfying = n_sat;
  rep->n_chosen = w;
  return w > 0 ? SPASM_OK : SPASM_NO_SOLUTION;
}

}  // namespace spasm

using namespace spasm;

struct spasm_model : public spasm::Model {};

extern "C" {

const char* spasm_last_error(void) { return spasm::last_error(); }
int spasm_version(void) { return 1; }

int spasm_trim(void) {
  spasm::pinned_trim();
  return SPASM_OK;
}

int64_t spasm_abi_sizeof(const char* type_name) {
  if (type_name == nullptr) return -1;
  const std::string n(type_name);
  if (n == "spasm_solve_config") return sizeof(spasm_solve_config);
  if (n == "spasm_solve_report") return sizeof(spasm_solve_report);
  if (n == "spasm_chain") return sizeof(spasm_chain);
  if (n == "spasm_traj_desc") return sizeof(spasm_traj_desc);
  if (n == "spasm_al_config") return sizeof(spasm_al_config);
  if (n == "spasm_al_result") return sizeof(spasm_al_result);
  return -1;
}

static int fill_bounds(Model& m, int D, const double* lower, const double* upper) {
  SPASM_REQUIRE(D >= 1 && D <= kMaxDim, "state dimension out of range (1..128)");
  for (int d = 0; d < D; ++d) {
    SPASM_REQUIRE(lower[d] <= upper[d], "lower bound exceeds upper bound");
    m.bounds.lo[d] = lower[d];
    m.bounds.hi[d] = upper[d];
  }
  return SPASM_OK;
}

}  // extern "C"

template <typename R>
static void fill_tetris(TetrisScene<R>& s, int n_bodies, const int32_t* spb, const double* lc, const double* rad,
                        int n_static, const double* sc, const double* sr, const double* sn, double wbb, double wbs,
                        double wh, double zs, int free_yaw, const Bounds64& b, int D) {
  std::memset(&s, 0, sizeof(s));
  s.n_bodies = n_bodies;
  s.n_static = n_static;
  s.free_yaw = free_yaw ? 1 : 0;
  s.dim = D;
  int off = 0;
  int uniform = n_bodies > 0 ? spb[0] : 0;
  for (int i = 0; i < n_bodies; ++i) {
    s.body_start[i] = off;
    off += spb[i];
    if (spb[i] != uniform) uniform = 0;
  }
  s.body_start[n_bodies] = off;
  s.n_mov = off;
  s.spb = (uniform == 1 || uniform == 2 || uniform == 4) ? uniform : 0;
  for (int a = 0; a < off; ++a) {
    s.lx[a] = (R)lc[3 * a];
    s.ly[a] = (R)lc[3 * a + 1];
    s.lz[a] = (R)lc[3 * a + 2];
    s.rad[a] = (R)rad[a];
  }
  for (int t = 0; t < n_static; ++t) {
    const double cx = sc[3 * t], cy = sc[3 * t + 1], cz = sc[3 * t + 2], r = sr[t];
    const double nx = sn[3 * t], ny = sn[3 * t + 1], nz = sn[3 * t + 2];
    s.sx[t] = (R)cx;
    s.sy[t] = (R)cy;
    s.sz[t] = (R)cz;
    s.sr[t] = (R)r;
    s.ax[t] = (R)(cx + r * nx);
    s.ay[t] = (R)(cy + r * ny);
    s.az[t] = (R)(cz + r * nz);
    s.nx[t] = (R)nx;
    s.ny[t] = (R)ny;
    s.nz[t] = (R)nz;
  }
  s.w_bb = (R)wbb;
  s.w_bs = (R)wbs;
  s.w_h = (R)wh;
  s.z_star = (R)zs;
  for (int d = 0; d < D; ++d) {
    s.lower[d] = (R)b.lo[d];
    s.upper[d] = (R)b.hi[d];
  }
}

// The fp32 tile kernel covers tetris scenes with 4 spheres per body of one radius, the 4
// box walls, fixed yaw and at most kTileMaxBodies bodies (stage1_tile.cuh).
static void fill_tile(Model& m, int n_bodies, const int32_t* spb, const double* lc, const double* rad, int n_static,
                      const double* sc, const double* sr, const double* sn, double wbb, double wbs, double wh,
                      double zs, int free_yaw) {
  m.tile_ok = false;
  if (free_yaw || n_bodies < 1 || n_bodies > kTileMaxBodies || n_static != kTileWalls) return;
  for (int i = 0; i < n_bodies; ++i)
    if (spb[i] != kTileSpb) return;
  const int S = n_bodies * kTileSpb;
  for (int a = 1; a < S; ++a)
    if (rad[a] != rad[0]) return;
  // walls must be box_wall_spheres' layout: normals +x, -x, +y, -y, one radius, one plane
  static const double kN[kTileWalls][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}};
  for (int w = 0; w < kTileWalls; ++w) {
    for (int k = 0; k < 3; ++k)
      if (sn[3 * w + k] != kN[w][k]) return;
    if (sr[w] != sr[0] || sc[3 * w + 2] != sc[2]) return;
  }
  if (sc[1] != sc[4] || sc[6] != sc[9]) return;
  TetrisTileScene& t = m.tile;
  std::memset(&t, 0, sizeof(t));
  t.n = n_bodies;
  for (int a = 0; a < S; ++a) {
    t.lx[a] = (float)lc[3 * a];
    t.ly[a] = (float)lc[3 * a + 1];
    t.lz[a] = (float)lc[3 * a + 2];
  }
  auto pack = [](float lo, float hi) {
    uint32_t l, h;
    std::memcpy(&l, &lo, 4);
    std::memcpy(&h, &hi, 4);
    return (unsigned long long)l | ((unsigned long long)h << 32);
  };
  for (int a = 0; a < S; a += 2) {
    t.px[a / 2] = pack(t.lx[a], t.lx[a + 1]);
    t.py[a / 2] = pack(t.ly[a], t.ly[a + 1]);
    t.pz[a / 2] = pack(t.lz[a], t.lz[a + 1]);
  }
  const double R = sr[0];
  for (int w = 0; w < kTileWalls; ++w) {
    const int axis = w < 2 ? 0 : 1;
    t.wall_a[w] = (float)(sc[3 * w + axis] + R * sn[3 * w + axis]);  // tangent point
  }
  t.wall_ay_x = (float)sc[1];
  t.wall_ax_y = (float)sc[6];
  t.wall_az = (float)sc[2];
  t.wr = (float)R;
  t.wr2 = (float)R * (float)R;
  t.two_wr = 2.f * (float)R;
  t.r = (float)rad[0];
  t.wa_x = pack(t.wall_a[0], t.wall_a[1]);
  t.wa_y = pack(t.wall_a[2], t.wall_a[3]);
  t.two_wr_pm = pack(t.two_wr, -t.two_wr);
  t.wr_pm = pack(t.wr, -t.wr);
  t.wr2_d = pack(t.wr2, t.wr2);
  t.wr_d = pack(t.wr, t.wr);
  t.r_d = pack(t.r, t.r);
  t.rs = 2.f * t.r;
  t.rs2 = t.rs * t.rs;
  t.rs_d = pack(t.rs, t.rs);
  t.m1_d = pack(-1.f, -1.f);
  t.tiny_d = pack(1e-30f, 1e-30f);
  t.w_bb = (float)wbb;
  t.w_bs = (float)wbs;
  t.k_bs_d = pack(-2.f * t.w_bs, -2.f * t.w_bs);
  t.w_h = (float)wh;
  t.z_star = (float)zs;
  for (int d = 0; d < 3 * n_bodies; ++d) {
    t.lower[d] = (float)m.bounds.lo[d];
    t.upper[d] = (float)m.bounds.hi[d];
  }
  m.tile_ok = true;
}

extern "C" {

int spasm_set_option(const char* key, int value) {
  SPASM_REQUIRE(key != nullptr, "null option key");
  if (std::strcmp(key, "graphs") == 0) {
    SPASM_REQUIRE(value == 0 || value == 1, "graphs must be 0 or 1");
    g_graphs = value;
    return SPASM_OK;
  }
  if (std::strcmp(key, "ik_cluster") == 0) {
    SPASM_REQUIRE(value == 0 || value == 1 || value == 2 || value == 4 || value == 8,
                  "ik_cluster must be 0 (auto), 1, 2, 4 or 8");
    g_ik_cluster = value;
    return SPASM_OK;
  }
  if (std::strcmp(key, "tower_lanes") == 0) {
    SPASM_REQUIRE(value == 0 || value == 1 || value == 2 || value == 4 || value == 8,
                  "tower_lanes must be 0 (auto), 1, 2, 4 or 8");
    g_tower_lanes = value;
    return SPASM_OK;
  }
  if (std::strcmp(key, "stage1_tile") == 0) {
    SPASM_REQUIRE(value >= -1 && value <= 4, "stage1_tile must be -1 (auto), 0 (off) or 1..4");
    g_stage1_tile = value;
    return SPASM_OK;
  }
  set_last_error(std::string("unknown option: ") + key);
  return SPASM_ERR_USAGE;
}

int spasm_tetris_model_create(spasm_model** out, int n_bodies, const int32_t* spheres_per_body,
                              const double* local_centers, const double* radii, int n_static,
                              const double* static_centers, const double* static_radii,
                              const double* static_normals, double w_block_block, double w_block_wall,
                              double w_height, double z_star, int free_yaw, const double* lower,
                              const double* upper) {
  SPASM_REQUIRE(out != nullptr, "null output handle");
  SPASM_REQUIRE(n_bodies >= 1 && n_bodies <= kMaxBodies, "n_bodies out of range (1..16)");
  SPASM_REQUIRE(n_static >= 0 && n_static <= kMaxStatic, "too many static spheres (max 32)");
  int total = 0;
  for (int i = 0; i < n_bodies; ++i) {
    SPASM_REQUIRE(spheres_per_body[i] >= 1, "every body needs at least one sphere");
    total += spheres_per_body[i];
  }
  SPASM_REQUIRE(total <= kMaxMov, "too many movable spheres (max 128)");
  const int D = n_bodies * (free_yaw ? 4 : 3);
  spasm_model* m = new (std::nothrow) spasm_model();
  SPASM_REQUIRE(m != nullptr, "out of host memory");
  m->kind = ModelKind::Tetris;
  m->dim = D;
  int rc = fill_bounds(*m, D, lower, upper);
  if (rc) {
    delete m;
    return rc;
  }
  fill_tetris<float>(m->tf, n_bodies, spheres_per_body, local_centers, radii, n_static, static_centers, static_radii,
                     static_normals, w_block_block, w_block_wall, w_height, z_star, free_yaw, m->bounds, D);
  fill_tetris<double>(m->td, n_bodies, spheres_per_body, local_centers, radii, n_static, static_centers,
                      static_radii, static_normals, w_block_block, w_block_wall, w_height, z_star, free_yaw,
                      m->bounds, D);
  fill_tile(*m, n_bodies, spheres_per_body, local_centers, radii, n_static, static_centers, static_radii,
            static_normals, w_block_block, w_block_wall, w_height, z_star, free_yaw);
  *out = m;
  return SPASM_OK;
}

}  // extern "C"

template <typename R>
static void fill_tower(TowerScene<R>& s, int nb, double side, double half, const double* tg, int no, const double* oc,
                       const double* orad, double ws, double wh, double wc, int free_yaw, const Bounds64& b, int D) {
  std::memset(&s, 0, sizeof(s));
  s.n_blocks = nb;
  s.n_obs = no;
  s.free_yaw = free_yaw ? 1 : 0;
  s.dim = D;
  s.side = (R)side;
  s.half = (R)half;
  s.radius = (R)(0.5 * side);
  for (int i = 0; i < nb; ++i) s.target[i] = (R)tg[i];
  for (int o = 0; o < no; ++o) {
    s.ox[o] = (R)oc[3 * o];
    s.oy[o] = (R)oc[3 * o + 1];
    s.oz[o] = (R)oc[3 * o + 2];
    s.orad[o] = (R)orad[o];
  }
  s.w_s = (R)ws;
  s.w_h = (R)wh;
  s.w_c = (R)wc;
  for (int d = 0; d < D; ++d) {
    s.lower[d] = (R)b.lo[d];
    s.upper[d] = (R)b.hi[d];
  }
}

extern "C" {

int spasm_tower_model_create(spasm_model** out, int n_blocks, double side, double footprint_halfwidth,
                             const double* height_targets, int n_obstacles, const double* obstacle_centers,
                             const double* obstacle_radii, double w_stability, double w_height,
                             double w_collision, int free_yaw, const double* lower, const double* upper) {
  SPASM_REQUIRE(out != nullptr, "null output handle");
  SPASM_REQUIRE(n_blocks >= 2 && n_blocks <= kMaxTowerBlocks, "n_blocks out of range (2..32)");
  SPASM_REQUIRE(n_obstacles >= 0 && n_obstacles <= kMaxObstacles, "too many obstacles (max 64)");
  SPASM_REQUIRE(side > 0, "cube side must be positive");
  const int D = n_blocks * (free_yaw ? 4 : 3);
  spasm_model* m = new (std::nothrow) spasm_model();
  SPASM_REQUIRE(m != nullptr, "out of host memory");
  m->kind = ModelKind::Tower;
  m->dim = D;
  int rc = fill_bounds(*m, D, lower, upper);
  if (rc) {
    delete m;
    return rc;
  }
  fill_tower<float>(m->wf, n_blocks, side, footprint_halfwidth, height_targets, n_obstacles, obstacle_centers,
                    obstacle_radii, w_stability, w_height, w_collision, free_yaw, m->bounds, D);
  fill_tower<double>(m->wd, n_blocks, side, footprint_halfwidth, height_targets, n_obstacles, obstacle_centers,
                     obstacle_radii, w_stability, w_height, w_collision, free_yaw, m->bounds, D);
  // fp32 tower tile kernel (stage1_tower_tile.cuh): fixed yaw, <= kTowerTileMaxBlocks cubes
  m->tower_tile_ok = !free_yaw && n_blocks >= 2 && n_blocks <= kTowerTileMaxBlocks && n_obstacles <= kMaxObstacles;
  if (m->tower_tile_ok) {
    TowerTileScene& t = m->tower_tile;
    std::memset(&t, 0, sizeof(t));
    t.n = n_blocks;
    t.n_obs = n_obstacles;
    t.side = m->wf.side;
    t.half = m->wf.half;
    t.radius = m->wf.radius;
    for (int i = 0; i < n_blocks; ++i) t.target[i] = m->wf.target[i];
    for (int o = 0; o < n_obstacles; ++o) {
      t.ox[o] = m->wf.ox[o];
      t.oy[o] = m->wf.oy[o];
      t.oz[o] = m->wf.oz[o];
      t.orad[o] = m->wf.orad[o];
    }
    t.w_s = m->wf.w_s;
    t.w_h = m->wf.w_h;
    t.w_c = m->wf.w_c;
    for (int d = 0; d < D; ++d) {
      t.lower[d] = m->wf.lower[d];
      t.upper[d] = m->wf.upper[d];
    }
  }
  *out = m;
  return SPASM_OK;
}

void spasm_model_destroy(spasm_model* model) {
  if (!model) return;
  pinned_put(model->pinned, model->pinned_bytes);
  if (model->gexec) cudaGraphExecDestroy(model->gexec);
  if (model->cap) cudaStreamDestroy(model->cap);
  if (model->rp_dev) cudaFree(model->rp_dev);
  if (model->rp_host) cudaFreeHost(model->rp_host);
  if (model->ev0) cudaEventDestroy(model->ev0);
  if (model->ev1) cudaEventDestroy(model->ev1);
  delete model;
}

int spasm_model_dimension(const spasm_model* model) { return model ? model->dim : -1; }


int spasm_evaluate(const spasm_model* model, int dtype, const void* values, int64_t P, int mode, void* costs,
                   void* stream) {
  SPASM_REQUIRE(model != nullptr, "null model");
  SPASM_REQUIRE(mode == SPASM_LINEAR || mode == SPASM_QUADRATIC, "unknown cost mode");
  SPASM_DTYPE_SWITCH(dtype, return launch_evaluate<R>(*model, static_cast<const R*>(values), P, mode,
                                                      static_cast<R*>(costs), as_stream(stream)););
}

int spasm_gradient(const spasm_model* model, int dtype, const void* values, int64_t P, int mode, void* grad,
                   void* stream) {
  SPASM_REQUIRE(model != nullptr, "null model");
  SPASM_REQUIRE(mode == SPASM_LINEAR || mode == SPASM_QUADRATIC, "unknown cost mode");
  SPASM_DTYPE_SWITCH(dtype, return launch_gradient<R>(*model, static_cast<const R*>(values), P, mode,
                                                      static_cast<R*>(grad), as_stream(stream)););
}

int spasm_pcg64_state(uint64_t seed, uint64_t restart, uint64_t out[4]) {
  SPASM_REQUIRE(out != nullptr, "null output");
  seedseq_pcg64(seed, &restart, 1, out);
  return SPASM_OK;
}

int spasm_sample(int dtype, int D, const double* lower, const double* upper, uint64_t seed, uint64_t restart,
                 int sampler, int64_t row_offset, int64_t N, const double* warm_dev, int64_t n_warm, void* values,
                 void* stream) {
  SPASM_REQUIRE(D >= 1 && D <= kMaxDim, "state dimension out of range (1..128)");
  SPASM_REQUIRE(N >= 0 && row_offset >= 0, "negative row range");
  Bounds64 b;
  for (int d = 0; d < D; ++d) {
    b.lo[d] = lower[d];
    b.hi[d] = upper[d];
  }
  const Pcg64State st = restart_state(seed, restart);
  SPASM_DTYPE_SWITCH(dtype, return launch_sample<R>(b, D, st, row_offset, nullptr, N, warm_dev, n_warm, sampler, seed,
                                                    (uint32_t)restart, static_cast<R*>(values), as_stream(stream)););
}

int spasm_sample_eval(const spasm_model* model, int dtype, uint64_t seed, uint64_t restart, int sampler,
                      int64_t row_offset, int64_t N, const double* warm_dev, int64_t n_warm, void* values, void* keys,
                      uint32_t* idx, void* stream) {
  SPASM_REQUIRE(model != nullptr, "null model");
  SPASM_REQUIRE(N >= 0 && row_offset >= 0, "negative row range");
  const Pcg64State st = restart_state(seed, restart);
  SPASM_DTYPE_SWITCH(dtype, return launch_sample_eval<R>(*model, st, row_offset, N, warm_dev, n_warm, sampler, seed,
                                                         (uint32_t)restart, static_cast<R*>(values),
                                                         static_cast<typename KeyOf<R>::type*>(keys), idx,
                                                         as_stream(stream)););
}

int spasm_step(int dtype, void* values, const void* grad, int64_t P, int D, double rate, const void* lower,
               const void* upper, uint8_t* flagged, void* stream) {
  SPASM_REQUIRE(rate >= 0, "rate must be >= 0");
  SPASM_DTYPE_SWITCH(dtype, return launch_step<R>(static_cast<R*>(values), static_cast<const R*>(grad), P, D, (R)rate,
                                                  static_cast<const R*>(lower), static_cast<const R*>(upper), flagged,
                                                  as_stream(stream)););
}

int spasm_descent_schedule(const spasm_model* model, int dtype, const void* src, const uint32_t* rows, int64_t M,
                           int k_lin, int k_quad, double eta_init, double alpha, double epsilon, void* out_values,
                           void* out_cost, uint8_t* flagged, uint32_t* flagged_count, void* trace_cost,
                           uint8_t* trace_sat, int n_traced, void* stream) {
  SPASM_REQUIRE(model != nullptr, "null model");
  SPASM_REQUIRE(k_lin >= 0 && k_quad >= 0, "step counts must be nonnegative");
  SPASM_DTYPE_SWITCH(dtype, return launch_schedule<R>(*model, static_cast<const R*>(src), rows, M, k_lin, k_quad,
                                                      eta_init, alpha, epsilon, static_cast<R*>(out_values),
                                                      static_cast<R*>(out_cost), flagged, flagged_count,
                                                      static_cast<R*>(trace_cost), trace_sat, n_traced,
                                                      StepRule{}, as_stream(stream)););
}

int64_t spasm_sort_workspace_bytes(int dtype, int64_t n) {
  const int64_t ksz = dtype == SPASM_F64 ? 8 : 4;
  const int64_t tiles = (n + 2047) / 2048 + 1;
  return align_up((size_t)(n * ksz)) + align_up((size_t)(n * 4)) + align_up((size_t)(tiles * 256 * 4));
}

int spasm_sort_pairs(int dtype, void* keys, uint32_t* vals, int64_t n, void* workspace, void* stream) {
  SPASM_REQUIRE(n >= 0 && n <= (int64_t)0xFFFFFFFF, "sort size out of range");
  if (n <= 1) return SPASM_OK;
  SPASM_REQUIRE(workspace != nullptr, "null sort workspace");
  const int64_t ksz = dtype == SPASM_F64 ? 8 : 4;
  char* w = static_cast<char*>(workspace);
  void* k1 = w;
  uint32_t* v1 = reinterpret_cast<uint32_t*>(w + align_up((size_t)(n * ksz)));
  unsigned int* hist = reinterpret_cast<unsigned int*>(w + align_up((size_t)(n * ksz)) + align_up((size_t)(n * 4)));
  cudaStream_t s = as_stream(stream);
  SPASM_DTYPE_SWITCH(dtype, {
    using K = typename KeyOf<R>::type;
    bool in1 = false;
    int r = launch_sort<R>(static_cast<K*>(keys), vals, static_cast<K*>(k1), v1, n, hist, &in1, s);
    if (r) return r;
    if (in1) {
      SPASM_CUDA_TRY(cudaMemcpyAsync(keys, k1, (size_t)(n * ksz), cudaMemcpyDeviceToDevice, s));
      SPASM_CUDA_TRY(cudaMemcpyAsync(vals, v1, (size_t)(n * 4), cudaMemcpyDeviceToDevice, s));
    }
    return SPASM_OK;
  });
}

int spasm_cost_keys(int dtype, const void* costs, int64_t P, double threshold, void* keys, uint32_t* vals,
                    uint32_t* n_below, void* stream) {
  SPASM_REQUIRE(P >= 0, "negative size");
  SPASM_DTYPE_SWITCH(dtype, {
    using K = typename KeyOf<R>::type;
    return launch_sat_keys<R>(static_cast<const R*>(costs), P, threshold, static_cast<K*>(keys), vals,
                              reinterpret_cast<unsigned int*>(n_below), as_stream(stream));
  });
}

int64_t spasm_solve_workspace_bytes(const spasm_model* model, int dtype, const spasm_solve_config* cfg,
                                    int64_t n_warm) {
  if (!model || !cfg) return -1;
  if (dtype == SPASM_F64) return (int64_t)make_layout<double>(model->dim, *cfg, n_warm).total;
  return (int64_t)make_layout<float>(model->dim, *cfg, n_warm).total;
}

int spasm_solve(const spasm_model* model, int dtype, const spasm_solve_config* cfg, const double* warm_host,
                int64_t n_warm, void* workspace, int64_t workspace_bytes, double* particles, double* costs,
                int64_t* indices, spasm_solve_report* report, void* trace_cost, uint8_t* trace_sat,
                int32_t* trace_ids, void* stream) {
  SPASM_REQUIRE(model != nullptr, "null model");
  int r = validate_cfg(cfg);
  if (r) return r;
  SPASM_REQUIRE(particles && costs && indices && report, "null output buffer");
  Model& m = const_cast<spasm_model&>(*model);
  SPASM_DTYPE_SWITCH(dtype, r = solve_launch<R>(m, *cfg, warm_host, n_warm, workspace, workspace_bytes,
                                                static_cast<R*>(trace_cost), trace_sat, trace_ids, as_stream(stream)););
  if (r) return r;
  return solve_collect(m, particles, costs, indices, report);
}

int spasm_solve_launch(const spasm_model* model, int dtype, const spasm_solve_config* cfg, const double* warm_host,
                       int64_t n_warm, void* workspace, int64_t workspace_bytes, void* stream) {
  SPASM_REQUIRE(model != nullptr, "null model");
  int r = validate_cfg(cfg);
  if (r) return r;
  Model& m = const_cast<spasm_model&>(*model);
  SPASM_DTYPE_SWITCH(dtype, return solve_launch<R>(m, *cfg, warm_host, n_warm, workspace, workspace_bytes, nullptr,
                                                   nullptr, nullptr, as_stream(stream)););
}

int spasm_solve_collect(const spasm_model* model, double* particles, double* costs, int64_t* indices,
                        spasm_solve_report* report) {
  SPASM_REQUIRE(model != nullptr, "null model");
  SPASM_REQUIRE(particles && costs && indices && report, "null output buffer");
  return solve_collect(const_cast<spasm_model&>(*model), particles, costs, indices, report);
}

int spasm_solve_device_rows(const spasm_model* model, const double** rows, const int32_t** n_rows) {
  SPASM_REQUIRE(model != nullptr && rows && n_rows, "null argument");
  const Model& m = *model;
  SPASM_REQUIRE(m.pend.res_dev != nullptr, "no launched solve");
  const ResLayout RL = res_layout(m.dim, m.pend.cfg.p_return);
  *rows = reinterpret_cast<const double*>(m.pend.res_dev + RL.fvals);
  *n_rows = reinterpret_cast<const int32_t*>(m.pend.res_dev) + 11;
  return SPASM_OK;
}

}  // extern "C"
