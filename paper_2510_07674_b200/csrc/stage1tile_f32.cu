// Dispatcher of the fp32 tetris tile kernels (stage1_tile.cuh, stage1tile_n<N>_f32.cu).
#include "stage1tile.hpp"

namespace spasm {

namespace {

// 4 lanes per particle measured fastest on B200 for every batch size (C3 tetris5 M =
// 8192: 53 us vs 213 us with one lane; C5 tetris8 M = 131072: 4.45 ms vs 6.5 ms, the
// one-lane N = 8 kernel overflows the instruction cache); it is the only variant built.
int auto_variant(int64_t) { return 4; }

}  // namespace

int launch_schedule_tile(const Model& m, const float* src, const uint32_t* rows, int64_t M, int k_lin, int k_quad,
                         double eta, double alpha, float* out_values, float* out_cost, uint8_t* flagged,
                         unsigned int* flagged_count, cudaStream_t s) {
  const int mode = stage1_tile_mode();
  if (!m.tile_ok || mode == 0 || M <= 0) return -1;
  const int variant = mode > 0 ? mode : auto_variant(M);
  const TetrisTileScene& sc = m.tile;
  // body counts without an instantiation fall back to the generic kernel
  switch (sc.n) {
    case 1: return launch_tile_n<1>(variant, sc, src, rows, M, k_lin, k_quad, eta, alpha, out_values, out_cost, flagged, flagged_count, s);
    case 4: return launch_tile_n<4>(variant, sc, src, rows, M, k_lin, k_quad, eta, alpha, out_values, out_cost, flagged, flagged_count, s);
    case 5: return launch_tile_n<5>(variant, sc, src, rows, M, k_lin, k_quad, eta, alpha, out_values, out_cost, flagged, flagged_count, s);
    case 6: return launch_tile_n<6>(variant, sc, src, rows, M, k_lin, k_quad, eta, alpha, out_values, out_cost, flagged, flagged_count, s);
    case 8: return launch_tile_n<8>(variant, sc, src, rows, M, k_lin, k_quad, eta, alpha, out_values, out_cost, flagged, flagged_count, s);
    default: return -1;
  }
}

int launch_sample_eval_tile(const Model& m, const Pcg64State& st, int64_t row_offset, int64_t rows_n,
                            const double* warm, int64_t n_warm, int use_philox, uint64_t seed, uint32_t restart,
                            float* values, uint32_t* keys, uint32_t* idx, cudaStream_t s) {
  if (!m.tile_ok || stage1_tile_mode() == 0 || rows_n <= 0) return -1;
  const TetrisTileScene& sc = m.tile;
  int r = launch_sample<float>(m.bounds, 3 * sc.n, st, row_offset, nullptr, rows_n, warm, n_warm, use_philox, seed,
                               restart, values, s);
  if (r) return r;
#define SPASM_TILE_KEYS_CASE(n) \
  case n: return launch_keys_tile_n<n>(sc, values, row_offset, rows_n, keys, idx, s);
  switch (sc.n) {
    SPASM_TILE_BODIES(SPASM_TILE_KEYS_CASE)
    default: return -1;
  }
#undef SPASM_TILE_KEYS_CASE
}

}  // namespace spasm
