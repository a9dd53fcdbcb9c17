// Declarations of the stage-1 launchers shared by the C-ABI translation units
// (capi.cu, shard.cu). The templates are explicitly instantiated once per precision in
// stage1_f32.cu / stage1_f64.cu (stage1_inst.inc) so each precision keeps its own
// compiler flags.
#pragma once
#include "model.hpp"
#include "rng.cuh"
#include "sort.cuh"

// Binds R to the arithmetic type selected by a SPASM_F32 / SPASM_F64 dtype argument.
#define SPASM_DTYPE_SWITCH(dtype, ...)                          \
  do {                                                          \
    if ((dtype) == SPASM_F32) {                                 \
      using R = float;                                          \
      __VA_ARGS__                                               \
    } else if ((dtype) == SPASM_F64) {                          \
      using R = double;                                         \
      __VA_ARGS__                                               \
    } else {                                                    \
      spasm::set_last_error("dtype must be SPASM_F32 or SPASM_F64"); \
      return SPASM_ERR_USAGE;                                   \
    }                                                           \
  } while (0)

namespace spasm {

int stage1_tile_mode();  // spasm_set_option("stage1_tile")
int tower_lanes_option();  // spasm_set_option("tower_lanes")
void seedseq_pcg64(uint64_t seed, const uint64_t* spawn_key, int n_spawn, uint64_t out[4]);

// ---- launchers (explicitly instantiated in stage1_f32.cu / stage1_f64.cu) ----------
template <typename R> int launch_evaluate(const Model&, const R*, int64_t, int, R*, cudaStream_t);
template <typename R> int launch_gradient(const Model&, const R*, int64_t, int, R*, cudaStream_t);
template <typename R>
int launch_sample_eval(const Model&, const Pcg64State&, int64_t, int64_t, const double*, int64_t, int, uint64_t,
                       uint32_t, R*, typename KeyOf<R>::type*, uint32_t*, cudaStream_t);
template <typename R>
int launch_schedule(const Model&, const R*, const uint32_t*, int64_t, int, int, double, double, double, R*, R*,
                    uint8_t*, unsigned int*, R*, uint8_t*, int, const StepRule&, cudaStream_t);
template <typename R>
int launch_sample(const Bounds64&, int, const Pcg64State&, int64_t, const uint32_t*, int64_t, const double*, int64_t,
                  int, uint64_t, uint32_t, R*, cudaStream_t);
template <typename R>
int launch_step(R*, const R*, int64_t, int, R, const R*, const R*, uint8_t*, cudaStream_t);
template <typename R>
int launch_sort(typename KeyOf<R>::type*, uint32_t*, typename KeyOf<R>::type*, uint32_t*, int64_t, unsigned int*,
                bool*, cudaStream_t);
template <typename R>
int launch_sat_keys(const R*, int64_t, double, typename KeyOf<R>::type*, uint32_t*, unsigned int*, cudaStream_t);

extern template int launch_evaluate<float>(const Model&, const float*, int64_t, int, float*, cudaStream_t);
extern template int launch_evaluate<double>(const Model&, const double*, int64_t, int, double*, cudaStream_t);

inline Pcg64State restart_state(uint64_t seed, uint64_t restart) {
  uint64_t o[4];
  seedseq_pcg64(seed, &restart, 1, o);
  Pcg64State s;
  s.state_hi = o[0];
  s.state_lo = o[1];
  s.inc_hi = o[2];
  s.inc_lo = o[3];
  return s;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace spasm
