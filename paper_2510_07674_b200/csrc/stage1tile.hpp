// Launch helpers of the fp32 tetris tile kernels (stage1_tile.cuh). Each body count N
// is instantiated in its own translation unit (stage1tile_n<N>_f32.cu, built with the
// fp32 flags) so the fully unrolled variants compile in parallel.
#pragma once
#include "stage1_launch.cuh"

namespace spasm {

template <int N>
int launch_tile_n(int variant, const TetrisTileScene& sc, const float* src, const uint32_t* rows, int64_t M, int k_lin,
                  int k_quad, double eta, double alpha, float* ov, float* oc, uint8_t* fl, unsigned int* fc,
                  cudaStream_t s);

template <int N>
int launch_keys_tile_n(const TetrisTileScene& sc, const float* values, int64_t row_offset, int64_t rows_n,
                       uint32_t* keys, uint32_t* idx, cudaStream_t s);

#define SPASM_TILE_BODIES(X) X(1) X(4) X(5) X(6) X(8)
#define SPASM_TILE_DECL(n)                                                                                        \
  extern template int launch_tile_n<n>(int, const TetrisTileScene&, const float*, const uint32_t*, int64_t, int, \
                                       int, double, double, float*, float*, uint8_t*, unsigned int*, cudaStream_t);
SPASM_TILE_BODIES(SPASM_TILE_DECL)
#define SPASM_TILE_SAMPLE_DECL(n)                                                                             \
  extern template int launch_keys_tile_n<n>(const TetrisTileScene&, const float*, int64_t, int64_t, uint32_t*, \
                                            uint32_t*, cudaStream_t);
SPASM_TILE_BODIES(SPASM_TILE_SAMPLE_DECL)

}  // namespace spasm
