// fp32 ("perf") instantiation of the stage-2 kernels.
#include "stage2_launch.cuh"
#define SPASM_R float
#include "stage2_inst.inc"

// Diagnostic: phase timer of the fp32 AL kernel (al_tile.cuh AlProf). enable = 1 turns it
// on, 0 off; out (optional, 12 doubles) receives the accumulated cycles per mark, then the
// counters are reset.
extern "C" int spasm_al_profile(int enable, double* out) {
  using namespace spasm;
  SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_al_prof_on, &enable, sizeof(int)));
  if (out) {
    unsigned long long h[12];
    SPASM_CUDA_TRY(cudaMemcpyFromSymbol(h, g_al_prof, sizeof(h)));
    for (int k = 0; k < 12; ++k) out[k] = (double)h[k];
    const unsigned long long z[12] = {0};
    SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_al_prof, z, sizeof(z)));
  }
  return SPASM_OK;
}
