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
  if (out) {  // out[0..11] phase times, out[12..19] tile arrivals, out[20..27] aux arrivals
    unsigned long long h[12], a[2][8];
    SPASM_CUDA_TRY(cudaMemcpyFromSymbol(h, g_al_prof, sizeof(h)));
    SPASM_CUDA_TRY(cudaMemcpyFromSymbol(a, g_al_arrive, sizeof(a)));
    for (int k = 0; k < 12; ++k) out[k] = (double)h[k];
    for (int k = 0; k < 8; ++k) {
      out[12 + k] = (double)a[0][k];
      out[20 + k] = (double)a[1][k];
    }
    const unsigned long long z[12] = {0}, za[2][8] = {{0}};
    SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_al_prof, z, sizeof(z)));
    SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_al_arrive, za, sizeof(za)));
  }
  return SPASM_OK;
}

// Diagnostic: per-warp own-work cycles of the fp32 AL kernel's phases (AlProf::arrive, lane
// 0 of every warp, summed over CTAs); out = 32 x 8 doubles [warp][phase] + 4 pick-polish
// counters (iterations, calls, calls at the iteration cap, max iterations), then reset.
extern "C" int spasm_al_profile_warps(double* out) {
  using namespace spasm;
  unsigned long long h[32][8];
  SPASM_CUDA_TRY(cudaMemcpyFromSymbol(h, g_al_warp, sizeof(h)));
  for (int w = 0; w < 32; ++w)
    for (int k = 0; k < 8; ++k) out[w * 8 + k] = (double)h[w][k];
  static const unsigned long long z[32][8] = {{0}};
  SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_al_warp, z, sizeof(z)));
  unsigned long long pol[4];
  SPASM_CUDA_TRY(cudaMemcpyFromSymbol(pol, g_al_polish, sizeof(pol)));
  for (int k = 0; k < 4; ++k) out[256 + k] = (double)pol[k];
  static const unsigned long long zp[4] = {0};
  SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_al_polish, zp, sizeof(zp)));
  return SPASM_OK;
}

// Diagnostic: k_ik_group counters (stage2_kernels.cuh g_ik_prof). enable 1/0; out (8
// doubles, optional) receives and resets them.
extern "C" int spasm_ik_profile(int enable, double* out) {
  using namespace spasm;
  SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_ik_prof_on, &enable, sizeof(int)));
  if (out) {
    unsigned long long h[8];
    SPASM_CUDA_TRY(cudaMemcpyFromSymbol(h, g_ik_prof, sizeof(h)));
    for (int k = 0; k < 8; ++k) out[k] = (double)h[k];
    static const unsigned long long z[8] = {0};
    SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_ik_prof, z, sizeof(z)));
  }
  return SPASM_OK;
}
