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

// Diagnostic: k_ik_group counters (stage2_kernels.cuh g_ik_prof). enable 1/0; out (12
// doubles, optional) receives and resets them.
extern "C" int spasm_ik_profile(int enable, double* out) {
  using namespace spasm;
  SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_ik_prof_on, &enable, sizeof(int)));
  if (out) {
    unsigned long long h[12];
    SPASM_CUDA_TRY(cudaMemcpyFromSymbol(h, g_ik_prof, sizeof(h)));
    for (int k = 0; k < 12; ++k) out[k] = (double)h[k];
    static const unsigned long long z[12] = {0};
    SPASM_CUDA_TRY(cudaMemcpyToSymbol(g_ik_prof, z, sizeof(z)));
  }
  return SPASM_OK;
}

// Self-test of the fp32 branch-free math against the reference routines, on the device:
// counts[0] = atan2_nobranch vs atan2f bit mismatches (n pseudo-random (y, x) pairs: raw bit
// patterns incl. zeros / infinities / NaNs, and small-range values), counts[1] = the
// normalize_yaw fold vs wrap_yaw in its fast range, counts[2] = the np.mod fold vs
// np_mod_pos in its fast range (NaN == NaN counts as equal).
namespace spasm {
__global__ void k_selftest_math(int64_t n, uint64_t seed, unsigned long long* bad) {
  unsigned long long b0 = 0, b1 = 0, b2 = 0;
  const float two_pi = 6.283185307179586476925286766559f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = ((uint64_t)i + seed) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    float y = __uint_as_float((unsigned)h), x = __uint_as_float((unsigned)(h >> 32));
    if (i & 1) {
      y = (float)((int)(h & 0xffff) - 32768) * 1e-4f;
      x = (float)((int)((h >> 16) & 0xffff) - 32768) * 1e-4f;
    }
    const float a = atan2f(y, x), c = atan2_nobranch(y, x);
    if (__float_as_uint(a) != __float_as_uint(c) && !(a != a && c != c)) ++b0;
    // yaw differences in (-2 pi, 2 pi) and joint offsets in [-pi, 4 pi): the fast ranges
    const float d = (float)((int)((h >> 20) & 0xfffff) - 524288) * (2.f * two_pi / 524288.f) * 0.999f;
    if (wrap_yaw_in_fast_range(d)) {
      const float w0 = wrap_yaw(d), w1 = wrap_yaw_finish(wrap_yaw_fold(d + 3.1415926535897932384626433832795f));
      if (__float_as_uint(w0) != __float_as_uint(w1)) ++b1;
    }
    const float m = (float)((int)((h >> 40) & 0xfffff)) * (5.f * 3.14159265f / 1048576.f) - 3.14159265f;
    if (np_mod_in_fast_range(m, two_pi)) {
      const float r0 = np_mod_pos(m, two_pi), r1 = np_mod_finish(m >= two_pi ? m - two_pi : m, two_pi);
      if (__float_as_uint(r0) != __float_as_uint(r1)) ++b2;
    }
  }
  atomicAdd(&bad[0], b0);
  atomicAdd(&bad[1], b1);
  atomicAdd(&bad[2], b2);
}
}  // namespace spasm

extern "C" int spasm_selftest_math(int64_t n, uint64_t seed, int64_t* counts) {
  using namespace spasm;
  SPASM_REQUIRE(n >= 0 && counts != nullptr, "n must be >= 0 and counts non-null");
  unsigned long long* d = nullptr;
  SPASM_CUDA_TRY(cudaMalloc(&d, 3 * sizeof(unsigned long long)));
  SPASM_CUDA_TRY(cudaMemset(d, 0, 3 * sizeof(unsigned long long)));
  k_selftest_math<<<4 * kNumSMs, 256>>>(n, seed, d);
  unsigned long long h[3];
  const cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  SPASM_CUDA_TRY(e);
  for (int k = 0; k < 3; ++k) counts[k] = (int64_t)h[k];
  return SPASM_OK;
}
