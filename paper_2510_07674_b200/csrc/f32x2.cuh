// Packed fp32 pairs (sm_100a FADD2 / FMUL2 / FFMA2): two independent values in one 64-bit
// register pair, one instruction for both lanes of the pair. Used by the stage-1 tile kernels
// (two sphere pairs of one particle) and the AL engine's fixed-obstacle pass (two obstacles
// of one sphere).
#pragma once
#include <cuda_runtime.h>

namespace spasm {

// ---- packed fp32 pairs (sm_100a FADD2/FMUL2/FFMA2) ----------------------------------
// Two sphere pairs of one particle share one 64-bit register pair; the scalar halves are
// plain registers (mov.b64 {lo, hi} is free aliasing), so per-component MUFU and selects
// cost nothing extra. Every op is a single PTX statement on .b64 values.
struct F2 {
  unsigned long long v;
};
__device__ __forceinline__ F2 f2_make(float lo, float hi) {
  F2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ F2 f2_dup(float a) { return f2_make(a, a); }
// mask ? a : b as one LOP3 on the bit patterns: a data select the compiler cannot turn
// into a branch (which would duplicate the unrolled pair code per mode)
__device__ __forceinline__ float pick(unsigned mask, float a, float b) {
  return __uint_as_float((mask & __float_as_uint(a)) | (~mask & __float_as_uint(b)));
}
__device__ __forceinline__ void f2_split(F2 a, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a.v));
}
__device__ __forceinline__ F2 f2_add(F2 a, F2 b) {
  F2 d;
  asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ F2 f2_sub(F2 a, F2 b) {
  F2 d;
  asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ F2 f2_mul(F2 a, F2 b) {
  F2 d;
  asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ F2 f2_fma(F2 a, F2 b, F2 c) {
  F2 d;
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return d;
}

}  // namespace spasm
