// Device random streams.
//
// PCG64 (XSL-RR 128/64, numpy's default BitGenerator) with O(log n) jump-ahead so
// every particle row draws exactly the numbers numpy's single centralized stream
// would hand it: row i of an (N, D) draw consumes outputs i*D .. i*D+D-1
// (reference: particle_opt.py:176-192, numpy Generator.uniform in C order).
//
// Philox4x32-10 is the counter-based stream for perf-mode extras (noise injection,
// north_star item 4); it is never used on a parity path.
#pragma once
#include <stdint.h>

namespace spasm {

typedef unsigned __int128 u128;

struct Pcg64State {
  uint64_t state_hi, state_lo;  // 128-bit LCG state
  uint64_t inc_hi, inc_lo;      // 128-bit odd increment
};

// The restart-dependent sampler inputs read from device memory instead of kernel arguments,
// so one captured CUDA graph of the stage-1 restart serves every restart (capi.cu).
struct RestartParams {
  Pcg64State st;
  uint64_t seed;
  uint32_t restart;
  uint32_t pad;
};

__host__ __device__ __forceinline__ u128 make_u128(uint64_t hi, uint64_t lo) {
  return ((u128)hi << 64) | (u128)lo;
}

#define SPASM_PCG_MULT_HI 0x2360ED051FC65DA4ull
#define SPASM_PCG_MULT_LO 0x4385DF649FCCF645ull

struct Pcg64 {
  u128 state, inc;

  __device__ __forceinline__ void init(const Pcg64State& s) {
    state = make_u128(s.state_hi, s.state_lo);
    inc = make_u128(s.inc_hi, s.inc_lo);
  }
  // Advance the LCG by `delta` steps (Brown's arbitrary-stride jump-ahead).
  __device__ __forceinline__ void advance(uint64_t delta) {
    u128 cur_mult = make_u128(SPASM_PCG_MULT_HI, SPASM_PCG_MULT_LO);
    u128 cur_plus = inc;
    u128 acc_mult = 1, acc_plus = 0;
    while (delta) {
      if (delta & 1) {
        acc_mult *= cur_mult;
        acc_plus = acc_plus * cur_mult + cur_plus;
      }
      cur_plus = (cur_mult + 1) * cur_plus;
      cur_mult *= cur_mult;
      delta >>= 1;
    }
    state = acc_mult * state + acc_plus;
  }
  // numpy pcg64_random_r: step, then XSL-RR output of the new state.
  __device__ __forceinline__ uint64_t next_u64() {
    state = state * make_u128(SPASM_PCG_MULT_HI, SPASM_PCG_MULT_LO) + inc;
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    uint64_t x = hi ^ lo;
    unsigned r = (unsigned)(state >> 122);
    return (x >> r) | (x << ((64u - r) & 63u));
  }
  // numpy next_double: 53 random bits scaled to [0, 1).
  __device__ __forceinline__ double next_double() {
    return (double)(next_u64() >> 11) * (1.0 / 9007199254740992.0);
  }
};

// ---- Philox4x32-10 ----------------------------------------------------------
struct Philox4x32 {
  static __device__ __forceinline__ uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  static __device__ __forceinline__ uint4 gen(uint4 ctr, uint2 key) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      ctr = round(ctr, key);
      key.x += 0x9E3779B9u;
      key.y += 0xBB67AE85u;
    }
    return ctr;
  }
  // uniform in [0,1) with 24 bits (fp32) from one 32-bit lane
  static __device__ __forceinline__ float u01(uint32_t v) { return (float)(v >> 8) * (1.0f / 16777216.0f); }
};

}  // namespace spasm
