// Device restatement of numpy's SeedSequence -> PCG64 seeding (bit_generator.pyx
// SeedSequence, pcg64.c pcg64_set_seed) for the streams the stage-2 path derives per
// target / per call:
//   np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(key,)))
// (reference robot.py:255-257 per IK target, bench.py:88-91 trajectory stream).
// Same algorithm as the host copy in seedseq.cpp; entropy <= 2 words, spawn key <= 2 words.
#pragma once
#include <stdint.h>

#include "rng.cuh"

namespace spasm {

__host__ __device__ inline Pcg64State seedseq_pcg64_dev(uint64_t seed, uint64_t key) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
  const uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t ent[8];
  int n = 0;
  // run entropy words (0 -> one zero word)
  if (seed == 0) {
    ent[n++] = 0u;
  } else {
    for (uint64_t v = seed; v; v >>= 32) ent[n++] = (uint32_t)(v & 0xFFFFFFFFu);
  }
  while (n < 4) ent[n++] = 0u;  // spawn key present: pad run entropy to the pool size
  if (key == 0) {
    ent[n++] = 0u;
  } else {
    for (uint64_t v = key; v; v >>= 32) ent[n++] = (uint32_t)(v & 0xFFFFFFFFu);
  }
  uint32_t hash_const = INIT_A;
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) {
    uint32_t value = ent[i] ^ hash_const;
    hash_const *= MULT_A;
    value *= hash_const;
    value ^= value >> 16;
    pool[i] = value;
  }
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) {
        uint32_t value = pool[s] ^ hash_const;
        hash_const *= MULT_A;
        value *= hash_const;
        value ^= value >> 16;
        uint32_t r = MIX_L * pool[d] - MIX_R * value;
        pool[d] = r ^ (r >> 16);
      }
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) {
      uint32_t value = ent[s] ^ hash_const;
      hash_const *= MULT_A;
      value *= hash_const;
      value ^= value >> 16;
      uint32_t r = MIX_L * pool[d] - MIX_R * value;
      pool[d] = r ^ (r >> 16);
    }
  uint32_t hc = INIT_B;
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4] ^ hc;
    hc *= MULT_B;
    v *= hc;
    v ^= v >> 16;
    w[i] = v;
  }
  uint64_t u[4];
  for (int i = 0; i < 4; ++i) u[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  const u128 mult = make_u128(SPASM_PCG_MULT_HI, SPASM_PCG_MULT_LO);
  const u128 initstate = make_u128(u[0], u[1]);
  const u128 inc = (make_u128(u[2], u[3]) << 1) | (u128)1u;
  u128 st = 0;
  st = st * mult + inc;
  st += initstate;
  st = st * mult + inc;
  Pcg64State out;
  out.state_hi = (uint64_t)(st >> 64);
  out.state_lo = (uint64_t)st;
  out.inc_hi = (uint64_t)(inc >> 64);
  out.inc_lo = (uint64_t)inc;
  return out;
}

}  // namespace spasm
