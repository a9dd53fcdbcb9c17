// Host restatement of numpy's SeedSequence -> PCG64 seeding, so the native solve loop
// derives each restart's stream exactly as the reference's
//   np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(restart,)))
// does (reference particle_opt.py:176-178; numpy bit_generator.pyx SeedSequence,
// pcg64.c pcg64_set_seed). Verified against numpy in tests/test_native_cpu.py.
#include <stdint.h>
#include <vector>

namespace spasm {

namespace {
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
constexpr int XSHIFT = 16;

void push_u32_words(std::vector<uint32_t>& v, uint64_t n) {
  if (n == 0) {
    v.push_back(0u);
    return;
  }
  while (n) {
    v.push_back((uint32_t)(n & 0xFFFFFFFFu));
    n >>= 32;
  }
}

typedef unsigned __int128 u128;
const u128 kMult = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}  // namespace

void seedseq_pcg64(uint64_t seed, const uint64_t* spawn_key, int n_spawn, uint64_t out[4]) {
  std::vector<uint32_t> run, spawn;
  push_u32_words(run, seed);
  for (int i = 0; i < n_spawn; ++i) push_u32_words(spawn, spawn_key[i]);
  if (!spawn.empty() && run.size() < 4) run.resize(4, 0u);
  std::vector<uint32_t> ent(run);
  ent.insert(ent.end(), spawn.begin(), spawn.end());

  uint32_t hash_const = INIT_A;
  auto hashmix = [&](uint32_t value) {
    value ^= hash_const;
    hash_const *= MULT_A;
    value *= hash_const;
    value ^= value >> XSHIFT;
    return value;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> XSHIFT;
    return r;
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (size_t s = 4; s < ent.size(); ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));

  // generate_state(4, uint64): 8 words from the pool, little-endian pairs
  uint32_t hc = INIT_B;
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hc;
    hc *= MULT_B;
    v *= hc;
    v ^= v >> XSHIFT;
    w[i] = v;
  }
  uint64_t u[4];
  for (int i = 0; i < 4; ++i) u[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  // pcg64_set_seed: state = u[0]:u[1], seq = u[2]:u[3]; pcg_setseq_128_srandom_r
  const u128 initstate = ((u128)u[0] << 64) | u[1];
  const u128 initseq = ((u128)u[2] << 64) | u[3];
  const u128 inc = (initseq << 1) | 1u;
  u128 st = 0;
  st = st * kMult + inc;
  st += initstate;
  st = st * kMult + inc;
  out[0] = (uint64_t)(st >> 64);
  out[1] = (uint64_t)st;
  out[2] = (uint64_t)(inc >> 64);
  out[3] = (uint64_t)inc;
}

}  // namespace spasm
