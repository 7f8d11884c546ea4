// numpy-compatible pair sampling for fit_variogram (kriging.py:278-286).
//
// The reference draws ``default_rng(seed).integers(0, m, max_pairs)`` twice.
// That is numpy's SeedSequence -> PCG64 (128-bit LCG, XSL-RR output) with
// 32-bit Lemire bounded draws whenever m - 1 fits in 32 bits; each 64-bit
// output is consumed as its low half, then its high half, and the buffered
// half carries over between the two ``integers`` calls.  A half h is accepted
// iff (h*m mod 2^32) >= (2^32 mod m) and then yields (h*m) >> 32, so the
// draw sequence is a stream compaction of accepted halves -- which is what
// the device kernel computes in parallel with LCG jump-ahead.
//
// The algorithms restated here are numpy's published ones (numpy 2.3:
// bit_generator.pyx SeedSequence, pcg64.h/pcg64.c, distributions.c
// buffered_bounded_lemire_uint32); there is no numpy code in this file.
#pragma once
#include <cstdint>
#include "vk_common.h"

namespace vk {

typedef unsigned __int128 u128;

struct Pcg64 {
  u128 state, inc;
};

// PCG_DEFAULT_MULTIPLIER_128
VK_HD u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

VK_HD uint64_t pcg_output(u128 s) {  // XSL-RR 128/64
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// State after ``delta`` LCG steps (Brown's jump-ahead, O(log delta)).
VK_HD u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// Raw 64-bit output number r (0-based) of a freshly seeded generator: numpy
// steps the LCG and then outputs the new state.
VK_HD uint64_t pcg_raw_at(const Pcg64& g, uint64_t r) {
  return pcg_output(pcg_advance(g.state, g.inc, r + 1));
}

// ---- SeedSequence(seed) -> PCG64 state (host only; O(1)) ------------------
inline uint32_t ss_hashmix(uint32_t value, uint32_t& hash_const) {
  value ^= hash_const;
  hash_const *= 0x931e8875u;
  value *= hash_const;
  value ^= value >> 16;
  return value;
}
inline uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  r ^= r >> 16;
  return r;
}

// numpy.random.PCG64(seed) for a non-negative integer seed.
inline Pcg64 pcg64_from_seed(uint64_t seed) {
  // entropy -> uint32 words, least significant first; 0 -> [0]
  uint32_t ent[2];
  int n_ent = 0;
  if (seed == 0) {
    ent[n_ent++] = 0;
  } else {
    while (seed) {
      ent[n_ent++] = (uint32_t)(seed & 0xffffffffu);
      seed >>= 32;
    }
  }
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n_ent ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  for (int s = 4; s < n_ent; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], hc));
  // generate_state(4, uint64): 8 uint32 words cycling over the pool
  uint32_t w[8];
  uint32_t hb = 0x8b51f9ddu;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= 0x58f38dedu;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  uint64_t v64[4];
  for (int i = 0; i < 4; ++i) v64[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  // pcg64_set_seed(state, seed=v64[0:2], inc=v64[2:4]); 128-bit = (hi<<64)|lo
  const u128 initstate = ((u128)v64[0] << 64) | v64[1];
  const u128 initseq = ((u128)v64[2] << 64) | v64[3];
  Pcg64 g;
  g.state = 0;
  g.inc = (initseq << 1) | 1u;
  g.state = g.state * pcg_mult() + g.inc;
  g.state += initstate;
  g.state = g.state * pcg_mult() + g.inc;
  return g;
}

// Lemire 32-bit acceptance test and value for a range m (= rng + 1).
// threshold = (2^32 - m) mod m  (distributions.c: (UINT32_MAX - rng) % rng_excl)
VK_HD uint32_t lemire_threshold(uint32_t m) { return (uint32_t)(0u - m) % m; }

}  // namespace vk
