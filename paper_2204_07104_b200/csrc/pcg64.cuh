// pcg64.cuh -- numpy's PCG64 (XSL-RR 128/64) on the device, with O(log n)
// jump-ahead so every thread can start at an arbitrary stream position.
//
// Stream convention (numpy _pcg64.pyx / pcg64.h): output m (m = 0, 1, ...) is
// XSL-RR of the state after m+1 LCG steps.  The buffered 32-bit draws that
// Generator.permutation / choice consume are position q = 2m (low half of
// output m) and q = 2m+1 (high half), in that order (pcg64_next32).
#pragma once
#include <stdint.h>

namespace sptk {

typedef unsigned __int128 u128;

struct Pcg64 {
  u128 state;
  u128 inc;
};

__host__ __device__ inline u128 pcg_mult() {
  return (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;
}

__host__ __device__ inline uint64_t pcg_xsl_rr(u128 s) {
  uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// LCG affine map for `delta` steps: state' = mult*state + plus.
__host__ __device__ inline void pcg_jump_coeffs(u128 inc, uint64_t delta, u128* mult, u128* plus) {
  u128 acc_m = 1, acc_p = 0, cur_m = pcg_mult(), cur_p = inc;
  while (delta) {
    if (delta & 1) {
      acc_m *= cur_m;
      acc_p = acc_p * cur_m + cur_p;
    }
    cur_p = (cur_m + 1) * cur_p;
    cur_m *= cur_m;
    delta >>= 1;
  }
  *mult = acc_m;
  *plus = acc_p;
}

// State after `delta` more steps.
__host__ __device__ inline u128 pcg_advance(const Pcg64& g, uint64_t delta) {
  u128 m, p;
  pcg_jump_coeffs(g.inc, delta, &m, &p);
  return m * g.state + p;
}

// 32-bit draw at stream position q.
__device__ inline uint32_t pcg_u32_at(const Pcg64& g, uint64_t q) {
  uint64_t out = pcg_xsl_rr(pcg_advance(g, (q >> 1) + 1));
  return (q & 1) ? (uint32_t)(out >> 32) : (uint32_t)out;
}

// numpy.random.SeedSequence(entropy) (pool size 4) -> PCG64 seeding
// (pcg64_set_seed -> pcg_setseq_128_srandom_r), as np.random.default_rng
// does it (trainer.py:196-198, trainer.py:214).  Entropy values are split
// into little-endian 32-bit words (0 -> one zero word); at most 64 words.
__host__ __device__ inline uint32_t ss_hashmix(uint32_t v, uint32_t* hc) {
  v ^= *hc;
  *hc *= 0x931e8875u;
  v *= *hc;
  v ^= v >> 16;
  return v;
}
__host__ __device__ inline uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  r ^= r >> 16;
  return r;
}
// returns the number of 32-bit words, or -1 if the entropy is too long
__host__ __device__ inline int seedseq_words(const uint64_t* ent, int n_ent, uint32_t* words, int cap) {
  int nw = 0;
  for (int e = 0; e < n_ent; ++e) {
    uint64_t x = ent[e];
    if (x == 0) {
      if (nw >= cap) return -1;
      words[nw++] = 0;
    }
    while (x) {
      if (nw >= cap) return -1;
      words[nw++] = (uint32_t)(x & 0xffffffffu);
      x >>= 32;
    }
  }
  return nw;
}
__host__ __device__ inline Pcg64 seedseq_pcg64(const uint32_t* words, int nw) {
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < nw ? words[i] : 0u, &hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = 4; s < nw; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(words[s], &hc));
  uint32_t out[8];
  uint32_t hb = 0x8b51f9ddu;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= 0x58f38dedu;
    v *= hb;
    v ^= v >> 16;
    out[i] = v;
  }
  uint64_t v64[4];
  for (int k = 0; k < 4; ++k) v64[k] = (uint64_t)out[2 * k] | ((uint64_t)out[2 * k + 1] << 32);
  const u128 initstate = ((u128)v64[0] << 64) | v64[1];
  const u128 initseq = ((u128)v64[2] << 64) | v64[3];
  Pcg64 g;
  g.inc = (initseq << 1) | 1u;
  g.state = 0;
  g.state = g.state * pcg_mult() + g.inc;
  g.state += initstate;
  g.state = g.state * pcg_mult() + g.inc;
  return g;
}

}  // namespace sptk
