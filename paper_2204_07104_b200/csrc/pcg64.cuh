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

}  // namespace sptk
