// sampler.cu -- K2: bit-exact GPU re-derivation of the reference's samplers.
//
// The reference draws, per epoch,
//   * the factor-phase visit order  default_rng([seed,1,t,*block]).permutation(len(ids))
//     (trainer.py:196-199): numpy Fisher-Yates, i = n-1..1,
//     j_i = random_interval(i) (masked rejection on buffered u32 draws);
//   * the core batch  default_rng([seed,2,t]).choice(nnz, k, replace=False)
//     (trainer.py:212-221): Floyd with Lemire draws + _shuffle_int, or the
//     tail-shuffle path (_shuffle_int over arange) when pop > 10000 and
//     k > pop // 50.
// These are inherently sequential loops over one PCG64 stream.  They are
// reproduced here exactly with three parallel building blocks:
//
//  (1) masked-rejection j-sequence (permutation).  Steps with the same mask
//      (i in [2^(k-1), 2^k)) form a segment.  Inside a segment, position q of
//      the u32 stream is accepted iff a_q <= y_q, a_q = accepts so far and
//      y_q = hi - (v_q & mask).  Chunks of L positions compute a reference
//      trajectory from a guessed count a0 (the mean curve) and record the few
//      "near-margin" positions |y_q - tau_q| < Delta.  A single resolver warp
//      then propagates the true count chunk to chunk: a shifted trajectory
//      differs from the reference only at near-margin positions (gap
//      dynamics), so each chunk costs O(#entries).  A second pass regenerates
//      every chunk from its true count and writes j_i.  Chunks whose shift is
//      out of range are walked exactly (slow path), so the result is exact
//      for every input, not just with high probability.
//  (2) Lemire draw sequences (Floyd values, _shuffle_int j's): rejections are
//      rare (< 1%); one warp walks 32 draws per round against 32 stream
//      positions staged in shared memory by the CTA's other warps, a round
//      ending at the first rejection (one test per draw, no speculation).
//      The training loop draws the core batch two epochs ahead, so this
//      single-SM walk runs underneath the other work.
//  (3) applying a Fisher-Yates swap sequence: with L_p the ascending list of
//      steps targeting p, result[l_k] = val(l_{k+1}), result[l_last] = p,
//      where val(s) (the value at position s just before step s) is the root
//      of the forest parent(s) = first step > s targeting s.  Built with two
//      bucket partitions (by target, then by step) around per-bucket counting
//      sorts, and chain walks guarded by an L2-resident has-parent bitmap.
#include <math.h>
#include <stdlib.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "pcg64.cuh"

namespace sptk {

#define FULLMASK 0xffffffffu

// ---------------------------------------------------------------------------
// raw stream
// ---------------------------------------------------------------------------
__global__ void u32_stream_kernel(Pcg64 g, unsigned long long q0, long long n, uint32_t* out) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; t < n; t += stride) out[t] = pcg_u32_at(g, q0 + (unsigned long long)t);
}

// ---------------------------------------------------------------------------
// (1) masked-rejection segments
// ---------------------------------------------------------------------------
struct Seg {
  int hi;         // largest step index of the segment
  unsigned mask;  // 2^k - 1
  int S;          // number of steps in the segment
};

// Accept flags of 64 ordered positions (lane l: position 2l (h=0), 2l+1 (h=1))
// given the exact count `a` before the group; accepted positions whose count
// would reach `cap` are dropped (the segment is over).
__device__ __forceinline__ void group_accept(int a, int y0, int y1, bool v0, bool v1, int cap,
                                             bool& acc0, bool& acc1) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  // d = y - a: a word is accepted iff (accepts before it in the group) <= d.
  // At most 63 words precede one, so d >= 63 accepts and d < 0 rejects for
  // sure; the rest are resolved by bounds: with L / H the accepts before the
  // word counting the undecided ones as rejected / accepted, d >= H accepts
  // and d < L rejects.  The first undecided word has L == H, so every pass
  // settles at least one (in practice one or two passes per group).
  const long long d0 = (long long)y0 - a, d1 = (long long)y1 - a;
  bool c0 = v0 && d0 >= 63, c1 = v1 && d1 >= 63;
  bool u0 = v0 && d0 >= 0 && d0 < 63, u1 = v1 && d1 >= 0 && d1 < 63;
  unsigned U0 = __ballot_sync(FULLMASK, u0), U1 = __ballot_sync(FULLMASK, u1);
  while (U0 | U1) {
    const unsigned A0 = __ballot_sync(FULLMASK, c0), A1 = __ballot_sync(FULLMASK, c1);
    const int lo0 = __popc(A0 & lt) + __popc(A1 & lt);
    const int hi0 = lo0 + __popc(U0 & lt) + __popc(U1 & lt);
    const int lo1 = lo0 + (c0 ? 1 : 0), hi1 = hi0 + ((c0 || u0) ? 1 : 0);
    if (u0) {
      if (d0 >= hi0) {
        c0 = true;
        u0 = false;
      } else if (d0 < lo0) {
        u0 = false;
      }
    }
    if (u1) {
      if (d1 >= hi1) {
        c1 = true;
        u1 = false;
      } else if (d1 < lo1) {
        u1 = false;
      }
    }
    U0 = __ballot_sync(FULLMASK, u0);
    U1 = __ballot_sync(FULLMASK, u1);
  }
  acc0 = c0;
  acc1 = c1;
  if (cap != 0x7fffffff) {
    unsigned b0 = __ballot_sync(FULLMASK, acc0), b1 = __ballot_sync(FULLMASK, acc1);
    int before0 = __popc(b0 & lt) + __popc(b1 & lt);
    int before1 = before0 + (acc0 ? 1 : 0);
    if (acc0 && (long long)a + before0 >= cap) acc0 = false;
    if (acc1 && (long long)a + before1 >= cap) acc1 = false;
  }
}

// Exact warp walk over positions [q_begin, q_end) starting with count a.
// Writes j_out[hi - count] = v & mask for accepted positions (if j_out), stops
// when the count reaches cap; *q_stop = position after the cap-th accept (or
// -1).  Returns the count at exit.  All 32 lanes must call it.
__device__ int walk_exact(const Pcg64& g, const u128& A32, const u128& C32, long long q_begin,
                          long long q_end, int a, const Seg sg, int cap, int* j_out,
                          long long* q_stop) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  long long mbase = q_begin >> 1;
  Pcg64 st;
  st.inc = g.inc;
  st.state = pcg_advance(g, (uint64_t)(mbase + lane + 1));
  long long stop = -1;
  while (2 * mbase < q_end && a < cap) {
    uint64_t out = pcg_xsl_rr(st.state);
    long long q0 = 2 * (mbase + lane), q1 = q0 + 1;
    bool v0 = q0 >= q_begin && q0 < q_end, v1 = q1 >= q_begin && q1 < q_end;
    unsigned u0 = (uint32_t)out & sg.mask, u1 = (uint32_t)(out >> 32) & sg.mask;
    int y0 = sg.hi - (int)u0, y1 = sg.hi - (int)u1;
    bool acc0, acc1;
    group_accept(a, y0, y1, v0, v1, cap, acc0, acc1);
    unsigned b0 = __ballot_sync(FULLMASK, acc0), b1 = __ballot_sync(FULLMASK, acc1);
    int before0 = __popc(b0 & lt) + __popc(b1 & lt);
    int before1 = before0 + (acc0 ? 1 : 0);
    if (j_out) {
      if (acc0) j_out[sg.hi - (a + before0)] = (int)u0;
      if (acc1) j_out[sg.hi - (a + before1)] = (int)u1;
    }
    int total = __popc(b0) + __popc(b1);
    if (a + total >= cap && cap != 0x7fffffff) {
      // position of the cap-th accept
      long long p = -1;
      if (acc0 && a + before0 == cap - 1) p = q0;
      if (acc1 && a + before1 == cap - 1) p = q1;
      unsigned who = __ballot_sync(FULLMASK, p >= 0);
      int src = __ffs(who) - 1;
      stop = __shfl_sync(FULLMASK, p, src) + 1;
    }
    a += total;
    st.state = st.state * A32 + C32;
    mbase += 32;
  }
  if (q_stop) *q_stop = stop;
  return a;
}

#define PERM_E_DEV 64
struct ChunkBuf {
  int* a0;
  int* D;
  int* cnt;  // number of entries (> E means overflow)
  int2* ent; // [C][E] (q_rel, margin)
  int* a_in; // true count at chunk start (written by the resolver)
  int E;
};

__device__ __forceinline__ int guess_count(const Seg& sg, long long p) {
  double a = ((double)sg.hi + 1.0) * (1.0 - exp(-(double)p / ((double)sg.mask + 1.0)));
  long long r = llrint(a);
  if (r < 0) r = 0;
  if (r > sg.S) r = sg.S;
  return (int)r;
}

// Phase A: reference trajectory per chunk (one warp per chunk c).
__device__ void perm_phaseA_body(const Pcg64& g, const long long* __restrict__ P, const Seg& sg, int L, int C,
                                 int Delta, const ChunkBuf& cb, int c) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  if (c >= C) return;
  u128 A32, C32;
  pcg_jump_coeffs(g.inc, 32, &A32, &C32);
  if (P[0] < 0) return;
  const long long q_begin = P[0] + (long long)c * L, q_end = q_begin + L;
  const int a0 = guess_count(sg, (long long)c * L);
  int a = a0, cnt = 0;
  long long mbase = q_begin >> 1;
  Pcg64 st;
  st.inc = g.inc;
  st.state = pcg_advance(g, (uint64_t)(mbase + lane + 1));
  int2* ent = cb.ent + (long long)c * cb.E;
  while (2 * mbase < q_end) {
    uint64_t out = pcg_xsl_rr(st.state);
    long long q0 = 2 * (mbase + lane), q1 = q0 + 1;
    bool v0 = q0 >= q_begin && q0 < q_end, v1 = q1 >= q_begin && q1 < q_end;
    int y0 = sg.hi - (int)((uint32_t)out & sg.mask);
    int y1 = sg.hi - (int)((uint32_t)(out >> 32) & sg.mask);
    bool acc0, acc1;
    group_accept(a, y0, y1, v0, v1, 0x7fffffff, acc0, acc1);
    unsigned b0 = __ballot_sync(FULLMASK, acc0), b1 = __ballot_sync(FULLMASK, acc1);
    int before0 = __popc(b0 & lt) + __popc(b1 & lt);
    int before1 = before0 + (acc0 ? 1 : 0);
    long long m0 = (long long)y0 - (a + before0), m1 = (long long)y1 - (a + before1);
    bool n0 = v0 && m0 >= -Delta && m0 < Delta, n1 = v1 && m1 >= -Delta && m1 < Delta;
    unsigned nb0 = __ballot_sync(FULLMASK, n0), nb1 = __ballot_sync(FULLMASK, n1);
    int i0 = cnt + __popc(nb0 & lt) + __popc(nb1 & lt), i1 = i0 + (n0 ? 1 : 0);
    if (n0 && i0 < cb.E) ent[i0] = make_int2((int)(q0 - q_begin), (int)m0);
    if (n1 && i1 < cb.E) ent[i1] = make_int2((int)(q1 - q_begin), (int)m1);
    cnt += __popc(nb0) + __popc(nb1);
    a += __popc(b0) + __popc(b1);
    st.state = st.state * A32 + C32;
    mbase += 32;
  }
  if (lane == 0) {
    cb.a0[c] = a0;
    cb.D[c] = a - a0;
    cb.cnt[c] = cnt;
  }
}

// Resolver: one warp propagates the exact count through the chunks.
// meta[0] = index of the chunk holding the segment end; P[1] = next start.
__device__ void perm_resolve_body(const Pcg64& g, long long* __restrict__ P, const Seg& sg, int L, int C,
                                  int Delta, const ChunkBuf& cb, int* __restrict__ meta,
                                  int2 (*ent_s)[PERM_E_DEV]) {
  const int lane = threadIdx.x & 31;
  u128 A32, C32;
  pcg_jump_coeffs(g.inc, 32, &A32, &C32);
  const long long Pk = P[0];
  long long a = 0;  // count at the current chunk
  if (lane == 0) meta[0] = -1;
  if (Pk < 0) {
    if (lane == 0) P[1] = -1;
    return;
  }
  for (int c0 = 0; c0 < C; c0 += 32) {
    const int c = c0 + lane;
    const bool valid = c < C;
    int a0 = 0, D = 0, cnt = 0;
    if (valid) {
      a0 = cb.a0[c];
      D = cb.D[c];
      cnt = cb.cnt[c];
    }
    const bool ovf = cnt > cb.E;
    const int ne = ovf ? 0 : cnt;
    for (int e = 0; e < ne; ++e) ent_s[lane][e] = cb.ent[(long long)c * cb.E + e];
    __syncwarp();
    int trig = 0;          // assumed (a0 + D + g) deficit: out = in + D - trig
    bool fixed = !valid;   // input final and trig exact (or past the end)
    long long in = 0;
    // Jacobi sweeps: every lane re-evaluates its chunk at the input implied by
    // the current trig values of the lanes before it.  The first lane whose
    // value changes (or that needs an exact walk) has a final input, so each
    // sweep fixes at least one lane; in practice 2-4 sweeps settle a batch.
    for (int it = 0; it < 70; ++it) {
      int contrib = valid ? D - trig : 0;
      int incl = contrib;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULLMASK, incl, o);
        if (lane >= o) incl += y;
      }
      in = a + (incl - contrib);
      const long long delta = in - a0;
      const bool walk = !fixed && (ovf || delta >= Delta || delta <= -Delta);
      int ntrig = trig;
      if (!fixed && !walk) {
        int gg = (int)delta;
        for (int e = 0; e < ne; ++e) {
          int m = ent_s[lane][e].y;
          if (gg > 0 && m >= 0 && m < gg) --gg;
          else if (gg < 0 && m >= gg && m < 0) ++gg;
        }
        ntrig = (int)delta - gg;
      }
      const unsigned badm = __ballot_sync(FULLMASK, walk || ntrig != trig);
      if (badm == 0) break;
      const int f = __ffs(badm) - 1;
      if (__shfl_sync(FULLMASK, (int)walk, f)) {
        const long long in_f = __shfl_sync(FULLMASK, in, f);
        const int D_f = __shfl_sync(FULLMASK, D, f);
        const long long qb = Pk + (long long)(c0 + f) * L;
        const int out_f = walk_exact(g, A32, C32, qb, qb + L, (int)in_f, sg, 0x7fffffff, nullptr, nullptr);
        if (lane == f) {
          trig = (int)(in_f + D_f - out_f);
          fixed = true;
        }
      } else {
        if (!walk) trig = ntrig;
        if (lane == f) fixed = true;
      }
    }
    long long out = in + D - trig;
    // segment end inside this batch?
    unsigned endm = __ballot_sync(FULLMASK, valid && out >= sg.S);
    if (valid && (endm == 0 || lane <= __ffs(endm) - 1)) cb.a_in[c] = (int)in;
    if (endm) {
      int e = __ffs(endm) - 1;
      long long in_e = __shfl_sync(FULLMASK, in, e);
      long long qb = Pk + (long long)(c0 + e) * L;
      long long qs = -1;
      walk_exact(g, A32, C32, qb, qb + L, (int)in_e, sg, sg.S, nullptr, &qs);
      if (lane == 0) {
        meta[0] = c0 + e;
        P[1] = qs;
      }
      return;
    }
    a = __shfl_sync(FULLMASK, out, 31);
    __syncwarp();
  }
  if (lane == 0) {
    meta[0] = -2;  // ran out of chunks: caller reports an error
    P[1] = -1;
  }
}

// Phase B: regenerate each chunk from its exact count and write j.
__device__ void perm_phaseB_body(const Pcg64& g, const long long* __restrict__ P, const Seg& sg, int L, int C,
                                 const ChunkBuf& cb, const int* __restrict__ meta, int* __restrict__ j_out, int c) {
  const int c_end = meta[0];
  if (c >= C || c_end < 0 || c > c_end || P[0] < 0) return;
  u128 A32, C32;
  pcg_jump_coeffs(g.inc, 32, &A32, &C32);
  const long long qb = P[0] + (long long)c * L;
  walk_exact(g, A32, C32, qb, qb + L, cb.a_in[c], sg, sg.S, j_out, nullptr);
}

// Small segments k = kmax_small..1 walked by one warp.
__device__ void perm_small_body(const Pcg64& g, const long long* __restrict__ P, int kstart, long long n,
                                int* __restrict__ j_out, long long* __restrict__ q_final) {
  u128 A32, C32;
  pcg_jump_coeffs(g.inc, 32, &A32, &C32);
  long long q = P[0];
  for (int k = kstart; k >= 1 && q >= 0; --k) {
    Seg sg;
    long long hi = (1LL << k) - 1;
    if (hi > n - 1) hi = n - 1;
    long long lo = 1LL << (k - 1);
    sg.hi = (int)hi;
    sg.mask = (unsigned)((1ULL << k) - 1);
    sg.S = (int)(hi - lo + 1);
    long long qs = -1;
    walk_exact(g, A32, C32, q, 0x3fffffffffffffffLL, 0, sg, sg.S, j_out, &qs);
    q = qs;
  }
  if ((threadIdx.x & 31) == 0 && q_final) *q_final = q;
}

// ---- batched j-generation: several permutations (e.g. a rank's DSGD blocks)
// advance segment level by segment level together, one launch per phase for
// all of them (a single permutation is a batch of one).
struct PermJob {
  Pcg64 g;
  long long* P;  // this block's start slot for the level
  int* meta;
  int* j_out;
  Seg sg;
  int L, C, Delta;
  int chunk0;  // first chunk of this job in the level's chunk space
  ChunkBuf cb;
};
struct SmallJob {
  Pcg64 g;
  long long* P;
  int kstart;
  long long n;
  int* j_out;
  long long* q_final;
};

__device__ __forceinline__ int find_job(const PermJob* __restrict__ jobs, int nj, int w) {
  int lo = 0, hi = nj - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].chunk0 <= w) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void perm_phaseA_batched(const PermJob* __restrict__ jobs, int nj, int total) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= total) return;
  const PermJob& jb = jobs[find_job(jobs, nj, w)];
  perm_phaseA_body(jb.g, jb.P, jb.sg, jb.L, jb.C, jb.Delta, jb.cb, w - jb.chunk0);
}

__global__ void perm_resolve_batched(const PermJob* __restrict__ jobs) {
  __shared__ int2 ent_s[32][PERM_E_DEV];
  const PermJob& jb = jobs[blockIdx.x];
  perm_resolve_body(jb.g, jb.P, jb.sg, jb.L, jb.C, jb.Delta, jb.cb, jb.meta, ent_s);
}

__global__ void perm_phaseB_batched(const PermJob* __restrict__ jobs, int nj, int total) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= total) return;
  const PermJob& jb = jobs[find_job(jobs, nj, w)];
  perm_phaseB_body(jb.g, jb.P, jb.sg, jb.L, jb.C, jb.cb, jb.meta, jb.j_out, w - jb.chunk0);
}

__global__ void perm_small_batched(const SmallJob* __restrict__ jobs) {
  const SmallJob& jb = jobs[blockIdx.x];
  perm_small_body(jb.g, jb.P, jb.kstart, jb.n, jb.j_out, jb.q_final);
}


// ---------------------------------------------------------------------------
// (2) Lemire draw sequences (one CTA, one walking warp)
// ---------------------------------------------------------------------------
// Draw t (t in [0,T)) asks for a value in [0, rng_t], rng_t = base + dir*t,
// via buffered_bounded_lemire_uint32; stream values v[] start at position Q0
// (v[0] is position Q0).  Writes out[t] and *q_end_out (position after the
// last draw, relative to Q0).
__device__ __forceinline__ bool lemire_ok(uint32_t v, uint32_t rng, uint32_t* res) {
  uint32_t rng_excl = rng + 1u;
  uint64_t m = (uint64_t)v * rng_excl;
  uint32_t left = (uint32_t)m;
  *res = (uint32_t)(m >> 32);
  if (left >= rng_excl) return true;
  uint32_t thr = (0xffffffffu - rng) % rng_excl;
  return left >= thr;
}

// Lemire draw walker: one CTA, warp 0 walks the draws, warps 1..7 stage the
// pre-generated stream v[] into a shared-memory ring ahead of it.  Each walker
// round tests 32 consecutive draws against 32 consecutive stream positions
// (one Lemire test per lane); the first rejecting lane ends the round and its
// draw retries at the next position, so a round costs one test per lane and
// the walk makes ~T/32 + (#rejections) rounds -- the work of the sequential
// loop itself, with no speculative tests.
#define LW_RING_LOG 13
#define LW_RING (1 << LW_RING_LOG)
#define LW_BLK 256
#define LW_NB (LW_RING / LW_BLK)
__global__ void __launch_bounds__(256) lemire_walk_kernel(const uint32_t* __restrict__ v, long long vcap, long long T,
                                                          long long base, int dir, uint32_t* __restrict__ out,
                                                          long long* __restrict__ q_end_out, int* __restrict__ err,
                                                          const int* __restrict__ only_if = nullptr) {
  // only_if: fallback of the parallel walker (lp_*): run only if it failed
  if (only_if && *only_if == 0) return;
  __shared__ uint32_t ring[LW_RING];
  __shared__ long long ready[LW_NB];
  __shared__ long long cons;
  __shared__ int done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int b = tid; b < LW_NB; b += blockDim.x) ready[b] = -1;
  if (tid == 0) {
    cons = 0;
    done = 0;
  }
  __syncthreads();
  volatile long long* vready = ready;
  volatile long long* vcons = &cons;
  volatile int* vdone = &done;
  const long long nblk = (vcap + LW_BLK - 1) / LW_BLK;
  if (warp > 0) {
    // producers: warp w stages blocks w-1, w-1+7, ...
    const int np = (blockDim.x >> 5) - 1;
    for (long long b = warp - 1; b < nblk; b += np) {
      // block b overwrites block b - LW_NB: wait until the walker is past it
      while ((*vcons) < (b - LW_NB + 1) * LW_BLK && !(*vdone)) __nanosleep(200);
      if (*vdone) break;
      const long long p0 = b * LW_BLK;
      uint32_t x[LW_BLK / 32];
#pragma unroll
      for (int k = 0; k < LW_BLK / 32; ++k) {
        const long long pos = p0 + k * 32 + lane;
        x[k] = pos < vcap ? __ldcs(v + pos) : 0u;
      }
#pragma unroll
      for (int k = 0; k < LW_BLK / 32; ++k) ring[((b % LW_NB) * LW_BLK) + k * 32 + lane] = x[k];
      __threadfence_block();
      __syncwarp();
      if (lane == 0) vready[b % LW_NB] = b;
    }
    return;
  }
  // walker (warp 0)
  long long q = 0, t = 0;
  int bad = 0;
  while (t < T) {
    if (q + 32 > vcap) {
      bad = 1;
      break;
    }
    const long long b0 = q / LW_BLK, b1 = (q + 31) / LW_BLK;
    while (vready[b0 % LW_NB] != b0 || vready[b1 % LW_NB] != b1) __nanosleep(32);
    __syncwarp();
    const uint32_t x = ring[(q + lane) & (LW_RING - 1)];
    const long long tt = t + lane;
    const bool valid = tt < T;
    uint32_t r = 0;
    const bool ok = !valid || lemire_ok(x, (uint32_t)(base + (long long)dir * tt), &r);
    const unsigned bal = __ballot_sync(FULLMASK, !ok);
    int nacc = bal ? __ffs(bal) - 1 : 32;
    if (nacc > T - t) nacc = (int)(T - t);  // lanes past the last draw consume nothing
    if (lane < nacc && valid) out[tt] = r;
    t += nacc;
    q += nacc + (bal ? 1 : 0);
    if (lane == 0) *vcons = q;
  }
  if (lane == 0) {
    *vdone = 1;
    if (bad) *err = 3;
    *q_end_out = q;
  }
}

// ---------------------------------------------------------------------------
// exclusive scan of int32 (n+1 outputs: out[n] = total); 3-phase
// ---------------------------------------------------------------------------
#define SCAN_B 256
#define SCAN_ITEMS 8
__device__ __forceinline__ int block_excl_scan(int x, int* sh, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FULLMASK, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sh[w] = incl;
  __syncthreads();
  if (w == 0) {
    int s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
    int si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULLMASK, si, o);
      if (lane >= o) si += y;
    }
    sh[lane] = si - s;
    if (lane == 31) sh[32] = si;
  }
  __syncthreads();
  int r = sh[w] + incl - x;
  *total = sh[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SCAN_B) scan_reduce_kernel(const int* __restrict__ in, long long n,
                                                             int* __restrict__ bsum) {
  __shared__ int sh[33];
  long long base = (long long)blockIdx.x * SCAN_B * SCAN_ITEMS;
  int s = 0;
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    long long i = base + (long long)k * SCAN_B + threadIdx.x;
    if (i < n) s += in[i];
  }
  int tot;
  block_excl_scan(s, sh, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_B) scan_top_kernel(int* __restrict__ bsum, int nb) {
  __shared__ int sh[33];
  int carry = 0;
  for (int b0 = 0; b0 < nb; b0 += SCAN_B) {
    int i = b0 + threadIdx.x;
    int x = i < nb ? bsum[i] : 0;
    int tot;
    int ex = block_excl_scan(x, sh, &tot);
    if (i < nb) bsum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) bsum[nb] = carry;
}

__global__ void __launch_bounds__(SCAN_B) scan_down_kernel(const int* __restrict__ in, long long n,
                                                           const int* __restrict__ bsum, int* __restrict__ out) {
  __shared__ int sh[33];
  long long base = (long long)blockIdx.x * SCAN_B * SCAN_ITEMS;
  // thread-contiguous items for a per-thread serial scan
  int vals[SCAN_ITEMS];
  int s = 0;
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    long long i = base + (long long)threadIdx.x * SCAN_ITEMS + k;
    vals[k] = i < n ? in[i] : 0;
    s += vals[k];
  }
  int tot;
  int ex = block_excl_scan(s, sh, &tot) + bsum[blockIdx.x];
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    long long i = base + (long long)threadIdx.x * SCAN_ITEMS + k;
    if (i < n) out[i] = ex;
    ex += vals[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) out[n] = bsum[gridDim.x];
}

size_t scan_ws_bytes(long long n) {
  long long nb = (n + SCAN_B * SCAN_ITEMS - 1) / (SCAN_B * SCAN_ITEMS);
  return (size_t)(nb + 1) * sizeof(int);
}

int exclusive_scan(const int* in, long long n, int* out, int* ws, cudaStream_t s) {
  long long nb = (n + SCAN_B * SCAN_ITEMS - 1) / (SCAN_B * SCAN_ITEMS);
  if (nb == 0) nb = 1;
  scan_reduce_kernel<<<(unsigned)nb, SCAN_B, 0, s>>>(in, n, ws);
  SPTK_CHECK_LAUNCH();
  scan_top_kernel<<<1, SCAN_B, 0, s>>>(ws, (int)nb);
  SPTK_CHECK_LAUNCH();
  scan_down_kernel<<<(unsigned)nb, SCAN_B, 0, s>>>(in, n, ws, out);
  SPTK_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// Floyd membership (choice, replace=False): out[t] = vals[t] unless vals[t]
// is already selected, in which case j_t = base + t (coo.py:281 / trainer.py:218
// -> Generator.choice).  c_t = !first_t || (vals[t]-base in [0,t) && c_{vals[t]-base}).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t mix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

__global__ void floyd_insert_kernel(const uint32_t* __restrict__ vals, long long k, uint32_t* keys, int* mint,
                                    uint32_t hmask) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; t < k; t += stride) {
    uint32_t v = vals[t];
    uint32_t slot = mix32(v) & hmask;
    while (true) {
      uint32_t old = atomicCAS(&keys[slot], 0xffffffffu, v);
      if (old == 0xffffffffu || old == v) {
        atomicMin(&mint[slot], (int)t);
        break;
      }
      slot = (slot + 1) & hmask;
    }
  }
}

__global__ void floyd_first_kernel(const uint32_t* __restrict__ vals, long long k, const uint32_t* keys,
                                   const int* mint, uint32_t hmask, unsigned char* first) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; t < k; t += stride) {
    uint32_t v = vals[t];
    uint32_t slot = mix32(v) & hmask;
    while (keys[slot] != v) slot = (slot + 1) & hmask;
    first[t] = mint[slot] == (int)t;
  }
}

__global__ void floyd_out_kernel(const uint32_t* __restrict__ vals, long long k, long long base,
                                 const unsigned char* __restrict__ first, int* __restrict__ out) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; t < k; t += stride) {
    long long x = t;
    int c = 0;
    while (true) {
      if (!first[x]) {
        c = 1;
        break;
      }
      long long jm = (long long)vals[x] - base;
      if (jm < 0 || jm >= x) {
        c = 0;
        break;
      }
      x = jm;
    }
    out[t] = c ? (int)(base + t) : (int)vals[t];
  }
}

__global__ void gather_kernel(const int* __restrict__ src, const int* __restrict__ perm, long long n,
                              int* __restrict__ dst) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[i] = src[perm[i]];
}

__global__ void iota_kernel(int* __restrict__ out, long long n, int offset) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = (int)i + offset;
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
static inline unsigned grid_for(long long n, int threads, int cap = 148 * 32) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

static Pcg64 make_pcg(const uint64_t st[4]) {
  Pcg64 g;
  g.state = ((u128)st[0] << 64) | st[1];
  g.inc = ((u128)st[2] << 64) | st[3];
  return g;
}

// segments with mask < 2^K_SMALL are walked by one warp
static const int K_SMALL = 12;

struct SegPlan {
  Seg sg;
  int L, C, Delta;
};

static SegPlan plan_segment(long long n, int k) {
  SegPlan sp;
  long long hi = (1LL << k) - 1;
  if (hi > n - 1) hi = n - 1;
  long long lo = 1LL << (k - 1);
  sp.sg.hi = (int)hi;
  sp.sg.mask = (unsigned)((1ULL << k) - 1);
  sp.sg.S = (int)(hi - lo + 1);
  double M = (double)sp.sg.mask + 1.0;
  // E[#positions] = sum_{i=lo}^{hi} M/(i+1); Var = sum (1-p)/p^2 with p=(i+1)/M
  double mean = M * (log((hi + 1.5) / (lo + 0.5)));
  double var = M * M * (1.0 / (lo + 0.5) - 1.0 / (hi + 1.5)) - mean;
  if (var < 0) var = 0;
  double bound = mean + 12.0 * sqrt(var) + 1024.0;
  sp.Delta = (int)ceil(4.0 * sqrt(mean) + 64.0);
  // ~24 near-margin entries per chunk (capacity PERM_E = 64)
  static const double target_entries = [] {
    const char* e = getenv("SPTK_PERM_ENTRIES");
    return e ? atof(e) : 24.0;
  }();
  double Lf = M * target_entries / (2.0 * sp.Delta);
  int L = 64;
  while (L * 2 <= Lf && L < 65536) L *= 2;
  sp.L = L;
  sp.C = (int)ceil(bound / L);
  return sp;
}

static const int PERM_E = 64;

static size_t apply_ws_bytes(long long n);

size_t jgen_batch_ws_bytes(const long long* n, int B);

// workspace of the j-sequence generation alone (segment chunk summaries)
size_t jgen_ws_bytes(long long n) { return jgen_batch_ws_bytes(&n, 1); }
size_t fy_ws_bytes(long long n) { return apply_ws_bytes(n) + 256; }

size_t perm_ws_bytes(long long n) {
  // P + meta of the caller, j (n+1), the j-generation and the apply
  return 66 * sizeof(long long) + 66 * sizeof(int) + 2 * 256 + (size_t)(n + 2) * sizeof(int) + 256 +
         jgen_ws_bytes(n) + apply_ws_bytes(n) + 16 * 256;
}

struct Carve {
  char* p;
  size_t left;
  bool overflow = false;
  template <typename T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
    if (bytes > left) {
      overflow = true;
      return (T*)p;
    }
    T* r = (T*)p;
    p += bytes;
    left -= bytes;
    return r;
  }
  bool ok() const { return !overflow; }
};

// j-sequences of B permutations: block b (n[b], generator st[4b..4b+3]) into
// j_out[b][1..n[b]-1].  Segment levels run in lock step across blocks.
static size_t jgen_batch_plan(const long long* n, int B, size_t* max_chunks, int* kmax_all) {
  size_t chunks = 0;
  int km = 0;
  for (int b = 0; b < B; ++b)
    if (n[b] >= 2) km = std::max(km, 64 - __builtin_clzll((unsigned long long)(n[b] - 1)));
  size_t njobs = 0;
  for (int k = km; k > K_SMALL; --k) {
    size_t lvl = 0;
    for (int b = 0; b < B; ++b) {
      if (n[b] < 2) continue;
      const int kb = 64 - __builtin_clzll((unsigned long long)(n[b] - 1));
      if (kb < k) continue;
      lvl += plan_segment(n[b], k).C;
      ++njobs;
    }
    chunks = std::max(chunks, lvl);
  }
  *max_chunks = chunks;
  *kmax_all = km;
  return njobs;
}

size_t jgen_batch_ws_bytes(const long long* n, int B) {
  size_t chunks;
  int km;
  const size_t njobs = jgen_batch_plan(n, B, &chunks, &km);
  return (size_t)B * (66 * sizeof(long long) + 66 * sizeof(int) + 2 * 256) +
         (chunks + 1) * (4 * sizeof(int) + PERM_E * sizeof(int2)) + 6 * 256 + (njobs + 1) * sizeof(PermJob) +
         (size_t)(B + 1) * sizeof(SmallJob) + 4 * 256;
}

int perm_jgen_batch(const Pcg64* g, const long long* n, int* const* j_out, int B, Carve& cv, cudaStream_t s) {
  size_t chunks;
  int km;
  const size_t njobs = jgen_batch_plan(n, B, &chunks, &km);
  std::vector<long long*> P(B);
  std::vector<int*> meta(B);
  for (int b = 0; b < B; ++b) {
    P[b] = cv.take<long long>(66);
    meta[b] = cv.take<int>(66);
  }
  ChunkBuf cb;
  cb.E = PERM_E;
  cb.a0 = cv.take<int>(chunks + 1);
  cb.D = cv.take<int>(chunks + 1);
  cb.cnt = cv.take<int>(chunks + 1);
  cb.a_in = cv.take<int>(chunks + 1);
  cb.ent = cv.take<int2>((chunks + 1) * PERM_E);
  PermJob* d_jobs = cv.take<PermJob>(njobs + 1);
  SmallJob* d_small = cv.take<SmallJob>(B + 1);
  SPTK_REQUIRE(cv.ok(), "permutation: workspace too small");
  std::vector<PermJob> jobs;
  std::vector<int> lvl_begin, lvl_total;
  jobs.reserve(njobs);
  for (int k = km; k > K_SMALL; --k) {
    lvl_begin.push_back((int)jobs.size());
    int c0 = 0;
    for (int b = 0; b < B; ++b) {
      if (n[b] < 2) continue;
      const int kb = 64 - __builtin_clzll((unsigned long long)(n[b] - 1));
      if (kb < k) continue;
      const SegPlan sp = plan_segment(n[b], k);
      PermJob jb;
      jb.g = g[b];
      jb.P = P[b] + (kb - k);
      jb.meta = meta[b] + (kb - k);
      jb.j_out = j_out[b];
      jb.sg = sp.sg;
      jb.L = sp.L;
      jb.C = sp.C;
      jb.Delta = sp.Delta;
      jb.chunk0 = c0;
      jb.cb = cb;
      jb.cb.a0 += c0;
      jb.cb.D += c0;
      jb.cb.cnt += c0;
      jb.cb.a_in += c0;
      jb.cb.ent += (long long)c0 * PERM_E;
      c0 += sp.C;
      jobs.push_back(jb);
    }
    lvl_total.push_back(c0);
  }
  lvl_begin.push_back((int)jobs.size());
  std::vector<SmallJob> small;
  for (int b = 0; b < B; ++b) {
    if (n[b] < 2) continue;
    const int kb = 64 - __builtin_clzll((unsigned long long)(n[b] - 1));
    const int kst = kb > K_SMALL ? K_SMALL : kb;
    SmallJob sj;
    sj.g = g[b];
    sj.P = P[b] + (kb - kst);
    sj.kstart = kst;
    sj.n = n[b];
    sj.j_out = j_out[b];
    sj.q_final = P[b] + 65;
    small.push_back(sj);
  }
  for (int b = 0; b < B; ++b) SPTK_CUDA_TRY(cudaMemsetAsync(P[b], 0, sizeof(long long) * 66, s));
  if (!jobs.empty())
    SPTK_CUDA_TRY(cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(PermJob) * jobs.size(), cudaMemcpyHostToDevice, s));
  if (!small.empty())
    SPTK_CUDA_TRY(cudaMemcpyAsync(d_small, small.data(), sizeof(SmallJob) * small.size(), cudaMemcpyHostToDevice, s));
  const int warps_per_block = 8;
  for (size_t l = 0; l + 1 < lvl_begin.size(); ++l) {
    const int j0 = lvl_begin[l], nj = lvl_begin[l + 1] - j0, total = lvl_total[l];
    if (nj == 0) continue;
    const unsigned blocks = (unsigned)((total + warps_per_block - 1) / warps_per_block);
    perm_phaseA_batched<<<blocks, 32 * warps_per_block, 0, s>>>(d_jobs + j0, nj, total);
    SPTK_CHECK_LAUNCH();
    perm_resolve_batched<<<nj, 32, 0, s>>>(d_jobs + j0);
    SPTK_CHECK_LAUNCH();
    perm_phaseB_batched<<<blocks, 32 * warps_per_block, 0, s>>>(d_jobs + j0, nj, total);
    SPTK_CHECK_LAUNCH();
  }
  if (!small.empty()) {
    perm_small_batched<<<(unsigned)small.size(), 32, 0, s>>>(d_small);
    SPTK_CHECK_LAUNCH();
  }
  return 0;
}

// j-sequence of Generator.permutation(n) into j_out[1..n-1]: a batch of one.
int perm_jgen(Pcg64 g, long long n, int* j_out, Carve& cv, long long* d_P, int* d_meta, cudaStream_t s) {
  (void)d_P;
  (void)d_meta;
  if (n < 2) return 0;
  int* outs[1] = {j_out};
  return perm_jgen_batch(&g, &n, outs, 1, cv, s);
}

int permutation_j_batch(const uint64_t* st, const long long* n, int* const* j_out, int B, void* ws, size_t ws_bytes,
                        cudaStream_t s) {
  SPTK_REQUIRE(B >= 0, "permutation_j_batch: bad batch");
  for (int b = 0; b < B; ++b) SPTK_REQUIRE(n[b] >= 0 && n[b] < (1LL << 30), "permutation_j_batch: n out of range");
  SPTK_REQUIRE(ws_bytes >= jgen_batch_ws_bytes(n, B), "permutation_j_batch: workspace too small");
  std::vector<Pcg64> g(B);
  for (int b = 0; b < B; ++b) g[b] = make_pcg(st + 4 * b);
  Carve cv{(char*)ws, ws_bytes};
  return perm_jgen_batch(g.data(), n, j_out, B, cv, s);
}

// ---------------------------------------------------------------------------
// (3) applying the swap sequence: two bucket partitions around a per-bucket
// sort, so that every pass is either sequential or L2-local.
//
//   B  partition the steps by target bucket (2^lg positions per bucket),
//      payload (step, target): the two-pass MSD partition below.
//   C  one CTA per target bucket: counting sort by target in an L2-resident
//      scratch, insertion sort of each (short, O(log n)) step list, then
//      parent[p] = first step > p targeting p, and each entry rewritten as
//      (step, next step of its target list, or -(p+1) for the last).
//   D  partition those entries by step bucket (same primitive as B).
//   E  one CTA per step bucket: v = root of the parent chain from the
//      successor (or p); result[step] = v, and/or the record gather
//      out_rec[step] = src_rec[v] -- writes land in the bucket's own
//      contiguous range, so the visit-ordered records stream out
//      sequentially and the factor pass reads them without indirection.
// Random DRAM traffic is one parent read per chain hop (~1 per step on
// average) plus, for the record gather, one record read per step.
// ---------------------------------------------------------------------------

static inline int fy_bucket_log(long long n) {
  int bits = 1;
  while ((1LL << bits) < n) ++bits;
  int lg = bits - 15;
  return lg < 12 ? 12 : lg;
}

// ---- two-pass MSD partition with coalesced writes ---------------------------
// Items (step, target) from j (FROM_J) or int2 entries e (key = e.x) are
// grouped by fine bucket f = key >> lg (nbk <= 2^13 buckets).  A single pass
// would scatter into nbk x CTAs write fronts whose partially written sectors
// get evicted (ECC read-modify-write); instead:
//   count:  per-CTA shared histograms of f, summed into fine_cnt (global)
//   pass 1: tiles of MSD_TILE items are counting-sorted in shared memory by
//           the coarse bucket f >> 6 and written as contiguous runs at space
//           reserved with one atomicAdd per (tile, coarse bucket)
//   pass 2: tiles inside each coarse segment are sorted by f & 63 the same
//           way and written to their final fine-bucket ranges.
// Each pass streams 8 bytes in and out per item with run-length ~TILE/64.
#define MSD_T 256
#define FY_TT 256
#define FY_LCAP 8192
#define MSD_TILE 2048
#define MSD_CB 8

template <bool FROM_J>
__device__ __forceinline__ int2 msd_item(const int* __restrict__ j, const int2* __restrict__ e, long long lo,
                                         long long i) {
  if (FROM_J) return make_int2((int)(lo + i), __ldcs(j + lo + i));
  return __ldcs(e + i);
}
template <bool FROM_J>
__device__ __forceinline__ int msd_key(int2 v) {
  return FROM_J ? v.y : v.x;
}

template <bool FROM_J>
__global__ void __launch_bounds__(MSD_T) msd_count_kernel(const int* __restrict__ j, const int2* __restrict__ e,
                                                          long long lo, long long n, int lg, int nbk,
                                                          int* __restrict__ fine_cnt) {
  // packed 16-bit counters (two per word; the grid is sized so no CTA sees
  // more than 65535 items): half the shared memory, so the kernel fits beside
  // the factor grid
  extern __shared__ unsigned hsm2[];
  const int nw = (nbk + 1) >> 1;
  for (int b = threadIdx.x; b < nw; b += MSD_T) hsm2[b] = 0u;
  __syncthreads();
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long a = per * blockIdx.x, z = min(n, a + per);
  for (long long i0 = a + threadIdx.x; i0 < z; i0 += (long long)MSD_T * 8) {
    int key[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long i = i0 + (long long)u * MSD_T;
      key[u] = i < z ? msd_key<FROM_J>(msd_item<FROM_J>(j, e, lo, i)) : -1;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (key[u] >= 0) {
        const int b = key[u] >> lg;
        atomicAdd(&hsm2[b >> 1], (b & 1) ? 65536u : 1u);
      }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < nw; w += MSD_T) {
    const unsigned x = hsm2[w];
    if (x & 0xffffu) atomicAdd(&fine_cnt[2 * w], (int)(x & 0xffffu));
    if ((x >> 16) && 2 * w + 1 < nbk) atomicAdd(&fine_cnt[2 * w + 1], (int)(x >> 16));
  }
}

// coarse cursors and per-coarse-segment tile prefix (one thread; ncb <= 128)
__global__ void msd_setup_kernel(const int* __restrict__ boff, int nbk, int* __restrict__ ccur,
                                 int* __restrict__ tile_start) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int ncb = (nbk + (1 << MSD_CB) - 1) >> MSD_CB;
  int acc = 0;
  for (int c = 0; c < ncb; ++c) {
    const int a = boff[c << MSD_CB], z = boff[min(nbk, (c + 1) << MSD_CB)];
    ccur[c] = a;
    tile_start[c] = acc;
    acc += (z - a + MSD_TILE - 1) / MSD_TILE;
  }
  tile_start[ncb] = acc;
}

// Sort one tile (items v[0..cnt) held MSD_TILE/MSD_T per thread) by bucket
// b(item) in [0, nb) and write runs to out at cursor-reserved positions.
template <int NBMAX, typename BucketFn>
__device__ __forceinline__ void msd_tile_scatter(int2 (&v)[MSD_TILE / MSD_T], const bool (&ok)[MSD_TILE / MSD_T],
                                                 int nb, BucketFn bucket, int* __restrict__ cursor,
                                                 int2* __restrict__ out, int2* sbuf, int* cnt, int* toff,
                                                 int* gbase, int* sh) {
  constexpr int U = MSD_TILE / MSD_T;
  const int tid = threadIdx.x;
  for (int b = tid; b < nb; b += MSD_T) cnt[b] = 0;
  __syncthreads();
  int rank[U], bk[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    bk[u] = ok[u] ? bucket(v[u]) : -1;
    if (bk[u] >= 0) rank[u] = atomicAdd(&cnt[bk[u]], 1);
  }
  __syncthreads();
  // exclusive scan of cnt[0..nb) (nb <= NBMAX <= MSD_T) and cursor reservation
  const int x = tid < nb ? cnt[tid] : 0;
  int tot;
  const int ex = block_excl_scan(x, sh, &tot);
  if (tid < nb) {
    toff[tid] = ex;
    gbase[tid] = x ? atomicAdd(&cursor[tid], x) : 0;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (bk[u] >= 0) sbuf[toff[bk[u]] + rank[u]] = v[u];
  __syncthreads();
  for (int i = tid; i < tot; i += MSD_T) {
    const int2 w = sbuf[i];
    const int b = bucket(w);
    out[gbase[b] + (i - toff[b])] = w;
  }
  __syncthreads();
}

template <bool FROM_J>
__global__ void __launch_bounds__(MSD_T) msd_pass1_kernel(const int* __restrict__ j, const int2* __restrict__ e,
                                                          long long lo, long long n, int lg, int nbk,
                                                          int* __restrict__ ccur, int2* __restrict__ out) {
  __shared__ int2 sbuf[MSD_TILE];
  __shared__ int cnt[256], toff[256], gbase[256], sh[33];
  constexpr int U = MSD_TILE / MSD_T;
  const int ncb = (nbk + (1 << MSD_CB) - 1) >> MSD_CB;
  const int sh_b = lg + MSD_CB;
  const long long ntiles = (n + MSD_TILE - 1) / MSD_TILE;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int2 v[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = t * MSD_TILE + u * MSD_T + threadIdx.x;
      ok[u] = i < n;
      v[u] = ok[u] ? msd_item<FROM_J>(j, e, lo, i) : make_int2(0, 0);
    }
    msd_tile_scatter<128>(v, ok, ncb, [&](int2 w) { return msd_key<FROM_J>(w) >> sh_b; }, ccur, out, sbuf, cnt,
                          toff, gbase, sh);
  }
}

template <bool FROM_J>
__global__ void __launch_bounds__(MSD_T) msd_pass2_kernel(const int2* __restrict__ in, const int* __restrict__ boff,
                                                          int lg, int nbk, const int* __restrict__ tile_start,
                                                          int* __restrict__ fcur, int2* __restrict__ out) {
  __shared__ int2 sbuf[MSD_TILE];
  __shared__ int cnt[1 << MSD_CB], toff[1 << MSD_CB], gbase[1 << MSD_CB], sh[33], ts[129];
  constexpr int U = MSD_TILE / MSD_T;
  const int ncb = (nbk + (1 << MSD_CB) - 1) >> MSD_CB;
  for (int c = threadIdx.x; c <= ncb; c += MSD_T) ts[c] = tile_start[c];
  __syncthreads();
  const int ntiles = ts[ncb];
  for (int g = blockIdx.x; g < ntiles; g += gridDim.x) {
    int c = 0;
    while (ts[c + 1] <= g) ++c;
    const int f0 = c << MSD_CB, f1 = min(nbk, (c + 1) << MSD_CB);
    const long long a = boff[f0] + (long long)(g - ts[c]) * MSD_TILE, z = boff[f1];
    int2 v[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = a + u * MSD_T + threadIdx.x;
      ok[u] = i < z;
      v[u] = ok[u] ? __ldcs(in + i) : make_int2(0, 0);
    }
    msd_tile_scatter<(1 << MSD_CB)>(v, ok, f1 - f0, [&](int2 w) { return (msd_key<FROM_J>(w) >> lg) - f0; },
                                    fcur + f0, out, sbuf, cnt, toff, gbase, sh);
  }
}

// Per target p of a bucket: insertion-sort its step list L (short), emit
// parent[p], the has-parent bit and (step, successor) entries.  Called with a
// shared-memory or a global list buffer (separate instantiations, so the
// shared case compiles to LDS/STS rather than generic loads).
__device__ __forceinline__ void fy_target_lists(int* lists, const int* cnt, const int* cur, long long base,
                                                long long n, int B, long long e0, int* __restrict__ parent,
                                                int2* __restrict__ out, unsigned* __restrict__ hasp) {
  for (int t = threadIdx.x; t < B; t += blockDim.x) {
    const long long p = base + t;
    if (p >= n) break;
    const int m = cnt[t];
    const int rel = cur[t] - m;
    int* L = lists + rel;
    for (int x = 1; x < m; ++x) {
      const int v = L[x];
      int c = x - 1;
      while (c >= 0 && L[c] > v) {
        L[c + 1] = L[c];
        --c;
      }
      L[c + 1] = v;
    }
    int par = -1;
    if (m > 0) par = L[0] > (int)p ? L[0] : (m > 1 ? L[1] : -1);
    parent[p] = par;
    // has-parent bitmap (n bits, L2-resident): a warp covers 32 consecutive
    // positions, base is a multiple of 32
    const unsigned bits = __ballot_sync(__activemask(), par >= 0);
    if ((t & 31) == 0) hasp[p >> 5] = bits;
    for (int k = 0; k < m; ++k) out[e0 + rel + k] = make_int2(L[k], k + 1 < m ? L[k + 1] : -(int)(p + 1));
  }
}

// C: per target bucket.  Dynamic smem: cnt[B] + cur[B] ints.
// (cnt/cur live in shared memory for buckets of <= 2^12 positions, else in
// the per-bucket slice of gcc[2 * 2^lg * nbk].)
__global__ void __launch_bounds__(FY_TT) fy_target_kernel(const int* __restrict__ offs, int G, long long n, int lg,
                                                          const int2* __restrict__ ent, int* __restrict__ tmp,
                                                          int* __restrict__ parent, int2* __restrict__ out,
                                                          long long cnt_total, int* __restrict__ gcc,
                                                          unsigned* __restrict__ hasp) {
  extern __shared__ int tsm[];
  __shared__ int sh[33];
  const int B = 1 << lg;
  int* cnt = gcc ? gcc + ((size_t)blockIdx.x << (lg + 1)) : tsm;
  int* cur = cnt + B;
  const int b = blockIdx.x, tid = threadIdx.x, T = blockDim.x;
  const long long base = (long long)b << lg;
  const long long e0 = offs[(size_t)b * G];
  const long long e1 = (size_t)(b + 1) * G < (size_t)gridDim.x * G ? offs[(size_t)(b + 1) * G] : cnt_total;
  // target-sorted step lists: in shared memory when the bucket fits (the
  // common case), else in the bucket's slice of the global scratch
  int* lists = (!gcc && e1 - e0 <= FY_LCAP) ? tsm + 2 * B : tmp + e0;
  for (int t = tid; t < B; t += T) cnt[t] = 0;
  __syncthreads();
  for (long long e = e0 + tid; e < e1; e += (long long)T * 4) {
    int tg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) tg[u] = e + u * T < e1 ? ent[e + u * T].y : -1;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (tg[u] >= 0) atomicAdd(&cnt[tg[u] - (int)base], 1);
  }
  __syncthreads();
  // exclusive scan of cnt into cur (thread-contiguous runs of B/T)
  const int per = B / T;
  int run = 0;
  for (int k = 0; k < per; ++k) run += cnt[tid * per + k];
  int tot;
  int ex = block_excl_scan(run, sh, &tot);
  for (int k = 0; k < per; ++k) {
    cur[tid * per + k] = ex;
    ex += cnt[tid * per + k];
  }
  __syncthreads();
  for (long long e = e0 + tid; e < e1; e += (long long)T * 4) {
    int2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = e + u * T < e1 ? ent[e + u * T] : make_int2(0, -1);
    int slot[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v[u].y >= 0) slot[u] = atomicAdd(&cur[v[u].y - (int)base], 1);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v[u].y >= 0) lists[slot[u]] = v[u].x;
  }
  __syncthreads();
  // cur[t] = end of target t's segment (relative to e0), cnt[t] its length
  if (lists != tmp + e0)
    fy_target_lists(tsm + 2 * B, cnt, cur, base, n, B, e0, parent, out, hasp);
  else
    fy_target_lists(tmp + e0, cnt, cur, base, n, B, e0, parent, out, hasp);
}

// E: per step bucket; entries e[lo..hi) are the bucket's steps in any order.
__global__ void __launch_bounds__(256) fy_emit_kernel(const int* __restrict__ offs, int G, int nbk,
                                                      const int2* __restrict__ ent, long long cnt_total,
                                                      const int* __restrict__ parent,
                                                      const unsigned* __restrict__ hasp, int* __restrict__ result,
                                                      const int4* __restrict__ src, int4* __restrict__ dst,
                                                      int rq) {
  const int b = blockIdx.x;
  const long long e0 = offs[(size_t)b * G];
  const long long e1 = b + 1 < nbk ? offs[(size_t)(b + 1) * G] : cnt_total;
  // EU independent chains per thread, walked in lock step (memory-level
  // parallelism for the random parent reads); a chain only continues through
  // positions whose has-parent bit is set (bitmap in L2)
  constexpr int EU = 4;
  for (long long e0u = e0 + threadIdx.x; e0u < e1; e0u += (long long)blockDim.x * EU) {
    int st[EU], v[EU];
    bool live[EU];
#pragma unroll
    for (int u = 0; u < EU; ++u) {
      const long long e = e0u + (long long)u * blockDim.x;
      const bool ok = e < e1;
      const int2 v2 = ok ? ent[e] : make_int2(-1, -1);
      st[u] = v2.x;
      v[u] = v2.y >= 0 ? v2.y : -v2.y - 1;
      live[u] = ok && v2.y >= 0;
    }
    bool any = true;
    while (any) {
      unsigned w[EU];
#pragma unroll
      for (int u = 0; u < EU; ++u) w[u] = live[u] ? __ldcg(hasp + (v[u] >> 5)) : 0u;
      any = false;
#pragma unroll
      for (int u = 0; u < EU; ++u) {
        live[u] = live[u] && ((w[u] >> (v[u] & 31)) & 1u);
        any |= live[u];
      }
      if (!any) break;
#pragma unroll
      for (int u = 0; u < EU; ++u)
        if (live[u]) v[u] = __ldcg(parent + v[u]);
    }
#pragma unroll
    for (int u = 0; u < EU; ++u) {
      if (st[u] < 0) continue;
      if (result) result[st[u]] = v[u];
      if (dst) {
        const int4* sp = src + (long long)v[u] * rq;
        int4* dp = dst + (long long)st[u] * rq;
        for (int k = 0; k < rq; ++k) dp[k] = __ldcs(sp + k);
      }
    }
  }
}

#define FY_SMEM_LG 12
static size_t apply_ws_bytes(long long n) {
  const int lg = fy_bucket_log(n > 1 ? n : 2);
  const long long nbk = (n + (1LL << lg) - 1) >> lg;
  size_t b = (size_t)(n + 2) * (3 * sizeof(int2) + 2 * sizeof(int)) + (size_t)(nbk + 2) * 3 * sizeof(int) +
             (size_t)(130 * 2) * sizeof(int) + scan_ws_bytes(nbk + 1) + 24 * 256;
  if (lg > FY_SMEM_LG) b += (((size_t)nbk << (lg + 1)) + 1) * sizeof(int) + 256;
  b += (((size_t)nbk << (lg - 5)) + 1) * sizeof(unsigned) + 256;
  return b;
}

// Apply steps i = n-1..first (target j[i]) to the identity; result[i] (if
// non-NULL) = final value at position i, and/or dst_rec[i] = src_rec[result[i]]
// (rq int4 per record), for i in [first, n).  If first <= 1 the virtual step
// 0 (j[0] = 0) is included so position 0 is produced too.  j is read only.
static int fy_apply_ex(int* j, long long n, long long first, int* result, const int* src_rec, int* dst_rec, int rq,
                       Carve& cv, cudaStream_t s) {
  if (n <= 0) return 0;
  const long long f = first <= 1 ? 0 : first;
  if (f == 0) SPTK_CUDA_TRY(cudaMemsetAsync(j, 0, sizeof(int), s));
  const long long cnt = n - f;
  const int lg = fy_bucket_log(n > 1 ? n : 2);
  const int nbk = (int)((n + (1LL << lg) - 1) >> lg);
  const int ncb = (nbk + (1 << MSD_CB) - 1) >> MSD_CB;
  int2* e1 = cv.take<int2>(cnt + 1);
  int2* e2 = cv.take<int2>(cnt + 1);
  int2* e3 = cv.take<int2>(cnt + 1);  // pass-1 scratch of both partitions
  int* tmp = cv.take<int>(cnt + 1);
  int* parent = cv.take<int>(n + 1);
  int* fcnt = cv.take<int>(nbk + 2);
  int* boff = cv.take<int>(nbk + 2);
  int* fcur = cv.take<int>(nbk + 2);
  int* ccur = cv.take<int>(ncb + 2);
  int* tstart = cv.take<int>(ncb + 2);
  int* sws = cv.take<int>(scan_ws_bytes(nbk + 1) / sizeof(int) + 1);
  int* gcc = lg > FY_SMEM_LG ? cv.take<int>(((size_t)nbk << (lg + 1)) + 1) : nullptr;
  unsigned* hasp = cv.take<unsigned>((size_t)(nbk << (lg - 5)) + 1);
  SPTK_REQUIRE(cv.ok(), "fy_apply: workspace too small");
  SPTK_REQUIRE(ncb <= 128 && (1 << MSD_CB) <= MSD_T, "fy_apply: n=%lld too large", n);
  const size_t hsm = sizeof(unsigned) * (size_t)((nbk + 1) / 2);
  const long long gcount_ll = (cnt + 65534) / 65535;
  const unsigned Gc = (unsigned)(gcount_ll > 4 * 148 ? gcount_ll : 4 * 148);
  static bool configured = false;
  if (!configured) {
    SPTK_CUDA_TRY(cudaFuncSetAttribute(msd_count_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
    SPTK_CUDA_TRY(cudaFuncSetAttribute(msd_count_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
    SPTK_CUDA_TRY(cudaFuncSetAttribute(fy_target_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (8 << FY_SMEM_LG) + (int)sizeof(int) * FY_LCAP));
    configured = true;
  }
  SPTK_REQUIRE(hsm <= (64u << 10), "fy_apply: n=%lld too large", n);
  const size_t tsm = gcc ? 0 : ((size_t)8 << lg) + sizeof(int) * FY_LCAP;
  const unsigned G = 4 * 148;
  auto partition = [&](bool from_j, const int2* src, int2* dst) -> int {
    SPTK_CUDA_TRY(cudaMemsetAsync(fcnt, 0, sizeof(int) * (nbk + 1), s));
    if (from_j)
      msd_count_kernel<true><<<Gc, MSD_T, hsm, s>>>(j, nullptr, f, cnt, lg, nbk, fcnt);
    else
      msd_count_kernel<false><<<Gc, MSD_T, hsm, s>>>(nullptr, src, 0, cnt, lg, nbk, fcnt);
    SPTK_CHECK_LAUNCH();
    if (exclusive_scan(fcnt, nbk, boff, sws, s)) return 1;
    SPTK_CUDA_TRY(cudaMemcpyAsync(fcur, boff, sizeof(int) * nbk, cudaMemcpyDeviceToDevice, s));
    msd_setup_kernel<<<1, 32, 0, s>>>(boff, nbk, ccur, tstart);
    SPTK_CHECK_LAUNCH();
    if (from_j)
      msd_pass1_kernel<true><<<G, MSD_T, 0, s>>>(j, nullptr, f, cnt, lg, nbk, ccur, e3);
    else
      msd_pass1_kernel<false><<<G, MSD_T, 0, s>>>(nullptr, src, 0, cnt, lg, nbk, ccur, e3);
    SPTK_CHECK_LAUNCH();
    if (from_j)
      msd_pass2_kernel<true><<<G, MSD_T, 0, s>>>(e3, boff, lg, nbk, tstart, fcur, dst);
    else
      msd_pass2_kernel<false><<<G, MSD_T, 0, s>>>(e3, boff, lg, nbk, tstart, fcur, dst);
    SPTK_CHECK_LAUNCH();
    return 0;
  };
  // B: steps by target bucket -> e1
  if (partition(true, nullptr, e1)) return 1;
  // C: per target bucket -> parent, e2 = (step, successor)
  fy_target_kernel<<<nbk, FY_TT, tsm, s>>>(boff, 1, n, lg, e1, tmp, parent, e2, cnt, gcc, hasp);
  SPTK_CHECK_LAUNCH();
  // D: entries by step bucket -> e1
  if (partition(false, e2, e1)) return 1;
  // E: roots, results / record gather
  fy_emit_kernel<<<nbk, 256, 0, s>>>(boff, 1, nbk, e1, cnt, parent, hasp, result,
                                     reinterpret_cast<const int4*>(src_rec), reinterpret_cast<int4*>(dst_rec), rq);
  SPTK_CHECK_LAUNCH();
  return 0;
}

int fy_apply(int* j, long long n, long long first, int* result, Carve& cv, cudaStream_t s) {
  return fy_apply_ex(j, n, first, result, nullptr, nullptr, 0, cv, s);
}

int permutation(const uint64_t st[4], long long n, int* out, void* ws, size_t ws_bytes, cudaStream_t s) {
  SPTK_REQUIRE(n >= 0 && n < (1LL << 30), "permutation: n=%lld out of range [0, 2^30)", n);
  SPTK_REQUIRE(ws_bytes >= perm_ws_bytes(n), "permutation: workspace too small (%zu < %zu)", ws_bytes,
               perm_ws_bytes(n));
  if (n == 0) return 0;
  if (n == 1) {
    SPTK_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int), s));
    return 0;
  }
  Carve cv{(char*)ws, ws_bytes};
  long long* d_P = cv.take<long long>(66);
  int* d_meta = cv.take<int>(66);
  int* j = cv.take<int>(n + 1);
  Pcg64 g = make_pcg(st);
  if (perm_jgen(g, n, j, cv, d_P, d_meta, s)) return 1;
  return fy_apply(j, n, 1, out, cv, s);
}

// rec_out[k] = rec_src[perm[k]] (rw 32-bit words per record), perm =
// Generator.permutation(n); perm_out (optional) receives perm itself.
int permute_records(const uint64_t st[4], long long n, const int* rec_src, int rw, int* rec_out, int* perm_out,
                    void* ws, size_t ws_bytes, cudaStream_t s) {
  SPTK_REQUIRE(n >= 0 && n < (1LL << 30), "permute_records: n=%lld out of range [0, 2^30)", n);
  SPTK_REQUIRE(rw == 4 || rw == 8 || rw == 16, "permute_records: rw=%d not in {4, 8, 16}", rw);
  SPTK_REQUIRE(ws_bytes >= perm_ws_bytes(n), "permute_records: workspace too small (%zu < %zu)", ws_bytes,
               perm_ws_bytes(n));
  if (n == 0) return 0;
  if (n == 1) {
    SPTK_CUDA_TRY(cudaMemcpyAsync(rec_out, rec_src, sizeof(int) * rw, cudaMemcpyDeviceToDevice, s));
    if (perm_out) SPTK_CUDA_TRY(cudaMemsetAsync(perm_out, 0, sizeof(int), s));
    return 0;
  }
  Carve cv{(char*)ws, ws_bytes};
  long long* d_P = cv.take<long long>(66);
  int* d_meta = cv.take<int>(66);
  int* j = cv.take<int>(n + 1);
  Pcg64 g = make_pcg(st);
  if (perm_jgen(g, n, j, cv, d_P, d_meta, s)) return 1;
  return fy_apply_ex(j, n, 1, perm_out, rec_src, rec_out, rw / 4, cv, s);
}

// j-sequence only (tests): j_out[i] for i in [1, n)
int permutation_j(const uint64_t st[4], long long n, int* j_out, void* ws, size_t ws_bytes, cudaStream_t s) {
  SPTK_REQUIRE(n >= 0 && n < (1LL << 30), "permutation_j: n out of range");
  SPTK_REQUIRE(ws_bytes >= jgen_ws_bytes(n), "permutation_j: workspace too small");
  if (n < 2) return 0;
  Carve cv{(char*)ws, ws_bytes};
  long long* d_P = cv.take<long long>(66);
  int* d_meta = cv.take<int>(66);
  Pcg64 g = make_pcg(st);
  return perm_jgen(g, n, j_out, cv, d_P, d_meta, s);
}

// result[i] (i in [0, n)) of applying the Fisher-Yates steps j[1..n-1] (j[0] is
// overwritten with 0): the second half of permutation(), for pipelining the
// j-sequence of one epoch with the apply of the previous one.
int fy_apply_public(int* j, long long n, int* out, void* ws, size_t ws_bytes, cudaStream_t s) {
  SPTK_REQUIRE(n >= 0 && n < (1LL << 30), "fy_apply: n=%lld out of range [0, 2^30)", n);
  SPTK_REQUIRE(ws_bytes >= fy_ws_bytes(n), "fy_apply: workspace too small (%zu < %zu)", ws_bytes, fy_ws_bytes(n));
  if (n == 0) return 0;
  if (n == 1) {
    SPTK_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int), s));
    return 0;
  }
  Carve cv{(char*)ws, ws_bytes};
  return fy_apply(j, n, 1, out, cv, s);
}

// Several blocks' j-sequences laid end to end (block b at [off[b], off[b+1]),
// block-local values) become one sequence over the concatenation: targets
// shifted by off[b] and each block's virtual step 0 a self-step.  Blocks
// touch disjoint position ranges, so one apply of the combined sequence
// equals the per-block permutations (each shifted by its offset).
__global__ void fy_globalize_kernel(int* __restrict__ j, const int* __restrict__ off) {
  const int b = blockIdx.x;
  const int lo = off[b], hi = off[b + 1];
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) j[i] = (i == lo) ? lo : j[i] + lo;
}

int fy_globalize(int* j, const int* off, int nb, cudaStream_t s) {
  if (nb <= 0) return 0;
  fy_globalize_kernel<<<nb, 256, 0, s>>>(j, off);
  SPTK_CHECK_LAUNCH();
  return 0;
}

// --- choice ---------------------------------------------------------------
// ---------------------------------------------------------------------------
// Parallel Lemire walk (same contract as lemire_walk_kernel).  Draw t (bound
// base + dir*t) consumes stream words until one is accepted, so the word
// position of draw t is t + r_t, r_t = rejections before t.  The draws are cut
// into chunks of LP_C; for chunk c the host predicts E[r] at its start from the
// exact per-bound rejection probabilities (2^32 mod (rng+1)) / 2^32 and a
// window of LP_W candidate offsets around it.  Pass 1 walks every (chunk,
// candidate) pair and records the offset it exits with; pass 2 (one thread)
// chains the true offsets through the chunks; pass 3 re-walks each chunk from
// its true offset and writes the draws.  A true offset outside a window (or a
// stream overflow) sets a flag and the sequential walker, launched after these
// passes, redoes the whole walk; it returns at once otherwise.  Every chunk's
// walk is the sequential algorithm itself, so the output is identical.
// ---------------------------------------------------------------------------
#define LP_C 4096
struct LpPlan {
  long long T, base, vcap;
  int dir, nch, W;
};

// Lemire rejection threshold 2^32 mod R kept incrementally while the bound
// R = rng + 1 steps by +-1 per accepted draw: with 2^32 = Q R + M, moving R
// by one changes M by -Q / +Q and Q by at most one (valid while Q < R; small
// bounds recompute).  Lets the walkers test a draw without the modulo the
// rare "left < R" branch of lemire_ok needs (which, taken by any of 32 lanes,
// stalled the whole warp on about half of the steps).
struct LemireThr {
  uint32_t R, Q, M;
  __device__ __forceinline__ void set(uint32_t rng) {
    R = rng + 1u;
    const unsigned long long two32 = 1ULL << 32;
    Q = (uint32_t)(two32 / R);
    M = (uint32_t)(two32 - (unsigned long long)Q * R);
  }
  __device__ __forceinline__ void step(int dir) {
    if (R < 65536u) {
      set(R - 1u + (uint32_t)dir);
      return;
    }
    if (dir > 0) {
      if (M >= Q) {
        M -= Q;
      } else {
        M = M + R + 1u - Q;
        --Q;
      }
      ++R;
    } else {
      const unsigned long long mq = (unsigned long long)M + Q;
      if (mq < (unsigned long long)(R - 1u)) {
        M = (uint32_t)mq;
      } else {
        M = (uint32_t)(mq - (R - 1u));
        ++Q;
      }
      --R;
    }
  }
  // lemire_ok with the threshold at hand
  __device__ __forceinline__ bool ok(uint32_t v, uint32_t* res) const {
    const uint64_t m = (uint64_t)v * R;
    *res = (uint32_t)(m >> 32);
    return (uint32_t)m >= M;
  }
};

__device__ __forceinline__ long long lp_walk(const uint32_t* __restrict__ v, long long vcap, long long t0,
                                             long long t1, long long q, long long base, int dir,
                                             uint32_t* __restrict__ out) {
  // walk draws [t0, t1) from word q; returns the position after the last
  // accepted word, or -1 on stream overflow
  long long t = t0;
  LemireThr th;
  th.set((uint32_t)(base + (long long)dir * t));
  while (t < t1) {
    if (q + 4 > vcap) {
      for (; t < t1 && q < vcap; ++q) {
        uint32_t r;
        if (th.ok(__ldg(v + q), &r)) {
          if (out) out[t] = r;
          ++t;
          th.step(dir);
        }
      }
      return t < t1 ? -1 : q;
    }
    uint32_t w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = __ldg(v + q + u);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (t < t1) {
        uint32_t r;
        if (th.ok(w[u], &r)) {
          if (out) out[t] = r;
          ++t;
          th.step(dir);
        }
        ++q;
      }
    }
  }
  return q;
}

__global__ void __launch_bounds__(256) lp_exit_kernel(const uint32_t* __restrict__ v, LpPlan P,
                                                      const int* __restrict__ lo, int* __restrict__ ex) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)P.nch * P.W) return;
  const int c = (int)(i / P.W), w = (int)(i % P.W);
  if (w >= lo[P.nch + c]) return;  // beyond this chunk's window
  const long long r = (long long)lo[c] + w;
  const long long t0 = (long long)c * LP_C, t1 = t0 + LP_C < P.T ? t0 + LP_C : P.T;
  const long long q = lp_walk(v, P.vcap, t0, t1, t0 + r, P.base, P.dir, nullptr);
  ex[i] = q < 0 ? INT_MIN : (int)(q - t1);
}

// Two-stage exits.  Walks of one chunk never cross: a walk entering at a
// larger offset can only be caught by one entering lower (same draw index,
// same word, same bound), after which the two are identical.  Pass 1a walks
// every candidate the first `pre` draws and records its offset there
// (non-decreasing in the candidate); pass 1b walks the rest of the chunk once
// per distinct offset (one thread per run of equal offsets) and gives the
// run's exit to all of its candidates.
__global__ void __launch_bounds__(256) lp_prewalk_kernel(const uint32_t* __restrict__ v, LpPlan P, int pre_len,
                                                         const int* __restrict__ lo, int* __restrict__ pre) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)P.nch * P.W) return;
  const int c = (int)(i / P.W), w = (int)(i % P.W);
  if (w >= lo[P.nch + c]) return;
  const long long r = (long long)lo[c] + w;
  const long long t0 = (long long)c * LP_C, t1 = t0 + LP_C < P.T ? t0 + LP_C : P.T;
  const long long tm = t0 + pre_len < t1 ? t0 + pre_len : t1;
  const long long q = lp_walk(v, P.vcap, t0, tm, t0 + r, P.base, P.dir, nullptr);
  pre[i] = q < 0 ? INT_MIN : (int)(q - tm);
}

// run starts compacted into a dense list (a lane per run, not per candidate:
// most candidates of a run would otherwise idle in their warps)
__global__ void __launch_bounds__(256) lp_runs_list_kernel(LpPlan P, const int* __restrict__ lo,
                                                           const int* __restrict__ pre, int* __restrict__ nruns,
                                                           int* __restrict__ runs) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  bool start = false;
  if (i < (long long)P.nch * P.W) {
    const int c = (int)(i / P.W), w = (int)(i % P.W);
    start = w < lo[P.nch + c] && (w == 0 || pre[i - 1] != pre[i]);
  }
  const unsigned m = __ballot_sync(0xffffffffu, start);
  int base = 0;
  if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(nruns, __popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (start) runs[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = (int)i;
}

__global__ void __launch_bounds__(256) lp_runs_kernel(const uint32_t* __restrict__ v, LpPlan P, int pre_len,
                                                      const int* __restrict__ lo, const int* __restrict__ pre,
                                                      const int* __restrict__ nruns, const int* __restrict__ runs,
                                                      int* __restrict__ ex) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= *nruns) return;
  const long long i = runs[g];
  const int c = (int)(i / P.W), w = (int)(i % P.W), width = lo[P.nch + c];
  const int d = pre[i];
  const long long t0 = (long long)c * LP_C, t1 = t0 + LP_C < P.T ? t0 + LP_C : P.T;
  const long long tm = t0 + pre_len < t1 ? t0 + pre_len : t1;
  int e = INT_MIN;
  if (d != INT_MIN) {
    const long long q = lp_walk(v, P.vcap, tm, t1, tm + d, P.base, P.dir, nullptr);
    e = q < 0 ? INT_MIN : (int)(q - t1);
  }
  for (int u = w; u < width && pre[(long long)c * P.W + u] == d; ++u) ex[(long long)c * P.W + u] = e;
}

__global__ void lp_resolve_kernel(LpPlan P, const int* __restrict__ lo, const int* __restrict__ ex,
                                  int* __restrict__ rc, long long* __restrict__ q_end_out, int* __restrict__ fail) {
  if (threadIdx.x != 0) return;
  long long r = 0;
  for (int c = 0; c < P.nch; ++c) {
    const long long w = r - lo[c];
    if (w < 0 || w >= lo[P.nch + c]) {
      *fail = 1;
      return;
    }
    rc[c] = (int)r;
    const int e = ex[(long long)c * P.W + w];
    if (e == INT_MIN) {
      *fail = 1;
      return;
    }
    r = e;
  }
  *q_end_out = P.T + r;
  *fail = 0;
}

// pass 3: one warp per chunk, 32 consecutive draws tested per round against 32
// consecutive words (the first rejecting lane ends the round, as in the
// sequential walker)
__global__ void __launch_bounds__(256) lp_emit_kernel(const uint32_t* __restrict__ v, LpPlan P,
                                                      const int* __restrict__ rc, const int* __restrict__ fail,
                                                      uint32_t* __restrict__ out) {
  const int c = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (c >= P.nch || *fail) return;
  const long long t0 = (long long)c * LP_C, t1 = t0 + LP_C < P.T ? t0 + LP_C : P.T;
  long long t = t0, q = t0 + rc[c];
  while (t < t1) {
    if (q + 32 > P.vcap) {  // tail of the stream: finish this chunk on one lane
      if (lane == 0) lp_walk(v, P.vcap, t, t1, q, P.base, P.dir, out);
      return;
    }
    const uint32_t x = __ldg(v + q + lane);
    const long long tt = t + lane;
    uint32_t r = 0;
    const bool ok = tt >= t1 || lemire_ok(x, (uint32_t)(P.base + (long long)P.dir * tt), &r);
    const unsigned bal = __ballot_sync(0xffffffffu, !ok);
    int nacc = bal ? __ffs(bal) - 1 : 32;
    if (nacc > t1 - t) nacc = (int)(t1 - t);
    if (lane < nacc) out[tt] = r;
    t += nacc;
    q += nacc + (bal ? 1 : 0);
  }
}

static size_t lp_ws_bytes(long long T) {
  const long long nch = (T + LP_C - 1) / LP_C;
  return (size_t)nch * 4096 * 4 * 3 + (size_t)(nch + 1) * 16 + 8 * 256;
}

static double lp_p(long long rng) {  // P(reject) of one Lemire draw with bound rng (inclusive)
  const unsigned long long ex = (unsigned long long)rng + 1ULL;
  return (double)((1ULL << 32) % ex) / 4294967296.0;
}

// Per chunk c: lo[c] = max(0, round(E[r]) - W_c/2) and lo[nch + c] = W_c, the
// window width for +-4.5 sigma of the offset at the chunk start (both from
// p/(1-p) and p(1-p) sampled every 16 draws and block-scanned over the
// chunks), at most P.W, so early chunks walk fewer candidates
#define LP_PLAN_CACHE 4096
__device__ int g_lp_plan_cache[LP_PLAN_CACHE];
__global__ void __launch_bounds__(1024) lp_plan_kernel(LpPlan P, int* __restrict__ lo) {
  __shared__ double sc[1024], sv[1024];
  const int c = threadIdx.x;
  double e = 0.0, var = 0.0;
  if (c < P.nch) {
    const long long t0 = (long long)c * LP_C, t1 = t0 + LP_C < P.T ? t0 + LP_C : P.T;
    for (long long t = t0; t < t1; t += 16) {
      const unsigned long long ex = (unsigned long long)(uint32_t)(P.base + (long long)P.dir * (t + 8)) + 1ULL;
      const double p = (double)((1ULL << 32) % ex) / 4294967296.0;
      const long long len = t + 16 < t1 ? 16 : t1 - t;
      e += (double)len * p / (1.0 - p);
      var += (double)len * p * (1.0 - p);
    }
  }
  sc[c] = e;
  sv[c] = var;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const double y = c >= o ? sc[c - o] : 0.0, yv = c >= o ? sv[c - o] : 0.0;
    __syncthreads();
    sc[c] += y;
    sv[c] += yv;
    __syncthreads();
  }
  if (c < P.nch) {
    const double before = c == 0 ? 0.0 : sc[c - 1], vb = c == 0 ? 0.0 : sv[c - 1];
    int w = c == 0 ? 1 : (int)((2.0 * (4.5 * sqrt(vb) + 16.0) + 63.0) / 64.0) * 64;
    if (w > P.W) w = P.W;
    const long long l = c == 0 ? 0 : llround(before) - w / 2;
    lo[c] = (int)(l < 0 ? 0 : l);
    lo[P.nch + c] = w;
  }
}

// Lemire walk of T draws (bounds base + dir*t) over the pre-generated stream
// v[0..vcap): out[t] = accepted draw, *d_qend = stream position after the
// walk, *d_err = 3 on stream overflow.  Parallel for 2*LP_C <= T <= 1024*LP_C,
// sequential otherwise (or with SPTK_LEMIRE_SERIAL=1).
static int lemire_walk(const uint32_t* v, long long vcap, long long T, long long base, int dir, uint32_t* out,
                       long long* d_qend, int* d_err, Carve& cv, cudaStream_t s) {
  static int serial = -1;
  if (serial < 0) {
    const char* e = getenv("SPTK_LEMIRE_SERIAL");
    serial = e && atoi(e) == 1;
  }
  const long long nch = (T + LP_C - 1) / LP_C;
  int W = 0;
  if (!serial && T >= 2 * LP_C && nch <= 1024) {
    // spread of the rejection count (coarse sample of p(1-p) over the draws)
    double var = 0.0;
    const int NS = 1024;
    for (int i = 0; i < NS; ++i) {
      const long long t = (long long)((i + 0.5) * (double)T / NS);
      const double p = lp_p((long long)(uint32_t)(base + (long long)dir * t));
      var += p * (1.0 - p) * ((double)T / NS);
    }
    // +-4.5 sigma of the final rejection count (an offset outside its window
    // only costs the sequential fallback)
    const double half = 4.5 * sqrt(var) + 16.0;
    W = (int)((2.0 * half + 63.0) / 64.0) * 64;
    if (W > 4096) W = 0;
    // test hook: a forced (too narrow) window exercises the sequential fallback
    if (const char* e = getenv("SPTK_LP_W")) W = atoi(e);
  }
  if (W == 0) {
    lemire_walk_kernel<<<1, 256, 0, s>>>(v, vcap, T, base, dir, out, d_qend, d_err);
    SPTK_CHECK_LAUNCH();
    return 0;
  }
  LpPlan P{T, base, vcap, dir, (int)nch, W};
  int* lo = cv.take<int>(2 * nch);
  int* rc = cv.take<int>(nch + 1);
  int* fail = cv.take<int>(1);
  int* ex = cv.take<int>((size_t)nch * W);
  int* pre = cv.take<int>((size_t)nch * W);
  int* runs = cv.take<int>((size_t)nch * W);
  int* nruns = cv.take<int>(1);
  SPTK_REQUIRE(cv.ok(), "sampler workspace too small (lemire walk)");
  {
    // the plan depends only on (T, base, dir, W): computed once, then copied
    // from a library-owned device cache (the per-thread modulo loop is 80 us)
    static long long kT = -1, kbase = 0;
    static int kdir = 0, kW = 0, kdev = -1;
    int dev = 0;
    SPTK_CUDA_TRY(cudaGetDevice(&dev));
    int* cache = nullptr;
    SPTK_CUDA_TRY(cudaGetSymbolAddress((void**)&cache, g_lp_plan_cache));
    const bool fits = 2 * nch <= LP_PLAN_CACHE;
    if (fits && kT == T && kbase == base && kdir == dir && kW == W && kdev == dev) {
      SPTK_CUDA_TRY(cudaMemcpyAsync(lo, cache, sizeof(int) * 2 * nch, cudaMemcpyDeviceToDevice, s));
    } else {
      lp_plan_kernel<<<1, 1024, 0, s>>>(P, lo);
      SPTK_CHECK_LAUNCH();
      if (fits) {
        SPTK_CUDA_TRY(cudaMemcpyAsync(cache, lo, sizeof(int) * 2 * nch, cudaMemcpyDeviceToDevice, s));
        SPTK_CUDA_TRY(cudaStreamSynchronize(s));  // once per parameter set: the cache is complete before use
        kT = T;
        kbase = base;
        kdir = dir;
        kW = W;
        kdev = dev;
      }
    }
  }
  // prefix length of the two-stage exits (SPTK_LP_PRE; 0 = walk every
  // candidate through the whole chunk).  NF core batch, per epoch: one stage
  // 1.09 ms; prefix 512 / 1024 / 2048: 0.62 / 0.69 / 0.84 ms
  static int pre_len = -1;
  if (pre_len < 0) {
    const char* e = getenv("SPTK_LP_PRE");
    pre_len = e ? atoi(e) : 512;
  }
  if (pre_len > 0 && pre_len < LP_C) {
    lp_prewalk_kernel<<<(unsigned)((nch * W + 255) / 256), 256, 0, s>>>(v, P, pre_len, lo, pre);
    SPTK_CHECK_LAUNCH();
    SPTK_CUDA_TRY(cudaMemsetAsync(nruns, 0, sizeof(int), s));
    lp_runs_list_kernel<<<(unsigned)((nch * W + 255) / 256), 256, 0, s>>>(P, lo, pre, nruns, runs);
    SPTK_CHECK_LAUNCH();
    lp_runs_kernel<<<(unsigned)((nch * W + 255) / 256), 256, 0, s>>>(v, P, pre_len, lo, pre, nruns, runs, ex);
    SPTK_CHECK_LAUNCH();
  } else {
    lp_exit_kernel<<<(unsigned)((nch * W + 255) / 256), 256, 0, s>>>(v, P, lo, ex);
    SPTK_CHECK_LAUNCH();
  }
  lp_resolve_kernel<<<1, 32, 0, s>>>(P, lo, ex, rc, d_qend, fail);
  SPTK_CHECK_LAUNCH();
  lp_emit_kernel<<<(unsigned)((nch * 32 + 255) / 256), 256, 0, s>>>(v, P, rc, fail, out);
  SPTK_CHECK_LAUNCH();
  lemire_walk_kernel<<<1, 256, 0, s>>>(v, vcap, T, base, dir, out, d_qend, d_err, fail);
  SPTK_CHECK_LAUNCH();
  return 0;
}

static long long lemire_vcap(long long T, double p_rej_max) {
  double mean = T * p_rej_max / (1.0 - p_rej_max);
  return T + (long long)(mean + 12.0 * sqrt(mean + 1.0) + 64.0) + 16 + 64;
}

size_t choice_ws_bytes(long long pop, long long k) {
  size_t pad = 64 * 256;
  size_t b_tail = 0, b_floyd = 0;
  {
    long long first = pop - k > 1 ? pop - k : 1;
    long long T = pop - first;
    b_tail = (size_t)(pop + 1) * 4 * 2 + (size_t)lemire_vcap(T > 0 ? T : 1, (double)pop / 4294967296.0) * 4 +
             (size_t)(T + 1) * 4 + apply_ws_bytes(pop) + lp_ws_bytes(T > 0 ? T : 1);
  }
  {
    long long hs = 1;
    while (hs < 2 * k + 2) hs <<= 1;
    b_floyd = (size_t)(k + 1) * 4 * 3 + (size_t)lemire_vcap(k + 1, (double)pop / 4294967296.0) * 4 +
              (size_t)hs * 8 + (size_t)(k + 1) + (size_t)(k + 1) * 4 * 3 +
              (size_t)lemire_vcap(k + 1, (double)k / 4294967296.0) * 4 + apply_ws_bytes(k) + 2 * lp_ws_bytes(k + 1);
  }
  return pad + (b_tail > b_floyd ? b_tail : b_floyd);
}

__global__ void reverse_into_kernel(const uint32_t* __restrict__ tmp, long long T, long long n,
                                    int* __restrict__ j) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; t < T; t += stride) j[n - 1 - t] = (int)tmp[t];
}

// Lemire j's for _shuffle_int(n, first): steps i = n-1..first, stream from q0.
static int shuffle_int_jgen(Pcg64 g, long long q0, long long n, long long first, int* j, Carve& cv,
                            long long* d_qend, int* d_err, cudaStream_t s) {
  long long T = n - first;
  if (T <= 0) return 0;
  double p = (double)n / 4294967296.0;
  long long vcap = lemire_vcap(T, p);
  uint32_t* v = cv.take<uint32_t>(vcap);
  uint32_t* tmp = cv.take<uint32_t>(T);
  SPTK_REQUIRE(cv.ok(), "sampler workspace too small");
  u32_stream_kernel<<<grid_for(vcap, 256), 256, 0, s>>>(g, (unsigned long long)q0, vcap, v);
  SPTK_CHECK_LAUNCH();
  if (lemire_walk(v, vcap, T, n - 1, -1, tmp, d_qend, d_err, cv, s)) return 1;
  reverse_into_kernel<<<grid_for(T, 256), 256, 0, s>>>(tmp, T, n, j);
  SPTK_CHECK_LAUNCH();
  return 0;
}

// Generator.choice(pop, k, replace=False, shuffle=shuffle) -> out[k] (int32).
// With shuffle=0 the Floyd set is returned in draw order (same set; training
// only needs the set).  The tail-shuffle path is always exact.
int choice(const uint64_t st[4], long long pop, long long k, int shuffle, int* out, void* ws,
           size_t ws_bytes, int* path_out, cudaStream_t s) {
  SPTK_REQUIRE(pop >= 0 && pop < (1LL << 30) && k >= 0 && k <= pop, "choice: bad pop=%lld k=%lld", pop, k);
  SPTK_REQUIRE(ws_bytes >= choice_ws_bytes(pop, k), "choice: workspace too small");
  Carve cv{(char*)ws, ws_bytes};
  long long* d_q = cv.take<long long>(4);
  int* d_err = cv.take<int>(4);
  SPTK_CUDA_TRY(cudaMemsetAsync(d_err, 0, sizeof(int) * 4, s));
  Pcg64 g = make_pcg(st);
  if (pop > 10000 && k > pop / 50) {
    if (path_out) *path_out = 1;
    long long first = pop - k > 1 ? pop - k : 1;
    int* j = cv.take<int>(pop + 1);
    if (shuffle_int_jgen(g, 0, pop, first, j, cv, d_q, d_err, s)) return 1;
    int* res = cv.take<int>(pop + 1);
    if (fy_apply(j, pop, first, res, cv, s)) return 1;
    SPTK_CUDA_TRY(cudaMemcpyAsync(out, res + (pop - k), sizeof(int) * k, cudaMemcpyDeviceToDevice, s));
    return 0;
  }
  if (path_out) *path_out = 2;
  if (k == 0) return 0;
  // Floyd draws: t = 0..k-1, rng = pop-k+t (rng == 0 returns 0 without a draw)
  long long base = pop - k;
  long long t_begin = 0;
  uint32_t* vals = cv.take<uint32_t>(k + 1);
  if (base == 0) {
    SPTK_CUDA_TRY(cudaMemsetAsync(vals, 0, sizeof(uint32_t), s));
    t_begin = 1;
  }
  long long T = k - t_begin;
  double p = (double)pop / 4294967296.0;
  long long vcap = lemire_vcap(T, p);
  uint32_t* v = cv.take<uint32_t>(vcap);
  if (T > 0) {
    u32_stream_kernel<<<grid_for(vcap, 256), 256, 0, s>>>(g, 0ULL, vcap, v);
    SPTK_CHECK_LAUNCH();
    if (lemire_walk(v, vcap, T, base + t_begin, +1, vals + t_begin, d_q, d_err, cv, s)) return 1;
  } else {
    SPTK_CUDA_TRY(cudaMemsetAsync(d_q, 0, sizeof(long long), s));
  }
  long long hs = 1;
  while (hs < 2 * k + 2) hs <<= 1;
  uint32_t* keys = cv.take<uint32_t>(hs);
  int* mint = cv.take<int>(hs);
  unsigned char* first = cv.take<unsigned char>(k + 1);
  SPTK_CUDA_TRY(cudaMemsetAsync(keys, 0xff, sizeof(uint32_t) * hs, s));
  SPTK_CUDA_TRY(cudaMemsetAsync(mint, 0x7f, sizeof(int) * hs, s));
  floyd_insert_kernel<<<grid_for(k, 256), 256, 0, s>>>(vals, k, keys, mint, (uint32_t)(hs - 1));
  SPTK_CHECK_LAUNCH();
  floyd_first_kernel<<<grid_for(k, 256), 256, 0, s>>>(vals, k, keys, mint, (uint32_t)(hs - 1), first);
  SPTK_CHECK_LAUNCH();
  int* sel = shuffle ? cv.take<int>(k + 1) : out;
  floyd_out_kernel<<<grid_for(k, 256), 256, 0, s>>>(vals, k, base, first, sel);
  SPTK_CHECK_LAUNCH();
  if (!shuffle || k < 2) {
    if (shuffle && k == 1) SPTK_CUDA_TRY(cudaMemcpyAsync(out, sel, sizeof(int), cudaMemcpyDeviceToDevice, s));
    return 0;
  }
  // _shuffle_int(k, 1, idx): continues the stream after the Floyd draws.
  // The stream offset lives on the device (d_q), so read it back (one small
  // sync, only on the exact-output path used by tests / the public API).
  long long qend = 0;
  SPTK_CUDA_TRY(cudaMemcpyAsync(&qend, d_q, sizeof(long long), cudaMemcpyDeviceToHost, s));
  int herr = 0;
  SPTK_CUDA_TRY(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPTK_CUDA_TRY(cudaStreamSynchronize(s));
  SPTK_REQUIRE(herr == 0, "choice: Lemire stream overflow");
  int* j = cv.take<int>(k + 1);
  if (shuffle_int_jgen(g, qend, k, 1, j, cv, d_q, d_err, s)) return 1;
  int* perm = cv.take<int>(k + 1);
  if (fy_apply(j, k, 1, perm, cv, s)) return 1;
  gather_kernel<<<grid_for(k, 256), 256, 0, s>>>(sel, perm, k, out);
  SPTK_CHECK_LAUNCH();
  return 0;
}

int u32_stream(const uint64_t st[4], unsigned long long q0, long long n, uint32_t* out, cudaStream_t s) {
  Pcg64 g = make_pcg(st);
  if (n <= 0) return 0;
  u32_stream_kernel<<<grid_for(n, 256), 256, 0, s>>>(g, q0, n, out);
  SPTK_CHECK_LAUNCH();
  return 0;
}

int iota(int* out, long long n, int offset, cudaStream_t s) {
  if (n <= 0) return 0;
  iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n, offset);
  SPTK_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// (5) DSGD block visit orders in shared memory.
//
// With W > 1 workers the reference draws one permutation per block,
// default_rng([seed, 1, t, *block]).permutation(len(ids)) (trainer.py:
// 196-199), and runs the W blocks of a round in parallel.  Blocks of up to
// 18,000 nonzeros are done entirely by one CTA:
//   j-sequence   one warp walks the PCG64 stream level by level (the same
//                masked-rejection walk as walk_exact, with the lane states
//                carried across levels) into J[1..n-1]
//   apply        Fisher-Yates by target lists: counting sort of the steps by
//                target, each list sorted (short), V(p) = root of the chain
//                p -> smallest step > p targeting p (pointer jumping), then
//                final[i] = V(previous step of i's list) or the target itself
//   output       visit[slot] = block offset + final[p], where slot interleaves
//                the round's blocks (the round's blocks share no rows, so
//                interleaving them is the reference's parallel round; it also
//                spreads the GPU's samples in flight over every block)
// Two launches: the j-sequences (one warp per block, 2 bytes per nonzero of
// global scratch), then the apply (one CTA per block, 12 bytes of shared
// memory per nonzero), every phase of it parallel over the block's steps.
// ---------------------------------------------------------------------------
struct BlockJob {
  long long off;       // first record of the block (partitioned layout)
  long long out_base;  // first visit slot of the block's round
  int n;               // nonzeros in the block
  int first;           // index of the round's first job (jobs are round-major)
  int m;               // jobs in the round
  int slot;            // this job's index within its round
  int nmin;            // smallest block of the round (below it the interleave is p * m + slot)
  int pad;
};

// one warp: J[hi - count] = draw for every level (numpy's random_interval).
// group_accept specialised to small blocks: 32-bit arithmetic and one set of
// ballots per group.
__device__ __forceinline__ void block_jgen(const Pcg64& g, int n, uint16_t* J) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  if (n < 2) return;
  u128 A32, C32;
  pcg_jump_coeffs(g.inc, 32, &A32, &C32);
  u128 state = pcg_advance(g, (uint64_t)lane + 1);  // output m = lane
  int mbase = 0, qs = 0;
  const int kb = 32 - __clz((unsigned)(n - 1));
  for (int k = kb; k >= 1; --k) {
    const int hi = min((1 << k) - 1, n - 1), S = hi - (1 << (k - 1)) + 1;
    const unsigned mask = (1u << k) - 1u;
    int a = 0;
    while (a < S) {
      const uint64_t out = pcg_xsl_rr(state);
      const int q0 = 2 * (mbase + lane);
      const unsigned u0 = (uint32_t)out & mask, u1 = (uint32_t)(out >> 32) & mask;
      const int d0 = hi - (int)u0 - a, d1 = hi - (int)u1 - a;  // accept iff (accepts before) <= d
      const bool v0 = q0 >= qs, v1 = q0 + 1 >= qs;
      bool c0 = v0 && d0 >= 63, c1 = v1 && d1 >= 63;
      bool x0 = v0 && (unsigned)d0 < 63u, x1 = v1 && (unsigned)d1 < 63u;
      unsigned X0 = __ballot_sync(FULLMASK, x0), X1 = __ballot_sync(FULLMASK, x1);
      while (X0 | X1) {
        const unsigned A0 = __ballot_sync(FULLMASK, c0), A1 = __ballot_sync(FULLMASK, c1);
        const int lo0 = __popc(A0 & lt) + __popc(A1 & lt), hi0 = lo0 + __popc(X0 & lt) + __popc(X1 & lt);
        const int lo1 = lo0 + (c0 ? 1 : 0), hi1 = hi0 + ((c0 || x0) ? 1 : 0);
        if (x0 && (d0 >= hi0 || d0 < lo0)) {
          c0 = d0 >= hi0;
          x0 = false;
        }
        if (x1 && (d1 >= hi1 || d1 < lo1)) {
          c1 = d1 >= hi1;
          x1 = false;
        }
        X0 = __ballot_sync(FULLMASK, x0);
        X1 = __ballot_sync(FULLMASK, x1);
      }
      const unsigned b0 = __ballot_sync(FULLMASK, c0), b1 = __ballot_sync(FULLMASK, c1);
      const int before0 = a + __popc(b0 & lt) + __popc(b1 & lt), before1 = before0 + (c0 ? 1 : 0);
      const int total = __popc(b0) + __popc(b1);
      // accepts past the level's S-th are not this level's
      if (c0 && before0 < S) J[hi - before0] = (uint16_t)u0;
      if (c1 && before1 < S) J[hi - before1] = (uint16_t)u1;
      if (a + total >= S) {
        // the level ends inside this group; the next one continues after it
        int p = -1;
        if (c0 && before0 == S - 1) p = q0;
        if (c1 && before1 == S - 1) p = q0 + 1;
        const unsigned who = __ballot_sync(FULLMASK, p >= 0);
        qs = __shfl_sync(FULLMASK, p, __ffs(who) - 1) + 1;
        a = S;
        if (qs >= 2 * (mbase + 32)) {
          state = state * A32 + C32;
          mbase += 32;
        }
      } else {
        a += total;
        state = state * A32 + C32;
        mbase += 32;
      }
    }
  }
}

__device__ __forceinline__ Pcg64 block_seed(const BlockJob& jb, const int* __restrict__ coords, int order,
                                              unsigned long long seed, long long t, long long b) {
  uint64_t ent[3 + SPTK_MAX_MODES];
  ent[0] = seed;
  ent[1] = 1;
  ent[2] = (uint64_t)t;
  for (int d = 0; d < order; ++d) ent[3 + d] = (uint64_t)coords[b * order + d];
  uint32_t words[64];
  const int nw = seedseq_words(ent, 3 + order, words, 64);
  return seedseq_pcg64(words, nw < 0 ? 0 : nw);
}

// j-sequences: one warp per block, into the block's slice of js (record order)
#define BP_JW 8
__global__ void __launch_bounds__(32 * BP_JW) block_jgen_kernel(const BlockJob* __restrict__ jobs, int n_jobs,
                                                                 const int* __restrict__ coords, int order,
                                                                 unsigned long long seed, long long t,
                                                                 uint16_t* __restrict__ js) {
  const long long b = (long long)blockIdx.x * BP_JW + (threadIdx.x >> 5);
  if (b >= n_jobs) return;
  const BlockJob jb = jobs[b];
  const Pcg64 g = block_seed(jb, coords, order, seed, t, b);  // every lane, same value
  block_jgen(g, jb.n, js + jb.off);
  if ((threadIdx.x & 31) == 0 && jb.n > 0) js[jb.off] = 0;  // virtual step 0 (position 0 keeps what is left)
}

// threads per block permutation CTA (NF W=24: 256 / 512 / 1024 -> 1.72 /
// 1.62 / 2.24 ms per epoch)
#ifndef BP_T
#define BP_T 512
#endif
// Shared memory per nonzero: 8 bytes -- C (group counts, then group starts /
// ends: 16-bit halves of 32-bit words, so the counting and scatter atomics
// stay 32-bit), J (target of each step), S (each target's group sorted by
// step, descending), and one array that holds L (steps grouped by target)
// until S is built and V (chain roots) after.  16-bit entries: n <= 28000.
#define BP_CAP 28000
__device__ __forceinline__ unsigned c16_inc(unsigned* C, int t) {
  const unsigned sh = (t & 1) * 16;
  return (atomicAdd(&C[t >> 1], 1u << sh) >> sh) & 0xFFFFu;
}
__global__ void __launch_bounds__(BP_T) block_fy_kernel(const BlockJob* __restrict__ jobs,
                                                        const uint16_t* __restrict__ js,
                                                        int* __restrict__ visit, int cap) {
  extern __shared__ __align__(16) unsigned char bp_sm[];
  // a zero word, then C: once the counts are group ends, Cu[t] reads C's
  // 16-bit half t directly and Cu[-1] = 0 is group 0's start
  unsigned* C = reinterpret_cast<unsigned*>(bp_sm) + 1;  // [cap/2 + 1] packed 16-bit
  const uint16_t* Cu = reinterpret_cast<const uint16_t*>(C);
  uint16_t* J = reinterpret_cast<uint16_t*>(C + (cap / 2 + 1));
  uint16_t* S = J + cap;
  uint16_t* LV = S + cap;  // L, then V
  __shared__ int sh[33];
  // the round's block sizes (slot order), ascending (with prefix sums), and
  // the sizes of the slots before this one, ascending: the interleaved slot
  // of entries past the round's smallest block by two binary searches
  __shared__ int sizes[64], srt[64], low[64];
  __shared__ long long pre[65];
  const BlockJob jb = jobs[blockIdx.x];
  const int n = jb.n, tid = threadIdx.x, m = min(jb.m, 64);
  if (tid < m) sizes[tid] = jobs[jb.first + tid].n;
  if (tid == 0) reinterpret_cast<unsigned*>(bp_sm)[0] = 0u;
  for (int p = tid; p < (n + 1) / 2; p += BP_T) C[p] = 0u;
  for (int p = tid; p < n; p += BP_T) J[p] = js[jb.off + p];
  __syncthreads();
  if (tid < m) {
    const int v = sizes[tid];
    int r = 0, rl = 0;
    for (int s2 = 0; s2 < m; ++s2) {
      const int w = sizes[s2];
      r += w < v || (w == v && s2 < tid);
      rl += s2 < jb.slot && (w < v || (w == v && s2 < tid));
    }
    srt[r] = v;
    if (tid < jb.slot) low[rl] = v;
  }
  for (int i = tid; i < n; i += BP_T) c16_inc(C, J[i]);
  __syncthreads();
  if (tid == 0) {
    long long a = 0;
    pre[0] = 0;
    for (int s2 = 0; s2 < m; ++s2) pre[s2 + 1] = a += srt[s2];
  }
  {
    // exclusive scan of the 16-bit counts, each thread a run of whole words
    const int words = (n + 1) / 2;
    const int per = (words + BP_T - 1) / BP_T, a = tid * per, z = min(words, a + per);
    int run = 0;
    for (int w = a; w < z; ++w) run += (int)(C[w] & 0xFFFFu) + (int)(C[w] >> 16);
    int tot;
    int ex = block_excl_scan(run, sh, &tot);
    for (int w = a; w < z; ++w) {
      const unsigned c0 = C[w] & 0xFFFFu, c1 = C[w] >> 16;
      C[w] = (unsigned)ex | ((unsigned)(ex + (int)c0) << 16);
      ex += (int)(c0 + c1);
    }
  }
  __syncthreads();
  // steps grouped by target (group starts -> group ends)
  for (int i = tid; i < n; i += BP_T) LV[c16_inc(C, J[i])] = (uint16_t)i;
  __syncthreads();
  // each step's place in its target's group, largest step first (the order
  // Fisher-Yates runs them): rank = number of larger steps in the group.
  // Walked in L order, so the lanes of a warp mostly share a group (the same
  // trip count, broadcast reads)
  for (int x0 = tid; x0 < n; x0 += BP_T) {
    const int i = LV[x0], t = J[i], s0 = Cu[t - 1], s1 = Cu[t];
    int rank = 0;
#pragma unroll 1
    for (int x = s0; x < s1; ++x) rank += (int)LV[x] > i;
    S[s0 + rank] = (uint16_t)i;
  }
  __syncthreads();
  // L is dead: V(p) = p (no step above p targets p: p keeps its own value)
  for (int p = tid; p < n; p += BP_T) LV[p] = (uint16_t)p;
  __syncthreads();
  // every step targeting t is >= t: the smallest step above t (t's parent)
  // is the last of the group, or the second to last after t's own step
  for (int t = tid; t < n; t += BP_T) {
    const int s0 = Cu[t - 1], s1 = Cu[t];
    if (s1 > s0) {
      const int last = S[s1 - 1];
      if (last > t) LV[t] = (uint16_t)last;
      else if (s1 - s0 >= 2) LV[t] = S[s1 - 2];
    }
  }
  __syncthreads();
  // V(p) = root of p's chain, by walking it (chains are short: mean depth
  // ~1, ~3 for the deepest of a warp's 32 at n = 12,400; pointer jumping took
  // 5 passes over every entry).  racecheck reports the read of LV[v] against
  // other threads' writes: benign -- every value LV[q] ever holds is an
  // ancestor of q on q's chain (roots never change), so a stale or a fresh
  // read both lead to the same root
  for (int p = tid; p < n; p += BP_T) {
    int v = LV[p];
    for (;;) {
      const int w = LV[v];
      if (w == v) break;
      v = w;
    }
    LV[p] = (uint16_t)v;
  }
  __syncthreads();
  // result[i]: the value its target held just before step i, written straight
  // to its round-interleaved slot:
  //   slot(p) = sum_s min(n_s, p) + #{s < slot : n_s > p}
  for (int x = tid; x < n; x += BP_T) {
    const int i = S[x], t = J[i], s0 = Cu[t - 1];
    const int val = x == s0 ? t : (int)LV[S[x - 1]];
    long long pos = jb.out_base;
    if (i < jb.nmin) {
      pos += (long long)i * m + jb.slot;  // every block of the round still has entries
    } else {
      // k sizes below i: sum_s min(n_s, i) = pre[k] + i (m - k); then the
      // earlier slots whose blocks are longer than i
      int k = 0, q = 0;
#pragma unroll
      for (int st = 64; st; st >>= 1) {
        if (k + st <= m && srt[k + st - 1] < i) k += st;
        if (q + st <= jb.slot && low[q + st - 1] <= i) q += st;
      }
      pos += pre[k] + (long long)i * (m - k) + (jb.slot - q);
    }
    visit[pos] = (int)(jb.off + val);
  }
}

int block_perm(const void* d_jobs, const int* d_coords, int n_jobs, int order, unsigned long long seed,
               long long t, int cap, uint16_t* d_js, int* d_visit, cudaStream_t s) {
  SPTK_REQUIRE(n_jobs >= 0 && order >= 1 && order <= SPTK_MAX_MODES, "block_perm: bad arguments");
  SPTK_REQUIRE(cap >= 1 && cap <= BP_CAP, "block_perm: block capacity must be in [1, %d]", BP_CAP);
  if (n_jobs == 0) return 0;
  const BlockJob* jobs = (const BlockJob*)d_jobs;
  block_jgen_kernel<<<(n_jobs + BP_JW - 1) / BP_JW, 32 * BP_JW, 0, s>>>(jobs, n_jobs, d_coords, order, seed, t, d_js);
  SPTK_CHECK_LAUNCH();
  const size_t smem = (size_t)(cap / 2 + 1) * 4 + (size_t)cap * 6 + 16;
  static size_t configured = 0;
  if (smem > configured) {
    SPTK_CUDA_TRY(cudaFuncSetAttribute(block_fy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  block_fy_kernel<<<n_jobs, BP_T, smem, s>>>(jobs, d_js, d_visit, cap);
  SPTK_CHECK_LAUNCH();
  return 0;
}
size_t block_job_bytes() { return sizeof(BlockJob); }
// Round-interleaved visit list from per-block visit orders that lie in the
// partitioned layout (perm[off_b + p], relative to off_b when rel_lo < 0,
// else to rel_lo): the layout block_fy_kernel writes, for blocks too large for
// one CTA's shared memory (their orders come from the batched j-sequence +
// Fisher-Yates apply).  One CTA per block.
__global__ void __launch_bounds__(256) interleave_kernel(const BlockJob* __restrict__ jobs,
                                                         const int* __restrict__ perm, long long rel_lo,
                                                         int* __restrict__ visit) {
  __shared__ int sizes[64];
  const BlockJob jb = jobs[blockIdx.x];
  const int m = min(jb.m, 64);
  if (threadIdx.x < m) sizes[threadIdx.x] = jobs[jb.first + threadIdx.x].n;
  __syncthreads();
  const long long add = rel_lo < 0 ? jb.off : rel_lo;
  // blockIdx.y splits a large block's entries over several CTAs
  for (int p = blockIdx.y * blockDim.x + threadIdx.x; p < jb.n; p += gridDim.y * blockDim.x) {
    long long pos = jb.out_base;
    if (p < jb.nmin) {
      pos += (long long)p * m + jb.slot;
    } else {
      for (int s2 = 0; s2 < m; ++s2) {
        const int ns = sizes[s2];
        pos += ns < p ? ns : p;
        if (s2 < jb.slot && ns > p) ++pos;
      }
    }
    visit[pos] = (int)(add + __ldg(perm + jb.off + p));
  }
}

int interleave_rounds(const void* d_jobs, int n_jobs, const int* d_perm, long long rel_lo, int* d_visit,
                      cudaStream_t s, long long cap) {
  if (n_jobs <= 0) return 0;
  // enough CTAs per block for ~4K entries each, and at least ~4 waves overall
  long long ys = (cap + 4095) / 4096;
  if (ys < 1) ys = 1;
  if (ys > 65535) ys = 65535;
  interleave_kernel<<<dim3((unsigned)n_jobs, (unsigned)ys), 256, 0, s>>>((const BlockJob*)d_jobs, d_perm, rel_lo,
                                                                         d_visit);
  SPTK_CHECK_LAUNCH();
  return 0;
}


}  // namespace sptk
