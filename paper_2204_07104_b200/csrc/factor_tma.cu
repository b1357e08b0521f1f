// factor_tma.cu -- K3 v6: the tcgen05 factor kernel with its row traffic on TMA.
//
// Same per-sample update as factor_tc2_kernel (_loops.py:17-63, Hogwild over
// the visit order; c refresh folded into the gs round through G_n = B_n^T B_n):
//
//   c_n  = A_n[tile] . B_n           (128 x R)  one MMA round per tile
//   gs_n = W_n . B_n^T,  h_n = W_n . G_n           one MMA round per mode
//   a'   = a - gamma(-x gs + lambda a + (a.gs) gs),  c_n' = (1 - gamma lambda) c_n + gamma (x - a.gs) h_n
//
// What changes against v2 is where the bytes move:
//  * rows are gathered by the tensor memory accelerator: a 2-D tensor map per
//    factor matrix and `tile::gather4` (four arbitrary rows per instruction)
//    write straight into a K-major operand tile in the swizzled layout whose
//    swizzle span is one row (32 / 64 B for J = 8 / 16), completing on an
//    mbarrier -- no per-lane cp.async, no load/store-pipe traffic;
//  * rows go back the same way: cold (large) modes as `tile::scatter4` stores
//    of the updated rows, hot (small) modes as one bulk fp32 add-reduction of
//    the 64-byte delta per sample (atomic at L2, nothing lost);
//  * W_n is written to TMEM (tcgen05.st) and used as the MMA's A operand from
//    there, so it never touches shared memory;
//  * the only CTA-wide barrier per mode is the one that hands W_n to the MMA.
// Thread t <-> sample t <-> TMEM lane t <-> row t of every operand tile; the
// swizzle keeps each row inside its own 16*J-byte span, so a thread reads and
// rewrites its row without conflicts and without touching other rows.
#include "common.cuh"
#include "factor_tc_util.cuh"
#include "kernels.cuh"
#include "tc.cuh"

#include <cudaTypedefs.h>

#include <atomic>
#include <stdio.h>
#include <stdlib.h>

namespace sptk {

template <int N>
struct TmaMaps {
  CUtensorMap m[N];
};

template <int N>
struct TmaParams {
  long long foff[N];
  float gam[N];
  float lam[N];
  long long* dbg;         // optional per-phase clock stamps of block 0 (long long[16][16])
  unsigned atomic_mask;   // bit n: mode-n rows are written back as add-reduced deltas (hot modes)
  unsigned early_mask;    // bit n: the next tile's mode-n rows are gathered while this tile runs
  int bulk_red;           // hot deltas as one bulk add-reduction per sample (TMA unit) instead of red.add.v4
};

// DSGD across GPUs, fused into the factor kernel (sptk_factor_pass_dsgd):
// the rank's visit list holds its blocks round after round, each round padded
// to whole 128-sample tiles (padding entries -1).  A tile of round r >= 1
// starts only once the rotated block of round r has landed (*ready >= gen0 +
// r, written by the sending rank over NVLink); the CTA that finishes the last
// tile of round r copies the block this rank hands on to its next owner
// (peer stores) and raises that rank's ready flag (release at system scope).
// (partition.py:100-117: consecutive rounds move one mode's blocks one rank
// along the ring.)
struct DsgdPush {
  long long row_lo;  // first row of the block
  long long nrows;   // 0: nothing to send after this round
  long long mode;
  float* dst;        // the receiving rank's copy of row row_lo (peer pointer)
  int* dst_ready;    // the receiving rank's ready flag (peer pointer)
  int* dst_gathered; // the receiving rank's epoch flag: its epoch-end exchange of epoch e-1 is written (peer)
};
struct DsgdParams {
  const long long* rstart;  // [n_rounds + 1] first visit slot of each round (multiples of 128)
  const long long* rend;    // [n_rounds] end of each round's valid samples
  const DsgdPush* push;     // [n_rounds]
  int* done;                // [n_rounds] finished tiles (zeroed by the launcher)
  int* ready;               // this rank's flag: rounds whose incoming block has landed
  int n_rounds;
  int gen0;                 // global round number of this epoch's round 0
  int epoch;                // the receiver's epoch flag must be >= this before a push lands
};

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_sys(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int N, int J, int R>
struct TmaCfg {
  static constexpr int M = 128;
  static constexpr int ROWB = J * 4;       // bytes per row = swizzle span
  static constexpr int SLOT = M * J;       // floats per operand tile
  static constexpr int NSLOT = N + 1;      // + a second slot for the last mode (only when it is gathered early)
  static constexpr int OFF_A = 0;          // slots first: 1024-byte aligned
  static constexpr int OFF_BT = OFF_A + N * SLOT;      // N x (R rows x J), canonical
  static constexpr int OFF_BN = OFF_BT + N * R * J;    // N x (J rows x R)
  static constexpr int OFF_G = OFF_BN + N * J * R;     // N x (R rows x R)
  static constexpr int OFF_BAR = (OFF_G + N * R * R + 1) & ~1;  // NSLOT + 1 mbarriers
  static constexpr int OFF_MISC = OFF_BAR + 2 * (NSLOT + 1);     // TMEM address, tile claim
  static constexpr int OFF_IDX = (OFF_MISC + 4 + 3) & ~3;         // [2][N][128] row indices (16-B aligned)
  static constexpr int RWC = N <= 3 ? 4 : (N <= 7 ? 8 : 16);     // record words
  static constexpr int OFF_RING = OFF_IDX + 2 * N * M;            // [2][128][RWC] records in flight (cp.async)
  static constexpr int OFF_SPARE = (OFF_RING + 2 * M * RWC + 255) & ~255;  // the spare slot, last (1024-B aligned)
  static constexpr size_t SMEM = (size_t)OFF_SPARE * 4 + 1024;          // + alignment slack
  static constexpr size_t SMEM_SPARE = SMEM + (size_t)SLOT * 4;
  // TMEM columns: the c round writes c_0..c_{N-1} at n*R; afterwards W at 0,
  // gs at R, h at R + J (c lives in registers by then)
  static constexpr int COL_W = 0, COL_G = R, COL_H = R + J;
  static constexpr int NEED = (N * R > 2 * R + J) ? N * R : 2 * R + J;
  static constexpr int TCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : 256;
};

// float offset of (row, 16-byte chunk q) in a swizzled operand tile of J-float rows
template <int J>
__device__ __forceinline__ int swz(int row, int q) {
  constexpr int CH = J / 4;
  return row * J + 4 * (q ^ (((row * J * 4) >> 7) & (CH - 1)));
}

template <int R>
__device__ __forceinline__ void tmem_st_row(uint32_t taddr, const float* v) {
  if (R % 16 == 0) {
#pragma unroll
    for (int q = 0; q < R / 16; ++q) tc::tmem_st16(taddr + 16 * q, v + 16 * q);
  } else {
#pragma unroll
    for (int q = 0; q < R / 8; ++q) tc::tmem_st8(taddr + 8 * q, v + 8 * q);
  }
}

__device__ unsigned g_tma_tile_ctr[64];

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(pred));
  return pred != 0;
}

#ifdef SPTK_TMA_STAMPS
#define TMA_STAMP(k)                                                                                       \
  do {                                                                                                     \
    if (p.dbg && blockIdx.x == 0 && tid == 0 && ntile < 16) p.dbg[ntile * 16 + (k)] = clock64();          \
  } while (0)
#else
#define TMA_STAMP(k) \
  do {               \
  } while (0)
#endif

// CTAs per SM the register budget is sized for: four (128 registers).  Five
// (96 registers, ~100 bytes of spill) measured slower at N = 3, J = 16: NF
// factor pass 7.8 -> 8.9 ms.
#ifndef SPTK_TMA_MINB_3_16
#define SPTK_TMA_MINB_3_16 4
#endif
template <int N, int J>
// Rank 8 at order 3 keeps less per sample (80 registers): six CTAs per SM.
// NF factor pass J=8 7.26 -> 5.27 ms, J=4 (rank-8 padding) 7.42 -> 5.40 ms.
// Order 6 at five CTAs (96 registers): with the record ring ~40 bytes of
// spill, O6 epoch 129.7 -> 121.0 ms (before the ring: ~100 bytes, 149 -> 153).
#ifndef SPTK_TMA_MINB_3_8
#define SPTK_TMA_MINB_3_8 6
#endif
#ifndef SPTK_TMA_MINB_6_8
#define SPTK_TMA_MINB_6_8 5
#endif
constexpr int tma_min_blocks() {
  return (N == 3 && J == 16) ? SPTK_TMA_MINB_3_16
                             : (N == 3 && J == 8) ? SPTK_TMA_MINB_3_8 : (N == 6 && J == 8) ? SPTK_TMA_MINB_6_8 : 4;
}
template <int N, int J, int R, bool HV, bool DS = false>
__global__ void __launch_bounds__(128, tma_min_blocks<N, J>())
    factor_tma_kernel(const int* __restrict__ rec, const int* __restrict__ visit, long long n_visit, long long base,
                      float* __restrict__ fac, const float* __restrict__ cor, const __grid_constant__ TmaParams<N> p,
                      const __grid_constant__ TmaMaps<N> maps, unsigned* __restrict__ tile_ctr,
                      const __grid_constant__ DsgdParams dp) {
  constexpr int RW = N <= 3 ? 4 : (N <= 7 ? 8 : 16);
  using C = TmaCfg<N, J, R>;
  extern __shared__ __align__(16) float sm_raw[];
  // operand tiles need 1024-byte alignment; offsetting the __shared__ array
  // itself keeps every access a shared-space one (LDS/STS)
  float* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u) / 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);  // [NSLOT]: row tiles landed
  uint64_t* mbar = full + C::NSLOT;                                 // MMA round done
  uint32_t* misc = reinterpret_cast<uint32_t*>(sm + C::OFF_MISC);   // [0] TMEM address, [1] tile claim
  int* ids = reinterpret_cast<int*>(sm + C::OFF_IDX);               // [2 tiles][N modes][128] row indices
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int ntile = 0;
  (void)ntile;

  for (int e = tid; e < N * J * R; e += 128) {
    const int n = e / (J * R), rem = e - n * (J * R), j = rem / R, r = rem - j * R;
    const float b = __ldg(cor + e);
    sm[C::OFF_BT + n * R * J + canon<R>(r, j)] = b;
    sm[C::OFF_BN + n * J * R + canon<J>(j, r)] = b;
  }
  for (int e = tid; e < N * R * R; e += 128) {
    const int n = e / (R * R), rem = e - n * (R * R), r = rem / R, r2 = rem - r * R;
    float g = 0.f;
    for (int j = 0; j < J; ++j) g = fmaf(__ldg(cor + n * J * R + j * R + r), __ldg(cor + n * J * R + j * R + r2), g);
    sm[C::OFF_G + n * R * R + canon<R>(r, r2)] = g;
  }
  if (tid == 0) {
    for (int s = 0; s <= C::NSLOT; ++s) tc::mbar_init(&full[s], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&misc[0], C::TCOLS);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = misc[0];
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t id_c = tc::idesc_tf32(128, R), id_g = tc::idesc_tf32(128, J), id_h = tc::idesc_tf32(128, R);
  const uint64_t pol_stream = tc::policy_evict_first();
  uint32_t mphase = 0, fphase = 0;  // fphase bit s: parity of slot s's next completion

  const unsigned early = p.early_mask;
  const int spare = (early >> (N - 1)) & 1u;  // the last mode double-buffers only when gathered early
  auto slot_of = [&](int n, int pb) { return (n == N - 1 && pb) ? N : n; };
  auto slot_off = [&](int s) { return s < N ? C::OFF_A + s * C::SLOT : C::OFF_SPARE; };
  auto slot_addr = [&](int s) { return sbase + 4u * (uint32_t)slot_off(s); };

  // Row indices of a tile, one int per (mode, sample), so that an elected lane
  // of each warp reads four rows with one LDS.128 and issues the warp's eight
  // gather4 / scatter4 operations in a uniform loop.  Past-the-end samples
  // carry row 0 (gathered, never written back).
  auto gather = [&](int n, int s, int par) {
    if (tid == 0) tc::mbar_expect_tx(&full[s], C::SLOT * 4);
    if (elect_one()) {
      const int4* id4 = reinterpret_cast<const int4*>(ids + (par * N + n) * 128 + warp * 32);
      const uint32_t dst = slot_addr(s) + warp * 32 * C::ROWB, bar = tc::smem_u32(&full[s]);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int4 r = id4[k];
        tc::tma_gather4(dst + 4 * k * C::ROWB, &maps.m[n], r.x, r.y, r.z, r.w, bar);
      }
    }
  };

  const long long G = gridDim.x;
  long long tile = blockIdx.x, t1 = tile + G, t2 = tile + 2 * G;
  if (tid == 0) misc[1] = atomicAdd(tile_ctr, 1u);
  // Records travel through a two-slot shared-memory ring (cp.async, issued
  // two tiles ahead) instead of registers: a thread keeps only its current and
  // next sample's value and validity; row indices are staged into ids[].
  // 127 -> 120 registers; NF W=20 factor pass 7.38 -> 7.20 ms (five CTAs per
  // SM at this size still spill ~56 bytes and ran slower: 7.58 ms).  The
  // cp.async here carries no L2 cache-hint operand: with one (evict_first
  // policy) the B200 raised "illegal instruction" on it.
  int* ring = reinterpret_cast<int*>(sm + C::OFF_RING);
  // DS: padding entries (-1) are invalid samples that read record 0
  auto fetch = [&](int q, int v, long long t) -> bool {
    bool ok = tile_valid(n_visit, t);
    if (DS) {
      ok = ok && v >= 0;
      v = v < 0 ? 0 : v;
    }
    const int* src = rec + (base + (long long)v) * RW;
    const uint32_t dst = tc::smem_u32(ring + (q * 128 + tid) * RW);
    tc::cp_async16_nohint(dst, src, 16u);
    if (RW >= 8) tc::cp_async16_nohint(dst + 16, src + 4, 16u);
    tc::cp_async_commit();
    return ok;
  };
  auto stage = [&](int q, bool ok, int par) -> float {
    const int4* r = reinterpret_cast<const int4*>(ring + (q * 128 + tid) * RW);
    int wv[8];
    const int4 w0 = r[0];
    wv[0] = w0.x, wv[1] = w0.y, wv[2] = w0.z, wv[3] = w0.w;
    if (RW >= 8) {
      const int4 w1 = r[1];
      wv[4] = w1.x, wv[5] = w1.y, wv[6] = w1.z, wv[7] = w1.w;
    }
#pragma unroll
    for (int n = 0; n < N; ++n) ids[(par * N + n) * 128 + tid] = ok ? wv[n] : 0;
    return __int_as_float(wv[N]);
  };
  int v2 = load_vis<HV>(visit, n_visit, t2, pol_stream);
  bool ok_cur = fetch(0, load_vis<HV>(visit, n_visit, tile, pol_stream), tile);
  bool ok_nxt = fetch(1, load_vis<HV>(visit, n_visit, t1, pol_stream), t1);
  asm volatile("cp.async.wait_group 1;" ::: "memory");
  float x_cur = stage(0, ok_cur, 0), x_nxt = 0.f;
  int rs = 1;  // ring slot of the next tile's record
  // DS round tracking: the round of this CTA's current tile (tiles only grow)
  int r_cur = 0, r_waited = 0, r_tiles = 0;
  auto adv = [&](int r, long long t) {
    while (r + 1 < dp.n_rounds && t * 128 >= dp.rstart[r + 1]) ++r;
    return r;
  };
  int pb = 0, par = 0;
  __syncwarp();
#pragma unroll
  for (int n = 0; n < N; ++n)
    if (early >> n & 1u) gather(n, slot_of(n, pb), 0);
  __syncthreads();
  long long t3 = 3 * G + misc[1];
  while (tile * 128 < n_visit) {
    TMA_STAMP(0);
    if (DS) {
      // a tile of a later round: its rotated block must have landed
      r_cur = adv(r_cur, tile);
      if (r_cur > r_waited) {
        if (tid == 0) {
          while (ld_relaxed_sys(dp.ready) < dp.gen0 + r_cur) __nanosleep(64);
          (void)ld_acquire_sys(dp.ready);
          fence_proxy_async_global();
        }
        __syncthreads();
        r_waited = r_cur;
      }
    }
    unsigned claim = 0;
    if (tid == 0) claim = atomicAdd(tile_ctr, 1u);
    // late modes (the hot ones by default) are read at the start of their own
    // tile, which keeps their Hogwild read-to-write window short
#pragma unroll
    for (int n = 0; n < N; ++n)
      if (!(early >> n & 1u)) gather(n, slot_of(n, pb), par);
    // the record of the tile after next into the free ring slot; the next
    // tile's (issued a tile ago) has landed: its indices for its early gathers
    // during this tile
    const bool ok_nn = fetch(rs ^ 1, v2, t2);
    v2 = load_vis<HV>(visit, n_visit, t3, pol_stream);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    x_nxt = stage(rs, ok_nxt, par ^ 1);
    const bool full_tile = (tile + 1) * 128 <= (DS ? dp.rend[r_cur] : n_visit);
    TMA_STAMP(1);
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const int s = slot_of(n, pb);
      tc::mbar_wait(&full[s], (fphase >> s) & 1u);
      fphase ^= 1u << s;
    }
    TMA_STAMP(2);
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const uint32_t a = slot_addr(slot_of(n, pb));
        const uint32_t b = sbase + 4u * (C::OFF_BT + n * R * J);
#pragma unroll
        for (int kk = 0; kk < J / 8; ++kk)
          tc::mma_tf32(tbase + n * R, tc::smem_desc_sw<C::ROWB>(a + 32 * kk),
                       tc::smem_desc(b + kk * 2 * (R * 16), R * 16, 128), id_c, kk > 0 ? 1u : 0u);
      }
      tc::mma_commit(mbar);
    }
    tc::mbar_wait(mbar, mphase);
    mphase ^= 1;
    tc::fence_after_sync();
    TMA_STAMP(3);
    float c[N][R];
#pragma unroll
    for (int n = 0; n < N; ++n) tc::tmem_ldh<R>(tlane + n * R, c[n]);

#pragma unroll
    for (int n = 0; n < N; ++n) {
      {
        float w[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float v = 0.f;
          bool first = true;
#pragma unroll
          for (int n0 = 0; n0 < N; ++n0)
            if (n0 != n) {
              v = first ? c[n0][r] : v * c[n0][r];
              first = false;
            }
          w[r] = v;
        }
        tmem_st_row<R>(tlane + C::COL_W, w);
      }
      tc::tmem_wait_st();
      // earlier write-backs have read their slots (slot n-1 is re-gathered below)
      tc::bulk_wait_read();
      tc::fence_before_sync();
      TMA_STAMP(4 + 3 * n);
      __syncthreads();
      TMA_STAMP(5 + 3 * n);
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t bn = sbase + 4u * (C::OFF_BN + n * J * R);
#pragma unroll
        for (int kk = 0; kk < R / 8; ++kk)
          tc::mma_tf32_ts(tbase + C::COL_G, tbase + C::COL_W + 8 * kk, tc::smem_desc(bn + kk * 2 * (J * 16), J * 16, 128),
                          id_g, kk > 0 ? 1u : 0u);
        // the refreshed c of the last mode is never read again: no h for it
        if (n < N - 1) {
          const uint32_t gg = sbase + 4u * (C::OFF_G + n * R * R);
#pragma unroll
          for (int kk = 0; kk < R / 8; ++kk)
            tc::mma_tf32_ts(tbase + C::COL_H, tbase + C::COL_W + 8 * kk,
                            tc::smem_desc(gg + kk * 2 * (R * 16), R * 16, 128), id_h, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(mbar);
      }
      // every thread is past its mode-(n-1) update and that mode's write-back
      // has read the slot: the next tile's rows can land there
      if (n >= 1 && n - 1 < N - 1 && (early >> (n - 1) & 1u)) gather(n - 1, n - 1, par ^ 1);
      if (n == N - 1 && spare) gather(N - 1, slot_of(N - 1, pb ^ 1), par ^ 1);
      tc::mbar_wait(mbar, mphase);
      mphase ^= 1;
      tc::fence_after_sync();
      TMA_STAMP(6 + 3 * n);
      float g[J];
      tc::tmem_ldh<J>(tlane + C::COL_G, g);
      float* slot = sm + slot_off(slot_of(n, pb));
      float a[J];
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(slot + swz<J>(tid, q));
        a[4 * q] = v.x;
        a[4 * q + 1] = v.y;
        a[4 * q + 2] = v.z;
        a[4 * q + 3] = v.w;
      }
      float inter = 0.f;
#pragma unroll
      for (int j = 0; j < J; ++j) inter = fmaf(a[j], g[j], inter);
      // a' = a - gamma (-x gs + lambda a + inter gs) = keep a + step gs
      const float gm = p.gam[n], lm = p.lam[n];
      const float keep = 1.f - gm * lm, step = gm * (x_cur - inter), shrink = -gm * lm;
      const bool red = p.atomic_mask >> n & 1u;
      if (red || !full_tile) {
        // own row in natural order (it stays inside the row's swizzle span):
        // the delta for add-reduced modes, the new row otherwise
#pragma unroll
        for (int q = 0; q < J / 4; ++q) {
          float v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 4 * q + u;
            v[u] = red ? fmaf(step, g[j], shrink * a[j]) : fmaf(step, g[j], keep * a[j]);
          }
          *reinterpret_cast<float4*>(slot + tid * J + 4 * q) = make_float4(v[0], v[1], v[2], v[3]);
        }
        if (red && !p.bulk_red) {
          // the warp's 32 deltas go out as red.add.v4 with CH = J/4 lanes per
          // row (one L2 request per row; concurrent updates all land)
          __syncwarp();
          constexpr int CH = J / 4, RPI = 32 / CH;
          const int cq = lane % CH, crow = lane / CH, wbase = tid & ~31;
          const int me = ok_cur ? ids[(par * N + n) * 128 + tid] : -1;
          int row[CH];
          float4 v[CH];
#pragma unroll
          for (int k = 0; k < CH; ++k) row[k] = __shfl_sync(0xffffffffu, me, k * RPI + crow);
#pragma unroll
          for (int k = 0; k < CH; ++k)
            v[k] = *reinterpret_cast<const float4*>(slot + (wbase + k * RPI + crow) * J + 4 * cq);
#pragma unroll
          for (int k = 0; k < CH; ++k)
            if (row[k] >= 0) tc::red_add_v4(fac + p.foff[n] + (long long)row[k] * J + 4 * cq, v[k]);
        } else {
          // one bulk add-reduction (delta) or store (new row) per sample
          tc::fence_async_smem();
          if (ok_cur) {
            float* dst = fac + p.foff[n] + (long long)ids[(par * N + n) * 128 + tid] * J;
            const uint32_t src = slot_addr(slot_of(n, pb)) + tid * C::ROWB;
            if (red)
              tc::bulk_red_add(dst, src, C::ROWB);
            else
              tc::bulk_store(dst, src, C::ROWB);
            tc::bulk_commit();
          }
        }
      } else {
        // new rows in place (swizzled), then the warp's rows go out as eight
        // scatter4 stores issued by one lane
#pragma unroll
        for (int q = 0; q < J / 4; ++q) {
          float v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = fmaf(step, g[4 * q + u], keep * a[4 * q + u]);
          *reinterpret_cast<float4*>(slot + swz<J>(tid, q)) = make_float4(v[0], v[1], v[2], v[3]);
        }
        tc::fence_async_smem();
        __syncwarp();
        if (elect_one()) {
          const int4* id4 = reinterpret_cast<const int4*>(ids + (par * N + n) * 128 + warp * 32);
          const uint32_t src = slot_addr(slot_of(n, pb)) + warp * 32 * C::ROWB;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int4 r = id4[k];
            tc::tma_scatter4(&maps.m[n], r.x, r.y, r.z, r.w, src + 4 * k * C::ROWB);
          }
          tc::bulk_commit();
        }
      }
      if (n < N - 1) {
        float h[R];
        tc::tmem_ldh<R>(tlane + C::COL_H, h);
#pragma unroll
        for (int r = 0; r < R; ++r) c[n][r] = fmaf(step, h[r], keep * c[n][r]);
      }
    }
    x_cur = x_nxt;
    ok_cur = ok_nxt;
    ok_nxt = ok_nn;
    rs ^= 1;
    tile = t1;
    t1 = t2;
    t2 = t3;
    pb ^= spare;
    par ^= 1;
    if (tid == 0) misc[1] = claim;
    if (DS) {
      ++r_tiles;
      if (!(tile * 128 < n_visit) || adv(r_cur, tile) != r_cur) {
        // this CTA's last tile of round r_cur: its row writes complete and
        // visible, then count its tiles; the round's last CTA forwards the
        // block.  Add-reduced (hot) rows need no drain here: the barrier orders
        // every thread's red.adds before thread 0's gpu-scope fence, which is
        // cumulative over them (the cooperative-groups grid barrier pattern;
        // a fence by every thread cost ~1 membar stall per issued instruction
        // at 8-way DSGD, where a CTA crosses a round every ~2.6 tiles).  A
        // pushed block written by bulk stores (a cold mode) is drained first.
        {
          const int pm = (int)dp.push[r_cur].mode;
          if (dp.push[r_cur].nrows > 0 && (!(p.atomic_mask >> pm & 1u) || p.bulk_red)) {
            tc::bulk_wait_all();
            fence_proxy_async_global();
          }
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          const int total = (int)((dp.rstart[r_cur + 1] - dp.rstart[r_cur]) / 128);
          const int c = atomicAdd(dp.done + r_cur, r_tiles) + r_tiles;
          __threadfence();
          misc[2] = (c == total && dp.push[r_cur].nrows > 0) ? 1u : 0u;
        }
        __syncthreads();
        if (misc[2]) {
          const DsgdPush ps = dp.push[r_cur];
          // the receiver must be past the previous epoch's block exchange,
          // which rewrites its replica (else this block would be overwritten)
          if (tid == 0)
            while (ld_relaxed_sys(ps.dst_gathered) < dp.epoch) __nanosleep(64);
          if (tid == 0) (void)ld_acquire_sys(ps.dst_gathered);
          __syncthreads();
          const long long nf4 = ps.nrows * J / 4;
          const float4* src = reinterpret_cast<const float4*>(fac + p.foff[ps.mode] + ps.row_lo * J);
          float4* dst = reinterpret_cast<float4*>(ps.dst);
          // eight loads in flight per thread (the receiver waits on this copy)
          long long e = tid;
          for (; e + 7 * 128 < nf4; e += 8 * 128) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + e + u * 128);
#pragma unroll
            for (int u = 0; u < 8; ++u) dst[e + u * 128] = v[u];
          }
          for (; e < nf4; e += 128) dst[e] = __ldcg(src + e);
          __threadfence_system();
          __syncthreads();
          if (tid == 0) atomicMax_system(ps.dst_ready, dp.gen0 + r_cur + 1);
        }
        r_tiles = 0;
      }
    }
    // late slots are re-gathered at the top of the next tile; the next c
    // round overwrites TMEM columns this tile's last loads read
    tc::bulk_wait_read();
    tc::fence_before_sync();
    TMA_STAMP(15);
    __syncthreads();
    t3 = 3 * G + misc[1];
    ++ntile;
  }
  tc::cp_async_wait_all();
  tc::bulk_wait_all();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, C::TCOLS);
  }
}
#undef TMA_STAMP

// ---------------------------------------------------------------------------
// v7: the v6 pipeline for J = R = 32 with two threads per sample.  256 threads
// own one 128-sample tile: warp w reads TMEM lane quadrant w % 4 (samples
// 32 (w % 4) .. +31) and owns column half h = w / 4 of every J- and R-vector,
// so a thread keeps c_n for 16 columns (48 registers, as v6 at J = 16).  Rows
// arrive by TMA gather4 into 128-byte-swizzled operand tiles; W_n goes to
// TMEM (each half its 16 columns) as the MMA's A operand; inter = a . gs is
// the current prediction sum_r W_n[r] c_n[r], whose halves are exchanged
// across the barrier that already precedes the MMA (as in v3).  The two warps
// of a lane quadrant meet at a named barrier before a cold mode's rows are
// scattered back (each wrote half of every row).  Records come through the
// shared-memory ring (warps 0-3 fetch and stage them).
// ---------------------------------------------------------------------------
template <int N, int J, int R>
struct Tma2Cfg {
  static constexpr int M = 128, H = J / 2;
  static constexpr int ROWB = J * 4;
  static constexpr int SLOT = M * J;
  static constexpr int RWC = N <= 3 ? 4 : (N <= 7 ? 8 : 16);
  static constexpr int OFF_A = 0;                               // N slots, 1024-B aligned
  static constexpr int OFF_BT = OFF_A + N * SLOT;
  static constexpr int OFF_BN = OFF_BT + N * R * J;
  static constexpr int OFF_G = OFF_BN + N * J * R;
  static constexpr int OFF_BAR = (OFF_G + N * R * R + 1) & ~1;  // N + 1 mbarriers
  static constexpr int OFF_MISC = OFF_BAR + 2 * (N + 1);
  static constexpr int OFF_IDX = (OFF_MISC + 4 + 3) & ~3;       // [2][N][128]
  static constexpr int OFF_X = OFF_IDX + 2 * N * M;             // [2][128] values
  static constexpr int OFF_PX = OFF_X + 2 * M;                  // [2 parity][2 halves][128]
  static constexpr int OFF_RING = (OFF_PX + 4 * M + 3) & ~3;    // [2][128][RWC]
  static constexpr int FLOATS = OFF_RING + 2 * M * RWC;
  static constexpr size_t SMEM = (size_t)FLOATS * 4 + 1024;
  static constexpr int COL_W = 0, COL_G = R, COL_H = R + J;
  static constexpr int NEED = (N * R > 2 * R + J) ? N * R : 2 * R + J;
  static constexpr int TCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : 256;
};

template <int N, int J, int R, bool HV>
__global__ void __launch_bounds__(256, 2)
    factor_tma2_kernel(const int* __restrict__ rec, const int* __restrict__ visit, long long n_visit, long long base,
                       float* __restrict__ fac, const float* __restrict__ cor, const __grid_constant__ TmaParams<N> p,
                       const __grid_constant__ TmaMaps<N> maps, unsigned* __restrict__ tile_ctr) {
  static_assert(J == R && J == 32, "v7 is the J = R = 32 kernel");
  constexpr int RW = N <= 3 ? 4 : (N <= 7 ? 8 : 16);
  using C = Tma2Cfg<N, J, R>;
  constexpr int H = C::H;
  extern __shared__ __align__(16) float sm_raw[];
  float* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u) / 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* mbar = full + N;
  uint32_t* misc = reinterpret_cast<uint32_t*>(sm + C::OFF_MISC);
  int* ids = reinterpret_cast<int*>(sm + C::OFF_IDX);
  float* xs = sm + C::OFF_X;
  float* px = sm + C::OFF_PX;
  int* ring = reinterpret_cast<int*>(sm + C::OFF_RING);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int qd = warp & 3, hf = warp >> 2, smp = 32 * qd + (tid & 31), c0 = hf * H;

  for (int e = tid; e < N * J * R; e += 256) {
    const int n = e / (J * R), rem = e - n * (J * R), j = rem / R, r = rem - j * R;
    const float b = __ldg(cor + e);
    sm[C::OFF_BT + n * R * J + canon<R>(r, j)] = b;
    sm[C::OFF_BN + n * J * R + canon<J>(j, r)] = b;
  }
  for (int e = tid; e < N * R * R; e += 256) {
    const int n = e / (R * R), rem = e - n * (R * R), r = rem / R, r2 = rem - r * R;
    float g = 0.f;
    for (int j = 0; j < J; ++j) g = fmaf(__ldg(cor + n * J * R + j * R + r), __ldg(cor + n * J * R + j * R + r2), g);
    sm[C::OFF_G + n * R * R + canon<R>(r, r2)] = g;
  }
  if (tid == 0) {
    for (int q = 0; q <= N; ++q) tc::mbar_init(&full[q], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&misc[0], C::TCOLS);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = misc[0];
  const uint32_t tlane = tbase + ((uint32_t)(qd * 32) << 16);
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t id_c = tc::idesc_tf32(128, R), id_g = tc::idesc_tf32(128, J), id_h = tc::idesc_tf32(128, R);
  const uint64_t pol_stream = tc::policy_evict_first();
  uint32_t mphase = 0, fphase = 0;
  const unsigned early = p.early_mask;
  auto slot_addr = [&](int q) { return sbase + 4u * (uint32_t)(C::OFF_A + q * C::SLOT); };

  // warps 0-3 gather their quadrant's 32 rows (8 gather4 by one lane)
  auto gather = [&](int n, int par) {
    if (tid == 0) tc::mbar_expect_tx(&full[n], C::SLOT * 4);
    if (hf == 0 && elect_one()) {
      const int4* id4 = reinterpret_cast<const int4*>(ids + (par * N + n) * 128 + qd * 32);
      const uint32_t dst = slot_addr(n) + qd * 32 * C::ROWB, bar = tc::smem_u32(&full[n]);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int4 r = id4[k];
        tc::tma_gather4(dst + 4 * k * C::ROWB, &maps.m[n], r.x, r.y, r.z, r.w, bar);
      }
    }
  };
  // records: warps 0-3 fetch (cp.async) and stage them (indices, value)
  auto fetch = [&](int q, int v, long long t) {
    if (hf == 0) {
      const int* src = rec + (base + (long long)v) * RW;
      const uint32_t dst = tc::smem_u32(ring + (q * 128 + smp) * RW);
      tc::cp_async16_nohint(dst, src, 16u);
      if (RW >= 8) tc::cp_async16_nohint(dst + 16, src + 4, 16u);
      tc::cp_async_commit();
    }
    (void)t;
  };
  auto stage = [&](int q, long long t, int par) {
    if (hf == 0) {
      const bool ok = tile_valid(n_visit, t) ;
      const int4* rr = reinterpret_cast<const int4*>(ring + (q * 128 + smp) * RW);
      int wv[8];
      const int4 w0 = rr[0];
      wv[0] = w0.x, wv[1] = w0.y, wv[2] = w0.z, wv[3] = w0.w;
      if (RW >= 8) {
        const int4 w1 = rr[1];
        wv[4] = w1.x, wv[5] = w1.y, wv[6] = w1.z, wv[7] = w1.w;
      }
#pragma unroll
      for (int n = 0; n < N; ++n) ids[(par * N + n) * 128 + smp] = ok ? wv[n] : 0;
      xs[par * 128 + smp] = __int_as_float(wv[N]);
    }
  };
  // valid(t) for this thread's sample (threads of both halves)
  auto valid_of = [&](long long t) { return t * 128 + smp < n_visit; };

  const long long G = gridDim.x;
  long long tile = blockIdx.x, t1 = tile + G, t2 = tile + 2 * G;
  if (tid == 0) misc[1] = atomicAdd(tile_ctr, 1u);
  int v2 = 0;
  {
    // sample smp of a tile (both halves compute the same visit entries;
    // only warps 0-3 use them)
    const long long k0 = tile * 128 + smp, k1 = t1 * 128 + smp, k2 = t2 * 128 + smp;
    auto vis = [&](long long k) -> int {
      k = k < n_visit ? k : n_visit - 1;
      return HV ? tc::ld_stream_s32(visit + k, pol_stream) : (int)k;
    };
    fetch(0, vis(k0), tile);
    fetch(1, vis(k1), t1);
    v2 = vis(k2);
  }
  if (hf == 0) asm volatile("cp.async.wait_group 1;" ::: "memory");
  stage(0, tile, 0);
  int rs = 1;
  int par = 0;
  __syncthreads();
#pragma unroll
  for (int n = 0; n < N; ++n)
    if (early >> n & 1u) gather(n, 0);
  long long t3 = 3 * G + misc[1];
  __syncthreads();
  while (tile * 128 < n_visit) {
    unsigned claim = 0;
    if (tid == 0) claim = atomicAdd(tile_ctr, 1u);
#pragma unroll
    for (int n = 0; n < N; ++n)
      if (!(early >> n & 1u)) gather(n, par);
    fetch(rs ^ 1, v2, t2);
    {
      long long k3 = t3 * 128 + smp;
      k3 = k3 < n_visit ? k3 : n_visit - 1;
      v2 = HV ? tc::ld_stream_s32(visit + k3, pol_stream) : (int)k3;
    }
    if (hf == 0) asm volatile("cp.async.wait_group 1;" ::: "memory");
    stage(rs, t1, par ^ 1);
    const bool full_tile = (tile + 1) * 128 <= n_visit;
    const bool ok = valid_of(tile);
    const float x = xs[par * 128 + smp];
#pragma unroll
    for (int n = 0; n < N; ++n) {
      tc::mbar_wait(&full[n], (fphase >> n) & 1u);
      fphase ^= 1u << n;
    }
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const uint32_t a = slot_addr(n);
        const uint32_t b = sbase + 4u * (C::OFF_BT + n * R * J);
#pragma unroll
        for (int kk = 0; kk < J / 8; ++kk)
          tc::mma_tf32(tbase + n * R, tc::smem_desc_sw<C::ROWB>(a + 32 * kk),
                       tc::smem_desc(b + kk * 2 * (R * 16), R * 16, 128), id_c, kk > 0 ? 1u : 0u);
      }
      tc::mma_commit(mbar);
    }
    tc::mbar_wait(mbar, mphase);
    mphase ^= 1;
    tc::fence_after_sync();
    float c[N][H];
#pragma unroll
    for (int n = 0; n < N; ++n) tc::tmem_ldh<H>(tlane + n * R + c0, c[n]);

#pragma unroll
    for (int n = 0; n < N; ++n) {
      float part = 0.f;
      {
        float w[H];
#pragma unroll
        for (int r = 0; r < H; ++r) {
          float v = 0.f;
          bool first = true;
#pragma unroll
          for (int n0 = 0; n0 < N; ++n0)
            if (n0 != n) {
              v = first ? c[n0][r] : v * c[n0][r];
              first = false;
            }
          w[r] = v;
          part = fmaf(v, c[n][r], part);
        }
        tc::tmem_st16(tlane + C::COL_W + c0, w);
      }
      px[((n & 1) * 2 + hf) * 128 + smp] = part;
      tc::tmem_wait_st();
      tc::bulk_wait_read();
      tc::fence_before_sync();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t bn = sbase + 4u * (C::OFF_BN + n * J * R);
#pragma unroll
        for (int kk = 0; kk < R / 8; ++kk)
          tc::mma_tf32_ts(tbase + C::COL_G, tbase + C::COL_W + 8 * kk,
                          tc::smem_desc(bn + kk * 2 * (J * 16), J * 16, 128), id_g, kk > 0 ? 1u : 0u);
        if (n < N - 1) {
          const uint32_t gg = sbase + 4u * (C::OFF_G + n * R * R);
#pragma unroll
          for (int kk = 0; kk < R / 8; ++kk)
            tc::mma_tf32_ts(tbase + C::COL_H, tbase + C::COL_W + 8 * kk,
                            tc::smem_desc(gg + kk * 2 * (R * 16), R * 16, 128), id_h, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(mbar);
      }
      if (n >= 1 && (early >> (n - 1) & 1u)) gather(n - 1, par ^ 1);
      const float inter = part + px[((n & 1) * 2 + (hf ^ 1)) * 128 + smp];
      tc::mbar_wait(mbar, mphase);
      mphase ^= 1;
      tc::fence_after_sync();
      float g[H];
      tc::tmem_ldh<H>(tlane + C::COL_G + c0, g);
      float* slot = sm + C::OFF_A + n * C::SLOT;
      float a[H];
#pragma unroll
      for (int q = 0; q < H / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(slot + swz<J>(smp, c0 / 4 + q));
        a[4 * q] = v.x;
        a[4 * q + 1] = v.y;
        a[4 * q + 2] = v.z;
        a[4 * q + 3] = v.w;
      }
      const float gm = p.gam[n], lm = p.lam[n];
      const float keep = 1.f - gm * lm, step = gm * (x - inter), shrink = -gm * lm;
      const bool red = p.atomic_mask >> n & 1u;
      if (red) {
        // hot mode: this thread's half of the delta, four add-reductions
        if (ok) {
          float* dst = fac + p.foff[n] + (long long)ids[(par * N + n) * 128 + smp] * J + c0;
#pragma unroll
          for (int q = 0; q < H / 4; ++q)
            tc::red_add_v4(dst + 4 * q, make_float4(fmaf(step, g[4 * q], shrink * a[4 * q]),
                                                     fmaf(step, g[4 * q + 1], shrink * a[4 * q + 1]),
                                                     fmaf(step, g[4 * q + 2], shrink * a[4 * q + 2]),
                                                     fmaf(step, g[4 * q + 3], shrink * a[4 * q + 3])));
        }
      } else {
        // cold mode: the new half-row in place (swizzled), the quadrant's two
        // warps meet, then one lane scatters the 32 rows (or, in a partial
        // tile, each valid sample's row goes out as one bulk store)
#pragma unroll
        for (int q = 0; q < H / 4; ++q) {
          float v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = fmaf(step, g[4 * q + u], keep * a[4 * q + u]);
          *reinterpret_cast<float4*>(slot + swz<J>(smp, c0 / 4 + q)) = make_float4(v[0], v[1], v[2], v[3]);
        }
        tc::fence_async_smem();
        asm volatile("bar.sync %0, 64;" ::"r"(1 + qd) : "memory");
        if (hf == 0) {
          if (full_tile) {
            if (elect_one()) {
              const int4* id4 = reinterpret_cast<const int4*>(ids + (par * N + n) * 128 + qd * 32);
              const uint32_t src = slot_addr(n) + qd * 32 * C::ROWB;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const int4 r = id4[k];
                tc::tma_scatter4(&maps.m[n], r.x, r.y, r.z, r.w, src + 4 * k * C::ROWB);
              }
              tc::bulk_commit();
            }
          } else if (ok) {
            // swizzled row -> natural order is a permutation of its 16-byte
            // chunks: one 16-byte bulk store per chunk
            float* dst = fac + p.foff[n] + (long long)ids[(par * N + n) * 128 + smp] * J;
#pragma unroll
            for (int q = 0; q < J / 4; ++q)
              tc::bulk_store(dst + 4 * q, slot_addr(n) + 4u * (uint32_t)swz<J>(smp, q), 16);
            tc::bulk_commit();
          }
        }
      }
      if (n < N - 1) {
        float h[H];
        tc::tmem_ldh<H>(tlane + C::COL_H + c0, h);
#pragma unroll
        for (int r = 0; r < H; ++r) c[n][r] = fmaf(step, h[r], keep * c[n][r]);
      }
    }
    tile = t1;
    t1 = t2;
    t2 = t3;
    par ^= 1;
    rs ^= 1;
    if (tid == 0) misc[1] = claim;
    tc::bulk_wait_read();
    tc::fence_before_sync();
    __syncthreads();
    t3 = 3 * G + misc[1];
  }
  tc::cp_async_wait_all();
  tc::bulk_wait_all();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, C::TCOLS);
  }
}

// ---------------------------------------------------------------- host side --
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int encode_fn() {
  if (g_encode) return 0;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    set_error("cuTensorMapEncodeTiled is not available from the driver");
    return 1;
  }
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  return 0;
}

// One tensor map per factor matrix: [rows][J] fp32, box = one row, swizzle
// span = one row (the operand-tile layout the MMA descriptors expect).
static int encode_row_map(CUtensorMap* m, float* base, long long rows, int J) {
  cuuint64_t dims[2] = {(cuuint64_t)J, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)J * 4};
  cuuint32_t box[2] = {(cuuint32_t)J, 1};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle sw = J == 8 ? CU_TENSOR_MAP_SWIZZLE_32B
                                : J == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                                          : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) for a %lld x %d factor matrix", (int)r, rows, J);
    return 1;
  }
  return 0;
}

static std::atomic<unsigned> g_tma_ctr_slot{0};
static const char* g_last_kernel = "none";
const char* last_factor_kernel() { return g_last_kernel; }
void note_factor_kernel(const char* name) { g_last_kernel = name; }

template <int N, int J, int R>
static int launch_tma(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                      const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s,
                      const DsgdParams* dsp = nullptr, int grid = 0) {
  using C = TmaCfg<N, J, R>;
  if (encode_fn()) return 1;
  (void)rw;
  TmaParams<N> p;
  for (int n = 0; n < N; ++n) {
    p.foff[n] = md.foff[n];
    p.gam[n] = gam[n];
    p.lam[n] = lam[n];
  }
  p.dbg = reinterpret_cast<long long*>(tc_debug_buffer());
  p.atomic_mask = hot_mode_mask(md);
  p.early_mask = ~p.atomic_mask & ((1u << N) - 1u);
  // Hot modes other than the last are gathered during the previous tile's
  // last mode round too (their read-to-write window grows by about one mode
  // round): NF W=24 factor pass 7.67 -> 7.34 ms, test RMSE 0.47839 ->
  // 0.47842 after 13 epochs; the last mode stays fresh at its tile's start
  // (also early: 7.28 ms, 0.47855)
  if (N == 3) p.early_mask |= ((1u << (N - 1)) - 1u);
  if (const char* e = getenv("SPTK_TMA_EARLY")) p.early_mask = (unsigned)strtoul(e, nullptr, 0) & ((1u << N) - 1u);
  // DSGD: only the stationary mode 0 may be gathered ahead of a round's wait
  if (dsp) p.early_mask &= 1u;
  {
    const char* e = getenv("SPTK_TMA_BULKRED");
    p.bulk_red = e ? atoi(e) : 0;
  }
  // tensor maps, re-encoded only when the model buffer changes
  static TmaMaps<N> maps;
  static const float* maps_fac = nullptr;
  static long long maps_foff[N];
  bool same = maps_fac == fac;
  for (int n = 0; n < N && same; ++n) same = maps_foff[n] == md.foff[n];
  if (!same) {
    for (int n = 0; n < N; ++n) {
      const long long end = n + 1 < N ? md.foff[n + 1] : md.fac_size;
      if (encode_row_map(&maps.m[n], fac + md.foff[n], (end - md.foff[n]) / J, J)) return 1;
      maps_foff[n] = md.foff[n];
    }
    maps_fac = fac;
  }
  auto kfn = dsp ? factor_tma_kernel<N, J, R, true, true>
                 : (visit ? factor_tma_kernel<N, J, R, true> : factor_tma_kernel<N, J, R, false>);
  const size_t smem = (p.early_mask >> (N - 1) & 1u) ? C::SMEM_SPARE : C::SMEM;
  static int per_sm = 0;
  static size_t per_sm_smem = 0;
  if (per_sm_smem != smem) {
    for (auto f : {factor_tma_kernel<N, J, R, true>, factor_tma_kernel<N, J, R, false>,
                   factor_tma_kernel<N, J, R, true, true>}) {
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_SPARE));
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    per_sm = resident_ctas((const void*)kfn, smem, C::TCOLS, false);
    per_sm_smem = smem;
  }
  const long long tiles = (n_visit + 127) / 128;
  // persistent grid minus the CTA slots left to the side-stream samplers
  // (order 3, J = 16: 32 slots, measured on the final code over 16 / 24 / 32 /
  // 40 / 48 / 64 / 148: NF epoch 9.30 / 9.16 / 9.06 / 9.11 / 9.13 / 9.15 /
  // 9.56 ms -- the samplers beside the pass gain more than the pass loses)
  int slots = (N == 3 && J >= 16) ? 32 : 148;
  if (const char* e = getenv("SPTK_SAMPLER_SLOTS")) slots = atoi(e);
  long long blocks = 148LL * per_sm - (per_sm >= 2 ? slots : 0);
  if (const char* e = getenv("SPTK_TC_GRID")) blocks = atoll(e);
  if (blocks > hogwild_cta_cap(n_visit, 128)) blocks = hogwild_cta_cap(n_visit, 128);
  // DSGD: a persistent grid (every CTA resident: a CTA may wait on a round
  // flag while earlier tiles are still running elsewhere); grid > 0 caps it
  // (two ranks sharing one GPU in the tests)
  if (dsp && grid > 0 && blocks > grid) blocks = grid;
  // grid < 0: the default grid divided by -grid (a rank of M-way DSGD keeps
  // the per-row concurrency of one GPU running the whole tensor)
  if (dsp && grid < 0) blocks = (blocks + (-grid) - 1) / (-grid);
  if (blocks < 1) blocks = 1;
  if (blocks > tiles) blocks = tiles;
  unsigned* ctr = nullptr;
  SPTK_CUDA_TRY(cudaGetSymbolAddress((void**)&ctr, g_tma_tile_ctr));
  ctr += g_tma_ctr_slot.fetch_add(1u) & 63u;
  SPTK_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
  DsgdParams dp{};
  if (dsp) {
    dp = *dsp;
    SPTK_CUDA_TRY(cudaMemsetAsync(dp.done, 0, sizeof(int) * dp.n_rounds, s));
  }
  kfn<<<(unsigned)blocks, 128, smem, s>>>(rec, visit, n_visit, base, fac, cor, p, maps, ctr, dp);
  SPTK_CHECK_LAUNCH();
  note_factor_kernel(dsp ? "factor_tma_kernel<dsgd>" : "factor_tma_kernel");
  return 0;
}

template <int N, int J, int R>
static int launch_tma2(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                       const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s) {
  using C = Tma2Cfg<N, J, R>;
  if (encode_fn()) return 1;
  (void)rw;
  TmaParams<N> p;
  for (int n = 0; n < N; ++n) {
    p.foff[n] = md.foff[n];
    p.gam[n] = gam[n];
    p.lam[n] = lam[n];
  }
  p.dbg = nullptr;
  p.atomic_mask = hot_mode_mask(md);
  p.early_mask = ~p.atomic_mask & ((1u << N) - 1u) & ~(1u << (N - 1));  // no spare slot: the last mode is late
  p.bulk_red = 0;
  static TmaMaps<N> maps;
  static const float* maps_fac = nullptr;
  static long long maps_foff[N];
  bool same = maps_fac == fac;
  for (int n = 0; n < N && same; ++n) same = maps_foff[n] == md.foff[n];
  if (!same) {
    for (int n = 0; n < N; ++n) {
      const long long end = n + 1 < N ? md.foff[n + 1] : md.fac_size;
      if (encode_row_map(&maps.m[n], fac + md.foff[n], (end - md.foff[n]) / J, J)) return 1;
      maps_foff[n] = md.foff[n];
    }
    maps_fac = fac;
  }
  auto kfn = visit ? factor_tma2_kernel<N, J, R, true> : factor_tma2_kernel<N, J, R, false>;
  static int per_sm = 0;
  if (!per_sm) {
    for (auto f : {factor_tma2_kernel<N, J, R, true>, factor_tma2_kernel<N, J, R, false>}) {
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    SPTK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 256, C::SMEM));
    if (per_sm < 1) per_sm = 1;
    if (getenv("SPTK_DEBUG")) fprintf(stderr, "[sptk] tma2 kernel smem=%zu -> %d CTAs/SM\n", C::SMEM, per_sm);
  }
  const long long tiles = (n_visit + 127) / 128;
  long long blocks = 148LL * per_sm;
  if (const char* e = getenv("SPTK_TC_GRID")) blocks = atoll(e);
  if (blocks > hogwild_cta_cap(n_visit, 128)) blocks = hogwild_cta_cap(n_visit, 128);
  if (blocks < 1) blocks = 1;
  if (blocks > tiles) blocks = tiles;
  unsigned* ctr = nullptr;
  SPTK_CUDA_TRY(cudaGetSymbolAddress((void**)&ctr, g_tma_tile_ctr));
  ctr += g_tma_ctr_slot.fetch_add(1u) & 63u;
  SPTK_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
  kfn<<<(unsigned)blocks, 256, C::SMEM, s>>>(rec, visit, n_visit, base, fac, cor, p, maps, ctr);
  SPTK_CHECK_LAUNCH();
  note_factor_kernel("factor_tma2_kernel");
  return 0;
}

// returns 1 if handled (uniform J = R in {8, 16}; N = 3, 4 at J = 16; N = 3, 6 at J = 8)
int try_factor_tma(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                   const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s, int* rc) {
  const int N = md.n_modes, R = md.rcore, J = md.jr[0];
  for (int n = 0; n < N; ++n)
    if (md.jr[n] != J) return 0;
  if (J != R || rw != rec_words(N)) return 0;
  static int tma2 = -1;
  if (tma2 < 0) {
    const char* e = getenv("SPTK_TMA2");
    tma2 = e ? atoi(e) : 0;
  }
  if (tma2 && N == 3 && J == 32) {
    *rc = launch_tma2<3, 32, 32>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s);
    return 1;
  }
#define SPTK_TMA_CASE(NN, JJ)                                                                    \
  if (N == NN && J == JJ) {                                                                      \
    *rc = launch_tma<NN, JJ, JJ>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s);      \
    return 1;                                                                                    \
  }
  SPTK_TMA_CASE(3, 16)
  SPTK_TMA_CASE(4, 16)
  SPTK_TMA_CASE(3, 8)
  SPTK_TMA_CASE(6, 8)
#undef SPTK_TMA_CASE
  return 0;
}

// One rank's whole epoch of DSGD rounds in one launch (see DsgdParams).
int factor_pass_dsgd(const int* rec, int rw, const int* visit, long long n_visit, float* fac, const float* cor,
                     const ModelDesc& md, const float* gam, const float* lam, const long long* rstart,
                     const long long* rend, const void* push, int* done, int* ready, int n_rounds, int gen0, int epoch,
                     int grid, cudaStream_t s) {
  const int N = md.n_modes, R = md.rcore, J = md.jr[0];
  for (int n = 0; n < N; ++n)
    SPTK_REQUIRE(md.jr[n] == J, "factor_pass_dsgd: needs uniform J (got J_%d = %d)", n, md.jr[n]);
  SPTK_REQUIRE(J == R && rw == rec_words(N), "factor_pass_dsgd: needs J == R and fp32 records");
  SPTK_REQUIRE(n_visit % 128 == 0, "factor_pass_dsgd: the visit list must be padded to whole tiles");
  SPTK_REQUIRE(n_rounds >= 1, "factor_pass_dsgd: no rounds");
  DsgdParams dp;
  dp.rstart = rstart;
  dp.rend = rend;
  dp.push = (const DsgdPush*)push;
  dp.done = done;
  dp.ready = ready;
  dp.n_rounds = n_rounds;
  dp.gen0 = gen0;
  dp.epoch = epoch;
#define SPTK_DSGD_CASE(NN, JJ)                                                                               \
  if (N == NN && J == JJ)                                                                                    \
    return launch_tma<NN, JJ, JJ>(rec, rw, visit, n_visit, 0, fac, cor, md, gam, lam, s, &dp, grid);
  SPTK_DSGD_CASE(3, 16)
  SPTK_DSGD_CASE(4, 16)
  SPTK_DSGD_CASE(3, 8)
  SPTK_DSGD_CASE(6, 8)
#undef SPTK_DSGD_CASE
  SPTK_REQUIRE(false, "factor_pass_dsgd: no fused DSGD kernel for order %d, J = R = %d", N, J);
}
size_t dsgd_push_bytes() { return sizeof(DsgdPush); }

__global__ void flag_store_kernel(int* flag, int value) { atomicMax_system(flag, value); }

int flag_store(int* flag, int value, cudaStream_t s) {
  flag_store_kernel<<<1, 1, 0, s>>>(flag, value);
  SPTK_CHECK_LAUNCH();
  return 0;
}

}  // namespace sptk
