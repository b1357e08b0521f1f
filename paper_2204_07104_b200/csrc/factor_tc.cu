// factor_tc.cu -- K3 on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Same update as factor_tps_kernel (_loops.py:17-63, Hogwild over the visit
// order), with the contractions moved to tcgen05.mma:
//
//   c_n  = A_n[tile] (128 x J) . B_n        (128 x R)   K = J
//   gs_n = W_n       (128 x R) . B_n^T      (128 x J)   K = R,  W_n = prod_{n0!=n} c_n0
//   c_n' = A_n'      (128 x J) . B_n        refresh after the row update
//
// One CTA owns a tile of 128 consecutive visit positions; thread t <-> sample
// t <-> TMEM lane t, so every elementwise step (products, residual, row update)
// is register-local and the accumulators come back with one tcgen05.ld per 16
// columns.  Operands are staged in shared memory in the K-major no-swizzle
// canonical layout; B(n) (and its transpose) stay resident for the whole
// launch.  TF32 inputs with fp32 accumulation; SPLIT = 3xTF32 (hi*hi + hi*lo +
// lo*hi), which restores ~fp32 accuracy of the products at 3x the (cheap)
// tensor work.  One elected thread issues the MMAs and commits to an mbarrier.
#include "common.cuh"
#include "kernels.cuh"
#include "tc.cuh"
#include "factor_tc_util.cuh"

#include <stdio.h>
#include <stdlib.h>

#include <atomic>

namespace sptk {

template <int N>
struct TcParams {
  long long foff[N];
  float gam[N];
  float lam[N];
  float* dbg;  // optional per-sample dump of the first tile (debug hook)
  unsigned atomic_mask;  // bit n: mode-n rows are written as red.add deltas (hot, small modes)
  int prefetch;          // v2: gather the next tile's rows during this tile (1) or at its start (0)
  int defer_wb;          // v2: write mode n's rows back while mode n+1's MMA runs
};

static float* g_tc_debug = nullptr;
__device__ unsigned g_tile_ctr[64];
// rotating pool index, shared by every host thread that launches
static std::atomic<unsigned> g_tc_ctr_slot{0};

template <int N, int J, int R, bool SPLIT>
struct TcCfg {
  static constexpr int M = 128;
  static constexpr int NB = SPLIT ? 2 : 1;
  static constexpr int BT = R * J;  // B_n^T: R rows x J (K)
  static constexpr int BN = J * R;  // B_n  : J rows x R (K)
  static constexpr int AT = M * J;
  static constexpr int WT = M * R;
  static constexpr int OFF_BT = 0;
  static constexpr int OFF_BN = OFF_BT + N * NB * BT;
  static constexpr int OFF_AT = OFF_BN + N * NB * BN;
  static constexpr int OFF_WT = OFF_AT + N * NB * AT;
  static constexpr int FLOATS = OFF_WT + NB * WT;
  static constexpr int NEED = N * R + J;
  static constexpr int TCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  // + 16 bytes for the mbarrier and the TMEM address slot
  static constexpr size_t SMEM = (size_t)FLOATS * 4 + 16;
};


__device__ __forceinline__ float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

// write one 4-float K chunk of row `row` (hi and, if SPLIT, lo copies)
template <int ROWS, bool SPLIT>
__device__ __forceinline__ void put4(float* base_hi, int lo_off, int row, int k0, float4 v) {
  float* p = base_hi + canon<ROWS>(row, k0);
  if (SPLIT) {
    float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
    float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
    *reinterpret_cast<float4*>(p) = h;
    *reinterpret_cast<float4*>(p + lo_off) = l;
  } else {
    *reinterpret_cast<float4*>(p) = v;
  }
}

template <int ROWS, bool SPLIT>
__device__ __forceinline__ float4 get4(const float* base_hi, int lo_off, int row, int k0) {
  const float* p = base_hi + canon<ROWS>(row, k0);
  float4 h = *reinterpret_cast<const float4*>(p);
  if (SPLIT) {
    float4 l = *reinterpret_cast<const float4*>(p + lo_off);
    h.x += l.x;
    h.y += l.y;
    h.z += l.z;
    h.w += l.w;
  }
  return h;
}

// D[dcol..] (+)= A(128 x K) . B(NR x K)^T over K in steps of 8 (tf32), with the
// 3xTF32 split when SPLIT.
template <int NR, int K, bool SPLIT>
__device__ __forceinline__ void issue_gemm(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi, uint32_t b_lo,
                                           uint32_t idesc) {
#pragma unroll
  for (int kk = 0; kk < K / 8; ++kk) {
    const uint32_t ao = kk * 2 * (128 * 16), bo = kk * 2 * (NR * 16);
    const uint64_t ah = tc::smem_desc(a_hi + ao, 128 * 16, 128);
    const uint64_t bh = tc::smem_desc(b_hi + bo, NR * 16, 128);
    tc::mma_tf32(d_tmem, ah, bh, idesc, kk > 0 ? 1u : 0u);
    if (SPLIT) {
      const uint64_t al = tc::smem_desc(a_lo + ao, 128 * 16, 128);
      const uint64_t bl = tc::smem_desc(b_lo + bo, NR * 16, 128);
      tc::mma_tf32(d_tmem, ah, bl, idesc, 1u);
      tc::mma_tf32(d_tmem, al, bh, idesc, 1u);
    }
  }
}

template <int N, int J, int R, bool SPLIT, int RW>
__global__ void __launch_bounds__(128, 1)
    factor_tc_kernel(const int* __restrict__ rec, const int* __restrict__ visit, long long n_visit, long long base,
                     float* __restrict__ fac, const float* __restrict__ cor, TcParams<N> p) {
  using C = TcCfg<N, J, R, SPLIT>;
  // Everything lives in the dynamic segment.  Only 16-byte alignment is assumed
  // (the no-swizzle canonical layout needs no more); assuming more lets the
  // compiler fold away low address bits that are not zero at run time.
  extern __shared__ __align__(16) float sm[];
  uint64_t& mbar = *reinterpret_cast<uint64_t*>(sm + C::FLOATS);
  uint32_t& tslot = *reinterpret_cast<uint32_t*>(sm + C::FLOATS + 2);
  const int tid = threadIdx.x, warp = tid >> 5;

  // resident operands: B_n^T (rows r, K j) and B_n (rows j, K r), hi/lo
  for (int e = tid; e < N * J * R; e += 128) {
    const int n = e / (J * R), rem = e - n * (J * R), j = rem / R, r = rem - j * R;
    const float b = __ldg(cor + e);
    const float h = SPLIT ? tf32_hi(b) : b;
    float* bt = sm + C::OFF_BT + n * C::NB * C::BT;
    float* bn = sm + C::OFF_BN + n * C::NB * C::BN;
    bt[canon<R>(r, j)] = h;
    bn[canon<J>(j, r)] = h;
    if (SPLIT) {
      bt[C::BT + canon<R>(r, j)] = b - h;
      bn[C::BN + canon<J>(j, r)] = b - h;
    }
  }
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tslot, C::TCOLS);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tslot;
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t id_c = tc::idesc_tf32(128, R), id_g = tc::idesc_tf32(128, J);
  uint32_t phase = 0;

  for (long long tile = blockIdx.x; tile * 128 < n_visit; tile += gridDim.x) {
    const long long k = tile * 128 + tid;
    const bool valid = k < n_visit;
    int idx[N];
    float x = 0.f;
    if (valid) {
      const int* rp = rec + (base + (visit ? (long long)__ldg(visit + k) : k)) * RW;
      int wv[8];
      int4 w0 = __ldg(reinterpret_cast<const int4*>(rp));
      wv[0] = w0.x;
      wv[1] = w0.y;
      wv[2] = w0.z;
      wv[3] = w0.w;
      if (RW >= 8) {
        int4 w1 = __ldg(reinterpret_cast<const int4*>(rp) + 1);
        wv[4] = w1.x;
        wv[5] = w1.y;
        wv[6] = w1.z;
        wv[7] = w1.w;
      }
#pragma unroll
      for (int n = 0; n < N; ++n) idx[n] = wv[n];
      x = __int_as_float(wv[N]);
    } else {
#pragma unroll
      for (int n = 0; n < N; ++n) idx[n] = 0;
    }
    // gather rows into the A tiles
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const float4* src = reinterpret_cast<const float4*>(fac + p.foff[n] + (long long)idx[n] * J);
      float* at = sm + C::OFF_AT + n * C::NB * C::AT;
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
        float4 v = valid ? __ldcg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        put4<128, SPLIT>(at, C::AT, tid, 4 * q, v);
      }
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const uint32_t a = sbase + 4 * (C::OFF_AT + n * C::NB * C::AT);
        const uint32_t b = sbase + 4 * (C::OFF_BT + n * C::NB * C::BT);
        issue_gemm<R, J, SPLIT>(tbase + n * R, a, a + 4 * C::AT, b, b + 4 * C::BT, id_c);
      }
      tc::mma_commit(&mbar);
    }
    tc::mbar_wait(&mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    float c[N][R];
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int q = 0; q < R / 16; ++q) tc::tmem_ld16(tlane + n * R + 16 * q, &c[n][16 * q]);
    const bool dump = p.dbg != nullptr && tile == blockIdx.x && blockIdx.x == 0;
    if (dump)
      for (int n = 0; n < N; ++n)
        for (int r = 0; r < R; ++r) p.dbg[tid * (2 * N * R + N * J) + n * R + r] = c[n][r];

#pragma unroll
    for (int n = 0; n < N; ++n) {
      // W_n = prod_{n0 != n} c_n0 (reference order), into the W tile
      float* wt = sm + C::OFF_WT;
#pragma unroll
      for (int q = 0; q < R / 4; ++q) {
        float w4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float w = 1.f;
#pragma unroll
          for (int n0 = 0; n0 < N; ++n0)
            if (n0 != n) w *= c[n0][4 * q + u];
          w4[u] = w;
        }
        put4<128, SPLIT>(wt, C::WT, tid, 4 * q, make_float4(w4[0], w4[1], w4[2], w4[3]));
      }
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t a = sbase + 4 * C::OFF_WT;
        const uint32_t b = sbase + 4 * (C::OFF_BN + n * C::NB * C::BN);
        issue_gemm<J, R, SPLIT>(tbase + N * R, a, a + 4 * C::WT, b, b + 4 * C::BN, id_g);
        tc::mma_commit(&mbar);
      }
      tc::mbar_wait(&mbar, phase);
      phase ^= 1;
      tc::fence_after_sync();
      float g[J];
#pragma unroll
      for (int q = 0; q < J / 16; ++q) tc::tmem_ld16(tlane + N * R + 16 * q, &g[16 * q]);
      if (dump)
        for (int j = 0; j < J; ++j) p.dbg[tid * (2 * N * R + N * J) + N * R + n * J + j] = g[j];
      // row update (register-local)
      float* at = sm + C::OFF_AT + n * C::NB * C::AT;
      float a[J];
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
        float4 v = get4<128, SPLIT>(at, C::AT, tid, 4 * q);
        a[4 * q] = v.x;
        a[4 * q + 1] = v.y;
        a[4 * q + 2] = v.z;
        a[4 * q + 3] = v.w;
      }
      float inter = 0.f;
#pragma unroll
      for (int j = 0; j < J; ++j) inter = fmaf(a[j], g[j], inter);
      const float gm = p.gam[n], lm = p.lam[n];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        float gr = -x * g[j] + lm * a[j] + inter * g[j];
        a[j] -= gm * gr;
      }
      if (valid) {
        float4* dst = reinterpret_cast<float4*>(fac + p.foff[n] + (long long)idx[n] * J);
        if (p.atomic_mask >> n & 1u) {
#pragma unroll
          for (int q = 0; q < J / 4; ++q) {
            float4 o = get4<128, SPLIT>(at, C::AT, tid, 4 * q);
            tc::red_add_v4(reinterpret_cast<float*>(dst + q), make_float4(a[4 * q] - o.x, a[4 * q + 1] - o.y,
                                                                          a[4 * q + 2] - o.z, a[4 * q + 3] - o.w));
          }
        } else {
#pragma unroll
          for (int q = 0; q < J / 4; ++q)
            __stcg(dst + q, make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]));
        }
      }
      if (n < N - 1) {
#pragma unroll
        for (int q = 0; q < J / 4; ++q)
          put4<128, SPLIT>(at, C::AT, tid, 4 * q, make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]));
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        if (tid == 0) {
          tc::fence_after_sync();
          const uint32_t aa = sbase + 4 * (C::OFF_AT + n * C::NB * C::AT);
          const uint32_t b = sbase + 4 * (C::OFF_BT + n * C::NB * C::BT);
          issue_gemm<R, J, SPLIT>(tbase + n * R, aa, aa + 4 * C::AT, b, b + 4 * C::BT, id_c);
          tc::mma_commit(&mbar);
        }
        tc::mbar_wait(&mbar, phase);
        phase ^= 1;
        tc::fence_after_sync();
#pragma unroll
        for (int q = 0; q < R / 16; ++q) tc::tmem_ld16(tlane + n * R + 16 * q, &c[n][16 * q]);
        if (dump)
          for (int r = 0; r < R; ++r) p.dbg[tid * (2 * N * R + N * J) + N * R + N * J + n * R + r] = c[n][r];
      }
    }
    // all TMEM reads and smem reads of this tile done before the next tile
    tc::fence_before_sync();
    __syncthreads();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, C::TCOLS);
  }
}



// ----------------------------------------------------------------------------
// v2 (TF32, the default throughput kernel): 1 + N tensor rounds per tile.
// The c_n refresh after the row update is folded into the same round as gs:
//   a' = (1 - g*l) a + g (x - inter) gs   =>   c_n' = (1 - g*l) c_n + g (x - inter) (W_n . G_n)
// with G_n = B_n^T B_n (R x R, resident), so one MMA round per mode yields
// both gs = W_n . B_n^T and h = W_n . G_n.  Rows of the next tile are gathered
// with cp.async straight into the canonical A layout of the idle buffer while
// the current tile computes; the record/visit streams use L2 evict_first and
// the factor rows L2 evict_last so the 32 MB model stays L2-resident.
// ----------------------------------------------------------------------------
template <int N, int J, int R>
struct Tc2Cfg {
  static constexpr int M = 128;
  static constexpr int OFF_BT = 0;                       // N x (R rows x J)
  static constexpr int OFF_BN = OFF_BT + N * R * J;      // N x (J rows x R)
  static constexpr int OFF_G = OFF_BN + N * J * R;       // N x (R rows x R)
  static constexpr int OFF_A = OFF_G + N * R * R;        // N x (128 x J)
  static constexpr int OFF_W = OFF_A + N * M * J;        // 128 x R
  static constexpr int OFF_BAR = OFF_W + M * R;          // mbarrier (2 words), TMEM slot, claim slot
  // the last mode's second slot, allocated only when that mode is gathered
  // ahead of its tile (a cold last mode); NF's and Y4's last modes are hot
  static constexpr int OFF_SPARE = OFF_BAR + 4;
  static constexpr int FLOATS = OFF_SPARE;
  static constexpr int NEED = (N * R > J + R) ? N * R : J + R;
  static constexpr int TCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr size_t SMEM = (size_t)FLOATS * 4;
  static constexpr size_t SMEM_SPARE = SMEM + (size_t)M * J * 4;
};


template <int N, int J, int R, bool HV>
__global__ void __launch_bounds__(128, (N * (J + R) <= 128 ? 4 : 2))
    factor_tc2_kernel(const int* __restrict__ rec, const int* __restrict__ visit, long long n_visit, long long base,
                      float* __restrict__ fac, const float* __restrict__ cor, TcParams<N> p,
                      unsigned* __restrict__ tile_ctr) {
  // debug hook: per-phase clock64 stamps of block 0 / thread 0 for 16 tiles
  long long* stamps = reinterpret_cast<long long*>(p.dbg);
  int ntile = 0;
#define TC2_STAMP(k)                                                              \
  do {                                                                            \
    if (stamps && blockIdx.x == 0 && threadIdx.x == 0 && ntile < 16) stamps[ntile * 16 + (k)] = clock64(); \
  } while (0)

  constexpr int RW = N <= 3 ? 4 : (N <= 7 ? 8 : 16);
  using C = Tc2Cfg<N, J, R>;
  extern __shared__ __align__(16) float sm[];
  uint64_t& mbar = *reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint32_t& tslot = *reinterpret_cast<uint32_t*>(sm + C::OFF_BAR + 2);
  const int tid = threadIdx.x, warp = tid >> 5;

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
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tslot, C::TCOLS);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tslot;
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t id_c = tc::idesc_tf32(128, R), id_g = tc::idesc_tf32(128, J), id_h = tc::idesc_tf32(128, R);
  const uint64_t pol_keep = tc::policy_evict_last(), pol_stream = tc::policy_evict_first();
  uint32_t phase = 0;

  // A-tile slot of mode n: modes 0..N-2 have one slot each, the last mode
  // alternates between two (pb).
  auto a_off = [&](int n, int pb) { return n == N - 1 && pb ? C::OFF_SPARE : C::OFF_A + n * 128 * J; };
  // Row gather of one mode for this warp's 32 samples: CH = J/4 lanes share a
  // row (one 16-byte chunk each), so one cp.async instruction covers 32/CH
  // whole rows and L1 merges each row into a single L2 request.
  constexpr int CH = J / 4, RPI = 32 / CH;
  // (lane -> (row, chunk) with the chunk fastest.  The row-fastest mapping has
  // 4x fewer shared wavefronts per access but measured 4% slower: ncu 11.95 ->
  // 12.43 ms, more short-scoreboard stalls)
  const int lane = tid & 31, wbase = tid & ~31, cq = lane % CH, crow = lane / CH;
  auto issue_mode = [&](const RecReg<N, RW>& rr, int n, int pb) {
    const uint32_t dst = sbase + 4 * a_off(n, pb);
    // no L2::cache_hint operand here: with it ptxas 12.9 pairs the global
    // descriptor with an odd uniform register (desc[UR1]) in this loop, which
    // traps as an illegal instruction (the rows are L2-resident anyway)
    // all row indices first (one shuffle per chunk: invalid samples carry
    // -1), then the copies, so no copy waits on a shuffle issued after it
    const int me = rr.valid ? rr.idx[n] : -1;
    int row[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) row[k] = __shfl_sync(0xffffffffu, me, k * RPI + crow);
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int sl = k * RPI + crow;
      const float* src = fac + p.foff[n] + (long long)(row[k] < 0 ? 0 : row[k]) * J + 4 * cq;
      tc::cp_async16_nohint(dst + 4 * canon<128>(wbase + sl, 4 * cq), src, row[k] >= 0 ? 16u : 0u);
    }
  };

  // Cooperative write-back of mode n's parked rows (new values, or deltas for
  // red.add modes) from slot (n, pb): CH lanes per row, 16 bytes each.
  auto flush_mode = [&](const RecReg<N, RW>& rr, int n, int pbs) {
    const float* at = sm + a_off(n, pbs);
    const bool red = p.atomic_mask >> n & 1u;
    if (red && (p.atomic_mask >> 31)) return;  // SPTK_DEBUG_DROP_HOT
    // shuffles and shared loads of every chunk first, then the stores
    const int me = rr.valid ? rr.idx[n] : -1;
    int row[CH];
    float4 v[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) row[k] = __shfl_sync(0xffffffffu, me, k * RPI + crow);
#pragma unroll
    for (int k = 0; k < CH; ++k) v[k] = *reinterpret_cast<const float4*>(at + canon<128>(wbase + k * RPI + crow, 4 * cq));
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      float* dst = fac + p.foff[n] + (long long)row[k] * J + 4 * cq;
      if (row[k] >= 0) {
        if (red)
          tc::red_add_v4(dst, v[k]);
        else
          tc::st_v4_hint(dst, v[k], pol_keep);
      }
    }
  };

  // Software pipeline over this CTA's tiles: visit entries three tiles ahead,
  // records two ahead (registers), factor rows one ahead: the next tile's
  // mode-n rows are gathered (cp.async into the canonical A layout) as soon as
  // this tile's last read of its mode-n slot is behind a barrier, and the
  // last mode has two slots so its gather is issued at the start of the
  // tile.  The Hogwild read-to-write window is therefore about one tile.
  // The first three tiles of a CTA are blockIdx + {0,1,2}*G; later ones are
  // claimed from a per-launch counter (claim issued at the start of a tile,
  // consumed at its end), so CTAs that start late (another stream's kernel
  // holding the SM) or run slow simply take fewer tiles.
  const long long G = gridDim.x;
  uint32_t& s_claim = *reinterpret_cast<uint32_t*>(sm + C::OFF_BAR + 3);
  long long tile = blockIdx.x, t1 = tile + G, t2 = tile + 2 * G;
  if (tid == 0) s_claim = atomicAdd(tile_ctr, 1u);
  RecReg<N, RW> cur, nxt;
  int v2 = load_vis<HV>(visit, n_visit, t2, pol_stream);
  load_rec<N, RW>(cur, rec, load_vis<HV>(visit, n_visit, tile, pol_stream), tile_valid(n_visit, tile), base,
                  pol_stream);
  load_rec<N, RW>(nxt, rec, load_vis<HV>(visit, n_visit, t1, pol_stream), tile_valid(n_visit, t1), base, pol_stream);
  int pb = 0;
  // Prefetched modes (bit n of pfm) are gathered one tile ahead; the others
  // at the start of their own tile.  Default: prefetch only the modes written
  // with plain stores (large, rarely shared rows); the hot red.add modes are
  // read fresh, which keeps their Hogwild staleness to one tile (measured on
  // the NF bench tensor: prefetching the hot modes costs ~1.5% test RMSE).
  const unsigned pfm = p.prefetch == 0 ? 0u : p.prefetch == 2 ? ~0u : ~p.atomic_mask;
  // late-prefetched modes (prefetch == 3: the hot modes): gathered for the
  // next tile once this tile reaches its last mode, i.e. a fraction of a
  // tile early instead of a whole tile
  const unsigned lpm = p.prefetch == 3 ? p.atomic_mask : 0u;
  const unsigned fresh = ~(pfm | lpm);
  // the last mode alternates between two slots only when gathered ahead
  const int pbm = ((pfm | lpm) >> (N - 1) & 1u) ? 1 : 0;
#pragma unroll
  for (int n = 0; n < N; ++n)
    if ((pfm | lpm) >> n & 1u) issue_mode(cur, n, pb);
  tc::cp_async_commit();
  __syncthreads();
  long long t3 = 3 * G + s_claim;
  while (tile * 128 < n_visit) {
    TC2_STAMP(0);
    unsigned claim = 0;
    if (tid == 0) claim = atomicAdd(tile_ctr, 1u);
#pragma unroll
    for (int n = 0; n < N; ++n)
      if (fresh >> n & 1u) issue_mode(cur, n, pb);
    tc::cp_async_commit();
    RecReg<N, RW> nnxt;
    load_rec<N, RW>(nnxt, rec, v2, tile_valid(n_visit, t2), base, pol_stream);
    v2 = load_vis<HV>(visit, n_visit, t3, pol_stream);
    TC2_STAMP(1);
    tc::cp_async_wait_all();
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    TC2_STAMP(2);
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const uint32_t a = sbase + 4 * a_off(n, pb);
        const uint32_t b = sbase + 4 * (C::OFF_BT + n * R * J);
        issue_gemm<R, J, false>(tbase + n * R, a, 0, b, 0, id_c);
      }
      tc::mma_commit(&mbar);
    }
    // the next tile's last-mode rows go to the other slot right away
    if (pfm >> (N - 1) & 1u) issue_mode(nxt, N - 1, pb ^ 1);
    TC2_STAMP(3);
    tc::mbar_wait(&mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    TC2_STAMP(4);
    float c[N][R];
#pragma unroll
    for (int n = 0; n < N; ++n) tc::tmem_ldh<R>(tlane + n * R, c[n]);

#pragma unroll
    for (int n = 0; n < N; ++n) {
      float* wt = sm + C::OFF_W;
#pragma unroll
      for (int q = 0; q < R / 4; ++q) {
        float w4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float w = 1.f;
#pragma unroll
          for (int n0 = 0; n0 < N; ++n0)
            if (n0 != n) w *= c[n0][4 * q + u];
          w4[u] = w;
        }
        *reinterpret_cast<float4*>(wt + canon<128>(tid, 4 * q)) = make_float4(w4[0], w4[1], w4[2], w4[3]);
      }
      tc::fence_async_smem();
      tc::fence_before_sync();
      TC2_STAMP(5 + 3 * n);
      __syncthreads();
      TC2_STAMP(6 + 3 * n);
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t a = sbase + 4 * C::OFF_W;
        issue_gemm<J, R, false>(tbase, a, 0, sbase + 4 * (C::OFF_BN + n * J * R), 0, id_g);
        // the refreshed c of the last mode is never read again: no h for it
        if (n < N - 1) issue_gemm<R, R, false>(tbase + J, a, 0, sbase + 4 * (C::OFF_G + n * R * R), 0, id_h);
        tc::mma_commit(&mbar);
      }
      // Deferred write-back of mode n-1 (parked before the barrier above): it
      // runs while this mode's MMA executes.  Then that slot is free for the
      // next tile's rows.
      if (p.defer_wb && n >= 1) flush_mode(cur, n - 1, pb);
      if (n >= 1 && n - 1 < N - 1 && (pfm >> (n - 1) & 1u)) issue_mode(nxt, n - 1, 0);
      if (n == N - 1 && lpm) {
        // every thread is past modes 0..N-2 of this tile: their slots and the
        // spare last-mode slot are free
#pragma unroll
        for (int m = 0; m < N; ++m)
          if (lpm >> m & 1u) issue_mode(nxt, m, m == N - 1 ? (pb ^ 1) : 0);
      }
      tc::mbar_wait(&mbar, phase);
      phase ^= 1;
      tc::fence_after_sync();
      TC2_STAMP(7 + 3 * n);
      float g[J];
      tc::tmem_ldh<J>(tlane, g);
      float* at = sm + a_off(n, pb);
      float a[J];
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
        float4 v = *reinterpret_cast<const float4*>(at + canon<128>(tid, 4 * q));
        a[4 * q] = v.x;
        a[4 * q + 1] = v.y;
        a[4 * q + 2] = v.z;
        a[4 * q + 3] = v.w;
      }
      float inter = 0.f;
#pragma unroll
      for (int j = 0; j < J; ++j) inter = fmaf(a[j], g[j], inter);
      const float gm = p.gam[n], lm = p.lam[n];
      // Row write-back through the (now dead) A slot: each thread parks its
      // new row (or, for red.add modes, its delta) in its own slot row, then
      // CH lanes per row write 16-byte chunks so each row is one request.
      const bool red = p.atomic_mask >> n & 1u;
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
        float d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * q + u;
          const float gr = -cur.x * g[j] + lm * a[j] + inter * g[j];
          d[u] = -gm * gr;
          a[j] += d[u];
        }
        const float4 v = red ? make_float4(d[0], d[1], d[2], d[3])
                             : make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
        *reinterpret_cast<float4*>(at + canon<128>(tid, 4 * q)) = v;
      }
      if (!p.defer_wb || n == N - 1) {
        __syncwarp();
        flush_mode(cur, n, pb);
      }
      if (n < N - 1) {
        float h[R];
        tc::tmem_ldh<R>(tlane + J, h);
        const float keep = 1.f - gm * lm, step = gm * (cur.x - inter);
#pragma unroll
        for (int r = 0; r < R; ++r) c[n][r] = fmaf(step, h[r], keep * c[n][r]);
      }
    }
    tc::cp_async_commit();
    cur = nxt;
    nxt = nnxt;
    tile = t1;
    t1 = t2;
    t2 = t3;
    pb ^= pbm;
    if (tid == 0) s_claim = claim;
    TC2_STAMP(15);
    __syncthreads();
    t3 = 3 * G + s_claim;
    ++ntile;
  }
#undef TC2_STAMP
  tc::cp_async_wait_all();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, C::TCOLS);
  }
}

// ----------------------------------------------------------------------------
// v3: the v2 update with two threads per sample.  256 threads own one
// 128-sample tile: warp w reads TMEM lane quadrant w % 4 (samples
// 32(w%4)..+31) and owns column half h = w / 4 of every J- or R-vector, so
// each thread's elementwise chain (products, update, refresh, write-back) is
// half as long and twice as many warps cover a tile.  The only cross-thread
// quantity, inter = a . gs, equals sum_r W_n[r] c_n[r] (the current
// prediction), so each thread adds its half of that sum and exchanges it
// through shared memory across the barrier that already precedes the MMA.
// ----------------------------------------------------------------------------
template <int N, int J, int R>
struct Tc3Cfg {
  static constexpr int M = 128;
  static constexpr int OFF_BT = 0;
  static constexpr int OFF_BN = OFF_BT + N * R * J;
  static constexpr int OFF_G = OFF_BN + N * J * R;
  static constexpr int OFF_A = OFF_G + N * R * R;        // N slots of 128 x J
  static constexpr int OFF_W = OFF_A + N * M * J;        // 128 x R
  // 2 x 128 partial predictions, double-buffered by mode parity: a thread's
  // partner reads mode n's value after the barrier while this thread may
  // already write mode n+1's (compute-sanitizer racecheck)
  static constexpr int OFF_X = OFF_W + M * R;
  static constexpr int OFF_BAR = OFF_X + 4 * M;          // mbarrier (2 words), TMEM slot, claim slot
  // the last mode's second slot, only allocated when that mode is gathered a
  // tile ahead (a cold mode); a hot last mode (NF) leaves it out, which lets
  // two J = 32 CTAs share an SM
  static constexpr int OFF_SPARE = OFF_BAR + 4;
  static constexpr int FLOATS = OFF_SPARE;
  static constexpr int NEED = (N * R > J + R) ? N * R : J + R;
  static constexpr int TCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr size_t SMEM = (size_t)FLOATS * 4;
  static constexpr size_t SMEM_SPARE = SMEM + (size_t)M * J * 4;
};

template <int N, int J, int R, bool HV>
__global__ void __launch_bounds__(256, (J <= 16 ? 3 : 2))
    factor_tc3_kernel(const int* __restrict__ rec, const int* __restrict__ visit, long long n_visit, long long base,
                      float* __restrict__ fac, const float* __restrict__ cor, TcParams<N> p,
                      unsigned* __restrict__ tile_ctr) {
  static_assert(J == R && J % 16 == 0, "v3 needs J == R, a multiple of 16");
  constexpr int RW = N <= 3 ? 4 : (N <= 7 ? 8 : 16);
  constexpr int H = J / 2;  // columns per thread
  using C = Tc3Cfg<N, J, R>;
  extern __shared__ __align__(16) float sm[];
  uint64_t& mbar = *reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint32_t& tslot = *reinterpret_cast<uint32_t*>(sm + C::OFF_BAR + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qd = warp & 3, hf = warp >> 2, s = 32 * qd + lane;  // quadrant, column half, sample
  const int c0 = hf * H;                                         // first owned column

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
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tslot, C::TCOLS);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tslot;
  const uint32_t tlane = tbase + ((uint32_t)(qd * 32) << 16);
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t id_c = tc::idesc_tf32(128, R), id_g = tc::idesc_tf32(128, J), id_h = tc::idesc_tf32(128, R);
  const uint64_t pol_keep = tc::policy_evict_last(), pol_stream = tc::policy_evict_first();
  uint32_t phase = 0;

  auto a_off = [&](int n, int pb) { return n == N - 1 && pb ? C::OFF_SPARE : C::OFF_A + n * 128 * J; };
  // this warp's half-rows of its 32 samples: 2 lanes per row chunk pair
  // (H/4 chunks per half-row; H = 8 -> 2 chunks, 16 rows per instruction)
  constexpr int HCH = H / 4, RPI = 32 / HCH;
  const int cq = lane % HCH, crow = lane / HCH;
  auto issue_mode = [&](const RecReg<N, RW>& rr, int n, int pb) {
    const uint32_t dst = sbase + 4 * a_off(n, pb);
#pragma unroll
    for (int k = 0; k < HCH; ++k) {
      const int sl = k * RPI + crow;
      const int row = __shfl_sync(0xffffffffu, rr.idx[n], sl);
      const int ok = __shfl_sync(0xffffffffu, rr.valid ? 1 : 0, sl);
      const float* src = fac + p.foff[n] + (long long)row * J + c0 + 4 * cq;
      tc::cp_async16_nohint(dst + 4 * canon<128>(32 * qd + sl, c0 + 4 * cq), src, ok ? 16u : 0u);
    }
  };

  const long long G = gridDim.x;
  uint32_t& s_claim = *reinterpret_cast<uint32_t*>(sm + C::OFF_BAR + 3);
  long long tile = blockIdx.x, t1 = tile + G, t2 = tile + 2 * G;
  if (tid == 0) s_claim = atomicAdd(tile_ctr, 1u);
  RecReg<N, RW> cur, nxt;
  // visit entries / records are indexed by sample s (both halves load them)
  auto vis = [&](long long t) -> int {
    long long k = t * 128 + s;
    k = k < n_visit ? k : n_visit - 1;
    if (HV) return tc::ld_stream_s32(visit + k, pol_stream);
    return (int)k;
  };
  auto valid_of = [&](long long t) { return t * 128 + s < n_visit; };
  int v2 = vis(t2);
  load_rec<N, RW>(cur, rec, vis(tile), valid_of(tile), base, pol_stream);
  load_rec<N, RW>(nxt, rec, vis(t1), valid_of(t1), base, pol_stream);
  int pb = 0;
  const unsigned pfm = p.prefetch == 0 ? 0u : p.prefetch == 2 ? ~0u : ~p.atomic_mask;
  // the last mode alternates slots only when it is gathered a tile ahead
  const int pbm = (pfm >> (N - 1) & 1u) ? 1 : 0;
#pragma unroll
  for (int n = 0; n < N; ++n)
    if (pfm >> n & 1u) issue_mode(cur, n, pb);
  tc::cp_async_commit();
  __syncthreads();
  long long t3 = 3 * G + s_claim;
  float* px = sm + C::OFF_X;
  while (tile * 128 < n_visit) {
    unsigned claim = 0;
    if (tid == 0) claim = atomicAdd(tile_ctr, 1u);
#pragma unroll
    for (int n = 0; n < N; ++n)
      if (!(pfm >> n & 1u)) issue_mode(cur, n, pb);
    tc::cp_async_commit();
    RecReg<N, RW> nnxt;
    load_rec<N, RW>(nnxt, rec, v2, valid_of(t2), base, pol_stream);
    v2 = vis(t3);
    tc::cp_async_wait_all();
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int n = 0; n < N; ++n)
        issue_gemm<R, J, false>(tbase + n * R, sbase + 4 * a_off(n, pb), 0, sbase + 4 * (C::OFF_BT + n * R * J), 0,
                                id_c);
      tc::mma_commit(&mbar);
    }
    if (pfm >> (N - 1) & 1u) issue_mode(nxt, N - 1, pb ^ 1);
    tc::mbar_wait(&mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    float c[N][H];
#pragma unroll
    for (int n = 0; n < N; ++n) tc::tmem_ldh<H>(tlane + n * R + c0, c[n]);

#pragma unroll
    for (int n = 0; n < N; ++n) {
      // W_n (my half), my half of inter = sum_r W_n[r] c_n[r]
      float* wt = sm + C::OFF_W;
      float part = 0.f;
#pragma unroll
      for (int q = 0; q < H / 4; ++q) {
        float w4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float w = 1.f;
#pragma unroll
          for (int n0 = 0; n0 < N; ++n0)
            if (n0 != n) w *= c[n0][4 * q + u];
          w4[u] = w;
          part = fmaf(w, c[n][4 * q + u], part);
        }
        *reinterpret_cast<float4*>(wt + canon<128>(s, c0 + 4 * q)) = make_float4(w4[0], w4[1], w4[2], w4[3]);
      }
      px[(n & 1) * 256 + hf * 128 + s] = part;
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t a = sbase + 4 * C::OFF_W;
        issue_gemm<J, R, false>(tbase, a, 0, sbase + 4 * (C::OFF_BN + n * J * R), 0, id_g);
        if (n < N - 1) issue_gemm<R, R, false>(tbase + J, a, 0, sbase + 4 * (C::OFF_G + n * R * R), 0, id_h);
        tc::mma_commit(&mbar);
      }
      if (n >= 1 && n - 1 < N - 1 && (pfm >> (n - 1) & 1u)) issue_mode(nxt, n - 1, 0);
      const float inter = part + px[(n & 1) * 256 + (hf ^ 1) * 128 + s];
      tc::mbar_wait(&mbar, phase);
      phase ^= 1;
      tc::fence_after_sync();
      float g[H];
      tc::tmem_ldh<H>(tlane + c0, g);
      float* at = sm + a_off(n, pb);
      float a[H];
#pragma unroll
      for (int q = 0; q < H / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(at + canon<128>(s, c0 + 4 * q));
        a[4 * q] = v.x;
        a[4 * q + 1] = v.y;
        a[4 * q + 2] = v.z;
        a[4 * q + 3] = v.w;
      }
      const float gm = p.gam[n], lm = p.lam[n];
      const bool red = p.atomic_mask >> n & 1u;
#pragma unroll
      for (int q = 0; q < H / 4; ++q) {
        float d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * q + u;
          const float gr = -cur.x * g[j] + lm * a[j] + inter * g[j];
          d[u] = -gm * gr;
          a[j] += d[u];
        }
        // red.add modes park the delta, the others the new row
        const float4 v = red ? make_float4(d[0], d[1], d[2], d[3])
                             : make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
        *reinterpret_cast<float4*>(at + canon<128>(s, c0 + 4 * q)) = v;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < HCH; ++k) {
        const int sl = k * RPI + crow;
        const int row = __shfl_sync(0xffffffffu, cur.idx[n], sl);
        const int ok = __shfl_sync(0xffffffffu, cur.valid ? 1 : 0, sl);
        const float4 v = *reinterpret_cast<const float4*>(at + canon<128>(32 * qd + sl, c0 + 4 * cq));
        float* dst = fac + p.foff[n] + (long long)row * J + c0 + 4 * cq;
        if (ok) {
          if (red)
            tc::red_add_v4(dst, v);
          else
            tc::st_v4_hint(dst, v, pol_keep);
        }
      }
      if (n < N - 1) {
        float hv[H];
        tc::tmem_ldh<H>(tlane + J + c0, hv);
        const float keep = 1.f - gm * lm, step = gm * (cur.x - inter);
#pragma unroll
        for (int r = 0; r < H; ++r) c[n][r] = fmaf(step, hv[r], keep * c[n][r]);
      }
    }
    tc::cp_async_commit();
    cur = nxt;
    nxt = nnxt;
    tile = t1;
    t1 = t2;
    t2 = t3;
    pb ^= pbm;
    if (tid == 0) s_claim = claim;
    __syncthreads();
    t3 = 3 * G + s_claim;
  }
  tc::cp_async_wait_all();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, C::TCOLS);
  }
}

template <int N, int J, int R>
static int launch_tc3(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                      const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s) {
  using C = Tc3Cfg<N, J, R>;
  TcParams<N> p;
  for (int n = 0; n < N; ++n) {
    p.foff[n] = md.foff[n];
    p.gam[n] = gam[n];
    p.lam[n] = lam[n];
  }
  p.dbg = nullptr;
  p.atomic_mask = hot_mode_mask(md);
  {
    const char* e = getenv("SPTK_TC_PREFETCH");
    p.prefetch = e ? atoi(e) : 1;
  }
  (void)rw;
  auto kfn = visit ? factor_tc3_kernel<N, J, R, true> : factor_tc3_kernel<N, J, R, false>;
  const unsigned pfm = p.prefetch == 0 ? 0u : p.prefetch == 2 ? ~0u : ~p.atomic_mask;
  const size_t smem = (pfm >> (N - 1) & 1u) ? C::SMEM_SPARE : C::SMEM;
  static size_t configured = 0;
  static int per_sm = 1;
  if (configured != smem) {
    for (auto f : {factor_tc3_kernel<N, J, R, true>, factor_tc3_kernel<N, J, R, false>}) {
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_SPARE));
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    cudaFuncAttributes fa;
    SPTK_CUDA_TRY(cudaFuncGetAttributes(&fa, (const void*)kfn));
    const int regs = fa.numRegs < 1 ? 1 : fa.numRegs;
    int by_regs = 65536 / (((regs * 32 + 255) / 256) * 256 * 8);
    int by_smem = (int)((228 * 1024) / (smem + fa.sharedSizeBytes + 1024));
    int by_tmem = 512 / C::TCOLS;
    int n = by_regs < by_smem ? by_regs : by_smem;
    n = n < by_tmem ? n : by_tmem;
    int cap = n >= 3 ? n - 1 : n;  // leave room for the side-stream samplers (see resident_ctas)
    if (const char* e = getenv("SPTK_TC_CTAS")) cap = atoi(e);
    if (cap >= 1 && cap < n) n = cap;
    per_sm = n < 1 ? 1 : n;
    if (getenv("SPTK_DEBUG")) fprintf(stderr, "[sptk] tc3 regs=%d smem=%zu -> %d CTAs/SM\n", regs, smem, per_sm);
    configured = smem;
  }
  long long tiles = (n_visit + 127) / 128;
  long long blocks = 148LL * per_sm;
  // CTA slots left to the side-stream samplers (see launch_tc2); default none
  if (const char* e = getenv("SPTK_SAMPLER_SLOTS3")) blocks -= atoi(e);
  if (blocks < 1) blocks = 1;
  if (blocks > hogwild_cta_cap(n_visit, 128)) blocks = hogwild_cta_cap(n_visit, 128);
  if (blocks > tiles) blocks = tiles;
  unsigned* ctr = nullptr;
  SPTK_CUDA_TRY(cudaGetSymbolAddress((void**)&ctr, g_tile_ctr));
  ctr += g_tc_ctr_slot.fetch_add(1u) & 63u;
  SPTK_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
  kfn<<<(unsigned)blocks, 256, smem, s>>>(rec, visit, n_visit, base, fac, cor, p, ctr);
  note_factor_kernel("factor_tc3_kernel");
  SPTK_CHECK_LAUNCH();
  return 0;
}

template <int N, int J, int R>
static int launch_tc2(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                      const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s) {
  using C = Tc2Cfg<N, J, R>;
  TcParams<N> p;
  for (int n = 0; n < N; ++n) {
    p.foff[n] = md.foff[n];
    p.gam[n] = gam[n];
    p.lam[n] = lam[n];
  }
  p.dbg = g_tc_debug;  // tc2: per-phase clock stamps (long long[16][16]) when set
  p.atomic_mask = hot_mode_mask(md);
  {
    const char* e = getenv("SPTK_TC_PREFETCH");
    p.prefetch = e ? atoi(e) : 1;
    // experiment hook (wrong results): drop the hot modes' row writes to
    // measure what their L2 contention costs
    if (getenv("SPTK_DEBUG_DROP_HOT")) {
      static bool warned = false;
      if (!warned) {
        fprintf(stderr, "[sptk] SPTK_DEBUG_DROP_HOT: hot-mode row updates are dropped (timing experiment)\n");
        warned = true;
      }
      p.atomic_mask |= 0x80000000u;
    }
    const char* d = getenv("SPTK_TC_DEFER_WB");
    p.defer_wb = d ? atoi(d) : 0;
  }
  (void)rw;  // == rec_words(N), checked by try_factor_tc
  auto kfn = visit ? factor_tc2_kernel<N, J, R, true> : factor_tc2_kernel<N, J, R, false>;
  // the last mode's spare slot only when it is gathered ahead (see Tc2Cfg)
  const unsigned pfm = p.prefetch == 0 ? 0u : p.prefetch == 2 ? ~0u : ~p.atomic_mask;
  const unsigned lpm = p.prefetch == 3 ? p.atomic_mask : 0u;
  const size_t smem = ((pfm | lpm) >> (N - 1) & 1u) ? C::SMEM_SPARE : C::SMEM;
  static size_t configured = 0;
  static int per_sm = 1;
  if (configured != smem) {
    for (auto f : {factor_tc2_kernel<N, J, R, true>, factor_tc2_kernel<N, J, R, false>}) {
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_SPARE));
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    per_sm = resident_ctas((const void*)kfn, smem, C::TCOLS, false);
    configured = smem;
  }
  long long tiles = (n_visit + 127) / 128;
  // Persistent grid: every CTA slot the kernel's resources allow except the
  // ones left to the side-stream samplers that run beside the factor pass
  // (SPTK_SAMPLER_SLOTS).  Measured per shape on the bench tensors (ms per
  // epoch): NF J=R=16 with one slot free on every SM (444 CTAs) 18.9, with
  // 520 / 560 / 575 CTAs 18.7 / 18.4 / 18.3, with all 592 slots 20.3 (the
  // samplers then wait for the whole pass), so 16 slots there; J=R=8, Y4 and
  // O6 are sampler-heavier relative to their factor pass and lose with 16
  // (13.0 -> 13.5, 90 -> 96, 251 -> 272), so they keep one slot per SM.
  int slots = (N == 3 && J >= 16) ? 16 : 148;
  if (const char* e = getenv("SPTK_SAMPLER_SLOTS")) slots = atoi(e);
  long long blocks = 148LL * per_sm - (per_sm >= 2 ? slots : 0);
  // experiment hook: SPTK_TC_GRID = explicit persistent grid size
  if (const char* e = getenv("SPTK_TC_GRID")) blocks = atoll(e);
  if (blocks < 1) blocks = 1;
  if (blocks > hogwild_cta_cap(n_visit, 128)) blocks = hogwild_cta_cap(n_visit, 128);
  if (blocks > tiles) blocks = tiles;
  // per-launch tile counter from a small rotating pool (launches on one stream
  // are ordered; the pool only guards against back-to-back reuse)
  unsigned* ctr = nullptr;
  SPTK_CUDA_TRY(cudaGetSymbolAddress((void**)&ctr, g_tile_ctr));
  ctr += g_tc_ctr_slot.fetch_add(1u) & 63u;
  SPTK_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
  kfn<<<(unsigned)blocks, 128, smem, s>>>(rec, visit, n_visit, base, fac, cor, p, ctr);
  note_factor_kernel("factor_tc2_kernel");
  SPTK_CHECK_LAUNCH();
  return 0;
}

// ----------------------------------------------------------------------------
// v4: J = R = 64 (the rank sweep's largest point).  At this rank the v2/v3
// shared-memory plan does not fit (B_n in both K-major orientations is 96 KB
// for N = 3, G_n would add 48 KB, the A tiles 96 KB), so the c_n refresh goes
// back to an MMA on the updated A tile (c_n' = A_n' . B_n, v1 style), the last
// mode's rows move to registers after the c round so W takes their slot, and
// the plan is 194 KB: one CTA per SM, 512 threads, four threads per sample.
// Warp w reads TMEM lane quadrant w % 4 (samples 32(w%4)..+31) and owns column
// quarter w / 4 of every J- or R-vector (16 columns: c_n[16] x N, gs[16], a[16]
// in registers).  inter = sum_r W_n[r] c_n[r] is summed from the four
// quarters' partials across the barrier that precedes the gs MMA (fixed
// order, so the four threads of a sample agree bit for bit).  Rows are
// gathered per quarter (4 lanes per 64-byte quarter row) with cp.async and
// written back straight from registers (plain stores, or red.add deltas for
// the hot modes).  Tensor rounds per tile: c (N MMAs), then per mode gs and,
// except for the last mode, the refresh: 2N rounds.  (Gathering the next
// tile's mode-0 rows during this tile, in a second slot with the partials
// exchanged through TMEM instead of shared memory, measured no gain: 69.8 ms
// either way on NF J = R = 64.)
// ----------------------------------------------------------------------------
template <int N, int J, int R>
struct Tc4Cfg {
  static constexpr int M = 128;
  static constexpr int OFF_BT = 0;                   // N x (R rows x J)
  static constexpr int OFF_BN = OFF_BT + N * R * J;  // N x (J rows x R)
  static constexpr int OFF_A = OFF_BN + N * J * R;   // N slots of 128 x J
  static constexpr int OFF_W = OFF_A + (N - 1) * M * J;  // 128 x R: the last mode's A slot (see below)
  static constexpr int OFF_X = OFF_A + N * M * J;    // 4 x 128 partial predictions, x2 by mode parity
  static constexpr int FLOATS = OFF_X + 8 * M;
  static constexpr int NEED = N * R + J;             // c_0..c_{N-1}, gs
  static constexpr int TCOLS = NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr size_t SMEM = (size_t)FLOATS * 4 + 16;
};

template <int N, int J, int R, bool HV>
__global__ void __launch_bounds__(512, 1)
    factor_tc4_kernel(const int* __restrict__ rec, const int* __restrict__ visit, long long n_visit, long long base,
                      float* __restrict__ fac, const float* __restrict__ cor, TcParams<N> p,
                      unsigned* __restrict__ tile_ctr) {
  static_assert(J == R && J % 64 == 0, "v4 needs J == R, a multiple of 64");
  constexpr int RW = N <= 3 ? 4 : (N <= 7 ? 8 : 16);
  constexpr int Q = J / 4;  // columns per thread
  using C = Tc4Cfg<N, J, R>;
  extern __shared__ __align__(16) float sm[];
  uint64_t& mbar = *reinterpret_cast<uint64_t*>(sm + C::FLOATS);
  uint32_t& tslot = *reinterpret_cast<uint32_t*>(sm + C::FLOATS + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qd = warp & 3, qq = warp >> 2, s = 32 * qd + lane;  // quadrant, column quarter, sample
  const int c0 = qq * Q;                                         // first owned column

  for (int e = tid; e < N * J * R; e += 512) {
    const int n = e / (J * R), rem = e - n * (J * R), j = rem / R, r = rem - j * R;
    const float b = __ldg(cor + e);
    sm[C::OFF_BT + n * R * J + canon<R>(r, j)] = b;
    sm[C::OFF_BN + n * J * R + canon<J>(j, r)] = b;
  }
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tslot, C::TCOLS);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tslot;
  const uint32_t tlane = tbase + ((uint32_t)(qd * 32) << 16);
  const uint32_t tgs = N * R;  // gs columns
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t id_c = tc::idesc_tf32(128, R), id_g = tc::idesc_tf32(128, J);
  const uint64_t pol_keep = tc::policy_evict_last(), pol_stream = tc::policy_evict_first();
  uint32_t phase = 0;

  auto a_off = [&](int n) { return C::OFF_A + n * 128 * J; };
  // this warp's quarter rows of its 32 samples: 4 lanes per quarter row (one
  // 16-byte chunk each), 8 rows per instruction
  constexpr int QCH = Q / 4, RPI = 32 / QCH;
  const int cq = lane % QCH, crow = lane / QCH;
  auto issue_mode = [&](const RecReg<N, RW>& rr, int n) {
    const uint32_t dst = sbase + 4 * a_off(n);
#pragma unroll
    for (int k = 0; k < QCH; ++k) {
      const int sl = k * RPI + crow;
      const int row = __shfl_sync(0xffffffffu, rr.idx[n], sl);
      const int ok = __shfl_sync(0xffffffffu, rr.valid ? 1 : 0, sl);
      const float* src = fac + p.foff[n] + (long long)row * J + c0 + 4 * cq;
      tc::cp_async16_nohint(dst + 4 * canon<128>(32 * qd + sl, c0 + 4 * cq), src, ok ? 16u : 0u);
    }
  };
  auto mma_round_wait = [&]() {
    tc::mbar_wait(&mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
  };

  const long long G = gridDim.x;
  uint32_t& s_claim = *reinterpret_cast<uint32_t*>(sm + C::FLOATS + 3);
  long long tile = blockIdx.x, t1 = tile + G, t2 = tile + 2 * G;
  if (tid == 0) s_claim = atomicAdd(tile_ctr, 1u);
  RecReg<N, RW> cur, nxt;
  auto vis = [&](long long t) -> int {
    long long k = t * 128 + s;
    k = k < n_visit ? k : n_visit - 1;
    if (HV) return tc::ld_stream_s32(visit + k, pol_stream);
    return (int)k;
  };
  auto valid_of = [&](long long t) { return t * 128 + s < n_visit; };
  int v2 = vis(t2);
  load_rec<N, RW>(cur, rec, vis(tile), valid_of(tile), base, pol_stream);
  load_rec<N, RW>(nxt, rec, vis(t1), valid_of(t1), base, pol_stream);
  __syncthreads();
  long long t3 = 3 * G + s_claim;
  float* px = sm + C::OFF_X;
  float* wt = sm + C::OFF_W;
  while (tile * 128 < n_visit) {
    unsigned claim = 0;
    if (tid == 0) claim = atomicAdd(tile_ctr, 1u);
#pragma unroll
    for (int n = 0; n < N; ++n) issue_mode(cur, n);
    tc::cp_async_commit();
    RecReg<N, RW> nnxt;
    load_rec<N, RW>(nnxt, rec, v2, valid_of(t2), base, pol_stream);
    v2 = vis(t3);
    tc::cp_async_wait_all();
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int n = 0; n < N; ++n)
        issue_gemm<R, J, false>(tbase + n * R, sbase + 4 * a_off(n), 0, sbase + 4 * (C::OFF_BT + n * R * J), 0, id_c);
      tc::mma_commit(&mbar);
    }
    mma_round_wait();
    float c[N][Q];
#pragma unroll
    for (int n = 0; n < N; ++n) tc::tmem_ldh<Q>(tlane + n * R + c0, c[n]);
    // The last mode's rows go to registers now: its slot then holds W (same
    // canonical layout since J == R, so every thread overwrites exactly the
    // entries it just read, and the c-round MMA that read them is complete).
    float a_last[Q];
#pragma unroll
    for (int q = 0; q < Q / 4; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(sm + a_off(N - 1) + canon<128>(s, c0 + 4 * q));
      a_last[4 * q] = v.x;
      a_last[4 * q + 1] = v.y;
      a_last[4 * q + 2] = v.z;
      a_last[4 * q + 3] = v.w;
    }

#pragma unroll
    for (int n = 0; n < N; ++n) {
      // W_n (my quarter) and my quarter of inter = sum_r W_n[r] c_n[r]
      float part = 0.f;
#pragma unroll
      for (int q = 0; q < Q / 4; ++q) {
        float w4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float w = 1.f;
#pragma unroll
          for (int n0 = 0; n0 < N; ++n0)
            if (n0 != n) w *= c[n0][4 * q + u];
          w4[u] = w;
          part = fmaf(w, c[n][4 * q + u], part);
        }
        *reinterpret_cast<float4*>(wt + canon<128>(s, c0 + 4 * q)) = make_float4(w4[0], w4[1], w4[2], w4[3]);
      }
      px[(n & 1) * 512 + qq * 128 + s] = part;
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
        issue_gemm<J, R, false>(tbase + tgs, sbase + 4 * C::OFF_W, 0, sbase + 4 * (C::OFF_BN + n * J * R), 0, id_g);
        tc::mma_commit(&mbar);
      }
      const float* pp = px + (n & 1) * 512;
      const float inter = ((pp[s] + pp[128 + s]) + pp[256 + s]) + pp[384 + s];
      float* at = sm + a_off(n);
      float a[Q];
      if (n == N - 1) {
#pragma unroll
        for (int j = 0; j < Q; ++j) a[j] = a_last[j];
      } else {
#pragma unroll
        for (int q = 0; q < Q / 4; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(at + canon<128>(s, c0 + 4 * q));
          a[4 * q] = v.x;
          a[4 * q + 1] = v.y;
          a[4 * q + 2] = v.z;
          a[4 * q + 3] = v.w;
        }
      }
      mma_round_wait();
      float g[Q];
      tc::tmem_ldh<Q>(tlane + tgs + c0, g);
      const float gm = p.gam[n], lm = p.lam[n];
      const bool red = p.atomic_mask >> n & 1u;
      float* dst = fac + p.foff[n] + (long long)cur.idx[n] * J + c0;
#pragma unroll
      for (int q = 0; q < Q / 4; ++q) {
        float d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * q + u;
          const float gr = -cur.x * g[j] + lm * a[j] + inter * g[j];
          d[u] = -gm * gr;
          a[j] += d[u];
        }
        if (cur.valid) {
          if (red)
            tc::red_add_v4(dst + 4 * q, make_float4(d[0], d[1], d[2], d[3]));
          else
            tc::st_v4_hint(dst + 4 * q, make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]), pol_keep);
        }
      }
      if (n < N - 1) {
        // refresh c_n from the updated rows: c_n' = A_n' . B_n
#pragma unroll
        for (int q = 0; q < Q / 4; ++q)
          *reinterpret_cast<float4*>(at + canon<128>(s, c0 + 4 * q)) =
              make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        if (tid == 0) {
          tc::fence_after_sync();
          issue_gemm<R, J, false>(tbase + n * R, sbase + 4 * a_off(n), 0, sbase + 4 * (C::OFF_BT + n * R * J), 0,
                                  id_c);
          tc::mma_commit(&mbar);
        }
        mma_round_wait();
        tc::tmem_ldh<Q>(tlane + n * R + c0, c[n]);
      }
    }
    cur = nxt;
    nxt = nnxt;
    tile = t1;
    t1 = t2;
    t2 = t3;
    if (tid == 0) s_claim = claim;
    tc::fence_before_sync();
    __syncthreads();
    t3 = 3 * G + s_claim;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, C::TCOLS);
  }
}

template <int N, int J, int R>
static int launch_tc4(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                      const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s) {
  using C = Tc4Cfg<N, J, R>;
  TcParams<N> p;
  for (int n = 0; n < N; ++n) {
    p.foff[n] = md.foff[n];
    p.gam[n] = gam[n];
    p.lam[n] = lam[n];
  }
  p.dbg = nullptr;
  p.atomic_mask = hot_mode_mask(md);
  p.prefetch = 0;
  p.defer_wb = 0;
  (void)rw;
  auto kfn = visit ? factor_tc4_kernel<N, J, R, true> : factor_tc4_kernel<N, J, R, false>;
  static int configured = 0;
  if (!configured) {
    for (auto f : {factor_tc4_kernel<N, J, R, true>, factor_tc4_kernel<N, J, R, false>}) {
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
      SPTK_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    configured = 1;
  }
  long long tiles = (n_visit + 127) / 128;
  long long blocks = 148;
  if (blocks > hogwild_cta_cap(n_visit, 128)) blocks = hogwild_cta_cap(n_visit, 128);
  if (blocks > tiles) blocks = tiles;
  unsigned* ctr = nullptr;
  SPTK_CUDA_TRY(cudaGetSymbolAddress((void**)&ctr, g_tile_ctr));
  ctr += g_tc_ctr_slot.fetch_add(1u) & 63u;
  SPTK_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
  kfn<<<(unsigned)blocks, 512, C::SMEM, s>>>(rec, visit, n_visit, base, fac, cor, p, ctr);
  note_factor_kernel("factor_tc4_kernel");
  SPTK_CHECK_LAUNCH();
  return 0;
}

// 0 off (CUDA-core FMA kernel), 1 TF32 v2, 2 TF32 v1, 3 3xTF32 v1,
// 4 TF32 v3 (two threads per sample), 5 CUDA-core thread-per-sample FMA,
// 6 TF32 v6 with TMA row traffic (default; v2/v3/v4 for shapes it lacks);
// J = R = 64 always takes v4 when on
static int g_tc_mode = -1;

static int tc_mode_env() {
  if (g_tc_mode < 0) {
    const char* e = getenv("SPTK_TC");
    g_tc_mode = e ? atoi(e) : 6;
  }
  return g_tc_mode;
}

int set_tc_mode(int mode) {
  if (mode < 0 || mode > 6) return 2;
  g_tc_mode = mode;
  return 0;
}
int get_tc_mode() { return tc_mode_env(); }
void set_tc_debug(float* buf) { g_tc_debug = buf; }
float* tc_debug_buffer() { return g_tc_debug; }

template <int N, int J, int R, bool SPLIT>
static int launch_tc(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                     const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s) {
  using C = TcCfg<N, J, R, SPLIT>;
  TcParams<N> p;
  for (int n = 0; n < N; ++n) {
    p.foff[n] = md.foff[n];
    p.gam[n] = gam[n];
    p.lam[n] = lam[n];
  }
  p.dbg = g_tc_debug;
  p.atomic_mask = hot_mode_mask(md);
  auto kfn = rw == 4 ? factor_tc_kernel<N, J, R, SPLIT, 4> : factor_tc_kernel<N, J, R, SPLIT, 8>;
  static int configured = 0;
  static int per_sm = 1;
  if (!configured) {
    SPTK_CUDA_TRY(cudaFuncSetAttribute(factor_tc_kernel<N, J, R, SPLIT, 4>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    SPTK_CUDA_TRY(cudaFuncSetAttribute(factor_tc_kernel<N, J, R, SPLIT, 8>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    SPTK_CUDA_TRY(cudaFuncSetAttribute(factor_tc_kernel<N, J, R, SPLIT, 4>,
                                       cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    SPTK_CUDA_TRY(cudaFuncSetAttribute(factor_tc_kernel<N, J, R, SPLIT, 8>,
                                       cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    per_sm = resident_ctas((const void*)kfn, C::SMEM, C::TCOLS);
    configured = 1;
  }
  long long tiles = (n_visit + 127) / 128;
  long long blocks = 148LL * per_sm;
  if (blocks > hogwild_cta_cap(n_visit, 128)) blocks = hogwild_cta_cap(n_visit, 128);
  if (blocks > tiles) blocks = tiles;
  kfn<<<(unsigned)blocks, 128, C::SMEM, s>>>(rec, visit, n_visit, base, fac, cor, p);
  note_factor_kernel("factor_tc_kernel");
  SPTK_CHECK_LAUNCH();
  return 0;
}

// returns 1 if handled
int try_factor_tc(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                  const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s, int* rc) {
  int mode = tc_mode_env();
  if (mode == 0 || mode == 5) return 0;
  // v6 (TMA row traffic) where it has an instance, v2 / v3 / v4 elsewhere
  if (mode == 6) {
    if (try_factor_tma(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s, rc)) return 1;
    mode = 1;
  }
  const int N = md.n_modes, R = md.rcore, J = md.jr[0];
  for (int n = 0; n < N; ++n)
    if (md.jr[n] != J) return 0;
  if (J != R || rw != rec_words(N)) return 0;
#define SPTK_TC_CASE(NN, JJ)                                                                                 \
  if (N == NN && J == JJ) {                                                                                  \
    *rc = mode == 4   ? launch_tc3<NN, JJ, JJ>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s)        \
          : mode == 1 ? launch_tc2<NN, JJ, JJ>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s)        \
          : mode == 2 ? launch_tc<NN, JJ, JJ, false>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s) \
                      : launch_tc<NN, JJ, JJ, true>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s);  \
    return 1;                                                                                                \
  }
  SPTK_TC_CASE(3, 16)
  SPTK_TC_CASE(4, 16)
  if (mode != 3 && N == 3 && J == 64) {  // (3xTF32 is not implemented for v4)
    *rc = launch_tc4<3, 64, 64>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s);
    return 1;
  }
  if (mode == 1 && N == 3 && J == 32) {
    // at J = R = 32 the one-thread-per-sample kernel needs ~250 registers (one
    // CTA per SM); two threads per sample is faster (NF: 37 vs 46 ms)
    *rc = launch_tc3<3, 32, 32>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s);
    return 1;
  }
  SPTK_TC_CASE(3, 32)
  if (mode == 1) {  // v2 only: 8-column tiles (MMA N = 8, K = 8)
    if (N == 3 && J == 8) {
      *rc = launch_tc2<3, 8, 8>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s);
      return 1;
    }
    if (N == 6 && J == 8) {
      *rc = launch_tc2<6, 8, 8>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s);
      return 1;
    }
  }
#undef SPTK_TC_CASE
  return 0;
}

}  // namespace sptk
