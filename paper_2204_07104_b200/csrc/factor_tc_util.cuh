// factor_tc_util.cuh -- pieces shared by the tcgen05 factor kernels
// (factor_tc.cu: v1-v4, factor_tma.cu: v6): operand layout, the per-thread
// record registers, and the launch-shape policies.
#pragma once
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc.cuh"

namespace sptk {

// float offset of element (row, k) in a K-major canonical operand with ROWS rows
template <int ROWS>
__device__ __forceinline__ int canon(int row, int k) {
  return (k >> 2) * (ROWS * 4) + (row >> 3) * 32 + (row & 7) * 4 + (k & 3);
}

template <int N, int RW>
struct RecReg {
  int idx[N];
  float x;
  bool valid;
};

// visit-list entry of this thread's sample in `tile` (-1 past the end)
// Returns the raw 32-bit entry: widening it here would make the compiler
// consume the load immediately (a sign extension right after the LDG), which
// exposed the full visit-gather latency at the start of every tile.
// (HV: a visit list is given; without one the k-th sample is record k.  A
// template flag, so no predicated select ever writes the loaded register.)
template <bool HV>
__device__ __forceinline__ int load_vis(const int* __restrict__ visit, long long n_visit, long long tile,
                                        uint64_t pol) {
  // unconditional (clamped) load; validity is recomputed from the tile index
  long long k = tile * 128 + threadIdx.x;
  k = k < n_visit ? k : n_visit - 1;
  if (HV) return tc::ld_stream_s32(visit + k, pol);
  return (int)k;
}
__device__ __forceinline__ bool tile_valid(long long n_visit, long long tile) {
  return tile * 128 + threadIdx.x < n_visit;
}

template <int N, int RW>
__device__ __forceinline__ void load_rec(RecReg<N, RW>& o, const int* __restrict__ rec, int v, bool valid,
                                         long long base, uint64_t pol) {
  // Unconditional load (past-the-end samples read the block's first record
  // and are masked by `valid` at use): a predicated load merged with a
  // default value would make the compiler wait for it right here, exposing
  // the record-gather latency instead of hiding it behind two tiles of work.
  o.valid = valid;
  const int* rp = rec + (base + (long long)v) * RW;
  int wv[8];
  int4 w0 = tc::ld_stream_v4(rp, pol);
  wv[0] = w0.x;
  wv[1] = w0.y;
  wv[2] = w0.z;
  wv[3] = w0.w;
  if (RW >= 8) {
    int4 w1 = tc::ld_stream_v4(rp + 4, pol);
    wv[4] = w1.x;
    wv[5] = w1.y;
    wv[6] = w1.z;
    wv[7] = w1.w;
  }
#pragma unroll
  for (int n = 0; n < N; ++n) o.idx[n] = wv[n];
  o.x = __int_as_float(wv[N]);
}

// CTAs of a 128-thread tcgen05 kernel that fit on one SM: registers, shared
// memory (228 KB per SM, 1 KB reserved per CTA) and TMEM (512 columns).
static inline int resident_ctas(const void* kfn, size_t smem, int tcols, bool leave_slot = true) {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kfn) != cudaSuccess) return 1;
  int regs = fa.numRegs < 1 ? 1 : fa.numRegs;
  int by_regs = 65536 / (((regs * 32 + 255) / 256) * 256 * 4);
  int by_smem = (int)((228 * 1024) / (smem + fa.sharedSizeBytes + 1024));
  int by_tmem = 512 / tcols;
  int n = by_regs < by_smem ? by_regs : by_smem;
  n = n < by_tmem ? n : by_tmem;
  // Default: one CTA per SM below the resource limit.  The training epoch
  // runs the next epoch's samplers on side streams; a persistent factor grid
  // that fills every SM locks them out until it drains, while one free slot
  // per SM lets them run underneath (NF bench: 19.6 ms vs 22.3 ms per epoch,
  // the factor pass itself 13.5 vs 11.2 ms).  SPTK_TC_CTAS overrides.
  int cap = leave_slot && n >= 4 ? n - 1 : n;
  if (const char* e = getenv("SPTK_TC_CTAS")) cap = atoi(e);
  if (cap >= 1 && cap < n) n = cap;
  if (getenv("SPTK_DEBUG")) fprintf(stderr, "[sptk] tc kernel regs=%d smem=%zu -> %d CTAs/SM\n", regs, smem, n);
  return n < 1 ? 1 : n;
}

// Modes with few rows take many concurrent updates per row; their row writes
// are issued as red.add deltas so no update is lost (Hogwild with atomic
// deltas).  Default: modes with fewer than 2^18 rows.  SPTK_ATOMIC_MASK
// overrides (bit n = mode n).
static inline unsigned hot_mode_mask(const ModelDesc& md) {
  if (const char* e = getenv("SPTK_ATOMIC_MASK")) return (unsigned)strtoul(e, nullptr, 0);
  unsigned m = 0;
  for (int n = 0; n < md.n_modes; ++n) {
    const long long end = n + 1 < md.n_modes ? md.foff[n + 1] : md.fac_size;
    const long long rows = (end - md.foff[n]) / (md.jr[n] > 0 ? md.jr[n] : 1);
    if (rows < (1LL << 18)) m |= 1u << n;
  }
  return m;
}

}  // namespace sptk
