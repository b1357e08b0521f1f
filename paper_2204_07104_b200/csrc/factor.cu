// factor.cu -- K3: the per-nonzero factor-row SGD update (Eq. 13).
//
// Restates _loops.factor_pass (_loops.py:17-63): for every visited sample and
// every mode n in ascending order,
//     c[n0,r] = A(n0)[i_n0,:] . B(n0)[:,r]                 (refreshed per mode)
//     gs[j]   = sum_r (prod_{n0!=n} c[n0,r]) * B(n)[j,r]
//     inter   = a . gs
//     a[j]   -= gamma_n * (-x*gs[j] + lambda_n*a[j] + inter*gs[j])
// Only the updated mode's c row changes between modes, so the kernels compute
// the c table once per sample and refresh one row per mode: (3N-1)*J*R FMAs
// per sample instead of the reference's (N^2+N)*J*R, with identical values.
//
// Three kernels:
//   * factor_tps_kernel<N,J,R,RW>  throughput mode, one thread per sample.
//     B(n) lives in the constant bank (uniform across the warp, so every FFMA
//     takes its B operand straight from c[][] with no shared-memory traffic),
//     rows are gathered with 16-byte L2 loads, Hogwild in visit order as in
//     cuFastTucker.
//   * factor_wps_kernel<T>         throughput mode for ranks without a
//     specialisation: one warp per sample, lanes over r and j (the paper's
//     warp-shuffle layout), B(n) in shared memory.
//   * factor_seq_kernel<T>         exact mode: reproduces the strictly
//     sequential loop (conflict-free prefixes of the visit list run in
//     parallel, the reference's operation order, no FMA contraction; fp32 or
//     fp64).
#include "common.cuh"
#include "kernels.cuh"

namespace sptk {

#define CONST_COR_MAX 12288
__constant__ float c_cor[CONST_COR_MAX];

template <int N>
struct TpsParams {
  long long foff[N];
  float gam[N];
  float lam[N];
};

// Software pipeline over the grid-stride samples: the visit entry two
// samples ahead and the record one sample ahead are in flight while the
// current sample computes (a thread's chain visit -> record -> rows would
// otherwise expose three memory latencies per sample).
template <int RW>
__device__ __forceinline__ void tps_load_rec(const int* __restrict__ rec, long long ri, int4& w0, int4& w1) {
  const int4* rp = reinterpret_cast<const int4*>(rec + ri * RW);
  w0 = __ldg(rp);
  if (RW >= 8) w1 = __ldg(rp + 1);
}

template <int N, int J, int R, int RW>
__global__ void __launch_bounds__(128, (J <= 4 ? 6 : (N * J <= 24 ? 5 : (J <= 8 ? 4 : 3))))
    factor_tps_kernel(const int* __restrict__ rec, const int* __restrict__ visit, long long n_visit,
                      long long base, float* __restrict__ fac, TpsParams<N> p) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long k0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  auto vis = [&](long long k) -> long long {
    const long long kc = k < n_visit ? k : n_visit - 1;
    return base + (visit ? (long long)__ldg(visit + kc) : kc);
  };
  long long v_next = vis(k0 + stride);
  int4 c0w = make_int4(0, 0, 0, 0), c1w = make_int4(0, 0, 0, 0);
  tps_load_rec<RW>(rec, vis(k0), c0w, c1w);
  for (long long k = k0; k < n_visit; k += stride) {
    int idx[N];
    float x;
    {
      int wv[RW];
      wv[0] = c0w.x;
      wv[1] = c0w.y;
      wv[2] = c0w.z;
      wv[3] = c0w.w;
      if (RW >= 8) {
        wv[4 % RW] = c1w.x;
        wv[5 % RW] = c1w.y;
        wv[6 % RW] = c1w.z;
        wv[7 % RW] = c1w.w;
      }
#pragma unroll
      for (int n = 0; n < N; ++n) idx[n] = wv[n];
      x = __int_as_float(wv[N]);
    }
    // next sample's record and the visit entry after it
    tps_load_rec<RW>(rec, v_next, c0w, c1w);
    v_next = vis(k + 2 * stride);
    float a[N][J];
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const float4* src = reinterpret_cast<const float4*>(fac + p.foff[n] + (long long)idx[n] * J);
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
        float4 v = __ldcg(src + q);
        a[n][4 * q] = v.x;
        a[n][4 * q + 1] = v.y;
        a[n][4 * q + 2] = v.z;
        a[n][4 * q + 3] = v.w;
      }
    }
    float c[N][R];
#pragma unroll
    for (int n = 0; n < N; ++n) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < J; ++j) acc = fmaf(a[n][j], c_cor[n * J * R + j * R + r], acc);
        c[n][r] = acc;
      }
    }
#pragma unroll
    for (int n = 0; n < N; ++n) {
      float gs[J];
#pragma unroll
      for (int j = 0; j < J; ++j) gs[j] = 0.f;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float w = 1.f;
#pragma unroll
        for (int n0 = 0; n0 < N; ++n0)
          if (n0 != n) w *= c[n0][r];
#pragma unroll
        for (int j = 0; j < J; ++j) gs[j] = fmaf(w, c_cor[n * J * R + j * R + r], gs[j]);
      }
      float inter = 0.f;
#pragma unroll
      for (int j = 0; j < J; ++j) inter = fmaf(a[n][j], gs[j], inter);
      const float gm = p.gam[n], lm = p.lam[n];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        float g = -x * gs[j] + lm * a[n][j] + inter * gs[j];
        a[n][j] -= gm * g;
      }
      float4* dst = reinterpret_cast<float4*>(fac + p.foff[n] + (long long)idx[n] * J);
#pragma unroll
      for (int q = 0; q < J / 4; ++q)
        __stcg(dst + q, make_float4(a[n][4 * q], a[n][4 * q + 1], a[n][4 * q + 2], a[n][4 * q + 3]));
      if (n < N - 1) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float acc = 0.f;
#pragma unroll
          for (int j = 0; j < J; ++j) acc = fmaf(a[n][j], c_cor[n * J * R + j * R + r], acc);
          c[n][r] = acc;
        }
      }
    }
  }
}

// ----------------------------------------------------------------------------
// factor_fma_kernel<N,J>: thread per sample on the CUDA cores (J = R), the
// tcgen05 kernels' Hogwild semantics (hot modes written as red.add deltas)
// with no tensor rounds or barriers: every thread runs its own sample's
// whole chain, so the SM's warps are independent.  B(n) sits in shared
// memory row-major (J x R) and is read as float4 broadcasts (4 FMAs per
// load); per sample (3N-1) J R FMAs (the c_n refresh recomputed from the
// updated row).  Records one sample ahead, visit entries two ahead.
// ----------------------------------------------------------------------------
// (a compiler-only memory barrier per row step: without it the fully unrolled
// loops hoist all N*J*R/4 shared loads of B to the top and spill)
#define SPTK_NO_HOIST() asm volatile("" ::: "memory")

template <int N, int J, bool HV>
__global__ void __launch_bounds__(128, (J <= 4 ? 8 : (J <= 8 ? 4 : 3)))
    factor_fma_kernel(const int* __restrict__ rec, const int* __restrict__ visit, long long n_visit, long long base,
                      float* __restrict__ fac, const float* __restrict__ cor, TpsParams<N> p, unsigned hot) {
  constexpr int R = J, RW = N <= 3 ? 4 : 8;
  __shared__ __align__(16) float Bs[N * J * R];  // B_n row-major (J x R)
  __shared__ __align__(16) float Bt[N * R * J];  // B_n^T (R x J)
  for (int i = threadIdx.x; i < N * J * R; i += blockDim.x) {
    const int n = i / (J * R), rem = i % (J * R), j = rem / R, r = rem % R;
    Bs[i] = cor[i];
    Bt[(n * R + r) * J + j] = cor[i];
  }
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long k0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  auto vis = [&](long long k) -> long long {
    const long long kc = k < n_visit ? k : n_visit - 1;
    return base + (HV ? (long long)__ldg(visit + kc) : kc);
  };
  long long v_next = vis(k0 + stride);
  int4 w0 = make_int4(0, 0, 0, 0), w1 = w0;
  tps_load_rec<RW>(rec, vis(k0), w0, w1);
  for (long long k = k0; k < n_visit; k += stride) {
    const int wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    int idx[N];
#pragma unroll
    for (int n = 0; n < N; ++n) idx[n] = wv[n];
    const float x = __int_as_float(wv[N]);
    tps_load_rec<RW>(rec, v_next, w0, w1);
    v_next = vis(k + 2 * stride);
    float a[N][J];
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const float4* src = reinterpret_cast<const float4*>(fac + p.foff[n] + (long long)idx[n] * J);
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
        const float4 v = __ldcg(src + q);
        a[n][4 * q] = v.x;
        a[n][4 * q + 1] = v.y;
        a[n][4 * q + 2] = v.z;
        a[n][4 * q + 3] = v.w;
      }
    }
    // c_n = a_n . B_n
    float c[N][R];
#pragma unroll
    for (int n = 0; n < N; ++n) {
#pragma unroll
      for (int r = 0; r < R; ++r) c[n][r] = 0.f;
#pragma unroll
      for (int j = 0; j < J; ++j)
#pragma unroll
        for (int r4 = 0; r4 < R / 4; ++r4) {
          const float4 b = *reinterpret_cast<const float4*>(Bs + (n * J + j) * R + 4 * r4);
          c[n][4 * r4] = fmaf(a[n][j], b.x, c[n][4 * r4]);
          c[n][4 * r4 + 1] = fmaf(a[n][j], b.y, c[n][4 * r4 + 1]);
          c[n][4 * r4 + 2] = fmaf(a[n][j], b.z, c[n][4 * r4 + 2]);
          c[n][4 * r4 + 3] = fmaf(a[n][j], b.w, c[n][4 * r4 + 3]);
          if (r4 == R / 4 - 1) SPTK_NO_HOIST();
        }
    }
#pragma unroll
    for (int n = 0; n < N; ++n) {
      // gs_j = sum_r W_r B_n[j][r] with W_r = prod_{n0 != n} c_n0[r] formed per
      // r (B_n^T rows: 4 j per load); inter = a . gs
      float gs[J];
#pragma unroll
      for (int j = 0; j < J; ++j) gs[j] = 0.f;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float wr = 1.f;
#pragma unroll
        for (int n0 = 0; n0 < N; ++n0)
          if (n0 != n) wr *= c[n0][r];
#pragma unroll
        for (int j4 = 0; j4 < J / 4; ++j4) {
          const float4 b = *reinterpret_cast<const float4*>(Bt + (n * R + r) * J + 4 * j4);
          gs[4 * j4] = fmaf(wr, b.x, gs[4 * j4]);
          gs[4 * j4 + 1] = fmaf(wr, b.y, gs[4 * j4 + 1]);
          gs[4 * j4 + 2] = fmaf(wr, b.z, gs[4 * j4 + 2]);
          gs[4 * j4 + 3] = fmaf(wr, b.w, gs[4 * j4 + 3]);
        }
        SPTK_NO_HOIST();
      }
      float inter = 0.f;
#pragma unroll
      for (int j = 0; j < J; ++j) inter = fmaf(a[n][j], gs[j], inter);
      const float gm = p.gam[n], lm = p.lam[n];
      const bool red = hot >> n & 1u;
      float4* dst = reinterpret_cast<float4*>(fac + p.foff[n] + (long long)idx[n] * J);
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
        float d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * q + u;
          const float g = -x * gs[j] + lm * a[n][j] + inter * gs[j];
          d[u] = -gm * g;
          a[n][j] += d[u];
        }
        if (red)
          atomicAdd(dst + q, make_float4(d[0], d[1], d[2], d[3]));
        else
          __stcg(dst + q, make_float4(a[n][4 * q], a[n][4 * q + 1], a[n][4 * q + 2], a[n][4 * q + 3]));
      }
      if (n < N - 1) {
#pragma unroll
        for (int r = 0; r < R; ++r) c[n][r] = 0.f;
#pragma unroll
        for (int j = 0; j < J; ++j)
#pragma unroll
          for (int r4 = 0; r4 < R / 4; ++r4) {
            const float4 b = *reinterpret_cast<const float4*>(Bs + (n * J + j) * R + 4 * r4);
            c[n][4 * r4] = fmaf(a[n][j], b.x, c[n][4 * r4]);
            c[n][4 * r4 + 1] = fmaf(a[n][j], b.y, c[n][4 * r4 + 1]);
            c[n][4 * r4 + 2] = fmaf(a[n][j], b.z, c[n][4 * r4 + 2]);
            c[n][4 * r4 + 3] = fmaf(a[n][j], b.w, c[n][4 * r4 + 3]);
            if (r4 == R / 4 - 1) SPTK_NO_HOIST();
          }
      }
    }
  }
}

// ----------------------------------------------------------------------------
// warp per sample (generic ranks, J <= 64, R <= 64), Hogwild
// ----------------------------------------------------------------------------
struct GamLam {
  double gam[SPTK_MAX_MODES];
  double lam[SPTK_MAX_MODES];
};

template <typename T>
__global__ void __launch_bounds__(256) factor_wps_kernel(const int* __restrict__ rec, int rw, int vo,
                                                         const int* __restrict__ visit, long long n_visit,
                                                         long long base, T* __restrict__ fac,
                                                         const T* __restrict__ cor, ModelDesc md, GamLam gl,
                                                         int scratch_per_warp) {
  extern __shared__ unsigned char smem_raw[];
  T* Bs = reinterpret_cast<T*>(smem_raw);
  for (int i = threadIdx.x; i < md.cor_size; i += blockDim.x) Bs[i] = cor[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int N = md.n_modes, R = md.rcore;
  T* scr = Bs + ((md.cor_size + 3) & ~3) + wib * scratch_per_warp;
  int aoff[SPTK_MAX_MODES];
  int tot = 0;
  for (int n = 0; n < N; ++n) {
    aoff[n] = tot;
    tot += md.jr[n];
  }
  T* a_s = scr;                // sum J
  T* c_s = scr + tot;          // N*R
  T* w_s = c_s + N * R;        // R
  T* g_s = w_s + R;            // max J
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long k = blockIdx.x * (long long)(blockDim.x >> 5) + wib; k < n_visit; k += nwarps) {
    const long long ri = base + (visit ? (long long)__ldg(visit + k) : k);
    const int* rp = rec + ri * rw;
    const T x = load_val<T>(rp, vo);
    for (int n = 0; n < N; ++n) {
      const int J = md.jr[n];
      const T* row = fac + md.foff[n] + (long long)__ldg(rp + n) * J;
      for (int j = lane; j < J; j += 32) a_s[aoff[n] + j] = __ldcg(row + j);
    }
    __syncwarp();
    for (int n0 = 0; n0 < N; ++n0) {
      const int J = md.jr[n0];
      for (int r = lane; r < R; r += 32) {
        T acc = 0;
        for (int j = 0; j < J; ++j) acc += a_s[aoff[n0] + j] * Bs[md.coff[n0] + j * R + r];
        c_s[n0 * R + r] = acc;
      }
    }
    __syncwarp();
    for (int n = 0; n < N; ++n) {
      const int J = md.jr[n];
      for (int r = lane; r < R; r += 32) {
        T w = 1;
        for (int n0 = 0; n0 < N; ++n0)
          if (n0 != n) w *= c_s[n0 * R + r];
        w_s[r] = w;
      }
      __syncwarp();
      T part = 0;
      for (int j = lane; j < J; j += 32) {
        T g = 0;
        for (int r = 0; r < R; ++r) g += w_s[r] * Bs[md.coff[n] + j * R + r];
        g_s[j] = g;
        part += a_s[aoff[n] + j] * g;
      }
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      const T inter = part;
      const T gm = (T)gl.gam[n], lm = (T)gl.lam[n];
      T* row = fac + md.foff[n] + (long long)__ldg(rp + n) * J;
      for (int j = lane; j < J; j += 32) {
        T av = a_s[aoff[n] + j];
        T gsj = g_s[j];
        T g = -x * gsj + lm * av + inter * gsj;
        av -= gm * g;
        a_s[aoff[n] + j] = av;
        __stcg(row + j, av);
      }
      __syncwarp();
      if (n < N - 1) {
        for (int r = lane; r < R; r += 32) {
          T acc = 0;
          for (int j = 0; j < J; ++j) acc += a_s[aoff[n] + j] * Bs[md.coff[n] + j * R + r];
          c_s[n * R + r] = acc;
        }
      }
      __syncwarp();
    }
  }
}

// ----------------------------------------------------------------------------
// sequential, exact reference operation order (no FMA contraction)
// ----------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

// One CTA walks the visit list in order.  Each step takes the next CAND
// samples, finds the longest prefix whose samples touch pairwise-distinct rows
// in every mode (__match_any_sync per mode), and updates that prefix in
// parallel, one thread per sample.  Samples in such a prefix commute exactly,
// so the result equals the strictly sequential reference loop, while ~sqrt(I)
// samples run concurrently.  Per-sample arithmetic follows _loops.py:31-62
// operation for operation, with no FMA contraction.
template <typename T>
__global__ void __launch_bounds__(32) factor_seq_kernel(const int* __restrict__ rec, int rw, int vo,
                                                        const int* __restrict__ visit, long long n_visit,
                                                        long long base, T* __restrict__ fac,
                                                        const T* __restrict__ cor, ModelDesc md, GamLam gl,
                                                        int cand, int per_thread) {
  extern __shared__ unsigned char smem_raw[];
  T* Bs = reinterpret_cast<T*>(smem_raw);
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < md.cor_size; i += 32) Bs[i] = cor[i];
  const int N = md.n_modes, R = md.rcore;
  int aoff[SPTK_MAX_MODES];
  int tot = 0;
  for (int n = 0; n < N; ++n) {
    aoff[n] = tot;
    tot += md.jr[n];
  }
  T* my = Bs + ((md.cor_size + 1) & ~1) + (size_t)lane * per_thread;
  T* a_s = my;             // sum J
  T* c_s = a_s + tot;      // N*R
  T* g_s = c_s + N * R;    // max J
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  long long pos = 0;
  while (pos < n_visit) {
    const long long k = pos + lane;
    const bool valid = lane < cand && k < n_visit;
    const int* rp = nullptr;
    unsigned conflict = 0;
    if (valid) rp = rec + (base + (visit ? (long long)visit[k] : k)) * rw;
    for (int n = 0; n < N; ++n) {
      int row = valid ? rp[n] : -1 - lane;
      unsigned peers = __match_any_sync(0xffffffffu, row);
      if (peers & lt) conflict |= 1u;
    }
    unsigned cm = __ballot_sync(0xffffffffu, conflict || !valid);
    int P = cm ? __ffs(cm) - 1 : 32;
    if (P == 0) P = 1;  // cannot happen for a valid lane 0; keeps progress
    if (lane < P && valid) {
      const T x = load_val<T>(rp, vo);
      for (int n = 0; n < N; ++n) {
        const int J = md.jr[n];
        volatile const T* row = fac + md.foff[n] + (long long)rp[n] * J;
        for (int j = 0; j < J; ++j) a_s[aoff[n] + j] = row[j];
      }
      for (int n0 = 0; n0 < N; ++n0) {
        const int J = md.jr[n0];
        for (int r = 0; r < R; ++r) {
          T acc = 0;
          for (int j = 0; j < J; ++j) acc = add_rn(acc, mul_rn(a_s[aoff[n0] + j], Bs[md.coff[n0] + j * R + r]));
          c_s[n0 * R + r] = acc;
        }
      }
      for (int n = 0; n < N; ++n) {
        const int J = md.jr[n];
        for (int j = 0; j < J; ++j) g_s[j] = 0;
        for (int r = 0; r < R; ++r) {
          T w = 1;
          for (int n0 = 0; n0 < N; ++n0)
            if (n0 != n) w = mul_rn(w, c_s[n0 * R + r]);
          for (int j = 0; j < J; ++j) g_s[j] = add_rn(g_s[j], mul_rn(w, Bs[md.coff[n] + j * R + r]));
        }
        T inter = 0;
        for (int j = 0; j < J; ++j) inter = add_rn(inter, mul_rn(a_s[aoff[n] + j], g_s[j]));
        const T gm = (T)gl.gam[n], lm = (T)gl.lam[n];
        T* row = fac + md.foff[n] + (long long)rp[n] * J;
        for (int j = 0; j < J; ++j) {
          T av = a_s[aoff[n] + j];
          T g = add_rn(add_rn(mul_rn(-x, g_s[j]), mul_rn(lm, av)), mul_rn(inter, g_s[j]));
          av = add_rn(av, -mul_rn(gm, g));
          a_s[aoff[n] + j] = av;
          row[j] = av;
        }
        if (n < N - 1) {
          for (int r = 0; r < R; ++r) {
            T acc = 0;
            for (int j = 0; j < J; ++j) acc = add_rn(acc, mul_rn(a_s[aoff[n] + j], Bs[md.coff[n] + j * R + r]));
            c_s[n * R + r] = acc;
          }
        }
      }
    }
    __threadfence_block();
    __syncwarp();
    pos += P;
  }
}

// ----------------------------------------------------------------------------
// host dispatch
// ----------------------------------------------------------------------------
static bool all_equal_j(const ModelDesc& md, int J) {
  for (int n = 0; n < md.n_modes; ++n)
    if (md.jr[n] != J) return false;
  return true;
}

template <int N, int J, int R>
static int launch_tps(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                      const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s) {
  TpsParams<N> p;
  for (int n = 0; n < N; ++n) {
    p.foff[n] = md.foff[n];
    p.gam[n] = gam[n];
    p.lam[n] = lam[n];
  }
  SPTK_CUDA_TRY(cudaMemcpyToSymbolAsync(c_cor, cor, sizeof(float) * N * J * R, 0, cudaMemcpyDeviceToDevice, s));
  const int threads = 128;
  long long blocks = (n_visit + threads - 1) / threads;
  const long long cap = 148LL * 3 * 8;
  if (blocks > cap) blocks = cap;
  if (blocks > hogwild_cta_cap(n_visit, threads)) blocks = hogwild_cta_cap(n_visit, threads);
  if (blocks < 1) blocks = 1;
  if (rw == 4)
    factor_tps_kernel<N, J, R, 4><<<(unsigned)blocks, threads, 0, s>>>(rec, visit, n_visit, base, fac, p);
  else
    factor_tps_kernel<N, J, R, 8><<<(unsigned)blocks, threads, 0, s>>>(rec, visit, n_visit, base, fac, p);
  note_factor_kernel("factor_tps_kernel");
  SPTK_CHECK_LAUNCH();
  return 0;
}

template <int N, int J>
static int launch_fma(const int* rec, const int* visit, long long n_visit, long long base, float* fac,
                      const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s) {
  TpsParams<N> p;
  for (int n = 0; n < N; ++n) {
    p.foff[n] = md.foff[n];
    p.gam[n] = gam[n];
    p.lam[n] = lam[n];
  }
  // hot modes (fewer than 2^18 rows): red.add deltas, as the tcgen05 kernels
  unsigned hot = 0;
  for (int n = 0; n < N; ++n) {
    const long long end = n + 1 < N ? md.foff[n + 1] : md.fac_size;
    if ((end - md.foff[n]) / J < (1LL << 18)) hot |= 1u << n;
  }
  if (const char* e = getenv("SPTK_ATOMIC_MASK")) hot = (unsigned)strtoul(e, nullptr, 0);
  int per_sm = J <= 4 ? 8 : (J <= 8 ? 4 : 3);
  if (const char* e = getenv("SPTK_TC_CTAS")) per_sm = atoi(e);
  long long blocks = 148LL * per_sm;
  const long long need = (n_visit + 127) / 128;
  if (blocks > need) blocks = need;
  if (blocks > hogwild_cta_cap(n_visit, 128)) blocks = hogwild_cta_cap(n_visit, 128);
  if (blocks < 1) blocks = 1;
  if (visit)
    factor_fma_kernel<N, J, true><<<(unsigned)blocks, 128, 0, s>>>(rec, visit, n_visit, base, fac, cor, p, hot);
  else
    factor_fma_kernel<N, J, false><<<(unsigned)blocks, 128, 0, s>>>(rec, visit, n_visit, base, fac, cor, p, hot);
  note_factor_kernel("factor_fma_kernel");
  SPTK_CHECK_LAUNCH();
  return 0;
}

// tc mode 5: the thread-per-sample CUDA-core kernel with red.add hot modes
static int try_fma(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                   const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s,
                   int* rc) {
  const int N = md.n_modes, R = md.rcore, J = md.jr[0];
  if (!all_equal_j(md, J) || J != R || rw != rec_words(N)) return 0;
  if (N == 3 && J == 16) {
    *rc = launch_fma<3, 16>(rec, visit, n_visit, base, fac, cor, md, gam, lam, s);
    return 1;
  }
  if (N == 3 && J == 8) {
    *rc = launch_fma<3, 8>(rec, visit, n_visit, base, fac, cor, md, gam, lam, s);
    return 1;
  }
  if (N == 3 && J == 4) {
    *rc = launch_fma<3, 4>(rec, visit, n_visit, base, fac, cor, md, gam, lam, s);
    return 1;
  }
  return 0;
}

// Ranks whose throughput factor pass runs on the CUDA-core FMA kernel
// instead of tcgen05 (bit r: J = R = r), from the measured crossover
// (DESIGN.md section 4); SPTK_FMA_RANKS="4,8" style overrides.
static bool fma_rank(int J) {
  static int mask = -1;
  if (mask < 0) {
    mask = 0;
    if (const char* e = getenv("SPTK_FMA_RANKS")) {
      const char* q = e;
      while (*q) {
        const int v = atoi(q);
        if (v > 0 && v < 31) mask |= 1 << v;
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
    }
  }
  return J > 0 && J < 31 && (mask >> J & 1);
}
int fma_rank_policy(int J) { return (get_tc_mode() == 5 || fma_rank(J)) ? 1 : 0; }

// returns 1 if handled (status in *rc), 0 if no specialisation
static int try_tps(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                   const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s,
                   int* rc) {
  const int N = md.n_modes, R = md.rcore, J = md.jr[0];
  if (!all_equal_j(md, J) || J != R) return 0;
  if (rw != rec_words(N)) return 0;
#define SPTK_TPS(NN, JJ)                                                                          \
  if (N == NN && J == JJ) {                                                                       \
    *rc = launch_tps<NN, JJ, JJ>(rec, rw, visit, n_visit, base, fac, cor, md, gam, lam, s);      \
    return 1;                                                                                     \
  }
  SPTK_TPS(3, 4)
  SPTK_TPS(3, 8)
  SPTK_TPS(3, 16)
  SPTK_TPS(4, 4)
  SPTK_TPS(4, 8)
  SPTK_TPS(4, 16)
  SPTK_TPS(6, 4)
  SPTK_TPS(6, 8)
#undef SPTK_TPS
  return 0;
}

template <typename T>
int factor_pass(const int* rec, int rw, const int* visit, long long n_visit, long long base, T* fac,
                const T* cor, const ModelDesc& md, const T* h_gammas, const T* h_lambdas, int mode,
                cudaStream_t s) {
  SPTK_REQUIRE(md.n_modes >= 2 && md.n_modes <= SPTK_MAX_MODES, "factor_pass: bad order %d", md.n_modes);
  if (n_visit <= 0) return 0;
  const bool f64 = sizeof(T) == 8;
  const int vo = rec_val_off(md.n_modes, f64);
  SPTK_REQUIRE(rw == rec_words_t(md.n_modes, f64), "factor_pass: record width %d does not match order %d", rw,
               md.n_modes);
  GamLam gl;
  for (int n = 0; n < md.n_modes; ++n) {
    gl.gam[n] = (double)h_gammas[n];
    gl.lam[n] = (double)h_lambdas[n];
  }
  int jmax = 0, tot = 0;
  for (int n = 0; n < md.n_modes; ++n) {
    jmax = md.jr[n] > jmax ? md.jr[n] : jmax;
    tot += md.jr[n];
  }
  if (mode == 1) {
    int per_thread = tot + md.n_modes * md.rcore + jmax + 2;
    per_thread = (per_thread + 1) & ~1;
    int cand = 32;
    size_t smem = sizeof(T) * ((size_t)((md.cor_size + 1) & ~1) + (size_t)per_thread * 32);
    SPTK_REQUIRE(smem <= 200 * 1024, "factor_pass(sequential): model ranks too large for shared memory");
    auto kfn = factor_seq_kernel<T>;
    SPTK_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kfn<<<1, 32, smem, s>>>(rec, rw, vo, visit, n_visit, base, fac, cor, md, gl, cand, per_thread);
  note_factor_kernel("factor_seq_kernel");
    SPTK_CHECK_LAUNCH();
    return 0;
  }
  if (!f64) {
    int rc = 0;
    if ((get_tc_mode() == 5 || fma_rank(md.jr[0])) &&
        try_fma(rec, rw, visit, n_visit, base, (float*)fac, (const float*)cor, md, (const float*)h_gammas,
                (const float*)h_lambdas, s, &rc))
      return rc;
    if (try_factor_tc(rec, rw, visit, n_visit, base, (float*)fac, (const float*)cor, md, (const float*)h_gammas,
                      (const float*)h_lambdas, s, &rc))
      return rc;
    if (md.cor_size <= CONST_COR_MAX &&
        try_tps(rec, rw, visit, n_visit, base, (float*)fac, (const float*)cor, md, (const float*)h_gammas,
                (const float*)h_lambdas, s, &rc))
      return rc;
  }
  SPTK_REQUIRE(jmax <= 1024 && md.rcore <= 1024, "factor_pass: ranks too large");
  int per_warp = tot + md.n_modes * md.rcore + md.rcore + jmax + 4;
  per_warp = (per_warp + 3) & ~3;
  int warps = 8;
  size_t smem = sizeof(T) * ((size_t)((md.cor_size + 3) & ~3) + (size_t)per_warp * warps);
  while (smem > 200 * 1024 && warps > 1) {
    warps /= 2;
    smem = sizeof(T) * ((size_t)((md.cor_size + 3) & ~3) + (size_t)per_warp * warps);
  }
  SPTK_REQUIRE(smem <= 200 * 1024, "factor_pass: model ranks too large for shared memory");
  auto kfn = factor_wps_kernel<T>;
      SPTK_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  long long blocks = (n_visit + warps - 1) / warps;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks > hogwild_cta_cap(n_visit, warps)) blocks = hogwild_cta_cap(n_visit, warps);
  kfn<<<(unsigned)blocks, 32 * warps, smem, s>>>(rec, rw, vo, visit, n_visit, base, fac, cor, md, gl, per_warp);
  note_factor_kernel("factor_wps_kernel");
  SPTK_CHECK_LAUNCH();
  return 0;
}

template int factor_pass<float>(const int*, int, const int*, long long, long long, float*, const float*,
                                const ModelDesc&, const float*, const float*, int, cudaStream_t);
template int factor_pass<double>(const int*, int, const int*, long long, long long, double*, const double*,
                                 const ModelDesc&, const double*, const double*, int, cudaStream_t);

}  // namespace sptk
