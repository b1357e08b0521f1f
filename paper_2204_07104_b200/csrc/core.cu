// core.cu -- K4 (core-gradient reduction) and K5 (core apply).
//
// K4 restates _loops.core_pass (_loops.py:66-104): against a frozen model,
//     acc[n][j][r] += (x_hat - x) * (prod_{n0!=n} c[n0,r]) * A(n)[i_n, j]
// summed over the core batch Psi (trainer.py:212-237).  This is a
// [J x |Psi|] . [|Psi| x R] reduction per mode.  Each CTA stages S samples at
// a time in shared memory (phase 1: one thread per sample computes its c table,
// residual and the coefficient vectors v_n[r] = resid * w_n[r]; phase 2: the
// CTA's threads own (n,j,r) outputs and reduce sum_s a_n[s][j] * v_n[s][r]
// over the staged samples), then writes one fp64 partial per CTA.  A second
// kernel sums the partials in CTA order (deterministic, fp64) -- the
// equivalent of the reference's chunk-order merge (trainer.py:238-240).
//
// EXACT = true is the verification mode: one CTA per reference chunk
// (np.array_split of Psi), samples accumulated one at a time in order with
// the reference's operation order and no FMA contraction, so that in fp64 the
// per-chunk accumulators equal the reference's bit for bit.
//
// K5 restates trainer.py:241-247 / core_sgd.py:62-79:
//     B(n) <- B(n) - gamma_b * (acc / denom + lambda_b * B(n)).
#include "common.cuh"
#include "kernels.cuh"

#include <stdlib.h>

namespace sptk {

template <typename T>
__device__ __forceinline__ T cmul(T a, T b);
template <>
__device__ __forceinline__ float cmul<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double cmul<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T cadd(T a, T b);
template <>
__device__ __forceinline__ float cadd<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double cadd<double>(double a, double b) { return __dadd_rn(a, b); }

template <typename T, bool EXACT>
__global__ void __launch_bounds__(256) core_pass_kernel(const int* __restrict__ rec, int rw, int vo,
                                                        const int* __restrict__ visit, const int* __restrict__ map,
                                                        long long n_visit, const T* __restrict__ fac,
                                                        const T* __restrict__ cor, ModelDesc md, int S,
                                                        double* __restrict__ partial, const long long* chunk_lo) {
  extern __shared__ unsigned char smem_raw[];
  T* Bs = reinterpret_cast<T*>(smem_raw);
  const int N = md.n_modes, R = md.rcore, CS = md.cor_size;
  int aoff[SPTK_MAX_MODES];
  int tot = 0;
  for (int n = 0; n < N; ++n) {
    aoff[n] = tot;
    tot += md.jr[n];
  }
  const int NR = N * R;
  T* sa = Bs + ((CS + 3) & ~3);  // [S][tot]
  T* sv = sa + (size_t)S * tot;  // [S][NR]
  T* sc = sv + (size_t)S * NR;   // [S][NR] c tables
  for (int i = threadIdx.x; i < CS; i += blockDim.x) Bs[i] = cor[i];
  double* out = partial + (size_t)blockIdx.x * CS;
  for (int o = threadIdx.x; o < CS; o += blockDim.x) out[o] = 0.0;
  __syncthreads();
  long long k_lo, k_hi, k_step;
  if (EXACT) {
    k_lo = chunk_lo[blockIdx.x];
    k_hi = chunk_lo[blockIdx.x + 1];
    k_step = S;
  } else {
    k_lo = (long long)blockIdx.x * S;
    k_hi = n_visit;
    k_step = (long long)gridDim.x * S;
  }
  for (long long kb = k_lo; kb < k_hi; kb += k_step) {
    const int t = threadIdx.x;
    const long long k = kb + t;
    // phase 1
    if (t < S) {
      T* my_a = sa + (size_t)t * tot;
      T* my_v = sv + (size_t)t * NR;
      T* my_c = sc + (size_t)t * NR;
      if (k < k_hi && (EXACT || k < n_visit)) {
        long long s = visit ? (long long)__ldg(visit + k) : k;
        long long ri = map ? (long long)__ldg(map + s) : s;
        const int* rp = rec + ri * rw;
        const T x = load_val<T>(rp, vo);
        for (int n = 0; n < N; ++n) {
          const int J = md.jr[n];
          const T* row = fac + md.foff[n] + (long long)__ldg(rp + n) * J;
          for (int j = 0; j < J; ++j) my_a[aoff[n] + j] = row[j];
        }
        for (int n0 = 0; n0 < N; ++n0) {
          const int J = md.jr[n0];
          for (int r = 0; r < R; ++r) {
            T dot = 0;
            for (int j = 0; j < J; ++j) dot = cadd(dot, cmul(my_a[aoff[n0] + j], Bs[md.coff[n0] + j * R + r]));
            my_c[n0 * R + r] = dot;
          }
        }
        T xhat = 0;
        for (int r = 0; r < R; ++r) {
          T p = 1;
          for (int n0 = 0; n0 < N; ++n0) p = cmul(p, my_c[n0 * R + r]);
          xhat = cadd(xhat, p);
        }
        const T resid = cadd(xhat, -x);
        for (int n = 0; n < N; ++n)
          for (int r = 0; r < R; ++r) {
            T w = 1;
            for (int n0 = 0; n0 < N; ++n0)
              if (n0 != n) w = cmul(w, my_c[n0 * R + r]);
            my_v[n * R + r] = cmul(resid, w);
          }
      } else {
        for (int i = 0; i < tot; ++i) my_a[i] = 0;
        for (int i = 0; i < NR; ++i) my_v[i] = 0;
      }
    }
    __syncthreads();
    // phase 2: thread owns outputs o; reduce over the staged samples in order
    int nval = S;
    if (kb + S > k_hi) nval = (int)(k_hi - kb);
    for (int o = threadIdx.x; o < CS; o += blockDim.x) {
      int n = 0;
      while (n + 1 < N && o >= md.coff[n + 1]) ++n;
      const int rel = o - md.coff[n];
      const int j = rel / R, r = rel % R;
      if (EXACT) {
        double acc = out[o];
        for (int s2 = 0; s2 < nval; ++s2)
          acc = cadd<double>(acc, cmul<double>((double)sv[(size_t)s2 * NR + n * R + r],
                                               (double)sa[(size_t)s2 * tot + aoff[n] + j]));
        out[o] = acc;
      } else {
        T acc = 0;
        for (int s2 = 0; s2 < nval; ++s2)
          acc += sv[(size_t)s2 * NR + n * R + r] * sa[(size_t)s2 * tot + aoff[n] + j];
        out[o] += (double)acc;
      }
    }
    __syncthreads();
  }
}

// acc[o] += sum_b partial[b][o]: one warp per output, lanes over b, fixed
// shuffle-tree order (deterministic).  Launch with 256-thread blocks.
__global__ void core_reduce_kernel(const double* __restrict__ partial, int nblocks, int CS, double* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  for (int o = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); o < CS; o += gridDim.x * (blockDim.x >> 5)) {
    double t = 0.0;
    for (int b = lane; b < nblocks; b += 32) t += partial[(size_t)b * CS + o];
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) t += __shfl_xor_sync(0xffffffffu, t, k);
    if (lane == 0) acc[o] += t;
  }
}

// total = acc_0 + acc_1 + ... (reference merge order) for the EXACT path
__global__ void core_reduce_ordered_kernel(const double* __restrict__ partial, int nblocks, int CS,
                                           double* __restrict__ acc) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < CS; o += gridDim.x * blockDim.x) {
    double t = partial[o];
    for (int b = 1; b < nblocks; ++b) t = __dadd_rn(t, partial[(size_t)b * CS + o]);
    acc[o] = __dadd_rn(acc[o], t);
  }
}

// ----------------------------------------------------------------------------
// Throughput K4 for uniform ranks (J_n = J for every mode), fp32:
// core_tp_kernel<N,J,R,RW>.  128 threads, 128 samples staged per round.
//   phase 1 (thread <-> sample): gather the N rows (16-byte loads), c[n][r]
//     against B in shared memory (broadcast reads), residual, coefficient
//     rows v_n[r] = resid * prod_{n0!=n} c[n0][r]; a_n and v_n go to the
//     stage as [sample][feature] rows.
//   phase 2 (register-tiled outer products): thread (n, j0..j0+3, r0..r0+3)
//     accumulates sum_s a_n[s][j] * v_n[s][r] over its half of the stage; the
//     two halves and the CTA's rounds are summed in registers, then one fp32
//     partial per CTA (converted to fp64) is written for the ordered reduce.
// Per sample: 4(N+1) record bytes + 4*N*J row bytes (B_c).
// ----------------------------------------------------------------------------
template <int N, int J, int R, int RW>
__global__ void __launch_bounds__(128, 4)
    core_tp_kernel(const int* __restrict__ rec, const int* __restrict__ visit, const int* __restrict__ map,
                   long long n_visit, const float* __restrict__ fac, const float* __restrict__ cor, ModelDesc md,
                   double* __restrict__ partial) {
  constexpr int S = 128;
  constexpr int F = N * J + N * R;  // stage row: a_0..a_{N-1}, v_0..v_{N-1}
  constexpr int FP = F + 4;         // padded row (16-byte aligned, shifts banks)
  constexpr int TJ = J / 4, TR = R / 4, TILES = N * TJ * TR;
  extern __shared__ __align__(16) float smc[];
  float* Bs = smc;                      // N*J*R
  float* st = smc + ((N * J * R + 3) & ~3);  // S x FP
  const int tid = threadIdx.x;
  for (int i = tid; i < N * J * R; i += 128) Bs[i] = cor[i];
  // phase-2 role: TILES <= 64: 64 tile owners x 2 sample halves; otherwise
  // every thread owns NT tiles over the whole stage.
  constexpr int HALVES = TILES <= 64 ? 2 : 1;
  constexpr int OWNERS = 128 / HALVES;
  constexpr int NT = (TILES + OWNERS - 1) / OWNERS;
  const int half = HALVES == 2 ? tid / 64 : 0, tl = HALVES == 2 ? tid % 64 : tid;
  int pn[NT], pj[NT], pr[NT];
  bool p2[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int ti = tl + t * OWNERS;
    p2[t] = ti < TILES;
    const int tt = p2[t] ? ti : 0;
    pn[t] = tt / (TJ * TR);
    const int rem = tt % (TJ * TR);
    pj[t] = 4 * (rem / TR);
    pr[t] = 4 * (rem % TR);
  }
  float acc[NT][4][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[t][u][v] = 0.f;
  __syncthreads();
  for (long long kb = (long long)blockIdx.x * S; kb < n_visit; kb += (long long)gridDim.x * S) {
    const long long k = kb + tid;
    float* row = st + tid * FP;
    if (k < n_visit) {
      const long long s = visit ? (long long)__ldg(visit + k) : k;
      const long long ri = map ? (long long)__ldg(map + s) : s;
      const int* rp = rec + ri * RW;
      int wv[RW];
      {
        const int4 w0 = __ldg(reinterpret_cast<const int4*>(rp));
        wv[0] = w0.x;
        wv[1] = w0.y;
        wv[2] = w0.z;
        wv[3] = w0.w;
        if (RW >= 8) {
          const int4 w1 = __ldg(reinterpret_cast<const int4*>(rp) + 1);
          wv[4 % RW] = w1.x;
          wv[5 % RW] = w1.y;
          wv[6 % RW] = w1.z;
          wv[7 % RW] = w1.w;
        }
      }
      const float x = __int_as_float(wv[N]);
      float c[N][R];
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const float4* src = reinterpret_cast<const float4*>(fac + md.foff[n] + (long long)wv[n] * J);
        float a[J];
#pragma unroll
        for (int q = 0; q < J / 4; ++q) {
          const float4 v = __ldg(src + q);
          a[4 * q] = v.x;
          a[4 * q + 1] = v.y;
          a[4 * q + 2] = v.z;
          a[4 * q + 3] = v.w;
          *reinterpret_cast<float4*>(row + n * J + 4 * q) = v;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) c[n][r] = 0.f;
#pragma unroll
        for (int j = 0; j < J; ++j) {
#pragma unroll
          for (int q = 0; q < R / 4; ++q) {
            const float4 b = *reinterpret_cast<const float4*>(Bs + n * J * R + j * R + 4 * q);
            c[n][4 * q] = fmaf(a[j], b.x, c[n][4 * q]);
            c[n][4 * q + 1] = fmaf(a[j], b.y, c[n][4 * q + 1]);
            c[n][4 * q + 2] = fmaf(a[j], b.z, c[n][4 * q + 2]);
            c[n][4 * q + 3] = fmaf(a[j], b.w, c[n][4 * q + 3]);
          }
        }
      }
      float xhat = 0.f;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float pr_ = c[0][r];
#pragma unroll
        for (int n = 1; n < N; ++n) pr_ *= c[n][r];
        xhat += pr_;
      }
      const float resid = xhat - x;
#pragma unroll
      for (int n = 0; n < N; ++n)
#pragma unroll
        for (int q = 0; q < R / 4; ++q) {
          float w4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float w = resid;
#pragma unroll
            for (int n0 = 0; n0 < N; ++n0)
              if (n0 != n) w *= c[n0][4 * q + u];
            w4[u] = w;
          }
          *reinterpret_cast<float4*>(row + N * J + n * R + 4 * q) = make_float4(w4[0], w4[1], w4[2], w4[3]);
        }
    } else {
#pragma unroll
      for (int q = 0; q < F / 4; ++q) *reinterpret_cast<float4*>(row + 4 * q) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if (!p2[t]) continue;
#pragma unroll 4
      for (int s2 = half * (S / HALVES); s2 < (half + 1) * (S / HALVES); ++s2) {
        const float* rr = st + s2 * FP;
        const float4 a4 = *reinterpret_cast<const float4*>(rr + pn[t] * J + pj[t]);
        const float4 v4 = *reinterpret_cast<const float4*>(rr + N * J + pn[t] * R + pr[t]);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[t][u][v] = fmaf(av[u], vv[v], acc[t][u][v]);
      }
    }
    __syncthreads();
  }
  // combine the sample halves through the (now idle) stage, write the partial
  float* red = st;
  if (HALVES == 2 && half == 1 && p2[0])
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) red[tl * 16 + u * 4 + v] = acc[0][u][v];
  __syncthreads();
  if (half == 0) {
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if (!p2[t]) continue;
      double* out = partial + (size_t)blockIdx.x * md.cor_size + md.coff[pn[t]];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          out[(pj[t] + u) * R + pr[t] + v] =
              (double)acc[t][u][v] + (HALVES == 2 ? (double)red[tl * 16 + u * 4 + v] : 0.0);
    }
  }
}

template <int N, int J, int R>
static int launch_core_tp(const int* rec, int rw, const int* visit, const int* map, long long n_visit,
                          const float* fac, const float* cor, const ModelDesc& md, double* acc, void* ws,
                          size_t ws_bytes, cudaStream_t s) {
  constexpr int S = 128, F = N * J + N * R, FP = F + 4;
  const size_t smem = sizeof(float) * (((N * J * R + 3) & ~3) + (size_t)S * FP);
  constexpr int RW = N <= 3 ? 4 : 8;  // rec_words(N); callers check rw
  auto kfn = core_tp_kernel<N, J, R, RW>;
  static bool configured = false;
  if (!configured) {
    SPTK_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  int per_sm = (int)((220 * 1024) / (smem + 1024));
  if (per_sm > 4) per_sm = 4;
  if (per_sm < 1) per_sm = 1;
  long long blocks = (n_visit + S - 1) / S;
  if (blocks > 148LL * per_sm) blocks = 148LL * per_sm;
  SPTK_REQUIRE(ws_bytes >= (size_t)blocks * md.cor_size * sizeof(double), "core_pass: workspace too small");
  double* partial = (double*)ws;
  kfn<<<(unsigned)blocks, 128, smem, s>>>(rec, visit, map, n_visit, fac, cor, md, partial);
  SPTK_CHECK_LAUNCH();
  core_reduce_kernel<<<(md.cor_size + 7) / 8, 256, 0, s>>>(partial, (int)blocks, md.cor_size, acc);
  SPTK_CHECK_LAUNCH();
  return 0;
}

// ----------------------------------------------------------------------------
// Throughput K4 for uniform ranks too wide for a thread-per-sample register
// tile (J = R = 64): core_wide_kernel<N,J,R,RW>.  256 threads, stages of 32
// samples.
//   phase 1: 8 threads per sample (a warp holds 4 samples); thread q gathers
//     J/8 columns of each row into the stage, then computes c_n[s][r] for its
//     R/8 columns against B in shared memory (row values are broadcast reads),
//     the prediction by a fixed-order butterfly over the 8 threads, and
//     v_n[s][r] = resid * prod_{n0!=n} c_n0[s][r] into the stage.
//   phase 2 (as core_tp_kernel): thread owns N*(J/4)*(R/4)/256 4x4 tiles of
//     sum_s a_n[s][j] v_n[s][r], accumulated in registers over the CTA's
//     stages; one fp64-converted partial per CTA for the ordered reduce.
// ----------------------------------------------------------------------------
template <int N, int J, int R, int RW>
__global__ void __launch_bounds__(256, 2)
    core_wide_kernel(const int* __restrict__ rec, const int* __restrict__ visit, const int* __restrict__ map,
                     long long n_visit, const float* __restrict__ fac, const float* __restrict__ cor, ModelDesc md,
                     double* __restrict__ partial) {
  constexpr int S = 32, TPS = 8, RQ = R / TPS, JQ = J / TPS;
  constexpr int F = N * J + N * R, FP = F + 4;
  constexpr int TJ = J / 4, TR = R / 4, TILES = N * TJ * TR, NT = (TILES + 255) / 256;
  static_assert(RQ % 4 == 0 && JQ % 4 == 0, "core_wide: J, R multiples of 32");
  extern __shared__ __align__(16) float smc[];
  float* Bs = smc;                            // N*J*R, row-major B_n[j][r]
  float* st = smc + ((N * J * R + 3) & ~3);  // S x FP
  const int tid = threadIdx.x, lane = tid & 31;
  const int sl = (tid >> 5) * 4 + (lane >> 3), q = lane & 7;  // stage sample, column eighth
  for (int i = tid; i < N * J * R; i += 256) Bs[i] = cor[i];
  int pn[NT], pj[NT], pr[NT];
  bool p2[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int ti = tid + t * 256;
    p2[t] = ti < TILES;
    const int tt = p2[t] ? ti : 0;
    pn[t] = tt / (TJ * TR);
    const int rem = tt % (TJ * TR);
    pj[t] = 4 * (rem / TR);
    pr[t] = 4 * (rem % TR);
  }
  float acc[NT][4][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[t][u][v] = 0.f;
  __syncthreads();
  float* row = st + sl * FP;
  for (long long kb = (long long)blockIdx.x * S; kb < n_visit; kb += (long long)gridDim.x * S) {
    const long long k = kb + sl;
    const bool ok = k < n_visit;
    float x = 0.f;
    if (ok) {
      const long long s = visit ? (long long)__ldg(visit + k) : k;
      const long long ri = map ? (long long)__ldg(map + s) : s;
      const int* rp = rec + ri * RW;
      int wv[RW];
      {
        const int4 w0 = __ldg(reinterpret_cast<const int4*>(rp));
        wv[0] = w0.x;
        wv[1] = w0.y;
        wv[2] = w0.z;
        wv[3] = w0.w;
        if (RW >= 8) {
          const int4 w1 = __ldg(reinterpret_cast<const int4*>(rp) + 1);
          wv[4 % RW] = w1.x;
          wv[5 % RW] = w1.y;
          wv[6 % RW] = w1.z;
          wv[7 % RW] = w1.w;
        }
      }
      x = __int_as_float(wv[N]);
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const float4* src = reinterpret_cast<const float4*>(fac + md.foff[n] + (long long)wv[n] * J + q * JQ);
#pragma unroll
        for (int u = 0; u < JQ / 4; ++u) *reinterpret_cast<float4*>(row + n * J + q * JQ + 4 * u) = __ldg(src + u);
      }
    } else {
#pragma unroll
      for (int n = 0; n < N; ++n)
#pragma unroll
        for (int u = 0; u < JQ / 4; ++u)
          *reinterpret_cast<float4*>(row + n * J + q * JQ + 4 * u) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();
    float c[N][RQ];
#pragma unroll
    for (int n = 0; n < N; ++n) {
#pragma unroll
      for (int r = 0; r < RQ; ++r) c[n][r] = 0.f;
#pragma unroll 8
      for (int j = 0; j < J; ++j) {
        const float a = row[n * J + j];
#pragma unroll
        for (int u = 0; u < RQ / 4; ++u) {
          const float4 b = *reinterpret_cast<const float4*>(Bs + n * J * R + j * R + q * RQ + 4 * u);
          c[n][4 * u] = fmaf(a, b.x, c[n][4 * u]);
          c[n][4 * u + 1] = fmaf(a, b.y, c[n][4 * u + 1]);
          c[n][4 * u + 2] = fmaf(a, b.z, c[n][4 * u + 2]);
          c[n][4 * u + 3] = fmaf(a, b.w, c[n][4 * u + 3]);
        }
      }
    }
    float xhat = 0.f;
#pragma unroll
    for (int r = 0; r < RQ; ++r) {
      float p = c[0][r];
#pragma unroll
      for (int n = 1; n < N; ++n) p *= c[n][r];
      xhat += p;
    }
    xhat += __shfl_xor_sync(0xffffffffu, xhat, 1);
    xhat += __shfl_xor_sync(0xffffffffu, xhat, 2);
    xhat += __shfl_xor_sync(0xffffffffu, xhat, 4);
    const float resid = ok ? xhat - x : 0.f;
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int u = 0; u < RQ / 4; ++u) {
        float w4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float w = resid;
#pragma unroll
          for (int n0 = 0; n0 < N; ++n0)
            if (n0 != n) w *= c[n0][4 * u + e];
          w4[e] = w;
        }
        *reinterpret_cast<float4*>(row + N * J + n * R + q * RQ + 4 * u) = make_float4(w4[0], w4[1], w4[2], w4[3]);
      }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if (!p2[t]) continue;
#pragma unroll 4
      for (int s2 = 0; s2 < S; ++s2) {
        const float* rr = st + s2 * FP;
        const float4 a4 = *reinterpret_cast<const float4*>(rr + pn[t] * J + pj[t]);
        const float4 v4 = *reinterpret_cast<const float4*>(rr + N * J + pn[t] * R + pr[t]);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[t][u][v] = fmaf(av[u], vv[v], acc[t][u][v]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if (!p2[t]) continue;
    double* out = partial + (size_t)blockIdx.x * md.cor_size + md.coff[pn[t]];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) out[(pj[t] + u) * R + pr[t] + v] = (double)acc[t][u][v];
  }
}

template <int N, int J, int R>
static int launch_core_wide(const int* rec, int rw, const int* visit, const int* map, long long n_visit,
                            const float* fac, const float* cor, const ModelDesc& md, double* acc, void* ws,
                            size_t ws_bytes, cudaStream_t s) {
  constexpr int S = 32, F = N * J + N * R, FP = F + 4;
  const size_t smem = sizeof(float) * (((N * J * R + 3) & ~3) + (size_t)S * FP);
  constexpr int RW = N <= 3 ? 4 : 8;
  (void)rw;
  auto kfn = core_wide_kernel<N, J, R, RW>;
  static bool configured = false;
  if (!configured) {
    SPTK_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  int per_sm = (int)((226 * 1024) / (smem + 1024));
  if (per_sm > 2) per_sm = 2;
  if (per_sm < 1) per_sm = 1;
  long long blocks = (n_visit + S - 1) / S;
  if (blocks > 148LL * per_sm) blocks = 148LL * per_sm;
  SPTK_REQUIRE(ws_bytes >= (size_t)blocks * md.cor_size * sizeof(double), "core_pass: workspace too small");
  double* partial = (double*)ws;
  kfn<<<(unsigned)blocks, 256, smem, s>>>(rec, visit, map, n_visit, fac, cor, md, partial);
  SPTK_CHECK_LAUNCH();
  core_reduce_kernel<<<(md.cor_size + 7) / 8, 256, 0, s>>>(partial, (int)blocks, md.cor_size, acc);
  SPTK_CHECK_LAUNCH();
  return 0;
}

// returns 1 if a specialised kernel handled the call
static int try_core_tp(const int* rec, int rw, const int* visit, const int* map, long long n_visit,
                       const float* fac, const float* cor, const ModelDesc& md, double* acc, void* ws,
                       size_t ws_bytes, cudaStream_t s, int* rc) {
  const int N = md.n_modes, J = md.jr[0], R = md.rcore;
  for (int n = 1; n < N; ++n)
    if (md.jr[n] != J) return 0;
  if (J != R || rw != rec_words(N)) return 0;
#define SPTK_CORE_CASE(NN, JJ)                                                                           \
  if (N == NN && J == JJ) {                                                                              \
    *rc = launch_core_tp<NN, JJ, JJ>(rec, rw, visit, map, n_visit, fac, cor, md, acc, ws, ws_bytes, s); \
    return 1;                                                                                            \
  }
  SPTK_CORE_CASE(3, 4)
  SPTK_CORE_CASE(3, 8)
  SPTK_CORE_CASE(3, 16)
  SPTK_CORE_CASE(3, 32)
  SPTK_CORE_CASE(4, 8)
  SPTK_CORE_CASE(4, 16)
  SPTK_CORE_CASE(6, 8)
#undef SPTK_CORE_CASE
  if (N == 3 && J == 64) {
    *rc = launch_core_wide<3, 64, 64>(rec, rw, visit, map, n_visit, fac, cor, md, acc, ws, ws_bytes, s);
    return 1;
  }
  return 0;
}

size_t core_ws_bytes(const ModelDesc& md) {
  // partials for up to 148*4 CTAs
  return (size_t)148 * 4 * md.cor_size * sizeof(double) + 4096;
}

static int pick_S(const ModelDesc& md, size_t elem, int* S_out, size_t* smem_out) {
  int tot = 0;
  for (int n = 0; n < md.n_modes; ++n) tot += md.jr[n];
  const int NR = md.n_modes * md.rcore;
  size_t fixed = elem * (size_t)((md.cor_size + 3) & ~3);
  size_t per = elem * (size_t)(tot + 2 * NR);
  int S = 256;
  while (S > 1 && fixed + per * S > 200 * 1024) S /= 2;
  *S_out = S;
  *smem_out = fixed + per * S;
  return fixed + per * S <= 200 * 1024;
}

template <typename T>
int core_pass(const int* rec, int rw, const int* visit, const int* map, long long n_visit, const T* fac,
              const T* cor, const ModelDesc& md, double* acc, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (n_visit <= 0) return 0;
  const bool f64 = sizeof(T) == 8;
  SPTK_REQUIRE(rw == rec_words_t(md.n_modes, f64), "core_pass: record width mismatch");
  if (!f64 && !getenv("SPTK_CORE_GENERIC")) {
    int rc = 0;
    if (try_core_tp(rec, rw, visit, map, n_visit, (const float*)fac, (const float*)cor, md, acc, ws, ws_bytes, s,
                    &rc))
      return rc;
  }
  int S;
  size_t smem;
  SPTK_REQUIRE(pick_S(md, sizeof(T), &S, &smem), "core_pass: model ranks too large");
  long long blocks = (n_visit + S - 1) / S;
  if (blocks > 148 * 4) blocks = 148 * 4;
  SPTK_REQUIRE(ws_bytes >= (size_t)blocks * md.cor_size * sizeof(double), "core_pass: workspace too small");
  double* partial = (double*)ws;
  auto kfn = core_pass_kernel<T, false>;
  SPTK_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kfn<<<(unsigned)blocks, 256, smem, s>>>(rec, rw, rec_val_off(md.n_modes, f64), visit, map, n_visit, fac, cor, md, S,
                                           partial, nullptr);
  SPTK_CHECK_LAUNCH();
  core_reduce_kernel<<<(md.cor_size + 7) / 8, 256, 0, s>>>(partial, (int)blocks, md.cor_size, acc);
  SPTK_CHECK_LAUNCH();
  return 0;
}

// Verification mode: chunk boundaries follow np.array_split(psi, n_chunks),
// each chunk's accumulator is the sample-ordered sum of _loops.py:92-103 and
// the chunks are merged in chunk order (trainer.py:238-240).  The per-sample
// terms are independent, only the sums are ordered, so the pass runs in
// segments of EXACT_SEG samples: phase 1 (every SM, one thread per sample)
// writes each sample's coefficient row v = resid * prod_{n0 != n} c[n0] and
// its factor rows a to a scratch table, phase 2 (one thread per (chunk,
// output)) extends that output's running sum over the segment's samples in
// order.  Bitwise equal to the one-CTA sequential walk it replaces.
#define EXACT_SEG 32768

template <typename T>
__global__ void __launch_bounds__(128) core_exact_terms_kernel(const int* __restrict__ rec, int rw, int vo,
                                                               const int* __restrict__ visit,
                                                               const int* __restrict__ map, long long k0, int cnt,
                                                               const T* __restrict__ fac, const T* __restrict__ cor,
                                                               ModelDesc md, T* __restrict__ tv, T* __restrict__ ta,
                                                               T* __restrict__ tc) {
  // term tables column-major (column stride EXACT_SEG): a thread's writes of
  // one column are coalesced with its neighbours', and the ordered sums read
  // each output's column as one contiguous stream
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  const int N = md.n_modes, R = md.rcore;
  constexpr long long S = EXACT_SEG;
  int aoff[SPTK_MAX_MODES];
  int tot = 0;
  for (int n = 0; n < N; ++n) {
    aoff[n] = tot;
    tot += md.jr[n];
  }
  T* my_a = ta + i;
  T* my_v = tv + i;
  T* my_c = tc + i;
  const long long k = k0 + i;
  const long long sid = visit ? (long long)__ldg(visit + k) : k;
  const long long ri = map ? (long long)__ldg(map + sid) : sid;
  const int* rp = rec + ri * rw;
  const T x = load_val<T>(rp, vo);
  for (int n = 0; n < N; ++n) {
    const int J = md.jr[n];
    const T* row = fac + md.foff[n] + (long long)__ldg(rp + n) * J;
    for (int j = 0; j < J; ++j) my_a[(aoff[n] + j) * S] = row[j];
  }
  for (int n0 = 0; n0 < N; ++n0) {
    const int J = md.jr[n0];
    for (int r = 0; r < R; ++r) {
      T dot = 0;
      for (int j = 0; j < J; ++j)
        dot = cadd(dot, cmul(my_a[(aoff[n0] + j) * S], __ldg(cor + md.coff[n0] + j * R + r)));
      my_c[(n0 * R + r) * S] = dot;
    }
  }
  T xhat = 0;
  for (int r = 0; r < R; ++r) {
    T pr = 1;
    for (int n0 = 0; n0 < N; ++n0) pr = cmul(pr, my_c[(n0 * R + r) * S]);
    xhat = cadd(xhat, pr);
  }
  const T resid = cadd(xhat, -x);
  for (int n = 0; n < N; ++n)
    for (int r = 0; r < R; ++r) {
      T w = 1;
      for (int n0 = 0; n0 < N; ++n0)
        if (n0 != n) w = cmul(w, my_c[(n0 * R + r) * S]);
      my_v[(n * R + r) * S] = cmul(resid, w);
    }
}

// One warp per (chunk blockIdx.y, output o): partial[c][o] += the segment's
// terms of chunk c in sample order.  The lanes load 32 consecutive samples'
// factors of the output's two columns (coalesced) and form the 32 products in
// parallel; the ordered sum then takes them one by one (shuffles issued ahead
// of the dependent additions).
template <typename T>
__global__ void __launch_bounds__(128) core_exact_sum_kernel(const T* __restrict__ tv, const T* __restrict__ ta,
                                                             long long k0, int cnt, const long long* __restrict__ lo,
                                                             ModelDesc md, double* __restrict__ partial) {
  const int CS = md.cor_size, c = blockIdx.y, lane = threadIdx.x & 31;
  const int o = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (o >= CS) return;
  long long a = lo[c], z = lo[c + 1];
  a = a > k0 ? a : k0;
  z = z < k0 + cnt ? z : k0 + cnt;
  if (a >= z) return;
  const int N = md.n_modes, R = md.rcore;
  int n = 0, aoffn = 0;
  while (n + 1 < N && o >= md.coff[n + 1]) ++n;
  for (int q = 0; q < n; ++q) aoffn += md.jr[q];
  const int rel = o - md.coff[n], j = rel / R, r = rel - (rel / R) * R;
  const T* pv = tv + (size_t)(n * R + r) * EXACT_SEG;
  const T* pa = ta + (size_t)(aoffn + j) * EXACT_SEG;
  double acc = partial[(size_t)c * CS + o];
  for (long long kb = a; kb < z; kb += 32) {
    const long long kk = kb + lane;
    const bool ok = kk < z;
    const double prod = ok ? cmul<double>((double)pv[kk - k0], (double)pa[kk - k0]) : 0.0;
    const int nk = (int)(z - kb < 32 ? z - kb : 32);
    double ps[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) ps[u] = __shfl_sync(0xffffffffu, prod, u);
#pragma unroll
    for (int u = 0; u < 32; ++u)
      if (u < nk) acc = cadd<double>(acc, ps[u]);
  }
  if (lane == 0) partial[(size_t)c * CS + o] = acc;
}

size_t core_exact_ws_bytes(const ModelDesc& md, int n_chunks) {
  int tot = 0;
  for (int n = 0; n < md.n_modes; ++n) tot += md.jr[n];
  const size_t NR = (size_t)md.n_modes * md.rcore;
  return (size_t)n_chunks * md.cor_size * sizeof(double) + sizeof(long long) * (n_chunks + 2) + 512 +
         (size_t)EXACT_SEG * (2 * NR + tot) * sizeof(double) + 768;
}

template <typename T>
int core_pass_exact(const int* rec, int rw, const int* visit, const int* map, long long n_visit, int n_chunks,
                    const T* fac, const T* cor, const ModelDesc& md, double* acc, void* ws, size_t ws_bytes,
                    cudaStream_t s) {
  if (n_visit <= 0) return 0;
  SPTK_REQUIRE(n_chunks >= 1 && n_chunks <= 1024, "core_pass_exact: bad chunk count");
  const bool f64 = sizeof(T) == 8;
  SPTK_REQUIRE(rw == rec_words_t(md.n_modes, f64), "core_pass_exact: record width mismatch");
  // np.array_split: first (n % k) chunks get one extra element; empty chunks dropped
  long long h_lo[1025];
  long long q = n_visit / n_chunks, rmd = n_visit % n_chunks, pos = 0;
  int nb = 0;
  for (int c = 0; c < n_chunks; ++c) {
    long long len = q + (c < rmd ? 1 : 0);
    if (len == 0) continue;
    h_lo[nb++] = pos;
    pos += len;
  }
  h_lo[nb] = pos;
  SPTK_REQUIRE(ws_bytes >= core_exact_ws_bytes(md, nb), "core_pass_exact: workspace too small");
  int tot = 0;
  for (int n = 0; n < md.n_modes; ++n) tot += md.jr[n];
  const size_t NR = (size_t)md.n_modes * md.rcore;
  char* w = (char*)ws;
  double* partial = (double*)w;
  w += ((size_t)nb * md.cor_size * sizeof(double) + 255) & ~(size_t)255;
  long long* d_lo = (long long*)w;
  w += (sizeof(long long) * (nb + 2) + 255) & ~(size_t)255;
  T* tv = (T*)w;
  w += ((size_t)EXACT_SEG * NR * sizeof(T) + 255) & ~(size_t)255;
  T* tc = (T*)w;
  w += ((size_t)EXACT_SEG * NR * sizeof(T) + 255) & ~(size_t)255;
  T* ta = (T*)w;
  SPTK_CUDA_TRY(cudaMemcpyAsync(d_lo, h_lo, sizeof(long long) * (nb + 1), cudaMemcpyHostToDevice, s));
  SPTK_CUDA_TRY(cudaMemsetAsync(partial, 0, (size_t)nb * md.cor_size * sizeof(double), s));
  const int vo = rec_val_off(md.n_modes, f64);
  for (long long k0 = 0; k0 < n_visit; k0 += EXACT_SEG) {
    const int cnt = (int)(n_visit - k0 < EXACT_SEG ? n_visit - k0 : EXACT_SEG);
    core_exact_terms_kernel<T><<<(cnt + 127) / 128, 128, 0, s>>>(rec, rw, vo, visit, map, k0, cnt, fac, cor, md, tv,
                                                                  ta, tc);
    SPTK_CHECK_LAUNCH();
    core_exact_sum_kernel<T><<<dim3((unsigned)((md.cor_size + 3) / 4), (unsigned)nb), 128, 0, s>>>(
        tv, ta, k0, cnt, d_lo, md, partial);
    SPTK_CHECK_LAUNCH();
  }
  core_reduce_ordered_kernel<<<(md.cor_size + 255) / 256, 256, 0, s>>>(partial, nb, md.cor_size, acc);
  SPTK_CHECK_LAUNCH();
  // (h_lo: a pageable host-to-device cudaMemcpyAsync returns once the source
  // has been staged, so the next call may overwrite it)
  return 0;
}

template <typename T>
__global__ void core_apply_kernel(T* __restrict__ cor, const double* __restrict__ acc, int CS, double gamma_b,
                                  double lambda_b, double denom) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < CS; o += gridDim.x * blockDim.x) {
    double b = (double)cor[o];
    double upd = __dadd_rn(__ddiv_rn(acc[o], denom), __dmul_rn(lambda_b, b));
    cor[o] = (T)__dadd_rn(b, -__dmul_rn(gamma_b, upd));
  }
}

template <typename T>
int core_apply(T* cor, const double* acc, int cor_size, double gamma_b, double lambda_b, double denom,
               cudaStream_t s) {
  core_apply_kernel<T><<<(cor_size + 255) / 256, 256, 0, s>>>(cor, acc, cor_size, gamma_b, lambda_b, denom);
  SPTK_CHECK_LAUNCH();
  return 0;
}

template int core_pass<float>(const int*, int, const int*, const int*, long long, const float*, const float*,
                              const ModelDesc&, double*, void*, size_t, cudaStream_t);
template int core_pass<double>(const int*, int, const int*, const int*, long long, const double*, const double*,
                               const ModelDesc&, double*, void*, size_t, cudaStream_t);
template int core_pass_exact<float>(const int*, int, const int*, const int*, long long, int, const float*,
                                    const float*, const ModelDesc&, double*, void*, size_t, cudaStream_t);
template int core_pass_exact<double>(const int*, int, const int*, const int*, long long, int, const double*,
                                     const double*, const ModelDesc&, double*, void*, size_t, cudaStream_t);
template int core_apply<float>(float*, const double*, int, double, double, double, cudaStream_t);
template int core_apply<double>(double*, const double*, int, double, double, double, cudaStream_t);

}  // namespace sptk
