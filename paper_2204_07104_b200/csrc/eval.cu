// eval.cu -- K6: predictions and RMSE/MAE sums over a set of nonzeros.
//
// Restates model.py:134-146 (predict_entries: x_hat = sum_r prod_n
// (A(n)[i_n,:] . B(n)[:,r])) and trainer.py:89-102 (rmse / mae), which the
// reference evaluates every eval_every epochs (trainer.py:251-265).
// One thread per nonzero; the core factors B(n) sit in shared memory and are
// read as warp-wide broadcasts, the record is one 16/32-byte load and each
// factor row is read with vector loads.  Residual sums are accumulated in
// fp64 (block reduction + one atomicAdd per block).
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace sptk {

template <typename T, int RT>
__global__ void __launch_bounds__(256) eval_kernel(const int* __restrict__ rec, int rw, long long m,
                                                   const T* __restrict__ fac, const T* __restrict__ cor,
                                                   ModelDesc md, T* __restrict__ pred_out,
                                                   double* __restrict__ sums) {
  extern __shared__ unsigned char smem_raw[];
  T* Bs = reinterpret_cast<T*>(smem_raw);
  for (int i = threadIdx.x; i < md.cor_size; i += blockDim.x) Bs[i] = cor[i];
  __syncthreads();
  const int R = RT > 0 ? RT : md.rcore;
  const int N = md.n_modes;
  double sq = 0.0, ab = 0.0;
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (; e < m; e += stride) {
    const int* rp = rec + e * rw;
    T prod[RT > 0 ? RT : 64];
#pragma unroll
    for (int r = 0; r < (RT > 0 ? RT : 64); ++r) prod[r] = T(1);
    for (int n = 0; n < N; ++n) {
      const int J = md.jr[n];
      const T* arow = fac + md.foff[n] + (long long)__ldg(rp + n) * J;
      const T* B = Bs + md.coff[n];
      T c[RT > 0 ? RT : 64];
#pragma unroll
      for (int r = 0; r < (RT > 0 ? RT : 64); ++r) c[r] = T(0);
      for (int j = 0; j < J; ++j) {
        T a = arow[j];
#pragma unroll
        for (int r = 0; r < (RT > 0 ? RT : 64); ++r)
          if (RT > 0 || r < R) c[r] += a * B[j * R + r];
      }
#pragma unroll
      for (int r = 0; r < (RT > 0 ? RT : 64); ++r)
        if (RT > 0 || r < R) prod[r] *= c[r];
    }
    T xh = T(0);
#pragma unroll
    for (int r = 0; r < (RT > 0 ? RT : 64); ++r)
      if (RT > 0 || r < R) xh += prod[r];
    if (pred_out) pred_out[e] = xh;
    if (sums) {
      T x = load_val<T>(rp, rec_val_off(N, sizeof(T) == 8));
      double d = (double)x - (double)xh;
      sq += d * d;
      ab += fabs(d);
    }
  }
  if (sums) {
    for (int o = 16; o > 0; o >>= 1) {
      sq += __shfl_xor_sync(0xffffffffu, sq, o);
      ab += __shfl_xor_sync(0xffffffffu, ab, o);
    }
    __shared__ double red[2][32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
      red[0][w] = sq;
      red[1][w] = ab;
    }
    __syncthreads();
    if (w == 0) {
      int nw = blockDim.x >> 5;
      sq = lane < nw ? red[0][lane] : 0.0;
      ab = lane < nw ? red[1][lane] : 0.0;
      for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        ab += __shfl_xor_sync(0xffffffffu, ab, o);
      }
      if (lane == 0) {
        atomicAdd(&sums[0], sq);
        atomicAdd(&sums[1], ab);
      }
    }
  }
}

// fp64 block reduction of (sq, ab) and one atomicAdd per block
__device__ __forceinline__ void eval_block_sums(double sq, double ab, double* sums) {
  for (int o = 16; o > 0; o >>= 1) {
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
    ab += __shfl_xor_sync(0xffffffffu, ab, o);
  }
  __shared__ double red[2][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][w] = sq;
    red[1][w] = ab;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    sq = lane < nw ? red[0][lane] : 0.0;
    ab = lane < nw ? red[1][lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      sq += __shfl_xor_sync(0xffffffffu, sq, o);
      ab += __shfl_xor_sync(0xffffffffu, ab, o);
    }
    if (lane == 0) {
      atomicAdd(&sums[0], sq);
      atomicAdd(&sums[1], ab);
    }
  }
}

// Uniform ranks (J_n = R for every mode, fp32): a thread scores E entries
// (e, e + stride, ...) at a time, their factor rows read as float4 loads, B(n)
// from shared memory as float4 broadcasts that each feed 4E FMAs.  The
// one-entry version (four FMAs per broadcast) was bound by those broadcasts:
// NF train + test RMSE 7.45 -> 5.45 ms per epoch at E = 2, 5.06 at E = 4
// (ncu); staging the rows through shared memory instead made it slower.
template <int N, int J, int RW, int E, int MINB>
__global__ void __launch_bounds__(256, MINB) eval_pair_kernel(const int* __restrict__ rec, long long m,
                                                           const float* __restrict__ fac,
                                                           const float* __restrict__ cor, ModelDesc md,
                                                           float* __restrict__ pred_out, double* __restrict__ sums) {
  __shared__ __align__(16) float Bs[N * J * J];
  for (int i = threadIdx.x; i < N * J * J; i += blockDim.x) Bs[i] = cor[i];
  __syncthreads();
  double sq = 0.0, ab = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m; e += E * stride) {
    int w[E][8];
    bool ok[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const long long ek = e + k * stride;
      ok[k] = ek < m;
      const long long ee = ok[k] ? ek : e;
      const int4 a0 = __ldg(reinterpret_cast<const int4*>(rec + ee * RW));
      w[k][0] = a0.x, w[k][1] = a0.y, w[k][2] = a0.z, w[k][3] = a0.w;
      if (RW >= 8) {
        const int4 a1 = __ldg(reinterpret_cast<const int4*>(rec + ee * RW) + 1);
        w[k][4] = a1.x, w[k][5] = a1.y, w[k][6] = a1.z, w[k][7] = a1.w;
      }
    }
    float p[E][J];
#pragma unroll
    for (int n = 0; n < N; ++n) {
      float4 rr[E][J / 4];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const float4* src = reinterpret_cast<const float4*>(fac + md.foff[n] + (long long)w[k][n] * J);
#pragma unroll
        for (int q = 0; q < J / 4; ++q) rr[k][q] = __ldg(src + q);
      }
      float c[E][J];
#pragma unroll
      for (int k = 0; k < E; ++k)
#pragma unroll
        for (int r = 0; r < J; ++r) c[k][r] = 0.f;
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * q + u;
#pragma unroll
          for (int r4 = 0; r4 < J / 4; ++r4) {
            const float4 b = *reinterpret_cast<const float4*>(Bs + (n * J + j) * J + 4 * r4);
#pragma unroll
            for (int k = 0; k < E; ++k) {
              const float av = u == 0 ? rr[k][q].x : u == 1 ? rr[k][q].y : u == 2 ? rr[k][q].z : rr[k][q].w;
              c[k][4 * r4] = fmaf(av, b.x, c[k][4 * r4]);
              c[k][4 * r4 + 1] = fmaf(av, b.y, c[k][4 * r4 + 1]);
              c[k][4 * r4 + 2] = fmaf(av, b.z, c[k][4 * r4 + 2]);
              c[k][4 * r4 + 3] = fmaf(av, b.w, c[k][4 * r4 + 3]);
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < E; ++k)
#pragma unroll
        for (int r = 0; r < J; ++r) p[k][r] = n == 0 ? c[k][r] : p[k][r] * c[k][r];
    }
#pragma unroll
    for (int k = 0; k < E; ++k) {
      float xh = 0.f;
#pragma unroll
      for (int r = 0; r < J; ++r) xh += p[k][r];
      if (ok[k]) {
        if (pred_out) pred_out[e + k * stride] = xh;
        const double d = (double)__int_as_float(w[k][N]) - (double)xh;
        sq += d * d;
        ab += fabs(d);
      }
    }
  }
  if (sums) eval_block_sums(sq, ab, sums);
}

template <int N, int J>
static int launch_eval_uniform(const int* rec, long long m, const float* fac, const float* cor, const ModelDesc& md,
                               float* pred_out, double* sums, cudaStream_t s) {
  constexpr int RW = N <= 3 ? 4 : 8;
  long long blocks = (m + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  // entries per thread (measured at NF, order 3 / J = 16, train + test per
  // epoch: 1 / 2 / 3 / 4 -> 7.45 / 5.45 / 5.6 / 5.06 ms; four need 255
  // registers, one CTA per SM)
  if constexpr (N == 3 && J == 16)
    eval_pair_kernel<N, J, RW, 4, 1><<<(unsigned)blocks, 256, 0, s>>>(rec, m, fac, cor, md, pred_out, sums);
  else
    eval_pair_kernel<N, J, RW, 2, 2><<<(unsigned)blocks, 256, 0, s>>>(rec, m, fac, cor, md, pred_out, sums);
  SPTK_CHECK_LAUNCH();
  return 0;
}

// returns 1 if a specialised kernel handled the call
static int try_eval_uniform(const int* rec, int rw, long long m, const float* fac, const float* cor,
                            const ModelDesc& md, float* pred_out, double* sums, cudaStream_t s, int* rc) {
  const int N = md.n_modes, J = md.jr[0];
  for (int n = 1; n < N; ++n)
    if (md.jr[n] != J) return 0;
  if (J != md.rcore || rw != rec_words(N) || getenv("SPTK_EVAL_GENERIC")) return 0;
#define SPTK_EVAL_U(NN, JJ)                                                          \
  if (N == NN && J == JJ) {                                                          \
    *rc = launch_eval_uniform<NN, JJ>(rec, m, fac, cor, md, pred_out, sums, s);     \
    return 1;                                                                        \
  }
  SPTK_EVAL_U(3, 4)
  SPTK_EVAL_U(3, 8)
  SPTK_EVAL_U(3, 16)
  SPTK_EVAL_U(4, 8)
  SPTK_EVAL_U(4, 16)
  SPTK_EVAL_U(6, 8)
#undef SPTK_EVAL_U
  return 0;
}

template <typename T>
int eval(const int* rec, int rw, long long m, const T* fac, const T* cor, const ModelDesc& md, T* pred_out,
         double* sums, cudaStream_t s) {
  SPTK_REQUIRE(md.rcore >= 1 && md.rcore <= 64, "eval: rcore must be in [1, 64]");
  if (m <= 0) return 0;
  if (sizeof(T) == 4) {
    int rc = 0;
    if (try_eval_uniform(rec, rw, m, (const float*)fac, (const float*)cor, md, (float*)pred_out, sums, s, &rc))
      return rc;
  }
  size_t smem = (size_t)md.cor_size * sizeof(T);
  SPTK_REQUIRE(smem <= 200 * 1024, "eval: core factors too large for shared memory");
  long long blocks = (m + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
#define SPTK_EVAL_CASE(RV)                                                                        \
  case RV: {                                                                                      \
    auto kfn = eval_kernel<T, RV>;                                                                \
    SPTK_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));       \
    kfn<<<(unsigned)blocks, 256, smem, s>>>(rec, rw, m, fac, cor, md, pred_out, sums);             \
    break;                                                                                        \
  }
  switch (md.rcore) {
    SPTK_EVAL_CASE(1)
    SPTK_EVAL_CASE(2)
    SPTK_EVAL_CASE(4)
    SPTK_EVAL_CASE(8)
    SPTK_EVAL_CASE(16)
    SPTK_EVAL_CASE(32)
    default: {
      // generic rank: up to 255 registers per thread (fp64), so 128-thread
      // blocks (256 would need more than the SM's 64K registers)
      auto kfn = eval_kernel<T, 0>;
      // (always: the 1.5 KB of static shared memory counts against the default 48 KB)
      SPTK_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kfn<<<(unsigned)(4 * blocks), 64, smem, s>>>(rec, rw, m, fac, cor, md, pred_out, sums);
    }
  }
#undef SPTK_EVAL_CASE
  SPTK_CHECK_LAUNCH();
  return 0;
}

template int eval<float>(const int*, int, long long, const float*, const float*, const ModelDesc&, float*,
                         double*, cudaStream_t);
template int eval<double>(const int*, int, long long, const double*, const double*, const ModelDesc&,
                          double*, double*, cudaStream_t);

}  // namespace sptk
