// eval.cu -- K6: predictions and RMSE/MAE sums over a set of nonzeros.
//
// Restates model.py:134-146 (predict_entries: x_hat = sum_r prod_n
// (A(n)[i_n,:] . B(n)[:,r])) and trainer.py:89-102 (rmse / mae), which the
// reference evaluates every eval_every epochs (trainer.py:251-265).
// One thread per nonzero; the core factors B(n) sit in shared memory and are
// read as warp-wide broadcasts, the record is one 16/32-byte load and each
// factor row is read with vector loads.  Residual sums are accumulated in
// fp64 (block reduction + one atomicAdd per block).
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

template <typename T>
int eval(const int* rec, int rw, long long m, const T* fac, const T* cor, const ModelDesc& md, T* pred_out,
         double* sums, cudaStream_t s) {
  SPTK_REQUIRE(md.rcore >= 1 && md.rcore <= 64, "eval: rcore must be in [1, 64]");
  if (m <= 0) return 0;
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
