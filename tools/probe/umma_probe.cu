// Standalone probe: one tcgen05.mma kind::tf32 (M=128, N=16, K=8 or 16) with
// known operands, several descriptor conventions; prints max error per variant.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include "../../paper_2204_07104_b200/csrc/tc.cuh"
using namespace sptk;

template <int ROWS>
__device__ int canonA(int row, int k) { return (k >> 2) * (ROWS * 4) + (row >> 3) * 32 + (row & 7) * 4 + (k & 3); }
template <int ROWS>
__device__ int canonB(int row, int k) { return (row >> 3) * (8 * 16) / 4 * 2 + (k >> 2) * 32 + (row & 7) * 4 + (k & 3); }  // alt: K chunks adjacent

__global__ void probe(const float* A, const float* B, float* D, int variant, int K) {
  __shared__ __align__(1024) float sa[128 * 16];
  __shared__ __align__(1024) float sb[16 * 16];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * K; e += 128) {
    int m = e / K, k = e % K;
    int off = (variant & 1) ? ((m >> 3) * (K * 8) + (k >> 2) * 32 + (m & 7) * 4 + (k & 3)) : canonA<128>(m, k);
    sa[off] = A[m * K + k];
  }
  for (int e = tid; e < 16 * K; e += 128) {
    int n = e / K, k = e % K;
    int off = (variant & 1) ? ((n >> 3) * (K * 8) + (k >> 2) * 32 + (n & 7) * 4 + (k & 3)) : canonA<16>(n, k);
    sb[off] = B[n * K + k];
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(&slot, 32);
  tc::fence_async_smem(); tc::fence_before_sync(); __syncthreads(); tc::fence_after_sync();
  uint32_t tb = slot;
  if (tid == 0) {
    uint32_t a = tc::smem_u32(sa), b = tc::smem_u32(sb);
    for (int kk = 0; kk < K / 8; ++kk) {
      uint32_t lboA, sboA, lboB, sboB, aoff, boff;
      if (variant & 1) {  // 8-row groups hold all K chunks contiguously
        lboA = 128; sboA = K * 32; lboB = 128; sboB = K * 32; aoff = kk * 256; boff = kk * 256;
      } else {
        lboA = 128 * 16; sboA = 128; lboB = 16 * 16; sboB = 128; aoff = kk * 2 * 128 * 16; boff = kk * 2 * 16 * 16;
      }
      if (variant & 2) { uint32_t t = lboA; lboA = sboA; sboA = t; t = lboB; lboB = sboB; sboB = t; }
      uint64_t da = tc::smem_desc(a + aoff, lboA, sboA);
      uint64_t db = tc::smem_desc(b + boff, lboB, sboB);
      tc::mma_tf32(tb, da, db, tc::idesc_tf32(128, 16), kk > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  float v[16];
  tc::tmem_ld16(tb + ((uint32_t)(warp * 32) << 16), v);
  for (int j = 0; j < 16; ++j) D[tid * 16 + j] = v[j];
  tc::fence_before_sync(); __syncthreads();
  if (warp == 0) { tc::fence_after_sync(); tc::tmem_dealloc(tb, 32); }
}


// D at column offset 16 (TMEM 64 cols), 3xTF32 split, K=16, random data
__device__ float hi32(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }
__global__ void probe_split(const float* A, const float* B, float* D, int split) {
  __shared__ __align__(1024) float sa[2][128 * 16];
  __shared__ __align__(1024) float sb[2][16 * 16];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  int tid = threadIdx.x, warp = tid >> 5;
  const int K = 16;
  for (int e = tid; e < 128 * K; e += 128) {
    int m = e / K, k = e % K; float v = A[m * K + k]; float h = split ? hi32(v) : v;
    sa[0][canonA<128>(m, k)] = h; sa[1][canonA<128>(m, k)] = v - h;
  }
  for (int e = tid; e < 16 * K; e += 128) {
    int n = e / K, k = e % K; float v = B[n * K + k]; float h = split ? hi32(v) : v;
    sb[0][canonA<16>(n, k)] = h; sb[1][canonA<16>(n, k)] = v - h;
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(&slot, 64);
  tc::fence_async_smem(); tc::fence_before_sync(); __syncthreads(); tc::fence_after_sync();
  uint32_t tb = slot;
  if (tid == 0) {
    for (int kk = 0; kk < 2; ++kk) {
      uint32_t ao = kk * 2 * 2048, bo = kk * 2 * 256;
      uint64_t ah = tc::smem_desc(tc::smem_u32(sa[0]) + ao, 2048, 128), al = tc::smem_desc(tc::smem_u32(sa[1]) + ao, 2048, 128);
      uint64_t bh = tc::smem_desc(tc::smem_u32(sb[0]) + bo, 256, 128), bl = tc::smem_desc(tc::smem_u32(sb[1]) + bo, 256, 128);
      tc::mma_tf32(tb + 16, ah, bh, tc::idesc_tf32(128, 16), kk > 0);
      if (split) { tc::mma_tf32(tb + 16, ah, bl, tc::idesc_tf32(128, 16), 1); tc::mma_tf32(tb + 16, al, bh, tc::idesc_tf32(128, 16), 1); }
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  float v[16];
  tc::tmem_ld16(tb + ((uint32_t)(warp * 32) << 16) + 16, v);
  for (int j = 0; j < 16; ++j) D[tid * 16 + j] = v[j];
  tc::fence_before_sync(); __syncthreads();
  if (warp == 0) { tc::fence_after_sync(); tc::tmem_dealloc(tb, 64); }
}

int main() {
  {
    float *A, *B, *D;
    cudaMallocManaged(&A, 128 * 16 * 4); cudaMallocManaged(&B, 16 * 16 * 4); cudaMallocManaged(&D, 128 * 16 * 4);
    srand(1);
    for (int i = 0; i < 128 * 16; ++i) A[i] = (float)rand() / RAND_MAX - 0.3f;
    for (int i = 0; i < 16 * 16; ++i) B[i] = (float)rand() / RAND_MAX - 0.4f;
    for (int split = 0; split < 2; ++split) {
      probe_split<<<1, 128>>>(A, B, D, split);
      cudaError_t e = cudaDeviceSynchronize();
      double err = 0;
      for (int m = 0; m < 128; ++m) for (int n = 0; n < 16; ++n) {
        double s = 0; for (int k = 0; k < 16; ++k) s += (double)A[m * 16 + k] * B[n * 16 + k];
        double d = fabs(s - D[m * 16 + n]); if (d > err) err = d;
      }
      printf("split=%d col-offset 16, K=16: %s max abs err %.3g\n", split, cudaGetErrorString(e), err);
    }
  }
  for (int K = 8; K <= 16; K += 8) {
    float *A, *B, *D;
    cudaMallocManaged(&A, 128 * 16 * 4); cudaMallocManaged(&B, 16 * 16 * 4); cudaMallocManaged(&D, 128 * 16 * 4);
    for (int m = 0; m < 128; ++m) for (int k = 0; k < K; ++k) A[m * K + k] = (float)((m * 7 + k * 3) % 11) - 5.0f;
    for (int n = 0; n < 16; ++n) for (int k = 0; k < K; ++k) B[n * K + k] = (float)((n * 5 + k * 2) % 7) - 3.0f;
    for (int variant = 0; variant < 2; ++variant) {
      memset(D, 0, 128 * 16 * 4);
      probe<<<1, 128>>>(A, B, D, variant, K);
      cudaError_t e = cudaDeviceSynchronize();
      double err = 0; int bad = 0;
      for (int m = 0; m < 128; ++m) for (int n = 0; n < 16; ++n) {
        double s = 0; for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
        double d = fabs(s - D[m * 16 + n]); if (d > err) err = d; if (d > 1e-3) ++bad;
      }
      printf("K=%d variant %d (%s%s): %s max err %.3g bad %d  D[0..3]=%g %g %g %g\n", K, variant,
             (variant & 1) ? "Kchunks-adjacent" : "Kchunks-strided", (variant & 2) ? ",swapLBO/SBO" : "",
             cudaGetErrorString(e), err, bad, D[0], D[1], D[2], D[3]);
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
