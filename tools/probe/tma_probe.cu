// Standalone probe for the TMA-gathered factor kernel's building blocks:
//  T1 tile::gather4 of factor rows into a swizzled (SW32/64/128 for J=8/16/32)
//     K-major slot; each thread reads its row back with the swizzle formula
//  T2 c = A_slot . B on tcgen05 with a swizzled K-major smem descriptor
//  T3 W written to TMEM (tcgen05.st) and used as the A operand (A in TMEM)
//  T4 tile::scatter4 store and add-reduce of the slot rows back to global
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_2204_07104_b200/csrc/tc.cuh"
using namespace sptk;

template <int ROWS>
__device__ int canon(int row, int k) { return (k >> 2) * (ROWS * 4) + (row >> 3) * 32 + (row & 7) * 4 + (k & 3); }

// physical float offset of (row, k) in a swizzled K-major slot with J floats per row
template <int J>
__device__ int swz(int row, int k) {
  constexpr int S = J * 4;                       // row bytes = swizzle span
  constexpr int MASK = S / 16 - 1;               // chunk-index mask
  const int chunk = (k >> 2) ^ (((S * row) >> 7) & MASK);
  return row * J + chunk * 4 + (k & 3);
}

template <int J>
__device__ uint64_t sw_desc(uint32_t saddr) {
  constexpr uint64_t layout = J == 8 ? 6 : J == 16 ? 4 : 2;  // SW32 / SW64 / SW128
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)((8 * J * 4) >> 4) << 32) |
         (1ULL << 46) | (layout << 61);
}

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                                        uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void scatter4(const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                                         uint32_t src, bool add) {
  if (add)
    asm volatile(
        "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, "
        "%5}], [%6];" ::"l"(map),
        "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(src)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
            map),
        "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(src)
        : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void mma_tmemA(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// J = R; B (J x R) row-major in global; rows: 128 indices
template <int J>
__global__ void probe(const __grid_constant__ CUtensorMap src, const __grid_constant__ CUtensorMap dst, const int* rows,
                      const float* B, float* out_rows, float* out_c, float* out_g, int add, float* gdst) {
  constexpr int R = J;
  __shared__ __align__(1024) float slot[128 * J];
  __shared__ __align__(1024) float bt[R * J];   // B^T as the N x K operand of c = A B
  __shared__ __align__(1024) float bn[J * R];   // B as the N x K operand of g = W B^T
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < J * R; e += 128) {
    const int j = e / R, r = e % R;
    bt[canon<R>(r, j)] = B[e];
    bn[canon<J>(j, r)] = B[e];
  }
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tslot, 128);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tb = tslot, tl = tb + ((uint32_t)(warp * 32) << 16);
  const uint32_t sbase = tc::smem_u32(slot);
  // T1: gather -- lanes 4k of every warp issue one gather4 for rows 4k..4k+3 of the warp
  if (tid == 0) expect_tx(&bar[0], 128 * J * 4);
  __syncthreads();
  const int me = rows[tid];
  const int r1 = __shfl_down_sync(~0u, me, 1), r2 = __shfl_down_sync(~0u, me, 2), r3 = __shfl_down_sync(~0u, me, 3);
  if ((lane & 3) == 0) gather4(sbase + tid * J * 4, &src, 0, me, r1, r2, r3, tc::smem_u32(&bar[0]));
  tc::mbar_wait(&bar[0], 0);
  for (int k = 0; k < J; ++k) out_rows[tid * J + k] = slot[swz<J>(tid, k)];
  // T2: c = A B
  tc::fence_before_sync();
  __syncthreads();
  if (tid == 0) {
    tc::fence_after_sync();
    for (int kk = 0; kk < J / 8; ++kk) {
      const uint64_t ad = sw_desc<J>(sbase + kk * 32);
      const uint64_t bd = tc::smem_desc(tc::smem_u32(bt) + kk * 2 * (R * 16), R * 16, 128);
      tc::mma_tf32(tb, ad, bd, tc::idesc_tf32(128, R), kk > 0);
    }
    tc::mma_commit(&bar[1]);
  }
  tc::mbar_wait(&bar[1], 0);
  tc::fence_after_sync();
  float c[R];
  tc::tmem_ldh<R>(tl, c);
  for (int r = 0; r < R; ++r) out_c[tid * R + r] = c[r];
  // T3: W = c (per thread, into TMEM cols R..2R), g = W . B^T (A from TMEM) into cols 2R..
  for (int q = 0; q < R / 16 || (R < 16 && q == 0); ++q) {
    if (R >= 16) tmem_st16(tl + R + 16 * q, c + 16 * q);
  }
  if (R == 8) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tl + R), "f"(c[0]),
                 "f"(c[1]), "f"(c[2]), "f"(c[3]), "f"(c[4]), "f"(c[5]), "f"(c[6]), "f"(c[7])
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  if (tid == 0) {
    tc::fence_after_sync();
    for (int kk = 0; kk < R / 8; ++kk) {
      const uint64_t bd = tc::smem_desc(tc::smem_u32(bn) + kk * 2 * (J * 16), J * 16, 128);
      mma_tmemA(tb + 2 * R, tb + R + kk * 8, bd, tc::idesc_tf32(128, J), kk > 0);
    }
    tc::mma_commit(&bar[1]);
  }
  tc::mbar_wait(&bar[1], 1);
  tc::fence_after_sync();
  float g[J];
  tc::tmem_ldh<J>(tl + 2 * R, g);
  for (int j = 0; j < J; ++j) out_g[tid * J + j] = g[j];
  // T4: rows += 1000 + k in the slot, then scatter / reduce back
  if (add == 3) {
    __syncthreads();
    for (int k = 0; k < J; ++k) slot[tid * J + k] = (float)(1000 + k);  // natural order
    tc::fence_async_smem();
    __syncthreads();
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst + (long long)me * J),
                 "r"(sbase + tid * J * 4), "r"(J * 4)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    add = 99;
  }
  for (int k = 0; k < J && add != 99; ++k) slot[swz<J>(tid, k)] = add ? (float)(1000 + k) : slot[swz<J>(tid, k)] + 1000 + k;
  tc::fence_async_smem();
  __syncthreads();
  if (add == 2) {  // one 2D tile reduce per row (box J x 1; the map un-swizzles)
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     &dst), "r"(0), "r"(me), "r"(sbase + tid * J * 4)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if ((lane & 3) == 0 && add != 99) {
    scatter4(&dst, 0, me, r1, r2, r3, sbase + tid * J * 4, add != 0);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tb, 128);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;

static CUtensorMap make_map(float* base, int rows, int J, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)J, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)J * 4};
  cuuint32_t box[2] = {(cuuint32_t)J, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUtensorMapSwizzle sw = J == 8 ? CU_TENSOR_MAP_SWIZZLE_32B : J == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d (box rows %d)\n", (int)r, box_rows);
  return m;
}


template <int J>
static int run(int box_rows, int add) {
  const int I = 1000, R = J;
  std::vector<float> F(I * J), B(J * R);
  for (int i = 0; i < I; ++i)
    for (int j = 0; j < J; ++j) F[i * J + j] = 0.001f * (i % 97) + 0.01f * j - 0.05f;
  for (int e = 0; e < J * R; ++e) B[e] = 0.02f * ((e * 7) % 13) - 0.1f;
  std::vector<int> rows(128);
  for (int t = 0; t < 128; ++t) rows[t] = (t * 389 + 17) % I;  // distinct
  float *dF, *dG, *dB, *o_rows, *o_c, *o_g;
  int* dr;
  cudaMalloc(&dF, I * J * 4);
  cudaMalloc(&dG, I * J * 4);
  cudaMalloc(&dB, J * R * 4);
  cudaMalloc(&o_rows, 128 * J * 4);
  cudaMalloc(&o_c, 128 * R * 4);
  cudaMalloc(&o_g, 128 * J * 4);
  cudaMalloc(&dr, 128 * 4);
  cudaMemcpy(dF, F.data(), I * J * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dG, F.data(), I * J * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), J * R * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, rows.data(), 128 * 4, cudaMemcpyHostToDevice);
  CUtensorMap ms = make_map(dF, I, J, box_rows), md = make_map(dG, I, J, box_rows);
  probe<J><<<1, 128>>>(ms, md, dr, dB, o_rows, o_c, o_g, add, dG);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("J=%d box_rows=%d add=%d: CUDA error %s\n", J, box_rows, add, cudaGetErrorString(e));
    exit(1);
  }
  std::vector<float> hr(128 * J), hc(128 * R), hg(128 * J), hG(I * J);
  cudaMemcpy(hr.data(), o_rows, hr.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc.data(), o_c, hc.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hg.data(), o_g, hg.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hG.data(), dG, hG.size() * 4, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0, e3 = 0, e4 = 0;
  for (int t = 0; t < 128; ++t) {
    const float* a = &F[rows[t] * J];
    for (int j = 0; j < J; ++j) e1 = fmax(e1, fabs(hr[t * J + j] - a[j]));
    std::vector<double> c(R, 0.0);
    for (int r = 0; r < R; ++r) {
      for (int j = 0; j < J; ++j) c[r] += (double)a[j] * B[j * R + r];
      e2 = fmax(e2, fabs(hc[t * R + r] - c[r]));
    }
    for (int j = 0; j < J; ++j) {
      double g = 0;
      for (int r = 0; r < R; ++r) g += (double)hc[t * R + r] * B[j * R + r];
      e3 = fmax(e3, fabs(hg[t * J + j] - g));
    }
    for (int j = 0; j < J; ++j) e4 = fmax(e4, fabs(hG[rows[t] * J + j] - (a[j] + 1000 + j)));
  }
  double e5 = 0;  // untouched rows unchanged
  std::vector<int> touched(I, 0);
  for (int t = 0; t < 128; ++t) touched[rows[t]] = 1;
  for (int i = 0; i < I; ++i)
    if (!touched[i])
      for (int j = 0; j < J; ++j) e5 = fmax(e5, fabs(hG[i * J + j] - F[i * J + j]));
  printf("J=%d box_rows=%d add=%d: gather %.3g  c(MMA, SW desc) %.3g  g(A in TMEM) %.3g  scatter %.3g  others %.3g\n",
         J, box_rows, add, e1, e2, e3, e4, e5);
  cudaFree(dF); cudaFree(dG); cudaFree(dB); cudaFree(o_rows); cudaFree(o_c); cudaFree(o_g); cudaFree(dr);
  return 0;
}

int main(int argc, char** argv) {
  const int box0 = argc > 1 ? atoi(argv[1]) : 1, add0 = argc > 2 ? atoi(argv[2]) : 0;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  if (!encode) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  run<16>(box0, add0);
  run<8>(box0, add0);
  run<32>(box0, add0);
  return 0;
}
