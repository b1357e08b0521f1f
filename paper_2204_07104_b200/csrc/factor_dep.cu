// factor_dep.cu -- K3 exact mode across the whole GPU (dependency-driven).
//
// The reference's factor phase is a strictly sequential loop over the visit
// list (_loops.py:17-63): sample k reads the rows A(n)[i_n(k)] as the last
// earlier sample touching each of those rows left them, and B is frozen for
// the whole phase.  So sample k depends only on its per-mode predecessors
//     pred_n(k) = max { k' < k : i_n(k') = i_n(k) }     (or none),
// and any schedule that runs every sample after its predecessors reproduces
// the sequential loop bit for bit (samples with no path between them touch
// disjoint rows, so their updates commute exactly).
//
//   1. predecessors: per mode, a stable radix sort of the visit positions by
//      row (K1's sort); pred_n of a sorted entry is its left neighbour when
//      that has the same row;
//   2. factor_dep_kernel: every resident warp claims the next visit position
//      from a global counter (positions are claimed in visit order by running
//      warps, so every predecessor of a claimed sample is held by a running
//      warp: no deadlock at any grid size), waits for its predecessors' done
//      flags (ld.acquire), updates the sample with the reference's operation
//      order (lanes over r / j, sums in the reference's index order, no FMA
//      contraction), writes the rows and publishes its flag (st.release).
// The critical path is the longest predecessor chain, not the visit length:
// cfg1's 90K samples have a longest chain of 563 (computed on the host for
// one visit order), against the ~2,800 conflict-free prefixes of the
// one-warp walker (factor_seq_kernel, kept for tiny visit lists).
#include "common.cuh"
#include "kernels.cuh"

namespace sptk {

namespace {

template <typename T>
__device__ __forceinline__ T dmul(T a, T b);
template <>
__device__ __forceinline__ float dmul<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double dmul<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T dadd(T a, T b);
template <>
__device__ __forceinline__ float dadd<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double dadd<double>(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void dep_keys_kernel(const int* __restrict__ rec, int rw, const int* __restrict__ visit, long long nv,
                                long long base, int mode, unsigned* __restrict__ keys, int* __restrict__ vals) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nv; k += stride) {
    const long long ri = base + (visit ? (long long)visit[k] : k);
    keys[k] = (unsigned)rec[ri * rw + mode];
    vals[k] = (int)k;
  }
}

__global__ void dep_pred_kernel(const unsigned* __restrict__ keys, const int* __restrict__ vals, long long nv,
                                int* __restrict__ pred) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += stride)
    pred[vals[i]] = (i > 0 && keys[i - 1] == keys[i]) ? vals[i - 1] : -1;
}

struct DepGamLam {
  double gam[SPTK_MAX_MODES];
  double lam[SPTK_MAX_MODES];
};

template <typename T>
__global__ void __launch_bounds__(128) factor_dep_kernel(const int* __restrict__ rec, int rw, int vo,
                                                         const int* __restrict__ visit, long long nv, long long base,
                                                         T* __restrict__ fac, const T* __restrict__ cor,
                                                         ModelDesc md, DepGamLam gl, const int* __restrict__ pred,
                                                         int* __restrict__ flags, unsigned long long* counter,
                                                         int per_warp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Bs = reinterpret_cast<T*>(smem_raw);
  for (int i = threadIdx.x; i < md.cor_size; i += blockDim.x) Bs[i] = cor[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int N = md.n_modes, R = md.rcore;
  int aoff[SPTK_MAX_MODES];
  int tot = 0;
  for (int n = 0; n < N; ++n) {
    aoff[n] = tot;
    tot += md.jr[n];
  }
  T* a_s = Bs + ((md.cor_size + 1) & ~1) + (size_t)warp * per_warp;  // sum J
  T* c_s = a_s + tot;                                                 // N*R
  T* w_s = c_s + N * R;                                               // R
  T* g_s = w_s + R;                                                   // max J
  while (true) {
    long long k = 0;
    if (lane == 0) k = (long long)atomicAdd(counter, 1ull);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= nv) break;
    const int* rp = rec + (base + (visit ? (long long)__ldg(visit + k) : k)) * rw;
    // the record is read-only: fetched before the wait
    const T x = load_val<T>(rp, vo);
    int rows[SPTK_MAX_MODES];
    for (int n = 0; n < N; ++n) rows[n] = __ldg(rp + n);
    // wait for the predecessors: lane n < N polls mode n's (one round trip
    // per poll for all modes together)
    {
      // relaxed polls (an acquire load invalidates the SM's L1 on every poll:
      // ncu showed 38% of the stall samples on that CCTL.IVALL), then one
      // acquire once every predecessor is seen done
      const int p = lane < N ? __ldg(pred + (long long)lane * nv + k) : -1;
      while (!__all_sync(0xffffffffu, p < 0 || ld_relaxed(flags + p) != 0)) {
      }
      if (p >= 0) (void)ld_acquire(flags + p);
      __syncwarp();
    }
    for (int n = 0; n < N; ++n) {
      const int J = md.jr[n];
      const T* row = fac + md.foff[n] + (long long)rows[n] * J;
      for (int j = lane; j < J; j += 32) a_s[aoff[n] + j] = __ldcg(row + j);
    }
    __syncwarp();
    for (int q = lane; q < N * R; q += 32) {
      const int n0 = q / R, r = q - n0 * R;
      const int J = md.jr[n0];
      T acc = 0;
      for (int j = 0; j < J; ++j) acc = dadd(acc, dmul(a_s[aoff[n0] + j], Bs[md.coff[n0] + j * R + r]));
      c_s[q] = acc;
    }
    __syncwarp();
    for (int n = 0; n < N; ++n) {
      const int J = md.jr[n];
      for (int r = lane; r < R; r += 32) {
        T w = 1;
        for (int n0 = 0; n0 < N; ++n0)
          if (n0 != n) w = dmul(w, c_s[n0 * R + r]);
        w_s[r] = w;
      }
      __syncwarp();
      for (int j = lane; j < J; j += 32) {
        T g = 0;
        for (int r = 0; r < R; ++r) g = dadd(g, dmul(w_s[r], Bs[md.coff[n] + j * R + r]));
        g_s[j] = g;
      }
      __syncwarp();
      T inter = 0;
      for (int j = 0; j < J; ++j) inter = dadd(inter, dmul(a_s[aoff[n] + j], g_s[j]));
      __syncwarp();
      const T gm = (T)gl.gam[n], lm = (T)gl.lam[n];
      T* row = fac + md.foff[n] + (long long)rows[n] * J;
      for (int j = lane; j < J; j += 32) {
        T av = a_s[aoff[n] + j];
        const T gsj = g_s[j];
        const T g = dadd(dadd(dmul(-x, gsj), dmul(lm, av)), dmul(inter, gsj));
        av = dadd(av, -dmul(gm, g));
        a_s[aoff[n] + j] = av;
        __stcg(row + j, av);
      }
      __syncwarp();
      if (n < N - 1) {
        for (int r = lane; r < R; r += 32) {
          T acc = 0;
          for (int j = 0; j < J; ++j) acc = dadd(acc, dmul(a_s[aoff[n] + j], Bs[md.coff[n] + j * R + r]));
          c_s[n * R + r] = acc;
        }
      }
      __syncwarp();
    }
    // publish: the warp's row stores (ordered before lane 0 by the warp
    // barrier), one gpu-scope fence (cumulative), then the flag
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      st_release(flags + k, 1);
    }
  }
}

struct Carve3 {
  char* p;
  size_t left;
  bool bad = false;
  template <typename U>
  U* take(size_t count) {
    size_t bytes = (count * sizeof(U) + 255) & ~(size_t)255;
    if (bytes > left) {
      bad = true;
      return (U*)p;
    }
    U* r = (U*)p;
    p += bytes;
    left -= bytes;
    return r;
  }
};

inline unsigned grid_for(long long n, int t) {
  long long g = (n + t - 1) / t;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)g;
}

}  // namespace

size_t factor_dep_ws_bytes(long long nv, int n_modes) {
  if (nv < 1) nv = 1;
  size_t b = 0;
  b += 4 * (((size_t)nv * 4 + 255) & ~(size_t)255);                 // keys x2, vals x2
  b += (((size_t)nv * n_modes * 4) + 255) & ~(size_t)255;            // pred
  b += (((size_t)nv * 4) + 255) & ~(size_t)255;                      // flags
  b += 256;                                                          // counter
  b += radix_ws_bytes(nv) + 256;
  return b;
}

template <typename T>
int factor_pass_dep(const int* rec, int rw, const int* visit, long long nv, long long base, T* fac, const T* cor,
                    const ModelDesc& md, const T* h_gammas, const T* h_lambdas, void* ws, size_t ws_bytes,
                    cudaStream_t s) {
  SPTK_REQUIRE(md.n_modes >= 2 && md.n_modes <= SPTK_MAX_MODES, "factor_pass_exact: bad order %d", md.n_modes);
  if (nv <= 0) return 0;
  SPTK_REQUIRE(nv < (1LL << 31), "factor_pass_exact: visit list too long");
  SPTK_REQUIRE(ws_bytes >= factor_dep_ws_bytes(nv, md.n_modes), "factor_pass_exact: workspace too small");
  const bool f64 = sizeof(T) == 8;
  const int N = md.n_modes;
  SPTK_REQUIRE(rw == rec_words_t(N, f64), "factor_pass_exact: record width %d does not match order %d", rw, N);
  Carve3 cv{(char*)ws, ws_bytes};
  unsigned* k0 = cv.take<unsigned>(nv);
  unsigned* k1 = cv.take<unsigned>(nv);
  int* v0 = cv.take<int>(nv);
  int* v1 = cv.take<int>(nv);
  int* pred = cv.take<int>((size_t)nv * N);
  int* flags = cv.take<int>(nv);
  unsigned long long* counter = cv.take<unsigned long long>(4);
  void* rws = cv.p;
  const size_t rws_bytes = cv.left;
  SPTK_REQUIRE(!cv.bad, "factor_pass_exact: workspace carve failed");
  for (int n = 0; n < N; ++n) {
    const long long rows = (((n + 1 < N) ? md.foff[n + 1] : md.fac_size) - md.foff[n]) / md.jr[n];
    int bits = 0;
    while ((1LL << bits) < rows) ++bits;
    dep_keys_kernel<<<grid_for(nv, 256), 256, 0, s>>>(rec, rw, visit, nv, base, n, k0, v0);
    SPTK_CHECK_LAUNCH();
    unsigned* ko = k0;
    int* vo = v0;
    if (bits > 0 && radix_sort_pairs(k0, v0, k1, v1, nv, bits, rws, rws_bytes, s, &ko, &vo)) return 1;
    dep_pred_kernel<<<grid_for(nv, 256), 256, 0, s>>>(ko, vo, nv, pred + (size_t)n * nv);
    SPTK_CHECK_LAUNCH();
  }
  SPTK_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int) * nv, s));
  SPTK_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
  DepGamLam gl;
  int jmax = 0, tot = 0;
  for (int n = 0; n < N; ++n) {
    gl.gam[n] = (double)h_gammas[n];
    gl.lam[n] = (double)h_lambdas[n];
    jmax = md.jr[n] > jmax ? md.jr[n] : jmax;
    tot += md.jr[n];
  }
  const int per_warp = (tot + N * md.rcore + md.rcore + jmax + 1) & ~1;
  const int threads = 128, warps = threads / 32;
  const size_t smem = sizeof(T) * ((size_t)((md.cor_size + 1) & ~1) + (size_t)per_warp * warps);
  SPTK_REQUIRE(smem <= 200 * 1024, "factor_pass_exact: model ranks too large for shared memory");
  auto kfn = factor_dep_kernel<T>;
  SPTK_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SPTK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, threads, smem));
  if (per_sm < 1) per_sm = 1;
  int dev = 0, sms = 148;
  SPTK_CUDA_TRY(cudaGetDevice(&dev));
  SPTK_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  long long blocks = (long long)sms * per_sm;
  const long long need = (nv + warps - 1) / warps;
  if (blocks > need) blocks = need;
  const int vo = rec_val_off(N, f64);
  kfn<<<(unsigned)blocks, threads, smem, s>>>(rec, rw, vo, visit, nv, base, fac, cor, md, gl, pred, flags, counter,
                                              per_warp);
  note_factor_kernel("factor_dep_kernel");
  SPTK_CHECK_LAUNCH();
  return 0;
}

template int factor_pass_dep<float>(const int*, int, const int*, long long, long long, float*, const float*,
                                    const ModelDesc&, const float*, const float*, void*, size_t, cudaStream_t);
template int factor_pass_dep<double>(const int*, int, const int*, long long, long long, double*, const double*,
                                     const ModelDesc&, const double*, const double*, void*, size_t, cudaStream_t);

}  // namespace sptk
