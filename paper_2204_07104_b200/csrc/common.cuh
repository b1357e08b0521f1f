// common.cuh -- shared helpers for the sptk CUDA library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#ifndef SPTK_MAX_MODES
#define SPTK_MAX_MODES 16
#endif

namespace sptk {

// Set by every entry point on failure; read through sptk_last_error().
void set_error(const char* fmt, ...);
// Counts kernels launched by this library (read through sptk_launch_count()).
void count_launch(int n = 1);

// Model layout shared by the factor / core / eval kernels.  This is the
// reference's packing (_loops.py:8-10, trainer.py:135-141): A(n) row i at
// fac[foff[n] + i*jr[n]], B(n)[j][r] at cor[coff[n] + j*rcore + r].
struct ModelDesc {
  int n_modes;
  int rcore;
  int jr[SPTK_MAX_MODES];
  long long foff[SPTK_MAX_MODES];
  int coff[SPTK_MAX_MODES];
  int cor_size;  // sum_n jr[n] * rcore
  long long fac_size;  // foff[n_modes]: total factor entries (rows of mode n = (foff[n+1]-foff[n])/jr[n])
};

// Nonzeros as packed AoS records of `rw` 32-bit words: idx[0..N) (int32)
// followed by the value (fp32 bits).  rw = 4 for N <= 3, 8 for N <= 7,
// 16 for N <= 15, so one record is one 16/32/64-byte aligned load.
struct MDims {
  long long d[SPTK_MAX_MODES];
};

struct RecDesc {
  const int* rec;
  int rw;
};

__host__ __device__ inline int rec_words(int n_modes) {
  return n_modes <= 3 ? 4 : (n_modes <= 7 ? 8 : 16);
}

// fp64 records (verification mode): the value is a double at an even word
// offset so that fp64 inputs reach the kernels unrounded.
__host__ __device__ inline int rec_val_off(int n_modes, bool f64) {
  return f64 ? ((n_modes + 1) & ~1) : n_modes;
}
__host__ __device__ inline int rec_words_t(int n_modes, bool f64) {
  if (!f64) return rec_words(n_modes);
  int need = rec_val_off(n_modes, true) + 2;
  int w = 4;
  while (w < need) w *= 2;
  return w;
}

template <typename T>
__device__ __forceinline__ T load_val(const int* rp, int vo);
template <>
__device__ __forceinline__ float load_val<float>(const int* rp, int vo) {
  return __int_as_float(__ldg(rp + vo));
}
template <>
__device__ __forceinline__ double load_val<double>(const int* rp, int vo) {
  return __ldg(reinterpret_cast<const double*>(rp + vo));
}

// Hogwild staleness bound for the throughput factor kernels: at most
// n_visit / SPAN samples in flight (SPAN = 64, SPTK_HOGWILD_SPAN overrides),
// i.e. a grid of at most that many samples / samples_per_cta CTAs.  Large
// visit lists (NF: 99M, 75K in flight) are unaffected; on small ones a full
// grid keeps a fifth of the epoch in flight and the add-reduced deltas of a
// hot row pile up (measured on a 400K-nonzero 3000x1200x300 tensor, one
// epoch: NaN with 75K samples in flight, test RMSE +4% with 19K, +0.5% with
// 4.7K, against the sequential reference).
static inline long long hogwild_cta_cap(long long n_visit, int samples_per_cta) {
  long long span = 64;
  if (const char* e = getenv("SPTK_HOGWILD_SPAN")) span = atoll(e);
  if (span < 1) return 1LL << 40;
  long long cap = n_visit / span / (samples_per_cta > 0 ? samples_per_cta : 1);
  return cap < 1 ? 1 : cap;
}

}  // namespace sptk

#define SPTK_CUDA_TRY(expr)                                                        \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::sptk::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                \
                        cudaGetErrorString(_e));                                   \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

#define SPTK_CHECK_LAUNCH()                                                        \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      ::sptk::set_error("%s:%d launch failed: %s", __FILE__, __LINE__,            \
                        cudaGetErrorString(_e));                                   \
      return 1;                                                                    \
    }                                                                              \
    ::sptk::count_launch();                                                        \
  } while (0)

#define SPTK_REQUIRE(cond, ...)                                                    \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      ::sptk::set_error(__VA_ARGS__);                                              \
      return 2;                                                                    \
    }                                                                              \
  } while (0)
