// capi.cu -- extern "C" entry points (include/sptk.h) and the host-side
// SeedSequence -> PCG64 seeding.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "../../include/sptk.h"
#include "common.cuh"
#include "kernels.cuh"
#include "pcg64.cuh"

#include <stdlib.h>

namespace sptk {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int n) { g_launches += n; }

static int build_model_desc(ModelDesc* md, const int64_t* h_foff, const int64_t* h_coff, const int64_t* h_jr,
                            int n_modes, int rcore) {
  SPTK_REQUIRE(n_modes >= 2 && n_modes <= SPTK_MAX_MODES, "order must be in [2, %d]", SPTK_MAX_MODES);
  SPTK_REQUIRE(rcore >= 1, "rcore must be >= 1");
  md->n_modes = n_modes;
  md->rcore = rcore;
  int cs = 0;
  for (int n = 0; n < n_modes; ++n) {
    SPTK_REQUIRE(h_jr[n] >= 1 && h_jr[n] <= 4096, "j_ranks out of range");
    md->jr[n] = (int)h_jr[n];
    md->foff[n] = h_foff[n];
    md->coff[n] = (int)h_coff[n];
    cs += md->jr[n] * rcore;
  }
  md->cor_size = cs;
  md->fac_size = h_foff[n_modes];
  return 0;
}

}  // namespace sptk

using namespace sptk;

template <typename T>
static int core_dispatch(const int32_t* d_rec, int rw, const int32_t* d_visit, const int32_t* d_map,
                         long long n_visit, const T* d_fac, const int64_t* h_foff, const T* d_cor,
                         const int64_t* h_coff, const int64_t* h_jr, int n_modes, int rcore, double* d_acc,
                         int exact_chunks, void* d_ws, size_t ws_bytes, void* stream) {
  ModelDesc md;
  if (build_model_desc(&md, h_foff, h_coff, h_jr, n_modes, rcore)) return 2;
  if (exact_chunks > 0)
    return core_pass_exact<T>(d_rec, rw, d_visit, d_map, n_visit, exact_chunks, d_fac, d_cor, md, d_acc, d_ws,
                              ws_bytes, (cudaStream_t)stream);
  return core_pass<T>(d_rec, rw, d_visit, d_map, n_visit, d_fac, d_cor, md, d_acc, d_ws, ws_bytes,
                      (cudaStream_t)stream);
}

extern "C" {

const char* sptk_last_error(void) { return g_err; }
int sptk_version(void) { return 100; }
long long sptk_launch_count(void) { return g_launches.load(); }
void sptk_reset_launch_count(void) { g_launches = 0; }
int sptk_record_words(int order, int f64_records) { return rec_words_t(order, f64_records != 0); }
int sptk_set_tc_mode(int mode) {
  SPTK_REQUIRE(set_tc_mode(mode) == 0, "tc mode must be 0 (FMA), 1 (TF32 v2), 2 (TF32 v1) or 3 (3xTF32)");
  return 0;
}
int sptk_get_tc_mode(void) { return get_tc_mode(); }
const char* sptk_last_factor_kernel(void) { return last_factor_kernel(); }
void sptk_debug_tc_buffer(float* d_buf) { set_tc_debug(d_buf); }

// numpy SeedSequence + PCG64 seeding (pcg64.cuh); used by the reference at
// trainer.py:196-198 and trainer.py:214 through np.random.default_rng.
int sptk_pcg64_seed(const uint64_t* h_entropy, int n_entropy, uint64_t h_state_out[4]) {
  uint32_t words[512];
  const int nw = seedseq_words(h_entropy, n_entropy, words, 512);
  SPTK_REQUIRE(nw >= 0, "entropy too long");
  const Pcg64 g = seedseq_pcg64(words, nw);
  h_state_out[0] = (uint64_t)(g.state >> 64);
  h_state_out[1] = (uint64_t)g.state;
  h_state_out[2] = (uint64_t)(g.inc >> 64);
  h_state_out[3] = (uint64_t)g.inc;
  return 0;
}

size_t sptk_block_job_bytes(void) { return block_job_bytes(); }

int sptk_block_perm(const void* d_jobs, const int32_t* d_coords, int n_jobs, int order, uint64_t seed, long long t,
                    int cap, uint16_t* d_js, int32_t* d_visit, void* stream) {
  return block_perm(d_jobs, d_coords, n_jobs, order, (unsigned long long)seed, t, cap, d_js, d_visit,
                    (cudaStream_t)stream);
}

int sptk_interleave_rounds(const void* d_jobs, int n_jobs, const int32_t* d_perm, long long rel_lo,
                           int32_t* d_visit, long long cap, void* stream) {
  return interleave_rounds(d_jobs, n_jobs, d_perm, rel_lo, d_visit, (cudaStream_t)stream, cap);
}

size_t sptk_permutation_ws_bytes(long long n) { return perm_ws_bytes(n); }

int sptk_permutation(const uint64_t h_state[4], long long n, int32_t* d_out, void* d_ws, size_t ws_bytes,
                     void* stream) {
  return permutation(h_state, n, d_out, d_ws, ws_bytes, (cudaStream_t)stream);
}

int sptk_permute_records(const uint64_t h_state[4], long long n, const int32_t* d_rec_src, int rw,
                         int32_t* d_rec_out, int32_t* d_perm_out, void* d_ws, size_t ws_bytes, void* stream) {
  return permute_records(h_state, n, d_rec_src, rw, d_rec_out, d_perm_out, d_ws, ws_bytes, (cudaStream_t)stream);
}

size_t sptk_permutation_j_ws_bytes(long long n) { return jgen_ws_bytes(n); }
size_t sptk_fy_apply_ws_bytes(long long n) { return fy_ws_bytes(n); }
int sptk_fy_apply(int32_t* d_j, long long n, int32_t* d_out, void* d_ws, size_t ws_bytes, void* stream) {
  return fy_apply_public(d_j, n, d_out, d_ws, ws_bytes, (cudaStream_t)stream);
}

int sptk_fy_globalize(int32_t* d_j, const int32_t* d_block_off, int n_blocks, void* stream) {
  return fy_globalize(d_j, d_block_off, n_blocks, (cudaStream_t)stream);
}

size_t sptk_permutation_j_batch_ws_bytes(const long long* h_n, int n_blocks) {
  return jgen_batch_ws_bytes(h_n, n_blocks);
}
int sptk_permutation_j_batch(const uint64_t* h_states, const long long* h_n, const long long* h_offsets,
                             int n_blocks, int32_t* d_j, void* d_ws, size_t ws_bytes, void* stream) {
  if (n_blocks <= 0) return 0;
  int** outs = (int**)malloc(sizeof(int*) * n_blocks);
  if (!outs) return 2;
  for (int b = 0; b < n_blocks; ++b) outs[b] = d_j + h_offsets[b];
  int rc = permutation_j_batch(h_states, h_n, outs, n_blocks, d_ws, ws_bytes, (cudaStream_t)stream);
  free(outs);
  return rc;
}

int sptk_permutation_j(const uint64_t h_state[4], long long n, int32_t* d_j, void* d_ws, size_t ws_bytes,
                       void* stream) {
  return permutation_j(h_state, n, d_j, d_ws, ws_bytes, (cudaStream_t)stream);
}

size_t sptk_choice_ws_bytes(long long pop, long long k) { return choice_ws_bytes(pop, k); }

int sptk_choice(const uint64_t h_state[4], long long pop, long long k, int shuffle, int32_t* d_out, void* d_ws,
                size_t ws_bytes, int* h_path_out, void* stream) {
  return choice(h_state, pop, k, shuffle, d_out, d_ws, ws_bytes, h_path_out, (cudaStream_t)stream);
}

int sptk_u32_stream(const uint64_t h_state[4], unsigned long long q0, long long n, uint32_t* d_out, void* stream) {
  return u32_stream(h_state, q0, n, d_out, (cudaStream_t)stream);
}

int sptk_h2d(void* d_dst, const void* h_src, size_t bytes, int threads) {
  return h2d(d_dst, h_src, bytes, threads);
}

size_t sptk_partition_ws_bytes(long long nnz, int order, long long m) { return partition_ws_bytes(nnz, order, m); }

int sptk_partition(const int64_t* d_idx, const double* d_vals, long long nnz, int order, const int64_t* h_dims,
                   long long m, int f64_records, int32_t* d_rec, int32_t* d_ids, int32_t* d_pos_of_id,
                   int32_t* d_block_off, void* d_ws, size_t ws_bytes, void* stream) {
  return partition((const long long*)d_idx, d_vals, nnz, order, (const long long*)h_dims, m, d_rec, d_ids,
                   d_pos_of_id, d_block_off, d_ws, ws_bytes, (cudaStream_t)stream, f64_records);
}

int sptk_h2d_pack(int32_t* d_rec, const int64_t* h_idx, const double* h_vals, long long nnz, int order,
                  int threads) {
  return h2d_pack_records(d_rec, (const long long*)h_idx, h_vals, nnz, order, rec_words(order), threads);
}

int sptk_partition_records(const int32_t* d_rec_src, long long nnz, int order, const int64_t* h_dims, long long m,
                           int32_t* d_rec_out, int32_t* d_ids, int32_t* d_pos_of_id, int32_t* d_block_off, void* d_ws,
                           size_t ws_bytes, void* stream) {
  return partition_records(d_rec_src, rec_words(order), nnz, order, (const long long*)h_dims, m, d_rec_out, d_ids,
                           d_pos_of_id, d_block_off, d_ws, ws_bytes, (cudaStream_t)stream);
}

int sptk_pack_records(const int64_t* d_idx, const double* d_vals, long long nnz, int order, int f64_records,
                      int32_t* d_rec, void* stream) {
  return pack_records((const long long*)d_idx, d_vals, nnz, order, d_rec, (cudaStream_t)stream, f64_records);
}

int sptk_factor_pass(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit, long long base,
                     float* d_fac, const int64_t* h_foff, const float* d_cor, const int64_t* h_coff,
                     const int64_t* h_jr, int n_modes, int rcore, const double* h_gammas, const double* h_lambdas,
                     int mode, void* stream) {
  ModelDesc md;
  if (build_model_desc(&md, h_foff, h_coff, h_jr, n_modes, rcore)) return 2;
  float g[SPTK_MAX_MODES], l[SPTK_MAX_MODES];
  for (int n = 0; n < n_modes; ++n) {
    g[n] = (float)h_gammas[n];
    l[n] = (float)h_lambdas[n];
  }
  return factor_pass<float>(d_rec, rw, d_visit, n_visit, base, d_fac, d_cor, md, g, l, mode, (cudaStream_t)stream);
}

int sptk_factor_pass_f64(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit, long long base,
                         double* d_fac, const int64_t* h_foff, const double* d_cor, const int64_t* h_coff,
                         const int64_t* h_jr, int n_modes, int rcore, const double* h_gammas,
                         const double* h_lambdas, int mode, void* stream) {
  ModelDesc md;
  if (build_model_desc(&md, h_foff, h_coff, h_jr, n_modes, rcore)) return 2;
  return factor_pass<double>(d_rec, rw, d_visit, n_visit, base, d_fac, d_cor, md, h_gammas, h_lambdas, mode,
                             (cudaStream_t)stream);
}

int sptk_fma_rank(int j) { return fma_rank_policy(j); }

size_t sptk_factor_pass_exact_ws_bytes(long long n_visit, int n_modes) {
  return factor_dep_ws_bytes(n_visit, n_modes);
}

int sptk_factor_pass_exact(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit, long long base,
                           float* d_fac, const int64_t* h_foff, const float* d_cor, const int64_t* h_coff,
                           const int64_t* h_jr, int n_modes, int rcore, const double* h_gammas,
                           const double* h_lambdas, void* d_ws, size_t ws_bytes, void* stream) {
  ModelDesc md;
  if (build_model_desc(&md, h_foff, h_coff, h_jr, n_modes, rcore)) return 2;
  float g[SPTK_MAX_MODES], l[SPTK_MAX_MODES];
  for (int n = 0; n < n_modes; ++n) {
    g[n] = (float)h_gammas[n];
    l[n] = (float)h_lambdas[n];
  }
  return factor_pass_dep<float>(d_rec, rw, d_visit, n_visit, base, d_fac, d_cor, md, g, l, d_ws, ws_bytes,
                                (cudaStream_t)stream);
}

int sptk_factor_pass_exact_f64(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit,
                               long long base, double* d_fac, const int64_t* h_foff, const double* d_cor,
                               const int64_t* h_coff, const int64_t* h_jr, int n_modes, int rcore,
                               const double* h_gammas, const double* h_lambdas, void* d_ws, size_t ws_bytes,
                               void* stream) {
  ModelDesc md;
  if (build_model_desc(&md, h_foff, h_coff, h_jr, n_modes, rcore)) return 2;
  return factor_pass_dep<double>(d_rec, rw, d_visit, n_visit, base, d_fac, d_cor, md, h_gammas, h_lambdas, d_ws,
                                 ws_bytes, (cudaStream_t)stream);
}

int sptk_factor_pass_dsgd(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit, float* d_fac,
                          const int64_t* h_foff, const float* d_cor, const int64_t* h_coff, const int64_t* h_jr,
                          int n_modes, int rcore, const double* h_gammas, const double* h_lambdas,
                          const long long* d_rstart, const long long* d_rend, const void* d_push, int32_t* d_done,
                          int32_t* d_ready, int n_rounds, int gen0, int epoch, int grid, void* stream) {
  ModelDesc md;
  if (build_model_desc(&md, h_foff, h_coff, h_jr, n_modes, rcore)) return 2;
  float g[SPTK_MAX_MODES], l[SPTK_MAX_MODES];
  for (int n = 0; n < n_modes; ++n) {
    g[n] = (float)h_gammas[n];
    l[n] = (float)h_lambdas[n];
  }
  return factor_pass_dsgd(d_rec, rw, d_visit, n_visit, d_fac, d_cor, md, g, l, d_rstart, d_rend, d_push, d_done,
                          d_ready, n_rounds, gen0, epoch, grid, (cudaStream_t)stream);
}

size_t sptk_dsgd_push_bytes(void) { return dsgd_push_bytes(); }

int sptk_flag_store(int32_t* d_flag, int value, void* stream) {
  return flag_store(d_flag, value, (cudaStream_t)stream);
}

int sptk_shared_alloc(size_t bytes, void** d_ptr) {
  *d_ptr = nullptr;
  SPTK_CUDA_TRY(cudaMalloc(d_ptr, bytes));
  SPTK_CUDA_TRY(cudaMemset(*d_ptr, 0, bytes));
  return 0;
}

int sptk_shared_free(void* d_ptr) {
  SPTK_CUDA_TRY(cudaFree(d_ptr));
  return 0;
}

int sptk_ipc_get(void* d_ptr, unsigned char* h_handle) {
  cudaIpcMemHandle_t h;
  SPTK_CUDA_TRY(cudaIpcGetMemHandle(&h, d_ptr));
  memcpy(h_handle, &h, sizeof(h));
  return 0;
}

int sptk_ipc_open(const unsigned char* h_handle, void** d_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle, sizeof(h));
  *d_ptr = nullptr;
  SPTK_CUDA_TRY(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int sptk_ipc_close(void* d_ptr) {
  SPTK_CUDA_TRY(cudaIpcCloseMemHandle(d_ptr));
  return 0;
}

size_t sptk_core_ws_bytes(const int64_t* h_jr, int n_modes, int rcore, int exact_chunks) {
  size_t cs = 0;
  for (int n = 0; n < n_modes; ++n) cs += (size_t)h_jr[n] * rcore;
  size_t blocks = exact_chunks > 0 ? (size_t)exact_chunks : (size_t)148 * 4;
  size_t b = blocks * cs * sizeof(double) + sizeof(long long) * (blocks + 2) + 1024;
  if (exact_chunks > 0) {
    // segment scratch of the whole-GPU exact pass (core.cu: EXACT_SEG samples)
    size_t tot = 0;
    for (int n = 0; n < n_modes; ++n) tot += (size_t)h_jr[n];
    b += (size_t)32768 * (2 * (size_t)n_modes * rcore + tot) * sizeof(double) + 1024;
  }
  return b;
}

int sptk_core_pass(const int32_t* d_rec, int rw, const int32_t* d_visit, const int32_t* d_map, long long n_visit,
                   const float* d_fac, const int64_t* h_foff, const float* d_cor, const int64_t* h_coff,
                   const int64_t* h_jr, int n_modes, int rcore, double* d_acc, int exact_chunks, void* d_ws,
                   size_t ws_bytes, void* stream) {
  return core_dispatch<float>(d_rec, rw, d_visit, d_map, n_visit, d_fac, h_foff, d_cor, h_coff, h_jr, n_modes,
                              rcore, d_acc, exact_chunks, d_ws, ws_bytes, stream);
}

int sptk_core_pass_f64(const int32_t* d_rec, int rw, const int32_t* d_visit, const int32_t* d_map,
                       long long n_visit, const double* d_fac, const int64_t* h_foff, const double* d_cor,
                       const int64_t* h_coff, const int64_t* h_jr, int n_modes, int rcore, double* d_acc,
                       int exact_chunks, void* d_ws, size_t ws_bytes, void* stream) {
  return core_dispatch<double>(d_rec, rw, d_visit, d_map, n_visit, d_fac, h_foff, d_cor, h_coff, h_jr, n_modes,
                               rcore, d_acc, exact_chunks, d_ws, ws_bytes, stream);
}

int sptk_core_apply(float* d_cor, const double* d_acc, int cor_size, double gamma_b, double lambda_b, double denom,
                    void* stream) {
  return core_apply<float>(d_cor, d_acc, cor_size, gamma_b, lambda_b, denom, (cudaStream_t)stream);
}

int sptk_core_apply_f64(double* d_cor, const double* d_acc, int cor_size, double gamma_b, double lambda_b,
                        double denom, void* stream) {
  return core_apply<double>(d_cor, d_acc, cor_size, gamma_b, lambda_b, denom, (cudaStream_t)stream);
}

int sptk_eval(const int32_t* d_rec, int rw, long long m, const float* d_fac, const int64_t* h_foff,
              const float* d_cor, const int64_t* h_coff, const int64_t* h_jr, int n_modes, int rcore, float* d_pred,
              double* d_sums, void* stream) {
  ModelDesc md;
  if (build_model_desc(&md, h_foff, h_coff, h_jr, n_modes, rcore)) return 2;
  SPTK_REQUIRE(rw == rec_words_t(n_modes, false), "eval: record width mismatch");
  return eval<float>(d_rec, rw, m, d_fac, d_cor, md, d_pred, d_sums, (cudaStream_t)stream);
}

int sptk_eval_f64(const int32_t* d_rec, int rw, long long m, const double* d_fac, const int64_t* h_foff,
                  const double* d_cor, const int64_t* h_coff, const int64_t* h_jr, int n_modes, int rcore,
                  double* d_pred, double* d_sums, void* stream) {
  ModelDesc md;
  if (build_model_desc(&md, h_foff, h_coff, h_jr, n_modes, rcore)) return 2;
  SPTK_REQUIRE(rw == rec_words_t(n_modes, true), "eval_f64: record width mismatch");
  return eval<double>(d_rec, rw, m, d_fac, d_cor, md, d_pred, d_sums, (cudaStream_t)stream);
}

}  // extern "C"
