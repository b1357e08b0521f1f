// kernels.cuh -- internal host-side entry points shared between .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "common.cuh"

namespace sptk {

// sampler.cu
size_t perm_ws_bytes(long long n);
size_t jgen_ws_bytes(long long n);
size_t jgen_batch_ws_bytes(const long long* n, int B);
int permutation_j_batch(const uint64_t* st, const long long* n, int* const* j_out, int B, void* ws, size_t ws_bytes,
                        cudaStream_t s);
size_t fy_ws_bytes(long long n);
int fy_apply_public(int* j, long long n, int* out, void* ws, size_t ws_bytes, cudaStream_t s);
int fy_globalize(int* j, const int* off, int nb, cudaStream_t s);
int permutation(const uint64_t st[4], long long n, int* out, void* ws, size_t ws_bytes, cudaStream_t s);
int permute_records(const uint64_t st[4], long long n, const int* rec_src, int rw, int* rec_out, int* perm_out,
                    void* ws, size_t ws_bytes, cudaStream_t s);
int permutation_j(const uint64_t st[4], long long n, int* j_out, void* ws, size_t ws_bytes, cudaStream_t s);
size_t choice_ws_bytes(long long pop, long long k);
int choice(const uint64_t st[4], long long pop, long long k, int shuffle, int* out, void* ws,
           size_t ws_bytes, int* path_out, cudaStream_t s);
int block_perm(const void* d_jobs, const int* d_coords, int n_jobs, int order, unsigned long long seed,
               long long t, int cap, uint16_t* d_js, int* d_visit, cudaStream_t s);
size_t block_job_bytes();
int interleave_rounds(const void* d_jobs, int n_jobs, const int* d_perm, long long rel_lo, int* d_visit,
                      cudaStream_t s, long long cap);
int u32_stream(const uint64_t st[4], unsigned long long q0, long long n, uint32_t* out, cudaStream_t s);
int iota(int* out, long long n, int offset, cudaStream_t s);
size_t scan_ws_bytes(long long n);
int exclusive_scan(const int* in, long long n, int* out, int* ws, cudaStream_t s);

// partition.cu
int h2d(void* dst, const void* src, size_t bytes, int threads);
size_t partition_ws_bytes(long long nnz, int order, long long m);
int partition(const long long* idx64, const double* vals64, long long nnz, int order, const long long* h_dims,
              long long m, int* rec_out, int* ids_out, int* pos_of_id_out, int* block_off_out, void* ws,
              size_t ws_bytes, cudaStream_t s, int f64);
int pack_records(const long long* idx64, const double* vals64, long long nnz, int order, int* rec_out,
                 cudaStream_t s, int f64);
int partition_records(const int* rec_src, int rw, long long nnz, int order, const long long* h_dims, long long m,
                      int* rec_out, int* ids_out, int* pos_of_id_out, int* block_off_out, void* ws, size_t ws_bytes,
                      cudaStream_t s);
int h2d_pack_records(int* d_rec, const long long* h_idx, const double* h_vals, long long nnz, int order, int rw,
                     int threads);
size_t radix_ws_bytes(long long n);
int radix_sort_pairs(unsigned* k0, int* v0, unsigned* k1, int* v1, long long n, int bits, void* ws, size_t ws_bytes,
                     cudaStream_t s, unsigned** kout, int** vout);

// factor.cu
template <typename T>
int factor_pass(const int* rec, int rw, const int* visit, long long n_visit, long long base, T* fac,
                const T* cor, const ModelDesc& md, const T* h_gammas, const T* h_lambdas, int mode,
                cudaStream_t s);

int fma_rank_policy(int J);

// factor_dep.cu (exact mode across the GPU: predecessor-driven schedule)
size_t factor_dep_ws_bytes(long long nv, int n_modes);
template <typename T>
int factor_pass_dep(const int* rec, int rw, const int* visit, long long nv, long long base, T* fac, const T* cor,
                    const ModelDesc& md, const T* h_gammas, const T* h_lambdas, void* ws, size_t ws_bytes,
                    cudaStream_t s);

// factor_tc.cu (tcgen05 path; returns 1 if it handled the launch)
int try_factor_tc(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                  const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s, int* rc);

// factor_tma.cu (tcgen05 + TMA row traffic; returns 1 if it handled the launch)
int try_factor_tma(const int* rec, int rw, const int* visit, long long n_visit, long long base, float* fac,
                   const float* cor, const ModelDesc& md, const float* gam, const float* lam, cudaStream_t s, int* rc);
int factor_pass_dsgd(const int* rec, int rw, const int* visit, long long n_visit, float* fac, const float* cor,
                     const ModelDesc& md, const float* gam, const float* lam, const long long* rstart,
                     const long long* rend, const void* push, int* done, int* ready, int n_rounds, int gen0, int epoch,
                     int grid, cudaStream_t s);
size_t dsgd_push_bytes();
int flag_store(int* flag, int value, cudaStream_t s);
// name of the factor kernel the last factor_pass dispatched to
const char* last_factor_kernel();
void note_factor_kernel(const char* name);
float* tc_debug_buffer();

int set_tc_mode(int mode);
int get_tc_mode();
void set_tc_debug(float* buf);

// core.cu
size_t core_ws_bytes(const ModelDesc& md);
template <typename T>
int core_pass(const int* rec, int rw, const int* visit, const int* map, long long n_visit, const T* fac,
              const T* cor, const ModelDesc& md, double* acc, void* ws, size_t ws_bytes, cudaStream_t s);
template <typename T>
int core_pass_exact(const int* rec, int rw, const int* visit, const int* map, long long n_visit, int n_chunks,
                    const T* fac, const T* cor, const ModelDesc& md, double* acc, void* ws, size_t ws_bytes,
                    cudaStream_t s);
template <typename T>
int core_apply(T* cor, const double* acc, int cor_size, double gamma_b, double lambda_b, double denom,
               cudaStream_t s);

// eval.cu
template <typename T>
int eval(const int* rec, int rw, long long m, const T* fac, const T* cor, const ModelDesc& md, T* pred_out,
         double* sums, cudaStream_t s);

}  // namespace sptk
