/*
 * sptk.h -- C ABI of the B200-native stochastic sparse-Tucker SGD library
 * (libsptk.so, built for sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/sptucker).  The reference's Python driver
 * trainer.train (trainer.py:150-271) calls two numba kernels and numpy's
 * Generator; each of those is replaced here by a C entry point that a ctypes
 * binding (paper_2204_07104_b200/_lib.py) calls with
 * device pointers (torch tensors' data_ptr()) and a cudaStream_t:
 *
 *   _loops.factor_pass(idx, vals, visit, fac, foff, cor, coff, jr, rcore,
 *                      gammas, lambdas) -> 0            (_loops.py:17-18)
 *       -> sptk_factor_pass / sptk_factor_pass_f64
 *   _loops.core_pass(idx, vals, visit, fac, foff, cor, coff, jr, rcore,
 *                    acc, aoff) -> 0                     (_loops.py:66-67)
 *       -> sptk_core_pass / sptk_core_pass_f64 (aoff == coff, as at
 *          trainer.py:226-230), then the merge+apply of trainer.py:238-247
 *       -> sptk_core_apply / sptk_core_apply_f64
 *   np.random.default_rng([seed,1,t,*block]).permutation(len(ids))
 *                                                        (trainer.py:196-199)
 *       -> sptk_pcg64_seed + sptk_permutation
 *   np.random.default_rng([seed,2,t]).choice(nnz, k, replace=False)
 *                                                        (trainer.py:212-221)
 *       -> sptk_pcg64_seed + sptk_choice
 *   build_partition(tensor, m)                           (partition.py:47-81)
 *       -> sptk_partition (+ the device re-layout of the COO data)
 *   predict_entries / rmse / mae          (model.py:134-146, trainer.py:89-102)
 *       -> sptk_eval / sptk_eval_f64
 *
 * Conventions
 *   - d_* arguments are device pointers, h_* arguments are host pointers.
 *   - `stream` is a cudaStream_t (0 = legacy default stream).
 *   - Nonzeros live on the device as packed records: `rw` 32-bit words per
 *     nonzero, {i_0..i_{N-1} (int32), value}; the value is fp32 at word N
 *     (rw = 4/8/16 for N <= 3/7/15) or, for the fp64 verification entry points,
 *     an fp64 at word (N+1)&~1 (rw from sptk_record_words(N, 1)).  This packs
 *     the reference's (idx int64 [nnz,N], vals f64 [nnz]) pair so a gathered
 *     nonzero is one 16/32-byte load.
 *   - Model layout is the reference's (_loops.py:8-10): A(n) row i at
 *     fac[h_foff[n] + i*h_jr[n]], B(n)[j][r] at cor[h_coff[n] + j*rcore + r].
 *     h_foff / h_coff have order+1 entries, exactly the offsets the
 *     reference's _pack returns (trainer.py:135-141).
 *   - Every function returns 0 on success and nonzero on failure;
 *     sptk_last_error() describes the last failure.  The library never
 *     allocates device memory: callers pass workspaces sized by *_ws_bytes.
 */
#ifndef SPTK_H
#define SPTK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- introspection ---------------------------------------------------- */
const char* sptk_last_error(void);
int sptk_version(void);
long long sptk_launch_count(void);
void sptk_reset_launch_count(void);
int sptk_record_words(int order, int f64_records);
/* Throughput factor kernel for J = R in {16, 32}: 0 = CUDA-core FMA kernel,
 * 1 = tcgen05 TF32 with the folded refresh and cp.async row prefetch
 * (default), 2 = tcgen05 TF32 straight form, 3 = tcgen05 3xTF32 straight
 * form.  The environment variable SPTK_TC sets the initial value. */
int sptk_set_tc_mode(int mode);
int sptk_get_tc_mode(void);
/* Name of the factor kernel the most recent sptk_factor_pass dispatched to
 * (e.g. "factor_tma_kernel"); "none" before the first call.  Lets the caller
 * label measurements with the kernel that actually ran. */
const char* sptk_last_factor_kernel(void);
/* 1 if the throughput factor pass at uniform J = R = j runs on the CUDA-core
 * FMA kernel rather than tcgen05 (measured crossover; SPTK_FMA_RANKS). */
int sptk_fma_rank(int j);
/* test hook: per-sample dump of the first tcgen05 tile (c, gs, refreshed c). */
void sptk_debug_tc_buffer(float* d_buf);

/* ---- K2: samplers (bit-exact with numpy 2.x Generator/PCG64) ----------- */
/* default_rng(entropy).bit_generator state: {state_hi, state_lo, inc_hi, inc_lo}
 * (SeedSequence(entropy) -> PCG64 seeding), computed on the host. */
int sptk_pcg64_seed(const uint64_t* h_entropy, int n_entropy, uint64_t h_state_out[4]);

/* DSGD block visit orders (workers > 1), one CTA per block in shared memory:
 * for every block b of the table, default_rng([seed, 1, t, *coords[b]])
 * .permutation(n_b) (trainer.py:196-199, bit-exact), written as
 * visit[slot] = off_b + perm[p] at the round-interleaved slot
 * out_base_b + sum_s min(n_s, p) + #{s < slot_b : n_s > p} over the blocks s
 * of b's round.  d_jobs: n_jobs records of sptk_block_job_bytes() bytes
 * {int64 off, int64 out_base, int32 n, int32 first, int32 m, int32 slot, int32 nmin
 * (the round's smallest block), int32 pad},
 * round-major (first = index of the round's first job, m <= 64 jobs per round);
 * d_coords: n_jobs x order block coordinates; cap >= max n_b, <= 28000 (8 bytes
 * of shared memory per nonzero); d_js: uint16 scratch for the j-sequences, one
 * entry per record of the jobs (indexed like the records: off_b + p).
 * Replaces the per-block permutation + `visit = ids[perm]` of the round loop. */
size_t sptk_block_job_bytes(void);
int sptk_block_perm(const void* d_jobs, const int32_t* d_coords, int n_jobs, int order, uint64_t seed, long long t,
                    int cap, uint16_t* d_js, int32_t* d_visit, void* stream);
/* The same round-interleaved visit list from per-block visit orders already
 * in the partitioned layout (d_perm[off_b + p]; entries relative to off_b, or
 * to rel_lo when rel_lo >= 0; cap = the largest block, which sets how many CTAs
 * share a block): for blocks above sptk_block_perm's capacity,
 * whose orders come from sptk_permutation_j_batch + sptk_fy_apply. */
int sptk_interleave_rounds(const void* d_jobs, int n_jobs, const int32_t* d_perm, long long rel_lo,
                           int32_t* d_visit, long long cap, void* stream);
size_t sptk_permutation_ws_bytes(long long n);
/* d_out[n] (int32) = Generator.permutation(n) for the generator in h_state. */
int sptk_permutation(const uint64_t h_state[4], long long n, int32_t* d_out, void* d_ws, size_t ws_bytes,
                     void* stream);
/* Visit-ordered records: d_rec_out[k] = d_rec_src[perm[k]] (rw 32-bit words
 * each, rw in {4, 8, 16}) with perm = Generator.permutation(n) for h_state;
 * d_perm_out (may be NULL) also receives perm.  The factor phase's
 * `visit = ids[perm]` gather (trainer.py:196-199) fused into the sampler, so
 * the factor pass streams its block's records sequentially.  Workspace:
 * sptk_permutation_ws_bytes(n). */
int sptk_permute_records(const uint64_t h_state[4], long long n, const int32_t* d_rec_src, int rw,
                         int32_t* d_rec_out, int32_t* d_perm_out, void* d_ws, size_t ws_bytes, void* stream);
/* The two halves of sptk_permutation, for pipelining across epochs:
 * sptk_permutation_j writes the Fisher-Yates index sequence j_i (i = 1..n-1)
 * of permutation(n) (workspace sptk_permutation_j_ws_bytes(n)); sptk_fy_apply
 * applies such a sequence to the identity (d_j[0] is overwritten with 0;
 * workspace sptk_fy_apply_ws_bytes(n)), d_out[n] = the permutation. */
size_t sptk_permutation_j_ws_bytes(long long n);
int sptk_permutation_j(const uint64_t h_state[4], long long n, int32_t* d_j, void* d_ws, size_t ws_bytes,
                       void* stream);
/* Several blocks' j-sequences end to end (block b at [off[b], off[b+1]),
 * block-local values, off relative to d_j) -> one sequence for a single
 * sptk_fy_apply over the concatenation, whose result is every block's
 * permutation shifted by its offset (blocks touch disjoint positions).  One
 * apply per epoch instead of one per DSGD block. */
int sptk_fy_globalize(int32_t* d_j, const int32_t* d_block_off, int n_blocks, void* stream);
/* Batched first half: the j-sequences of n_blocks permutations (generator
 * states h_states[4b..4b+3], sizes h_n[b]) into d_j + h_offsets[b], all
 * blocks advancing segment level by segment level together (one launch per
 * phase for the batch instead of per block: the DSGD blocks of a rank). */
size_t sptk_permutation_j_batch_ws_bytes(const long long* h_n, int n_blocks);
int sptk_permutation_j_batch(const uint64_t* h_states, const long long* h_n, const long long* h_offsets,
                             int n_blocks, int32_t* d_j, void* d_ws, size_t ws_bytes, void* stream);
size_t sptk_fy_apply_ws_bytes(long long n);
int sptk_fy_apply(int32_t* d_j, long long n, int32_t* d_out, void* d_ws, size_t ws_bytes, void* stream);
size_t sptk_choice_ws_bytes(long long pop, long long k);
/* d_out[k] = Generator.choice(pop, k, replace=False).  shuffle=0 returns the
 * same set without the final _shuffle_int (the core phase only needs the
 * set).  *h_path_out = 1 (tail shuffle) or 2 (Floyd). */
int sptk_choice(const uint64_t h_state[4], long long pop, long long k, int shuffle, int32_t* d_out, void* d_ws,
                size_t ws_bytes, int* h_path_out, void* stream);
/* raw buffered 32-bit draws at stream positions q0..q0+n-1 (test hook). */
int sptk_u32_stream(const uint64_t h_state[4], unsigned long long q0, long long n, uint32_t* d_out, void* stream);

/* ---- host -> device upload of the input arrays ------------------------- */
/* Synchronous copy of `bytes` from pageable host memory (the reference hands
 * the COO tensor over as numpy arrays: SparseTensorCoo, coo.py:23-75) to
 * device memory through pinned staging buffers filled by `threads` host
 * threads (0: all hardware threads) with overlapped DMA.  The caller orders
 * it against its streams (the copy runs on internal streams). */
int sptk_h2d(void* d_dst, const void* h_src, size_t bytes, int threads);

/* ---- COO text ingestion (host) ---------------------------------------- */
/* load_coo(path, index_base) (coo.py:90-148), multi-threaded: the file is
 * memory-mapped and parsed by `threads` host threads (0: all hardware
 * threads) with the reference's grammar and error order.  Returns 0; 1 = the
 * reference's CooFormatError (sptk_last_error(): "line N: <message>", the
 * earliest bad line in file order; N = 0 for whole-file errors); 2 = OS error
 * (open/mmap); 3 = an index outside int64 (the reference's OverflowError).
 * On success *handle owns the entries: sptk_coo_text_dims reads the dims (the
 * "# dims:" header if any, else max index + 1) and sptk_coo_text_take copies
 * indices (int64 [nnz, order], 0-based, C order) and values (float64 [nnz])
 * in file order into caller memory and frees the handle. */
int sptk_coo_text_parse(const char* path, int index_base, int threads, void** handle, int64_t* nnz, int* order);
int sptk_coo_text_dims(void* handle, int64_t* dims, int* from_header);
int sptk_coo_text_take(void* handle, int64_t* indices, double* values, int threads);
void sptk_coo_text_free(void* handle);

/* ---- K1: partition + device layout ------------------------------------ */
size_t sptk_partition_ws_bytes(long long nnz, int order, long long m);
/* d_idx int64 [nnz, order], d_vals f64 [nnz] -> d_rec (block-grouped records),
 * d_ids[nnz] (source id of each record: the concatenated block_entries),
 * d_pos_of_id[nnz] (inverse), d_block_off[m^order + 1] (record offset of each
 * block key).  Any of d_ids / d_pos_of_id may be NULL. */
int sptk_partition(const int64_t* d_idx, const double* d_vals, long long nnz, int order, const int64_t* h_dims,
                   long long m, int f64_records, int32_t* d_rec, int32_t* d_ids, int32_t* d_pos_of_id,
                   int32_t* d_block_off, void* d_ws, size_t ws_bytes, void* stream);
/* The fp32 record path of the two calls above with the packing moved to the
 * host side of the upload: sptk_h2d_pack converts the COO arrays (int64
 * indices [nnz, order], float64 values; indices < 2^31) into fp32 records
 * {i_0..i_{N-1}, value} in the upload threads' pinned staging buffers and
 * DMAs those (16 bytes per nonzero at order <= 3 instead of 8N + 8);
 * sptk_partition_records then groups device records (source order) by block
 * exactly like sptk_partition (m == 1: in place, d_rec_out == d_rec_src). */
int sptk_h2d_pack(int32_t* d_rec, const int64_t* h_idx, const double* h_vals, long long nnz, int order, int threads);
int sptk_partition_records(const int32_t* d_rec_src, long long nnz, int order, const int64_t* h_dims, long long m,
                           int32_t* d_rec_out, int32_t* d_ids, int32_t* d_pos_of_id, int32_t* d_block_off, void* d_ws,
                           size_t ws_bytes, void* stream);
int sptk_pack_records(const int64_t* d_idx, const double* d_vals, long long nnz, int order, int f64_records,
                      int32_t* d_rec, void* stream);

/* ---- K3: factor-row SGD (one pass over a visit list) ------------------- */
/* record index of the k-th visited sample = base + d_visit[k] (d_visit may be
 * NULL: k).  mode 0 = throughput (Hogwild, visit order), 1 = deterministic
 * (strictly sequential, reference operation order). */
int sptk_factor_pass(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit, long long base,
                     float* d_fac, const int64_t* h_foff, const float* d_cor, const int64_t* h_coff,
                     const int64_t* h_jr, int n_modes, int rcore, const double* h_gammas, const double* h_lambdas,
                     int mode, void* stream);
int sptk_factor_pass_f64(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit, long long base,
                         double* d_fac, const int64_t* h_foff, const double* d_cor, const int64_t* h_coff,
                         const int64_t* h_jr, int n_modes, int rcore, const double* h_gammas,
                         const double* h_lambdas, int mode, void* stream);

/* Exact (sequential-equivalent) factor pass across the whole GPU: the result
 * equals mode 1 of sptk_factor_pass (the reference's strictly sequential
 * loop, _loops.py:17-63, bit for bit) but every sample runs as soon as the
 * earlier samples sharing one of its rows are done (per-mode predecessors
 * from a stable sort of the visit positions by row), so the critical path is
 * the longest row chain instead of the visit length.  d_ws: at least
 * sptk_factor_pass_exact_ws_bytes(n_visit, n_modes) bytes. */
size_t sptk_factor_pass_exact_ws_bytes(long long n_visit, int n_modes);
int sptk_factor_pass_exact(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit, long long base,
                           float* d_fac, const int64_t* h_foff, const float* d_cor, const int64_t* h_coff,
                           const int64_t* h_jr, int n_modes, int rcore, const double* h_gammas,
                           const double* h_lambdas, void* d_ws, size_t ws_bytes, void* stream);
int sptk_factor_pass_exact_f64(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit,
                               long long base, double* d_fac, const int64_t* h_foff, const double* d_cor,
                               const int64_t* h_coff, const int64_t* h_jr, int n_modes, int rcore,
                               const double* h_gammas, const double* h_lambdas, void* d_ws, size_t ws_bytes,
                               void* stream);

/* ---- multi-GPU DSGD, fused (one launch per rank per epoch) ------------- */
/* One rank's factor phase of a whole DSGD epoch (trainer.py:189-208 with the
 * rounds of partition.py:100-117 spread over processes/GPUs): d_visit holds
 * the rank's block of each round, round after round, each round padded with
 * -1 entries to whole 128-sample tiles; round r occupies
 * [d_rstart[r], d_rstart[r+1]) with valid samples below d_rend[r].  Tiles of
 * round r >= 1 start once *d_ready >= gen0 + r (the block rotated in for
 * round r has landed); after its last tile of round r the rank copies the
 * block described by d_push[r] (sptk_dsgd_push_bytes() bytes each: {int64
 * row_lo, int64 nrows, int64 mode, float* dst, int32* dst_ready, int32*
 * dst_gathered}; nrows = 0: none) to its next owner's model (peer pointer:
 * NVLink stores) -- once that rank's epoch flag *dst_gathered >= epoch, i.e.
 * its previous epoch-end exchange has been written -- and raises that rank's
 * ready flag to gen0 + r + 1 (release, system scope).  d_done:
 * n_rounds ints of scratch.  grid > 0 caps the persistent grid (all CTAs of
 * every rank sharing a GPU must be resident).  Uniform J = R, TMA kernel
 * shapes (order 3/4 at J = 16, 3/6 at J = 8); grid < 0 divides the default
 * grid by -grid (M-way DSGD: the per-row concurrency of one GPU). */
int sptk_factor_pass_dsgd(const int32_t* d_rec, int rw, const int32_t* d_visit, long long n_visit, float* d_fac,
                          const int64_t* h_foff, const float* d_cor, const int64_t* h_coff, const int64_t* h_jr,
                          int n_modes, int rcore, const double* h_gammas, const double* h_lambdas,
                          const long long* d_rstart, const long long* d_rend, const void* d_push, int32_t* d_done,
                          int32_t* d_ready, int n_rounds, int gen0, int epoch, int grid, void* stream);
size_t sptk_dsgd_push_bytes(void);
/* *d_flag = max(*d_flag, value) at system scope, in stream order (a rank's
 * epoch flag after its epoch-end exchange). */
int sptk_flag_store(int32_t* d_flag, int value, void* stream);
/* Device memory other processes can map (cudaMalloc'd, zeroed) and its CUDA
 * IPC handle (64 bytes); sptk_ipc_open maps a peer's allocation (peer access
 * enabled lazily: NVLink loads/stores on NVSwitch systems). */
int sptk_shared_alloc(size_t bytes, void** d_ptr);
int sptk_shared_free(void* d_ptr);
int sptk_ipc_get(void* d_ptr, unsigned char* h_handle);
int sptk_ipc_open(const unsigned char* h_handle, void** d_ptr);
int sptk_ipc_close(void* d_ptr);

/* ---- K4/K5: core gradient + apply ------------------------------------- */
size_t sptk_core_ws_bytes(const int64_t* h_jr, int n_modes, int rcore, int exact_chunks);
/* d_acc (fp64, layout coff) += sum over visited samples.  sample id of the
 * k-th entry = d_visit[k] (or k); record index = d_map[id] (or id).
 * exact_chunks = 0: throughput reduction; > 0: verification mode, the visit
 * list split like np.array_split(psi, exact_chunks), accumulated in order and
 * merged in chunk order (trainer.py:221-240). */
int sptk_core_pass(const int32_t* d_rec, int rw, const int32_t* d_visit, const int32_t* d_map, long long n_visit,
                   const float* d_fac, const int64_t* h_foff, const float* d_cor, const int64_t* h_coff,
                   const int64_t* h_jr, int n_modes, int rcore, double* d_acc, int exact_chunks, void* d_ws,
                   size_t ws_bytes, void* stream);
int sptk_core_pass_f64(const int32_t* d_rec, int rw, const int32_t* d_visit, const int32_t* d_map,
                       long long n_visit, const double* d_fac, const int64_t* h_foff, const double* d_cor,
                       const int64_t* h_coff, const int64_t* h_jr, int n_modes, int rcore, double* d_acc,
                       int exact_chunks, void* d_ws, size_t ws_bytes, void* stream);
/* B <- B - gamma_b * (acc/denom + lambda_b * B) over cor_size entries. */
int sptk_core_apply(float* d_cor, const double* d_acc, int cor_size, double gamma_b, double lambda_b, double denom,
                    void* stream);
int sptk_core_apply_f64(double* d_cor, const double* d_acc, int cor_size, double gamma_b, double lambda_b,
                        double denom, void* stream);

/* ---- K6: predictions / RMSE / MAE ------------------------------------- */
/* d_pred[m] (may be NULL) = predictions; d_sums[2] (may be NULL) +=
 * {sum (x - x_hat)^2, sum |x - x_hat|} in fp64. */
int sptk_eval(const int32_t* d_rec, int rw, long long m, const float* d_fac, const int64_t* h_foff,
              const float* d_cor, const int64_t* h_coff, const int64_t* h_jr, int n_modes, int rcore, float* d_pred,
              double* d_sums, void* stream);
int sptk_eval_f64(const int32_t* d_rec, int rw, long long m, const double* d_fac, const int64_t* h_foff,
                  const double* d_cor, const int64_t* h_coff, const int64_t* h_jr, int n_modes, int rcore,
                  double* d_pred, double* d_sums, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPTK_H */
