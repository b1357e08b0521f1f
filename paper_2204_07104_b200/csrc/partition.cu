// partition.cu -- K1: block partition and device re-layout of the COO data.
//
// Restates build_partition (partition.py:47-81): mode n is cut at
// floor(k * I_n / m); an entry's block component is the last cut <= its index
// (searchsorted(cuts, i, 'right') - 1); the block key is
// sum_n bucket_n * m^(N-1-n) (mode 0 most significant), and entries are
// grouped by a STABLE sort on the key so source order is kept inside every
// block.  The stable sort is an LSD radix sort (8-bit digits, per-tile
// histograms, ordered scan, stable scatter with warp match ranking).
//
// The grouped entries are then packed into the device layout the kernels
// read: one 16/32/64-byte record per nonzero {i_0..i_{N-1}, value} with
// int32 indices, blocks contiguous, plus block offsets and the inverse map
// (source id -> record) used by the core batch.
#include "common.cuh"
#include "kernels.cuh"

namespace sptk {

#define RX_THREADS 256
#define RX_ITEMS 8
#define RX_TILE (RX_THREADS * RX_ITEMS)

__global__ void keys_kernel(const long long* __restrict__ idx, long long nnz, int N, MDims md, long long m,
                            unsigned* __restrict__ keys) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; e < nnz; e += stride) {
    unsigned long long key = 0;
    for (int n = 0; n < N; ++n) {
      long long i = idx[e * N + n];
      long long d = md.d[n];
      // largest b in [0, m-1] with floor(b*d/m) <= i
      long long lo = 0, hi = m;
      while (hi - lo > 1) {
        long long mid = (lo + hi) >> 1;
        if ((mid * d) / m <= i) lo = mid;
        else hi = mid;
      }
      key = key * (unsigned long long)m + (unsigned long long)lo;
    }
    keys[e] = (unsigned)key;
  }
}

__global__ void __launch_bounds__(RX_THREADS) radix_hist_kernel(const unsigned* __restrict__ keys, long long n,
                                                                int shift, int ntiles, int* __restrict__ hist) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  long long base = (long long)blockIdx.x * RX_TILE;
  for (int k = 0; k < RX_ITEMS; ++k) {
    long long i = base + (long long)k * RX_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1);
  }
  __syncthreads();
  hist[(long long)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter of one 8-bit digit pass.  Each tile's elements are first
// ranked (warp match + per-warp counts, round by round, in source order) into
// a digit-sorted copy in shared memory, then written out so that consecutive
// threads store consecutive elements of the same digit (coalesced runs).
__global__ void __launch_bounds__(RX_THREADS) radix_scatter_kernel(const unsigned* __restrict__ kin,
                                                                   const int* __restrict__ vin, long long n,
                                                                   int shift, int ntiles,
                                                                   const int* __restrict__ offs,
                                                                   const int* __restrict__ hist,
                                                                   unsigned* __restrict__ kout,
                                                                   int* __restrict__ vout) {
  __shared__ int run[256];        // next local slot per digit
  __shared__ int lstart[256];     // tile-local start of each digit
  __shared__ int gstart[256];     // global start of each digit for this tile
  __shared__ int wcnt[RX_THREADS / 32][256];
  __shared__ unsigned sk[RX_TILE];
  __shared__ int sv[RX_TILE];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  {
    // tile-local exclusive scan of this tile's digit counts
    const int c = hist[(long long)threadIdx.x * ntiles + blockIdx.x];
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wcnt[0][w] = incl;
    __syncthreads();
    int pre = 0;
    for (int q = 0; q < w; ++q) pre += wcnt[0][q];
    lstart[threadIdx.x] = pre + incl - c;
    run[threadIdx.x] = pre + incl - c;
    gstart[threadIdx.x] = offs[(long long)threadIdx.x * ntiles + blockIdx.x];
    __syncthreads();
    for (int q = 0; q < RX_THREADS / 32; ++q) wcnt[q][threadIdx.x] = 0;
    __syncthreads();
  }
  const long long base = (long long)blockIdx.x * RX_TILE;
  const unsigned lt = (1u << lane) - 1u;
  for (int k = 0; k < RX_ITEMS; ++k) {
    long long i = base + (long long)k * RX_THREADS + threadIdx.x;
    bool valid = i < n;
    unsigned key = valid ? kin[i] : 0u;
    int val = valid ? vin[i] : 0;
    int d = valid ? (int)((key >> shift) & 255u) : 256 + lane;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int rank = __popc(peers & lt);
    if (valid && rank == 0) wcnt[w][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      int pre = 0;
      for (int q = 0; q < w; ++q) pre += wcnt[q][d];
      int pos = run[d] + pre + rank;
      sk[pos] = key;
      sv[pos] = val;
    }
    __syncthreads();
    {
      int dd = threadIdx.x;
      int add = 0;
      for (int q = 0; q < RX_THREADS / 32; ++q) {
        add += wcnt[q][dd];
        wcnt[q][dd] = 0;
      }
      run[dd] += add;
    }
    __syncthreads();
  }
  const long long cnt = (n - base) < RX_TILE ? (n - base) : RX_TILE;
  for (int e = threadIdx.x; e < cnt; e += RX_THREADS) {
    const unsigned key = sk[e];
    const int d = (key >> shift) & 255u;
    const long long g = (long long)gstart[d] + (e - lstart[d]);
    kout[g] = key;
    vout[g] = sv[e];
  }
}

__global__ void iota_i32_kernel(int* __restrict__ out, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = (int)i;
}

__global__ void key_count_kernel(const unsigned* __restrict__ keys, long long n, int* __restrict__ cnt) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) atomicAdd(&cnt[keys[i]], 1);
}

__global__ void block_off1_kernel(int* __restrict__ off, int nnz) {
  if (threadIdx.x == 0) {
    off[0] = 0;
    off[1] = nnz;
  }
}

__global__ void pack_kernel(const long long* __restrict__ idx, const double* __restrict__ vals,
                            const int* __restrict__ ids, long long nnz, int N, int rw, int f64,
                            int* __restrict__ rec, int* __restrict__ pos_of_id) {
  long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  const int vo = rec_val_off(N, f64 != 0);
  for (; p < nnz; p += stride) {
    long long id = ids ? ids[p] : p;
    int* r = rec + p * rw;
    for (int n = 0; n < N; ++n) r[n] = (int)idx[id * N + n];
    for (int q = N; q < rw; ++q) r[q] = 0;
    if (f64) {
      *reinterpret_cast<double*>(r + vo) = vals[id];
    } else {
      r[vo] = __float_as_int((float)vals[id]);
    }
    if (pos_of_id) pos_of_id[id] = (int)p;
  }
}

static inline unsigned gridn(long long n, int t) {
  long long g = (n + t - 1) / t;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (unsigned)g;
}

size_t partition_ws_bytes(long long nnz, int order, long long m) {
  if (m == 1) return 4096;  // one block: no keys, no sort (see partition)
  long long nkeys = 1;
  for (int n = 0; n < order; ++n) nkeys *= m;
  long long ntiles = (nnz + RX_TILE - 1) / RX_TILE + 1;
  size_t b = 0;
  b += (size_t)(nnz + 1) * 4 * 4;                 // keys x2, vals x2
  b += (size_t)(256 * ntiles + 2) * 4 * 2;        // hist + offs
  b += scan_ws_bytes(256 * ntiles + 1) + 4096;
  b += (size_t)(nkeys + 2) * 4 + scan_ws_bytes(nkeys + 1) + 4096;
  return b + 16 * 256;
}

struct Carve2 {
  char* p;
  size_t left;
  bool bad = false;
  template <typename T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
    if (bytes > left) {
      bad = true;
      return (T*)p;
    }
    T* r = (T*)p;
    p += bytes;
    left -= bytes;
    return r;
  }
};

int partition(const long long* idx64, const double* vals64, long long nnz, int order, const long long* h_dims,
              long long m, int* rec_out, int* ids_out, int* pos_of_id_out, int* block_off_out, void* ws,
              size_t ws_bytes, cudaStream_t s, int f64) {
  SPTK_REQUIRE(order >= 2 && order <= SPTK_MAX_MODES, "partition: bad order");
  SPTK_REQUIRE(m >= 1, "partition: m must be >= 1");
  long long nkeys = 1;
  for (int n = 0; n < order; ++n) {
    SPTK_REQUIRE(m <= h_dims[n], "partition: m=%lld exceeds mode %d dimension %lld", m, n, h_dims[n]);
    nkeys *= m;
    SPTK_REQUIRE(nkeys < (1LL << 31), "partition: too many blocks");
  }
  SPTK_REQUIRE(nnz >= 0 && nnz < (1LL << 31), "partition: nnz out of range");
  SPTK_REQUIRE(ws_bytes >= partition_ws_bytes(nnz, order, m), "partition: workspace too small");
  if (m == 1) {
    // One block holding every entry in source order (the stable sort of
    // all-equal keys is the identity): pack, ids = pos_of_id = iota,
    // block_off = {0, nnz}.  No key or sort buffers.
    const int rw1 = rec_words_t(order, f64 != 0);
    if (nnz > 0) {
      pack_kernel<<<gridn(nnz, 256), 256, 0, s>>>(idx64, vals64, nullptr, nnz, order, rw1, f64, rec_out, nullptr);
      SPTK_CHECK_LAUNCH();
      for (int* o : {ids_out, pos_of_id_out})
        if (o) {
          iota_i32_kernel<<<gridn(nnz, 256), 256, 0, s>>>(o, nnz);
          SPTK_CHECK_LAUNCH();
        }
    }
    block_off1_kernel<<<1, 32, 0, s>>>(block_off_out, (int)nnz);
    SPTK_CHECK_LAUNCH();
    return 0;
  }
  Carve2 cv{(char*)ws, ws_bytes};
  unsigned* k0 = cv.take<unsigned>(nnz + 1);
  unsigned* k1 = cv.take<unsigned>(nnz + 1);
  int* v0 = cv.take<int>(nnz + 1);
  int* v1 = cv.take<int>(nnz + 1);
  long long ntiles = (nnz + RX_TILE - 1) / RX_TILE;
  if (ntiles < 1) ntiles = 1;
  int* hist = cv.take<int>(256 * ntiles + 2);
  int* offs = cv.take<int>(256 * ntiles + 2);
  int* sws = cv.take<int>(scan_ws_bytes(256 * ntiles + 1) / 4 + 1);
  int* kcnt = cv.take<int>(nkeys + 2);
  int* sws2 = cv.take<int>(scan_ws_bytes(nkeys + 1) / 4 + 1);
  SPTK_REQUIRE(!cv.bad, "partition: workspace carve failed");
  const int rw = rec_words_t(order, f64 != 0);
  MDims md;
  for (int n = 0; n < order; ++n) md.d[n] = h_dims[n];
  if (nnz > 0) {
    keys_kernel<<<gridn(nnz, 256), 256, 0, s>>>(idx64, nnz, order, md, m, k0);
    SPTK_CHECK_LAUNCH();
    iota_i32_kernel<<<gridn(nnz, 256), 256, 0, s>>>(v0, nnz);
    SPTK_CHECK_LAUNCH();
    int bits = 0;
    while ((1LL << bits) < nkeys) ++bits;
    unsigned* kin = k0;
    unsigned* kout = k1;
    int* vin = v0;
    int* vout = v1;
    for (int shift = 0; shift < bits; shift += 8) {
      radix_hist_kernel<<<(unsigned)ntiles, RX_THREADS, 0, s>>>(kin, nnz, shift, (int)ntiles, hist);
      SPTK_CHECK_LAUNCH();
      if (exclusive_scan(hist, 256 * ntiles, offs, sws, s)) return 1;
      radix_scatter_kernel<<<(unsigned)ntiles, RX_THREADS, 0, s>>>(kin, vin, nnz, shift, (int)ntiles, offs, hist,
                                                                   kout, vout);
      SPTK_CHECK_LAUNCH();
      unsigned* tk = kin;
      kin = kout;
      kout = tk;
      int* tv = vin;
      vin = vout;
      vout = tv;
    }
    SPTK_CUDA_TRY(cudaMemsetAsync(kcnt, 0, sizeof(int) * (nkeys + 1), s));
    key_count_kernel<<<gridn(nnz, 256), 256, 0, s>>>(kin, nnz, kcnt);
    SPTK_CHECK_LAUNCH();
    if (exclusive_scan(kcnt, nkeys, block_off_out, sws2, s)) return 1;
    if (ids_out) SPTK_CUDA_TRY(cudaMemcpyAsync(ids_out, vin, sizeof(int) * nnz, cudaMemcpyDeviceToDevice, s));
    pack_kernel<<<gridn(nnz, 256), 256, 0, s>>>(idx64, vals64, vin, nnz, order, rw, f64, rec_out, pos_of_id_out);
    SPTK_CHECK_LAUNCH();
  } else {
    SPTK_CUDA_TRY(cudaMemsetAsync(block_off_out, 0, sizeof(int) * (nkeys + 1), s));
  }
  return 0;
}

size_t radix_ws_bytes(long long n) {
  long long ntiles = (n + RX_TILE - 1) / RX_TILE;
  if (ntiles < 1) ntiles = 1;
  return (size_t)(256 * ntiles + 2) * 4 * 2 + scan_ws_bytes(256 * ntiles + 1) + 4 * 256;
}

// Stable LSD radix sort of (key, value) pairs on the low `bits` key bits,
// ping-ponging between (k0, v0) and (k1, v1); *kout / *vout get the result.
int radix_sort_pairs(unsigned* k0, int* v0, unsigned* k1, int* v1, long long n, int bits, void* ws, size_t ws_bytes,
                     cudaStream_t s, unsigned** kout, int** vout) {
  SPTK_REQUIRE(ws_bytes >= radix_ws_bytes(n), "radix_sort_pairs: workspace too small");
  long long ntiles = (n + RX_TILE - 1) / RX_TILE;
  if (ntiles < 1) ntiles = 1;
  Carve2 cv{(char*)ws, ws_bytes};
  int* hist = cv.take<int>(256 * ntiles + 2);
  int* offs = cv.take<int>(256 * ntiles + 2);
  int* sws = cv.take<int>(scan_ws_bytes(256 * ntiles + 1) / 4 + 1);
  unsigned* kin = k0;
  unsigned* kb = k1;
  int* vin = v0;
  int* vb = v1;
  for (int shift = 0; shift < bits && n > 0; shift += 8) {
    radix_hist_kernel<<<(unsigned)ntiles, RX_THREADS, 0, s>>>(kin, n, shift, (int)ntiles, hist);
    SPTK_CHECK_LAUNCH();
    if (exclusive_scan(hist, 256 * ntiles, offs, sws, s)) return 1;
    radix_scatter_kernel<<<(unsigned)ntiles, RX_THREADS, 0, s>>>(kin, vin, n, shift, (int)ntiles, offs, hist, kb, vb);
    SPTK_CHECK_LAUNCH();
    unsigned* tk = kin;
    kin = kb;
    kb = tk;
    int* tv = vin;
    vin = vb;
    vb = tv;
  }
  *kout = kin;
  *vout = vin;
  return 0;
}

__global__ void rec_keys_kernel(const int* __restrict__ rec, int rw, long long nnz, int N, MDims md, long long m,
                                unsigned* __restrict__ keys, int* __restrict__ vals) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; e < nnz; e += stride) {
    unsigned long long key = 0;
    for (int n = 0; n < N; ++n) {
      const long long i = rec[e * rw + n];
      const long long d = md.d[n];
      long long lo = 0, hi = m;  // largest b in [0, m-1] with floor(b*d/m) <= i
      while (hi - lo > 1) {
        const long long mid = (lo + hi) >> 1;
        if ((mid * d) / m <= i) lo = mid;
        else hi = mid;
      }
      key = key * (unsigned long long)m + (unsigned long long)lo;
    }
    keys[e] = (unsigned)key;
    vals[e] = (int)e;
  }
}

__global__ void rec_gather_kernel(const int* __restrict__ src, int rw, const int* __restrict__ ids, long long nnz,
                                  int* __restrict__ dst, int* __restrict__ pos_of_id) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < nnz; p += stride) {
    const long long id = ids[p];
    const int4* s4 = reinterpret_cast<const int4*>(src + id * rw);
    int4* d4 = reinterpret_cast<int4*>(dst + p * rw);
    for (int q = 0; q < rw / 4; ++q) d4[q] = s4[q];
    if (pos_of_id) pos_of_id[id] = (int)p;
  }
}

// K1 from records already on the device in source order (sptk_h2d_pack):
// the same stable block grouping as partition(), keys read from the records'
// int32 indices; rec_out receives the grouped records (m == 1: rec_src is
// already the layout -- pass rec_out == rec_src).
int partition_records(const int* rec_src, int rw, long long nnz, int order, const long long* h_dims, long long m,
                      int* rec_out, int* ids_out, int* pos_of_id_out, int* block_off_out, void* ws, size_t ws_bytes,
                      cudaStream_t s) {
  SPTK_REQUIRE(order >= 2 && order <= SPTK_MAX_MODES, "partition_records: bad order");
  SPTK_REQUIRE(m >= 1, "partition_records: m must be >= 1");
  long long nkeys = 1;
  for (int n = 0; n < order; ++n) {
    SPTK_REQUIRE(m <= h_dims[n], "partition_records: m=%lld exceeds mode %d dimension %lld", m, n, h_dims[n]);
    nkeys *= m;
    SPTK_REQUIRE(nkeys < (1LL << 31), "partition_records: too many blocks");
  }
  SPTK_REQUIRE(nnz >= 0 && nnz < (1LL << 31), "partition_records: nnz out of range");
  SPTK_REQUIRE(ws_bytes >= partition_ws_bytes(nnz, order, m), "partition_records: workspace too small");
  if (m == 1) {
    SPTK_REQUIRE(rec_out == rec_src, "partition_records: m == 1 keeps the records in place (rec_out == rec_src)");
    if (nnz > 0)
      for (int* o : {ids_out, pos_of_id_out})
        if (o) {
          iota_i32_kernel<<<gridn(nnz, 256), 256, 0, s>>>(o, nnz);
          SPTK_CHECK_LAUNCH();
        }
    block_off1_kernel<<<1, 32, 0, s>>>(block_off_out, (int)nnz);
    SPTK_CHECK_LAUNCH();
    return 0;
  }
  SPTK_REQUIRE(rec_out != rec_src, "partition_records: m > 1 needs a separate output buffer");
  Carve2 cv{(char*)ws, ws_bytes};
  unsigned* k0 = cv.take<unsigned>(nnz + 1);
  unsigned* k1 = cv.take<unsigned>(nnz + 1);
  int* v0 = cv.take<int>(nnz + 1);
  int* v1 = cv.take<int>(nnz + 1);
  long long ntiles = (nnz + RX_TILE - 1) / RX_TILE;
  if (ntiles < 1) ntiles = 1;
  int* hist = cv.take<int>(256 * ntiles + 2);
  int* offs = cv.take<int>(256 * ntiles + 2);
  int* sws = cv.take<int>(scan_ws_bytes(256 * ntiles + 1) / 4 + 1);
  int* kcnt = cv.take<int>(nkeys + 2);
  int* sws2 = cv.take<int>(scan_ws_bytes(nkeys + 1) / 4 + 1);
  SPTK_REQUIRE(!cv.bad, "partition_records: workspace carve failed");
  MDims md;
  for (int n = 0; n < order; ++n) md.d[n] = h_dims[n];
  if (nnz > 0) {
    rec_keys_kernel<<<gridn(nnz, 256), 256, 0, s>>>(rec_src, rw, nnz, order, md, m, k0, v0);
    SPTK_CHECK_LAUNCH();
    int bits = 0;
    while ((1LL << bits) < nkeys) ++bits;
    unsigned* kin = k0;
    unsigned* kout = k1;
    int* vin = v0;
    int* vout = v1;
    for (int shift = 0; shift < bits; shift += 8) {
      radix_hist_kernel<<<(unsigned)ntiles, RX_THREADS, 0, s>>>(kin, nnz, shift, (int)ntiles, hist);
      SPTK_CHECK_LAUNCH();
      if (exclusive_scan(hist, 256 * ntiles, offs, sws, s)) return 1;
      radix_scatter_kernel<<<(unsigned)ntiles, RX_THREADS, 0, s>>>(kin, vin, nnz, shift, (int)ntiles, offs, hist,
                                                                   kout, vout);
      SPTK_CHECK_LAUNCH();
      unsigned* tk = kin;
      kin = kout;
      kout = tk;
      int* tv = vin;
      vin = vout;
      vout = tv;
    }
    SPTK_CUDA_TRY(cudaMemsetAsync(kcnt, 0, sizeof(int) * (nkeys + 1), s));
    key_count_kernel<<<gridn(nnz, 256), 256, 0, s>>>(kin, nnz, kcnt);
    SPTK_CHECK_LAUNCH();
    if (exclusive_scan(kcnt, nkeys, block_off_out, sws2, s)) return 1;
    if (ids_out) SPTK_CUDA_TRY(cudaMemcpyAsync(ids_out, vin, sizeof(int) * nnz, cudaMemcpyDeviceToDevice, s));
    rec_gather_kernel<<<gridn(nnz, 256), 256, 0, s>>>(rec_src, rw, vin, nnz, rec_out, pos_of_id_out);
    SPTK_CHECK_LAUNCH();
  } else {
    SPTK_CUDA_TRY(cudaMemsetAsync(block_off_out, 0, sizeof(int) * (nkeys + 1), s));
  }
  return 0;
}

int pack_records(const long long* idx64, const double* vals64, long long nnz, int order, int* rec_out,
                 cudaStream_t s, int f64) {
  if (nnz <= 0) return 0;
  pack_kernel<<<gridn(nnz, 256), 256, 0, s>>>(idx64, vals64, nullptr, nnz, order, rec_words_t(order, f64 != 0),
                                               f64, rec_out, nullptr);
  SPTK_CHECK_LAUNCH();
  return 0;
}

}  // namespace sptk
