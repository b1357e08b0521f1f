// upload.cu -- host -> device copy of large host arrays (the COO indices and
// values the reference's API hands over as numpy arrays, coo.py:23-75) at
// PCIe speed instead of the pageable-copy rate.
//
// A pageable cudaMemcpy is bounded by one host thread staging the bytes into
// the driver's pinned bounce buffer (~11 GB/s measured for the 2.4 GB NF index
// array).  Here T host threads each own a contiguous slice of the source, two
// pinned staging buffers and a stream: a thread copies the next piece of its
// slice into the idle buffer (after that buffer's previous DMA completed) and
// enqueues its DMA, so host copies of all threads and the DMAs overlap.  The
// staging buffers are allocated once per process and reused.  Synchronous on
// return, like the pageable copy it replaces.
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace sptk {

namespace {
constexpr size_t kPiece = 8u << 20;  // bytes per staging buffer
struct Lane {
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
};
std::mutex g_mu;
std::vector<Lane> g_lanes;
int g_dev = -1;

int ensure_lanes(int T) {
  int dev = 0;
  SPTK_CUDA_TRY(cudaGetDevice(&dev));
  if (g_dev != dev) {  // staging is per device (streams/events belong to one)
    for (auto& l : g_lanes) {
      for (int b = 0; b < 2; ++b) {
        if (l.buf[b]) cudaFreeHost(l.buf[b]);
        if (l.ev[b]) cudaEventDestroy(l.ev[b]);
      }
      if (l.st) cudaStreamDestroy(l.st);
    }
    g_lanes.clear();
    g_dev = dev;
  }
  while ((int)g_lanes.size() < T) {
    Lane l;
    for (int b = 0; b < 2; ++b) {
      SPTK_CUDA_TRY(cudaHostAlloc((void**)&l.buf[b], kPiece, cudaHostAllocDefault));
      SPTK_CUDA_TRY(cudaEventCreateWithFlags(&l.ev[b], cudaEventDisableTiming));
    }
    SPTK_CUDA_TRY(cudaStreamCreateWithFlags(&l.st, cudaStreamNonBlocking));
    g_lanes.push_back(l);
  }
  return 0;
}
}  // namespace

int h2d(void* dst, const void* src, size_t bytes, int threads) {
  if (bytes == 0) return 0;
  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (const char* e = getenv("SPTK_H2D_THREADS")) T = atoi(e);
  if (T < 1) T = 1;
  if (T > 32) T = 32;
  const size_t per = (bytes + T - 1) / T;
  if (per < kPiece) T = (int)((bytes + kPiece - 1) / kPiece);  // small copies: fewer lanes
  std::lock_guard<std::mutex> lk(g_mu);
  if (ensure_lanes(T)) return 1;
  int dev = g_dev;
  std::vector<int> rc(T, 0);
  std::vector<std::thread> th;
  const size_t slice = (bytes + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    th.emplace_back([&, t]() {
      cudaSetDevice(dev);
      Lane& l = g_lanes[t];
      const size_t lo = (size_t)t * slice, hi = lo + slice < bytes ? lo + slice : bytes;
      int b = 0;
      for (size_t off = lo; off < hi; off += kPiece, b ^= 1) {
        const size_t n = hi - off < kPiece ? hi - off : kPiece;
        if (cudaEventSynchronize(l.ev[b]) != cudaSuccess) { rc[t] = 1; return; }
        memcpy(l.buf[b], (const char*)src + off, n);
        if (cudaMemcpyAsync((char*)dst + off, l.buf[b], n, cudaMemcpyHostToDevice, l.st) != cudaSuccess ||
            cudaEventRecord(l.ev[b], l.st) != cudaSuccess) {
          rc[t] = 1;
          return;
        }
      }
      if (cudaStreamSynchronize(l.st) != cudaSuccess) rc[t] = 1;
    });
  }
  for (auto& x : th) x.join();
  for (int t = 0; t < T; ++t)
    if (rc[t]) {
      set_error("h2d: CUDA error in upload lane %d: %s", t, cudaGetErrorString(cudaGetLastError()));
      return 1;
    }
  return 0;
}

// The COO arrays packed into device records on the way: every lane converts
// its slice of nonzeros (int64 indices, float64 value) into the fp32 record
// layout {i_0..i_{N-1} (int32), value (fp32)} in its pinned staging buffer and
// DMAs that -- 16 bytes per nonzero over PCIe instead of 8N + 8 (NF: 1.6 GB
// instead of 3.2 GB).  Indices must fit int32 (checked by the caller).
int h2d_pack_records(int* d_rec, const long long* h_idx, const double* h_vals, long long nnz, int order, int rw,
                     int threads) {
  if (nnz <= 0) return 0;
  SPTK_REQUIRE(order >= 1 && order < rw, "h2d_pack_records: bad order %d for %d-word records", order, rw);
  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (const char* e = getenv("SPTK_H2D_THREADS")) T = atoi(e);
  if (T < 1) T = 1;
  if (T > 32) T = 32;
  const long long per_piece = (long long)(kPiece / ((size_t)rw * 4));
  if ((nnz + T - 1) / T < per_piece) T = (int)((nnz + per_piece - 1) / per_piece);
  std::lock_guard<std::mutex> lk(g_mu);
  if (ensure_lanes(T)) return 1;
  int dev = g_dev;
  std::vector<int> rc(T, 0);
  std::vector<std::thread> th;
  const long long slice = (nnz + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    th.emplace_back([&, t]() {
      cudaSetDevice(dev);
      Lane& l = g_lanes[t];
      const long long lo = (long long)t * slice, hi = lo + slice < nnz ? lo + slice : nnz;
      int b = 0;
      for (long long a = lo; a < hi; a += per_piece, b ^= 1) {
        const long long n = hi - a < per_piece ? hi - a : per_piece;
        if (cudaEventSynchronize(l.ev[b]) != cudaSuccess) {
          rc[t] = 1;
          return;
        }
        int* out = reinterpret_cast<int*>(l.buf[b]);
        for (long long k = 0; k < n; ++k) {
          const long long* ix = h_idx + (a + k) * order;
          int* r = out + k * rw;
          for (int q = 0; q < order; ++q) r[q] = (int)ix[q];
          const float v = (float)h_vals[a + k];
          memcpy(r + order, &v, 4);
          for (int q = order + 1; q < rw; ++q) r[q] = 0;
        }
        if (cudaMemcpyAsync(d_rec + a * rw, l.buf[b], (size_t)n * rw * 4, cudaMemcpyHostToDevice, l.st) !=
                cudaSuccess ||
            cudaEventRecord(l.ev[b], l.st) != cudaSuccess) {
          rc[t] = 1;
          return;
        }
      }
      if (cudaStreamSynchronize(l.st) != cudaSuccess) rc[t] = 1;
    });
  }
  for (auto& x : th) x.join();
  for (int t = 0; t < T; ++t)
    if (rc[t]) {
      set_error("h2d_pack_records: CUDA error in upload lane %d: %s", t, cudaGetErrorString(cudaGetLastError()));
      return 1;
    }
  return 0;
}

}  // namespace sptk
