// Pinned staging ring for the host entries (hostio.cuh).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>
#include "hostio.cuh"

namespace bse {
namespace {

constexpr size_t kStageBytes = size_t(128) << 20;  // per buffer
constexpr int kStageBufs = 2;
constexpr int kCopyThreads = 8;

struct Stage {
  char* buf[kStageBufs] = {};
  cudaEvent_t done[kStageBufs] = {};
  bool ready = false;
};

std::mutex g_mu;  // one staged transfer at a time per process

Stage& stage() {
  static Stage st;
  return st;
}

cudaError_t ensure(Stage& st) {
  if (st.ready) return cudaSuccess;
  for (int b = 0; b < kStageBufs; ++b) {
    cudaError_t e = cudaHostAlloc((void**)&st.buf[b], kStageBytes, cudaHostAllocPortable);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&st.done[b], cudaEventDisableTiming)) != cudaSuccess)
      return e;
  }
  st.ready = true;
  return cudaSuccess;
}

// copy `rows` rows of `row_bytes` (pitches dp, sp) with up to kCopyThreads threads
void par_copy(char* dst, size_t dp, const char* src, size_t sp, size_t row_bytes, size_t rows) {
  const size_t total = row_bytes * rows;
  const int nt = (int)std::min<size_t>(kCopyThreads, std::max<size_t>(1, total >> 22));
  auto work = [&](int t) {
    if (dp == row_bytes && sp == row_bytes) {
      const size_t per = (total + nt - 1) / nt;
      const size_t a = std::min(total, per * t), b = std::min(total, a + per);
      if (b > a) std::memcpy(dst + a, src + a, b - a);
      return;
    }
    for (size_t r = t; r < rows; r += nt) std::memcpy(dst + r * dp, src + r * sp, row_bytes);
  };
  if (nt == 1) {
    work(0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

}  // namespace

cudaError_t h2d_staged(void* dst, size_t dpitch, const void* src, size_t spitch,
                       size_t row_bytes, size_t rows, cudaStream_t s) {
  if (rows == 0 || row_bytes == 0) return cudaSuccess;
  std::lock_guard<std::mutex> lk(g_mu);
  Stage& st = stage();
  cudaError_t e = ensure(st);
  if (e != cudaSuccess) return e;
  const size_t rows_per = std::max<size_t>(1, kStageBytes / row_bytes);
  if (rows_per * row_bytes > kStageBytes)  // a single row larger than a stage buffer
    return cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, cudaMemcpyHostToDevice, s);
  int b = 0;
  for (size_t r0 = 0; r0 < rows; r0 += rows_per, b = (b + 1) % kStageBufs) {
    const size_t nr = std::min(rows_per, rows - r0);
    if ((e = cudaEventSynchronize(st.done[b])) != cudaSuccess) return e;  // buffer free
    par_copy(st.buf[b], row_bytes, static_cast<const char*>(src) + r0 * spitch, spitch, row_bytes,
             nr);
    if ((e = cudaMemcpy2DAsync(static_cast<char*>(dst) + r0 * dpitch, dpitch, st.buf[b], row_bytes,
                               row_bytes, nr, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return e;
    if ((e = cudaEventRecord(st.done[b], s)) != cudaSuccess) return e;
  }
  // the ring must not be refilled by another caller before these DMAs end
  for (int q = 0; q < kStageBufs; ++q)
    if ((e = cudaEventSynchronize(st.done[q])) != cudaSuccess) return e;
  return cudaSuccess;
}

cudaError_t d2h_staged(void* dst, size_t dpitch, const void* src, size_t spitch,
                       size_t row_bytes, size_t rows, cudaStream_t s) {
  if (rows == 0 || row_bytes == 0) return cudaSuccess;
  std::lock_guard<std::mutex> lk(g_mu);
  Stage& st = stage();
  cudaError_t e = ensure(st);
  if (e != cudaSuccess) return e;
  const size_t rows_per = std::max<size_t>(1, kStageBytes / row_bytes);
  if (rows_per * row_bytes > kStageBytes) {
    if ((e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, cudaMemcpyDeviceToHost,
                               s)) != cudaSuccess)
      return e;
    return cudaStreamSynchronize(s);
  }
  const size_t nchunks = (rows + rows_per - 1) / rows_per;
  // DMA chunk k into buffer k % 2; copy chunk k out of it while chunk k+1 lands
  auto issue = [&](size_t k) -> cudaError_t {
    const size_t r0 = k * rows_per, nr = std::min(rows_per, rows - r0);
    const int b = (int)(k % kStageBufs);
    cudaError_t ee = cudaMemcpy2DAsync(st.buf[b], row_bytes,
                                       static_cast<const char*>(src) + r0 * spitch, spitch,
                                       row_bytes, nr, cudaMemcpyDeviceToHost, s);
    if (ee == cudaSuccess) ee = cudaEventRecord(st.done[b], s);
    return ee;
  };
  if ((e = issue(0)) != cudaSuccess) return e;
  for (size_t k = 0; k < nchunks; ++k) {
    const int b = (int)(k % kStageBufs);
    if ((e = cudaEventSynchronize(st.done[b])) != cudaSuccess) return e;
    if (k + 1 < nchunks && (e = issue(k + 1)) != cudaSuccess) return e;
    const size_t r0 = k * rows_per, nr = std::min(rows_per, rows - r0);
    par_copy(static_cast<char*>(dst) + r0 * dpitch, dpitch, st.buf[b], row_bytes, row_bytes, nr);
  }
  return cudaSuccess;
}

}  // namespace bse
