// Pinned staging ring + host copy pool for uploads (see host_stage.hpp).
#include "host_stage.hpp"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "device.hpp"
#include "kernels.h"

namespace pdlp_host {
namespace {

constexpr size_t kDirectMax = size_t(1) << 20;  // below this: plain cudaMemcpyAsync
#ifndef PDLPH_STAGE_CHUNK_MB
#define PDLPH_STAGE_CHUNK_MB 8
#endif
#ifndef PDLPH_STAGE_SLOTS
#define PDLPH_STAGE_SLOTS 6
#endif
#ifndef PDLPH_STAGE_THREADS
#define PDLPH_STAGE_THREADS 12
#endif
constexpr size_t kChunk = size_t(PDLPH_STAGE_CHUNK_MB) << 20;  // bytes per ring slot
constexpr int kSlots = PDLPH_STAGE_SLOTS;                      // ring depth
constexpr size_t kMinPart = size_t(256) << 10;  // smallest per-thread memcpy

// Fixed pool of memcpy workers; run() splits one chunk copy across them and
// returns when every part is done (the caller copies part 0 itself).
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int workers = static_cast<int>(std::min<unsigned>(PDLPH_STAGE_THREADS, hw)) - 1;
    for (int i = 0; i < workers; ++i) threads_.emplace_back([this, i] { loop(i + 1); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int width() const { return static_cast<int>(threads_.size()) + 1; }

  // narrow: src holds len / 4 int64 values, dst receives them as saturated
  // int32 (len = destination bytes)
  void run(char* dst, const char* src, size_t len, bool narrow = false) {
    const int parts = static_cast<int>(
        std::max<size_t>(1, std::min<size_t>(width(), (len + kMinPart - 1) / kMinPart)));
    if (parts == 1) {
      narrow_ = narrow;
      dst_ = dst;
      src_ = src;
      len_ = len;
      parts_ = 1;
      copy_part(0);
      return;
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      dst_ = dst;
      src_ = src;
      len_ = len;
      narrow_ = narrow;
      parts_ = parts;
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    copy_part(0);
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void copy_part(int i) const {
    size_t per = (len_ + parts_ - 1) / parts_;
    per = (per + 7) & ~size_t(7);  // whole 4- and 8-byte elements per part
    const size_t lo = std::min(len_, per * i), hi = std::min(len_, lo + per);
    if (hi <= lo) return;
    if (!narrow_) {
      std::memcpy(dst_ + lo, src_ + lo, hi - lo);
      return;
    }
    int32_t* d = reinterpret_cast<int32_t*>(dst_ + lo);
    const int64_t* v = reinterpret_cast<const int64_t*>(src_) + lo / 4;
    const size_t n = (hi - lo) / 4;
    for (size_t k = 0; k < n; ++k) {
      const int64_t x = v[k];
      d[k] = x < 0 ? -1 : (x > INT32_MAX ? INT32_MAX : static_cast<int32_t>(x));
    }
  }
  void loop(int id) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> g(mu_);
      cv_.wait(g, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      if (id >= parts_) continue;
      g.unlock();
      copy_part(id);
      g.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }

  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t len_ = 0;
  bool narrow_ = false;
  int parts_ = 0;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct Ring {
  char* slot[kSlots] = {};
  // The last DMA that touched each slot (recorded on that call's stream):
  // a slot is reused only after it completes, so calls need not drain the
  // ring and successive uploads overlap.  Events belong to one device; a call
  // on another device waits for them and recreates them there.
  cudaEvent_t ev[kSlots] = {};
  bool pending[kSlots] = {};
  int device = -1;
  int next = 0;  // round-robin slot cursor
  CopyPool pool;
  std::mutex mu;  // one transfer at a time
  bool ok = false;
  Ring() {
    // Portable pinned memory: usable from every device's streams.  Kept for
    // the life of the process (freeing at exit races the runtime teardown).
    char* p = nullptr;
    if (cudaHostAlloc(reinterpret_cast<void**>(&p), kChunk * kSlots, cudaHostAllocPortable) !=
        cudaSuccess) {
      cudaGetLastError();
      return;
    }
    for (int i = 0; i < kSlots; ++i) slot[i] = p + kChunk * i;
    ok = true;
  }
  // Caller holds mu.
  void bind_device() {
    int d = 0;
    PDLP_CK(cudaGetDevice(&d));
    if (d == device) return;
    for (int k = 0; k < kSlots; ++k) {
      if (ev[k] != nullptr) {
        if (pending[k]) cudaEventSynchronize(ev[k]);
        cudaEventDestroy(ev[k]);
        ev[k] = nullptr;
      }
      pending[k] = false;
    }
    for (int k = 0; k < kSlots; ++k) {
      PDLP_CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    }
    device = d;
  }
  // Slot k is free for the host (its last DMA has completed).
  cudaError_t acquire(int k) {
    if (!pending[k]) return cudaSuccess;
    pending[k] = false;
    return cudaEventSynchronize(ev[k]);
  }
  cudaError_t release(int k, cudaStream_t s) {
    pending[k] = true;
    return cudaEventRecord(ev[k], s);
  }
};

Ring& ring() {
  static Ring* r = new Ring();  // intentionally leaked, see Ring()
  return *r;
}

// src bytes per destination byte: 2 when narrowing int64 -> int32
// PDLP_TIMING: time in slot waits vs host copies (stage_report()).
double g_wait_s = 0.0, g_copy_s = 0.0, g_bytes = 0.0;

void stage_h2d_impl(void* dst, const void* src, size_t bytes, cudaStream_t s, bool narrow) {
  Ring& R = ring();
  std::lock_guard<std::mutex> g(R.mu);
  R.bind_device();
  using C = std::chrono::steady_clock;
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  const size_t ratio = narrow ? 2 : 1;
  cudaError_t err = cudaSuccess;
  for (size_t off = 0; off < bytes && err == cudaSuccess; off += kChunk) {
    const int k = R.next;
    R.next = (R.next + 1) % kSlots;
    const size_t len = std::min(kChunk, bytes - off);
    const auto t0 = C::now();
    if ((err = R.acquire(k)) != cudaSuccess) break;
    const auto t1 = C::now();
    R.pool.run(R.slot[k], in + off * ratio, len, narrow);
    const auto t2 = C::now();
    g_wait_s += std::chrono::duration<double>(t1 - t0).count();
    g_copy_s += std::chrono::duration<double>(t2 - t1).count();
    g_bytes += static_cast<double>(len);
    if ((err = cudaMemcpyAsync(out + off, R.slot[k], len, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      break;
    err = R.release(k, s);
  }
  PDLP_CK(err);
}

}  // namespace

void stage_report(double* wait_s, double* copy_s, double* mbytes) {
  *wait_s = g_wait_s;
  *copy_s = g_copy_s;
  *mbytes = g_bytes / 1048576.0;
  g_wait_s = g_copy_s = g_bytes = 0.0;
}

// Page-locked host memory (cudaHostAlloc'd or registered, e.g. through
// pdlp_host_register): the copy engine reads it directly, so uploads from it
// skip the ring's host copies.
bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void stage_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (bytes <= kDirectMax || !ring().ok || is_pinned(src)) {
    PDLP_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  stage_h2d_impl(dst, src, bytes, s, false);
}

void stage_h2d_narrow(int32_t* dst, const int64_t* src, size_t count, cudaStream_t s) {
  if (count == 0) return;
  if (count * 8 > kDirectMax && is_pinned(src)) {
    // pinned source: DMA the 64-bit values into a device chunk, narrow there
    // (same saturation as the host path); stream order reuses the chunk
    const size_t chunk = std::min(count, size_t(32) << 20);
    int64_t* tmp = nullptr;  // allocated and freed on s: ordered after its last use
    PDLP_CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), chunk * 8, s));
    cudaError_t err = cudaSuccess;
    for (size_t off = 0; off < count && err == cudaSuccess; off += chunk) {
      const size_t n = std::min(chunk, count - off);
      err = cudaMemcpyAsync(tmp, src + off, n * 8, cudaMemcpyHostToDevice, s);
      if (err == cudaSuccess) {
        err = static_cast<cudaError_t>(pdlpk_narrow_i64(tmp, dst + off, static_cast<int64_t>(n), s));
      }
    }
    cudaFreeAsync(tmp, s);
    PDLP_CK(err);
    return;
  }
  if (!ring().ok || count * 8 <= kDirectMax) {
    // small: narrow on the host into a temporary, one pageable copy
    std::vector<int32_t> tmp(count);
    for (size_t k = 0; k < count; ++k) {
      const int64_t x = src[k];
      tmp[k] = x < 0 ? -1 : (x > INT32_MAX ? INT32_MAX : static_cast<int32_t>(x));
    }
    PDLP_CK(cudaMemcpyAsync(dst, tmp.data(), count * 4, cudaMemcpyHostToDevice, s));
    PDLP_CK(cudaStreamSynchronize(s));  // tmp dies here
    return;
  }
  stage_h2d_impl(dst, src, count * 4, s, true);
}

void stage_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  Ring& R = ring();
  if (bytes <= kDirectMax || !R.ok || is_pinned(dst)) {
    PDLP_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    PDLP_CK(cudaStreamSynchronize(s));
    return;
  }
  std::lock_guard<std::mutex> g(R.mu);
  R.bind_device();
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  const size_t chunks = (bytes + kChunk - 1) / kChunk;
  cudaError_t err = cudaSuccess;
  auto issue = [&](size_t c) {
    const int k = static_cast<int>(c % kSlots);
    const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
    if (err == cudaSuccess) err = R.acquire(k);  // an upload may still read it
    if (err == cudaSuccess) err = cudaMemcpyAsync(R.slot[k], in + off, len, cudaMemcpyDeviceToHost, s);
    if (err == cudaSuccess) err = R.release(k, s);
  };
  size_t issued = 0;
  for (; issued < chunks && issued < static_cast<size_t>(kSlots); ++issued) issue(issued);
  for (size_t c = 0; c < chunks && err == cudaSuccess; ++c) {
    const int k = static_cast<int>(c % kSlots);
    if ((err = R.acquire(k)) != cudaSuccess) break;
    const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
    R.pool.run(out + off, R.slot[k], len);
    if (issued < chunks) issue(issued++);  // the slot is free again
  }
  if (err != cudaSuccess) cudaStreamSynchronize(s);  // no DMA may outlive the ring lock
  PDLP_CK(err);
}

}  // namespace pdlp_host
