// Pinned staging ring + host copy pool for uploads (see host_stage.hpp).
#include "host_stage.hpp"

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "device.hpp"

namespace pdlp_host {
namespace {

constexpr size_t kDirectMax = size_t(1) << 20;  // below this: plain cudaMemcpyAsync
constexpr size_t kChunk = size_t(8) << 20;      // bytes per ring slot
constexpr int kSlots = 6;                       // ring depth
constexpr size_t kMinPart = size_t(256) << 10;  // smallest per-thread memcpy

// Fixed pool of memcpy workers; run() splits one chunk copy across them and
// returns when every part is done (the caller copies part 0 itself).
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int workers = static_cast<int>(std::min(12u, hw)) - 1;
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

  void run(char* dst, const char* src, size_t len) {
    const int parts = static_cast<int>(
        std::max<size_t>(1, std::min<size_t>(width(), (len + kMinPart - 1) / kMinPart)));
    if (parts == 1) {
      std::memcpy(dst, src, len);
      return;
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      dst_ = dst;
      src_ = src;
      len_ = len;
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
    const size_t per = (len_ + parts_ - 1) / parts_;
    const size_t lo = std::min(len_, per * i), hi = std::min(len_, lo + per);
    if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
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
  int parts_ = 0;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct Ring {
  char* slot[kSlots] = {};
  CopyPool pool;
  std::mutex mu;  // one upload at a time
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
};

Ring& ring() {
  static Ring* r = new Ring();  // intentionally leaked, see Ring()
  return *r;
}

}  // namespace

void stage_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (bytes <= kDirectMax) {
    PDLP_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  Ring& R = ring();
  if (!R.ok) {
    PDLP_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  std::lock_guard<std::mutex> g(R.mu);
  // Events belong to the current device, so they live for one upload; the
  // ring is drained before returning, which also frees the slots for the
  // next upload.
  cudaEvent_t ev[kSlots];
  for (int i = 0; i < kSlots; ++i) PDLP_CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  bool used[kSlots] = {};
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  cudaError_t err = cudaSuccess;
  int i = 0;
  for (size_t off = 0; off < bytes && err == cudaSuccess; off += kChunk, ++i) {
    const int k = i % kSlots;
    const size_t len = std::min(kChunk, bytes - off);
    if (used[k] && (err = cudaEventSynchronize(ev[k])) != cudaSuccess) break;
    R.pool.run(R.slot[k], in + off, len);
    if ((err = cudaMemcpyAsync(out + off, R.slot[k], len, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      break;
    err = cudaEventRecord(ev[k], s);
    used[k] = true;
  }
  for (int k = 0; k < kSlots; ++k) {
    if (used[k]) {
      const cudaError_t e = cudaEventSynchronize(ev[k]);
      if (err == cudaSuccess) err = e;
    }
    cudaEventDestroy(ev[k]);
  }
  PDLP_CK(err);
}

}  // namespace pdlp_host
