// Host-side RAII helpers for device memory, streams and events.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <map>
#include <mutex>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

namespace pdlp_host {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                    cudaGetErrorString(e) + ")");
  }
}

// Launchers in kernels.h return the cudaError_t of the launch (0 = success).
inline void check_launch(int rc, const char* what) {
  if (rc != 0) check_cuda(rc < 0 ? cudaErrorUnknown : static_cast<cudaError_t>(rc), what);
}

#define PDLP_CK(expr) ::pdlp_host::check_cuda((expr), #expr)
#define PDLP_LAUNCH(expr) ::pdlp_host::check_launch((expr), #expr)

// Stream-ordered allocation.  While an Engine is alive its stream is the
// thread's allocation stream: buffers come from the device's default memory
// pool (cudaMallocAsync) and go back to it in stream order, so a solve neither
// maps nor unmaps device memory once the pool is warm (the pool keeps what it
// holds, like a caching allocator; pdlp_trim_device_memory() returns it).
// Without an allocation stream DevBuf falls back to cudaMalloc/cudaFree.
inline thread_local cudaStream_t g_alloc_stream = nullptr;
// Host seconds spent in device allocations on this thread (phase report of
// the `logging` option).
inline thread_local double g_alloc_seconds = 0.0;

inline void retain_pool_memory(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  PDLP_CK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = ~0ull;
  PDLP_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  done[device] = true;
}

// Exact-size cache of stream-ordered blocks across solves (a caching layer
// over the pool): a released buffer goes into it with an event recorded on
// its stream; a later allocation of the same byte size on the same device
// takes it back after the allocating stream waits for that event.  Repeated
// solves of one problem then allocate nothing -- the pool's own reuse of
// blocks freed on another (since destroyed) stream still mapped memory,
// 2-5 ms per large buffer.  Bounded (PDLP_BLOCK_CACHE_MB, default 49152;
// 0 disables it); pdlp_trim_device_memory empties it; an allocation that
// fails empties it and retries.
class BlockCache {
 public:
  static BlockCache& get() {
    static BlockCache* c = new BlockCache();  // leaked: outlives static teardown
    return *c;
  }
  void* take(size_t bytes, cudaStream_t s) {
    if (cap_ == 0) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> g(mu_);
    auto it = free_.find(std::make_pair(dev, bytes));
    if (it == free_.end() || it->second.empty()) return nullptr;
    Block b = it->second.back();
    it->second.pop_back();
    held_ -= bytes;
    cudaStreamWaitEvent(s, b.ev, 0);
    cudaEventDestroy(b.ev);  // released once the wait is satisfied
    return b.p;
  }
  bool give(void* p, size_t bytes, cudaStream_t s) {
    if (cap_ == 0) return false;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    std::lock_guard<std::mutex> g(mu_);
    if (held_ + bytes > cap_) return false;
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (cudaEventRecord(ev, s) != cudaSuccess) {
      cudaGetLastError();
      cudaEventDestroy(ev);
      return false;
    }
    free_[std::make_pair(dev, bytes)].push_back(Block{p, ev});
    held_ += bytes;
    return true;
  }
  // Frees every cached block of `device` (-1: all devices).
  void trim(int device) {
    std::lock_guard<std::mutex> g(mu_);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto it = free_.begin(); it != free_.end();) {
      if (device >= 0 && it->first.first != device) {
        ++it;
        continue;
      }
      cudaSetDevice(it->first.first);
      for (Block& b : it->second) {
        cudaEventSynchronize(b.ev);
        cudaEventDestroy(b.ev);
        cudaFree(b.p);
        held_ -= it->first.second;
      }
      it = free_.erase(it);
    }
    cudaSetDevice(cur);
  }

 private:
  BlockCache() {
    const char* e = std::getenv("PDLP_BLOCK_CACHE_MB");
    const long long mb = e != nullptr ? std::atoll(e) : 49152;
    cap_ = mb > 0 ? static_cast<size_t>(mb) << 20 : 0;
  }
  struct Block {
    void* p;
    cudaEvent_t ev;
  };
  std::mutex mu_;
  std::map<std::pair<int, size_t>, std::vector<Block>> free_;
  size_t held_ = 0, cap_ = 0;
};

class AllocStreamScope {
 public:
  explicit AllocStreamScope(cudaStream_t s) : prev_(g_alloc_stream) { g_alloc_stream = s; }
  ~AllocStreamScope() { g_alloc_stream = prev_; }
  AllocStreamScope(const AllocStreamScope&) = delete;
  AllocStreamScope& operator=(const AllocStreamScope&) = delete;

 private:
  cudaStream_t prev_;
};

template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      s_ = o.s_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void alloc(size_t n) {
    release();
    n_ = n;
    if (n == 0) return;
    void* p = nullptr;
    // +64 bytes: the SpMV tile path bulk-copies 16-byte-aligned windows that
    // may extend up to 15 bytes past the last element, and the segmented
    // spans load 8-entry blocks that may extend 7 entries past it.
    s_ = g_alloc_stream;
    const auto t0 = std::chrono::steady_clock::now();
    if (s_ != nullptr) {
      const size_t bytes = n * sizeof(T) + 64;
      p = BlockCache::get().take(bytes, s_);
      if (p == nullptr && cudaMallocAsync(&p, bytes, s_) != cudaSuccess) {
        cudaGetLastError();  // out of memory: return the cached blocks, retry
        BlockCache::get().trim(-1);
        PDLP_CK(cudaMallocAsync(&p, bytes, s_));
      }
    } else {
      PDLP_CK(cudaMalloc(&p, n * sizeof(T) + 64));
    }
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    g_alloc_seconds += dt;
    static const bool debug = std::getenv("PDLP_ALLOC_DEBUG") != nullptr;
    if (debug && dt > 2e-3) {
      std::fprintf(stderr, "alloc %.1f MB took %.1f ms\n", n * sizeof(T) / 1048576.0, 1e3 * dt);
    }
    p_ = static_cast<T*>(p);
  }
  void release() {
    if (p_ != nullptr) {
      if (s_ != nullptr) {
        if (!BlockCache::get().give(p_, n_ * sizeof(T) + 64, s_)) cudaFreeAsync(p_, s_);
      } else {
        cudaFree(p_);
      }
    }
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void swap(DevBuf& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(s_, o.s_);
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;  // allocation stream (nullptr: cudaMalloc)
};

class Stream {
 public:
  Stream() { PDLP_CK(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking)); }
  ~Stream() {
    if (s_ != nullptr) cudaStreamDestroy(s_);
  }
  Stream(const Stream&) = delete;
  Stream& operator=(const Stream&) = delete;
  cudaStream_t get() const { return s_; }
  void sync() const { PDLP_CK(cudaStreamSynchronize(s_)); }

 private:
  cudaStream_t s_ = nullptr;
};

class Event {
 public:
  Event() { PDLP_CK(cudaEventCreate(&e_)); }
  ~Event() {
    if (e_ != nullptr) cudaEventDestroy(e_);
  }
  Event(const Event&) = delete;
  Event& operator=(const Event&) = delete;
  cudaEvent_t get() const { return e_; }
  void record(cudaStream_t s) { PDLP_CK(cudaEventRecord(e_, s)); }

 private:
  cudaEvent_t e_ = nullptr;
};

inline double elapsed_seconds(const Event& a, const Event& b) {
  float ms = 0.0f;
  PDLP_CK(cudaEventSynchronize(b.get()));
  PDLP_CK(cudaEventElapsedTime(&ms, a.get(), b.get()));
  return static_cast<double>(ms) * 1e-3;
}

}  // namespace pdlp_host

// NVTX phase ranges (tracing): upload / precondition / attempts /
// cadence / gap / polish.  nvtx3 is header-only and inert unless a profiler
// injects itself (ncu --nvtx, Nsight Systems); no library is linked.
namespace pdlp_host {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace pdlp_host
