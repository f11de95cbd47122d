// Host->device upload options for 384 MB of pageable input (the C1 bench
// inputs): pageable cudaMemcpy, cudaHostRegister + DMA (+ unregister), and
// the host memcpy bandwidth that bounds a pinned staging ring.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

using Clock = std::chrono::steady_clock;
static double ms(Clock::time_point a) {
  return std::chrono::duration<double, std::milli>(Clock::now() - a).count();
}

int main() {
  const size_t bytes = size_t(384) << 20;
  char* host = static_cast<char*>(std::malloc(bytes));
  for (size_t i = 0; i < bytes; i += 4096) host[i] = static_cast<char>(i);
  std::memset(host, 1, bytes);
  char* dev = nullptr;
  cudaMalloc(&dev, bytes);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaMemcpy(dev, host, 1 << 20, cudaMemcpyHostToDevice);  // warm up
  for (int rep = 0; rep < 2; ++rep) {
    auto t = Clock::now();
    cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice);
    std::printf("pageable cudaMemcpy: %.2f ms (%.1f GB/s)\n", ms(t), bytes / ms(t) / 1e6);
    t = Clock::now();
    cudaHostRegister(host, bytes, cudaHostRegisterDefault);
    const double reg = ms(t);
    cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    const double dma = ms(t) - reg;
    auto u = Clock::now();
    cudaHostUnregister(host);
    std::printf("register %.2f ms + DMA %.2f ms (%.1f GB/s) + unregister %.2f ms = %.2f ms\n", reg,
                dma, bytes / dma / 1e6, ms(u), ms(t));
    char* pin = nullptr;
    cudaHostAlloc(reinterpret_cast<void**>(&pin), size_t(64) << 20, cudaHostAllocPortable);
    for (int th : {1, 4, 8, 12, 16}) {
      t = Clock::now();
      std::vector<std::thread> ts;
      const size_t chunk = size_t(64) << 20;
      for (int k = 0; k < th; ++k) {
        ts.emplace_back([&, k] {
          for (size_t off = 0; off < bytes; off += chunk) {
            const size_t per = (chunk + th - 1) / th;
            const size_t lo = std::min(chunk, per * k), hi = std::min(chunk, lo + per);
            if (off + hi <= bytes) std::memcpy(pin + lo, host + off + lo, hi - lo);
          }
        });
      }
      for (auto& x : ts) x.join();
      std::printf("memcpy into pinned, %2d threads: %.2f ms (%.1f GB/s)\n", th, ms(t),
                  bytes / ms(t) / 1e6);
    }
    cudaFreeHost(pin);
  }
  std::printf("hw threads %u\n", std::thread::hardware_concurrency());
  return 0;
}
