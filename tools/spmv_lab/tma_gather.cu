// Probe (measurement only): random-row gather throughput of the TMA engine
// (cp.async.bulk.tensor.2d ... tile::gather4, sm_100a) against LSU gathers.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o tools/spmv_lab/tma_gather tools/spmv_lab/tma_gather.cu -lcuda
//   tools/spmv_lab/tma_gather [n_doubles] [count]
//
// The vector is viewed as a 2-D tensor of rows of 2 doubles (16 bytes); one
// gather4 fetches 4 arbitrary rows.  Each warp's lane 0 keeps S stages of G
// gather4 requests in flight on mbarriers; the warp sums what lands.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));      \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t hash32(uint32_t h) {
  h *= 0x9E3779B1u;
  h ^= h >> 15;
  h *= 0x85EBCA77u;
  h ^= h >> 13;
  return h;
}

template <int S, int G>
__global__ void __launch_bounds__(256) tma_gather_probe(const __grid_constant__ CUtensorMap tmap,
                                                        uint32_t rows, int64_t count, double* out) {
  // per warp: S stages x G gather4 x 4 rows x 16 bytes
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + w * S;
  unsigned char* buf = sm + 1024 + static_cast<size_t>(w) * S * G * 128;  // 128-B aligned destinations
  if (lane == 0) {
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t per_round = static_cast<int64_t>(G) * 4;  // rows per stage
  double acc = 0.0;
  int64_t round = 0;
  uint32_t phase[S] = {};
  auto issue = [&](int s, int64_t r) {
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + s)),
                   "r"(G * 64));
      for (int g = 0; g < G; ++g) {
        const uint32_t b = static_cast<uint32_t>(r * per_round + g * 4);
        const int r0 = hash32(b) % rows, r1 = hash32(b + 1) % rows, r2 = hash32(b + 2) % rows,
                  r3 = hash32(b + 3) % rows;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf + (s * G + g) * 128)),
            "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar + s))
            : "memory");
      }
    }
  };
  // rounds owned by this warp: gw, gw + nw, ... (each round = one stage)
  const int64_t rounds = count / per_round;
  int64_t next = gw;
  for (int s = 0; s < S && next < rounds; ++s, next += nw) issue(s, next);
  for (int64_t r = gw; r < rounds; r += nw, ++round) {
    const int s = static_cast<int>(round % S);
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
            smem_u32(bar + s)),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1u;
    const double* d = reinterpret_cast<const double*>(buf + s * G * 128);
    for (int i = lane; i < G * 8; i += 32) acc += d[(i >> 3) * 16 + (i & 7)];
    __syncwarp();
    if (next < rounds) {
      issue(s, next);
      next += nw;
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void lsu_probe(const double* __restrict__ v, uint32_t n, int64_t count, double* out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t b = tid * 8; b < count; b += nt * 8) {
    double g[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) g[u] = __ldg(v + hash32(static_cast<uint32_t>(b + u)) % n);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += g[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

template <class F>
float time_it(F&& f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  CK(cudaGetLastError());
  return ms * 1000.0f / reps;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 5000000;
  const int64_t count = argc > 2 ? atoll(argv[2]) : 165000000;
  double *v, *out;
  CK(cudaMalloc(&v, n * 8 + 64));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(v, 0, n * 8));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  CUtensorMap tmap;
  const uint32_t rows = static_cast<uint32_t>(n / 2);
  cuuint64_t gdim[2] = {2, rows};
  cuuint64_t gstride[1] = {16};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, v, gdim, gstride, box,
                                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    std::printf("cuTensorMapEncodeTiled failed: %d\n", (int)cr);
    return 1;
  }
  std::printf("n=%lld doubles (%.0f MB), %lld random rows per run\n", (long long)n, n * 8 / 1e6,
              (long long)count);
  float us = time_it([&] { lsu_probe<<<sms * 8, 256>>>(v, (uint32_t)n, count, out); }, 5);
  std::printf("LSU gathers (8 B):            %8.1f us  %6.1f G/s\n", us, count / us / 1e3);
  auto run = [&](auto ks, auto kg, int ctas_per_sm) {
    constexpr int S = decltype(ks)::value, G = decltype(kg)::value;
    const size_t smem = 1024 + 8ull * S * G * 128;
    auto k = tma_gather_probe<S, G>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    float t = time_it([&] { k<<<sms * ctas_per_sm, 256, smem>>>(tmap, rows, count, out); }, 5);
    std::printf("TMA gather4 S=%d G=%2d x%d/SM (%4zu KB): %8.1f us  %6.1f G rows/s\n", S, G, ctas_per_sm,
                smem / 1024, t, count / t / 1e3);
  };
  run(std::integral_constant<int, 2>{}, std::integral_constant<int, 8>{}, 1);
  run(std::integral_constant<int, 4>{}, std::integral_constant<int, 8>{}, 1);
  run(std::integral_constant<int, 4>{}, std::integral_constant<int, 16>{}, 1);
  run(std::integral_constant<int, 4>{}, std::integral_constant<int, 16>{}, 2);
  run(std::integral_constant<int, 8>{}, std::integral_constant<int, 16>{}, 2);
  run(std::integral_constant<int, 4>{}, std::integral_constant<int, 32>{}, 2);
  return 0;
}
