// Probe: which cp.async forms run on this device (bring-up of the async
// segmented-span prefetch).  Each kernel copies 16/4-byte pieces into smem
// and writes them back; the host checks the results and the error state.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <int MODE>
__global__ void k(const int4* src, int4* dst, const uint32_t* m, uint32_t* mo) {
  extern __shared__ __align__(128) unsigned char buf[];
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  int4* s = reinterpret_cast<int4*>(buf) + threadIdx.x;
  uint32_t* sm = reinterpret_cast<uint32_t*>(buf + 16 * blockDim.x) + threadIdx.x;
  if (MODE == 0) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(s)), "l"(src + threadIdx.x) : "memory");
  if (MODE == 1) asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(su(s)), "l"(src + threadIdx.x), "l"(pol) : "memory");
  if (MODE == 2) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su(sm)), "l"(m + threadIdx.x) : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (MODE < 2) dst[threadIdx.x] = *s; else mo[threadIdx.x] = *sm;
}
int main() {
  int4 *src, *dst; uint32_t *m, *mo;
  cudaMalloc(&src, 4096); cudaMalloc(&dst, 4096); cudaMalloc(&m, 1024); cudaMalloc(&mo, 1024);
  cudaMemset(src, 7, 4096); cudaMemset(m, 9, 1024);
  void (*ks[3])(const int4*, int4*, const uint32_t*, uint32_t*) = {k<0>, k<1>, k<2>};
  for (int i = 0; i < 3; ++i) {
    ks[i]<<<1, 64, 64 * 20>>>(src, dst, m, mo);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("mode %d: %s\n", i, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  // 50 KB of dynamic smem with the opt-in, as the seg kernels launch
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  k<1><<<148, 256, 50176>>>(src, dst, m, mo);
  std::printf("50KB: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
