// Minimal sm_100a async-copy helpers: 1D bulk copies (cp.async.bulk, the TMA
// engine without a tensor map) completing on shared-memory mbarriers.
#pragma once

#include <cstdint>

namespace pdlp {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Arrive (count 1) and add `bytes` to the transaction count of the phase.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Order earlier generic-proxy shared-memory accesses before later async-proxy
// (bulk copy) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Global -> shared bulk copy; dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 evict-first policy for data read once per pass.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Same, with an L2 cache-policy hint (a matrix stream, read once per pass:
// evict_first keeps it from pushing out the vector the consumers gather from
// and the operands the next pass reads).
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Stage elements [first, first + count) of a global array into shared memory
// with one bulk copy: the byte range is widened to 16-byte boundaries (every
// device array is allocated with >= 16 bytes of tail padding), and the
// returned pointer addresses element `first` inside the staged window.
template <class T>
__device__ __forceinline__ const T* stage_range(T* smem_window, const T* gsrc, int64_t first,
                                                int64_t count, uint64_t* bar, uint32_t& bytes_out) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(gsrc + first);
  const uintptr_t hi = reinterpret_cast<uintptr_t>(gsrc + first + count);
  const uintptr_t alo = lo & ~uintptr_t(15);
  const uintptr_t ahi = (hi + 15) & ~uintptr_t(15);
  const uint32_t bytes = static_cast<uint32_t>(ahi - alo);
  if (count > 0) bulk_g2s(smem_window, reinterpret_cast<const void*>(alo), bytes, bar);
  bytes_out = count > 0 ? bytes : 0u;
  return reinterpret_cast<const T*>(reinterpret_cast<const char*>(smem_window) + (lo - alo));
}

}  // namespace pdlp
