// Device-side scalar helpers shared by every kernel.
//
// All translation units are compiled with -fmad=false: the reference's dual
// update  y' = yhat - sigma*proj  (proj/include/pdhglp/step.hpp:85) relies on
// exact cancellation to keep y' in its sign cone, and FMA contraction breaks
// that (SURVEY.md §0 finding 6).  Where contraction is wanted (perf-mode SpMV
// accumulation) it is written explicitly as fma().
#pragma once

#include <cstdint>
#include <cstdlib>
#include <math_constants.h>

#include "kernels.h"  // tuning defaults (PDLPK_PDL, ...)

namespace pdlp {

constexpr int kWarp = 32;

__device__ __forceinline__ bool finite_d(double v) { return isfinite(v); }

// reference core.hpp:18-21 — product with 0 * (+-inf) = 0.
__device__ __forceinline__ double mul_zero_inf(double a, double b) {
  if (a == 0.0 || b == 0.0) return 0.0;
  return a * b;
}

// reference core.hpp:26-28 (NaN passes through, as in the reference).
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

// reference core.hpp:31-35.
__device__ __forceinline__ double interval_distance(double v, double lo, double hi) {
  if (v < lo) return lo - v;
  if (v > hi) return v - hi;
  return 0.0;
}

// std::max(acc, v) semantics: (acc < v) ? v : acc — NaN never wins.
__device__ __forceinline__ double max_keep(double acc, double v) {
  return (acc < v) ? v : acc;
}

// SignCone (problem.hpp:36-57): 0 Zero, 1 NonPos, 2 NonNeg, 3 Free.
enum Cone : int { kZero = 0, kNonPos = 1, kNonNeg = 2, kFree = 3 };

__device__ __forceinline__ int cone_of_bounds(double lo, double hi) {
  const bool lo_f = lo > -CUDART_INF;
  const bool hi_f = hi < CUDART_INF;
  if (lo_f && hi_f) return kFree;
  if (lo_f) return kNonNeg;
  if (hi_f) return kNonPos;
  return kZero;
}

// recession_cone (residuals.hpp:15-22): the opposite classification.
__device__ __forceinline__ int recession_cone(double lo, double hi) {
  const bool lo_f = lo > -CUDART_INF;
  const bool hi_f = hi < CUDART_INF;
  if (lo_f && hi_f) return kZero;
  if (lo_f) return kNonNeg;
  if (hi_f) return kNonPos;
  return kFree;
}

__device__ __forceinline__ double cone_project(double v, int cone) {
  switch (cone) {
    case kZero: return 0.0;
    case kNonPos: return v < 0.0 ? v : 0.0;
    case kNonNeg: return v > 0.0 ? v : 0.0;
    default: return v;
  }
}

// ----------------------------------------------------------- reductions ---
// Deterministic block reductions: fixed shuffle tree, fixed smem tree.

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max_keep(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum over a group of `width` consecutive lanes (width a power of two <= 32);
// the group's first lane holds the result.
template <int W>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, W);
  return v;
}

// Block-wide sum (blockDim.x a multiple of 32, <= 1024); result valid in
// thread 0.  `smem` needs blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? smem[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

__device__ __forceinline__ double block_max(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? smem[lane] : 0.0;
    r = warp_max(r);
  }
  return r;
}

// Streaming loads for data touched once per pass (matrix entries): evict
// first so the gathered dense operand keeps its L2 residency.
// L2 eviction priority for a vector that a later kernel gathers from (x-bar
// for the row pass): stores carry an evict_last policy on `frac` of the
// lines, so the streams around them (evict_first / .cs) go first.
__device__ __forceinline__ uint64_t l2_keep_policy(float frac) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(pol) : "f"(frac));
  return pol;
}
__device__ __forceinline__ void st_keep(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// Programmatic dependent launch (the attempt's three kernels).  pdl_wait()
// at the top of a kernel: block until the previous kernel of the stream has
// completed and its writes are visible (before any dependent read).
// pdl_trigger() once a CTA's main work is issued: the next kernel's CTAs may
// then launch onto SMs this CTA's tail leaves free.  Triggering at kernel
// start instead fills the SMs with waiting CTAs (measured: C1 6,440 ->
// 3,950 it/s).  Outside a PDL launch both are no-ops.
__device__ __forceinline__ void pdl_wait() {
#if PDLPK_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if PDLPK_PDL && PDLPK_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// The cadence's kernels (reductions, products): the same, when enabled.
__device__ __forceinline__ void pdl_wait_cadence() {
#if PDLPK_PDL && PDLPK_PDL_CADENCE
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger_cadence() {
#if PDLPK_PDL && PDLPK_PDL_CADENCE
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// <<<>>> or, with pdl, cudaLaunchKernelEx with programmatic stream
// serialization.  Only for kernels that begin with pdl_enter(): their wait
// keeps the dependence on the previous kernel of the stream.
// PDLP_NO_PDL=1 in the environment launches everything plainly (tests
// compare the two).
inline bool pdl_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("PDLP_NO_PDL");
    return e != nullptr && e[0] == '1';
  }();
  return off;
}

template <class... KArgs, class... Args>
inline void launch_pdl(bool pdl, void (*kern)(KArgs...), unsigned grid, unsigned block,
                       size_t smem, cudaStream_t s, Args... args) {
  if (!(PDLPK_PDL && pdl) || pdl_disabled()) {
    kern<<<grid, block, smem, s>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldcs(p); }
__device__ __forceinline__ int64_t ld_stream(const int64_t* p) { return __ldcs(p); }
__device__ __forceinline__ int4 ld_stream(const int4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
// Read-once matrix streams with an explicit L2 evict_first policy (pol from
// createpolicy), bypassing L1: they must not push the gathered vector out.
__device__ __forceinline__ int4 ld_stream_ef(const int4* p, uint64_t pol) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_stream_ef(const double2* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
// Gather with an explicit L2 policy (pol from createpolicy).
__device__ __forceinline__ double ld_gather_pol(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t l2_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Warm a line of global memory in L2 (the segmented spans' epilogue operands).
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

}  // namespace pdlp
