// Load-balanced CSR SpMV skeleton with a fused per-line epilogue.
//
// One launch covers three segments of CTAs (schedule built at upload time
// from the row lengths, see solver.cpp build_schedule):
//   [0, n_long)              one CTA per long line   (len >  t_med)
//   [.., + ceil(n_med/8))    one warp per medium line (t_short < len <= t_med)
//   [.., + short_blocks)     V-lane groups over every line with len <= t_short
//                            (grid-stride, warp-uniform trip counts)
// Each line's sum is produced by exactly one group with a fixed reduction
// tree, so results are deterministic run to run.  The epilogue functor sees
// (line, sum) once per line and accumulates its own per-thread partials.
//
// Matrix entries are streamed with evict-first loads; the dense operand goes
// through the read-only path so it stays L2-resident across the pass.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace pdlp {

constexpr int kSpmvThreads = 256;

// acc + a*b with the product rounded separately (the TU is built with
// -fmad=false): per-term rounding identical to the reference's
// `acc += value * x[idx]`, so a line whose terms one lane sums in storage
// order reproduces the reference bit for bit.  No cost: the pass is
// HBM-bound.
__device__ __forceinline__ double mac(double acc, double a, double b) { return acc + a * b; }

__host__ __device__ inline int64_t sched_blocks(const pdlpk_csr& A) {
  return A.n_long + (A.n_med + 7) / 8 + A.short_blocks;
}

template <class P, int V, class Epi>
__device__ __forceinline__ void sched_spmv(const pdlpk_csr& A, const double* __restrict__ vals,
                                           const double* __restrict__ v, Epi& epi) {
  const P* __restrict__ start = static_cast<const P*>(A.start);
  const int32_t* __restrict__ idx = A.index;
  int64_t b = blockIdx.x;
  if (b < A.n_long) {
    __shared__ double red_long[32];
    const int64_t r = A.long_rows[b];
    const int64_t lo = start[r], hi = start[r + 1];
    double acc = 0.0;
    int64_t k = lo + threadIdx.x;
    // two independent chains for memory-level parallelism
    double acc2 = 0.0;
    for (; k + kSpmvThreads < hi; k += 2 * kSpmvThreads) {
      const int32_t c0 = ld_stream(idx + k), c1 = ld_stream(idx + k + kSpmvThreads);
      const double a0 = ld_stream(vals + k), a1 = ld_stream(vals + k + kSpmvThreads);
      acc = mac(acc, a0, __ldg(v + c0));
      acc2 = mac(acc2, a1, __ldg(v + c1));
    }
    if (k < hi) acc = mac(acc, ld_stream(vals + k), __ldg(v + ld_stream(idx + k)));
    acc = block_sum(acc + acc2, red_long);
    if (threadIdx.x == 0) epi.line(r, acc);
    return;
  }
  b -= A.n_long;
  const int64_t med_blocks = (A.n_med + 7) / 8;
  if (b < med_blocks) {
    const int64_t w = b * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (w < A.n_med) {
      const int64_t r = A.med_rows[w];
      const int64_t lo = start[r], hi = start[r + 1];
      double acc = 0.0, acc2 = 0.0;
      int64_t k = lo + lane;
      for (; k + 32 < hi; k += 64) {
        const int32_t c0 = ld_stream(idx + k), c1 = ld_stream(idx + k + 32);
        const double a0 = ld_stream(vals + k), a1 = ld_stream(vals + k + 32);
        acc = mac(acc, a0, __ldg(v + c0));
        acc2 = mac(acc2, a1, __ldg(v + c1));
      }
      if (k < hi) acc = mac(acc, ld_stream(vals + k), __ldg(v + ld_stream(idx + k)));
      acc = warp_sum(acc + acc2);
      if (lane == 0) epi.line(r, acc);
    }
    return;
  }
  b -= med_blocks;
  constexpr int kGroupsPerWarp = 32 / V;
  constexpr int kGroupsPerBlock = kSpmvThreads / V;
  const int lane = threadIdx.x & 31;
  const int lig = lane % V;  // lane in group
  const int64_t stride = static_cast<int64_t>(A.short_blocks) * kGroupsPerBlock;
  const int64_t warp_first = b * kGroupsPerBlock + (threadIdx.x >> 5) * kGroupsPerWarp;
  for (int64_t wr = warp_first; wr < A.dim; wr += stride) {
    const int64_t r = wr + lane / V;
    double acc = 0.0;
    bool own = false;
    if (r < A.dim) {
      const int64_t lo = start[r], hi = start[r + 1];
      if (hi - lo <= A.t_short) {
        own = true;
        for (int64_t k = lo + lig; k < hi; k += V) {
          acc = mac(acc, ld_stream(vals + k), __ldg(v + ld_stream(idx + k)));
        }
      }
    }
    acc = group_sum<V>(acc);
    if (own && lig == 0) epi.line(r, acc);
  }
}

// Dispatch helper: calls F::template launch<P, V>() for the runtime (wide, vec).
template <class F>
inline int dispatch_pv(const pdlpk_csr& A, F&& f) {
  if (A.wide) {
    switch (A.vec) {
      case 1: return f.template go<int64_t, 1>();
      case 2: return f.template go<int64_t, 2>();
      case 4: return f.template go<int64_t, 4>();
      case 8: return f.template go<int64_t, 8>();
      case 16: return f.template go<int64_t, 16>();
      default: return f.template go<int64_t, 32>();
    }
  }
  switch (A.vec) {
    case 1: return f.template go<int32_t, 1>();
    case 2: return f.template go<int32_t, 2>();
    case 4: return f.template go<int32_t, 4>();
    case 8: return f.template go<int32_t, 8>();
    case 16: return f.template go<int32_t, 16>();
    default: return f.template go<int32_t, 32>();
  }
}

}  // namespace pdlp
