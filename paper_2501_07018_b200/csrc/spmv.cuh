// Load-balanced CSR SpMV skeleton with a fused per-line epilogue.
//
// One launch covers three segments of CTAs (schedule built at upload time
// from the line lengths, see solver.cpp build_schedule):
//   [0, n_long)                one CTA per long line    (len > kMedMax)
//   [.., + ceil(n_med/8))      one warp per medium line (kShortMax < len <= kMedMax),
//                              8 independent accumulator chains per lane
//   [.., + tile_blocks)        warp tiles of consecutive short lines
//                              (len <= kShortMax, <= kTileRows lines and
//                              <= kTileNnz entries per tile), grid-stride
// Tiles: the warp loads the tile's entries cooperatively (coalesced
// index/value streams, independent gathers), stores the rounded products
// value*x in shared memory, then each lane sums its own lines sequentially in
// storage order.  Because every product is rounded on its own and added in
// storage order starting from 0.0, a tiled line's sum is bit-identical to
// the reference's `acc += value * x[idx]` (kernels.hpp:30-59).
//
// Each line's sum is produced by exactly one group with a fixed order, so
// results are deterministic run to run.  The epilogue functor sees
// (line, sum) once per line and accumulates its own per-thread partials.
// Matrix entries are streamed with evict-first loads; the dense operand goes
// through the read-only path so it stays L2-resident across the pass.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace pdlp {

constexpr int kSpmvThreads = 256;
constexpr int kSpmvWarps = kSpmvThreads / 32;
constexpr int kShortMax = PDLPK_SHORT_MAX;  // longest tiled line
constexpr int kMedMax = PDLPK_MED_MAX;      // longest warp-per-line line
constexpr int kTileNnz = PDLPK_TILE_NNZ;    // entries per warp tile (4 KB of products)
constexpr int kTileRows = PDLPK_TILE_ROWS;
constexpr int kTileRowsPerLane = kTileRows / 32;
constexpr size_t kSpmvSmem = sizeof(double) * kSpmvWarps * kTileNnz;  // 32 KB / CTA

// acc + a*b with the product rounded separately (the TU is built with
// -fmad=false): per-term rounding identical to the reference.  No cost: the
// pass is HBM-bound.
__device__ __forceinline__ double mac(double acc, double a, double b) { return acc + a * b; }

// Segment mask of a layout: 1 long, 2 medium, 4 tiles.  Kernels are
// instantiated per mask so each pass only pays the registers of the paths it
// runs.  The tile segment is kept when nothing else exists so the grid is
// never empty (the column pass's last CTA makes the step decision).
__host__ __device__ inline int seg_mask(const pdlpk_csr& A) {
  int s = (A.n_long > 0 ? 1 : 0) | (A.n_med > 0 ? 2 : 0);
  if (A.n_tiles > 0 || s == 0) s |= 4;
  return s;
}

// Occupancy target per variant: tile variants keep a tile's index/value
// stream in registers (ILP), so they trade one CTA per SM for it.
__host__ __device__ constexpr int spmv_min_blocks(int seg) { return (seg & 4) ? 3 : 4; }

__host__ __device__ inline int64_t sched_blocks(const pdlpk_csr& A) {
  return A.n_long + (A.n_med + kSpmvWarps - 1) / kSpmvWarps +
         ((seg_mask(A) & 4) ? A.tile_blocks : 0);
}

template <class P, int Seg, class Epi>
__device__ __forceinline__ void sched_spmv(const pdlpk_csr& A, const double* __restrict__ vals,
                                           const double* __restrict__ v, Epi& epi) {
  const P* __restrict__ start = static_cast<const P*>(A.start);
  const int32_t* __restrict__ idx = A.index;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  int64_t b = blockIdx.x;
  if constexpr ((Seg & 1) != 0) {
  if (b < A.n_long) {
    __shared__ double red_long[32];
    const int64_t r = A.long_rows[b];
    const int64_t lo = start[r], hi = start[r + 1];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t k = lo + threadIdx.x;
    for (; k + 3 * kSpmvThreads < hi; k += 4 * kSpmvThreads) {
      int32_t c[4];
      double a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = ld_stream(idx + k + u * kSpmvThreads);
        a[u] = ld_stream(vals + k + u * kSpmvThreads);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = mac(acc[u], a[u], __ldg(v + c[u]));
    }
    for (; k < hi; k += kSpmvThreads) acc[0] = mac(acc[0], ld_stream(vals + k), __ldg(v + ld_stream(idx + k)));
    const double s = block_sum((acc[0] + acc[1]) + (acc[2] + acc[3]), red_long);
    if (threadIdx.x == 0) epi.line(r, s, epi.load(r));
    return;
  }
  }
  b -= A.n_long;
  const int64_t med_blocks = (A.n_med + kSpmvWarps - 1) / kSpmvWarps;
  if constexpr ((Seg & 2) != 0) {
  if (b < med_blocks) {
    const int64_t w = b * kSpmvWarps + warp;
    if (w < A.n_med) {
      const int64_t r = A.med_rows[w];
      typename Epi::Pre pre{};
      if (lane == 0) pre = epi.load(r);
      const int64_t lo = start[r], hi = start[r + 1];
      double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      int64_t k = lo + lane;
      for (; k + 7 * 32 < hi; k += 8 * 32) {
        int32_t c[8];
        double a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          c[u] = ld_stream(idx + k + u * 32);
          a[u] = ld_stream(vals + k + u * 32);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = mac(acc[u], a[u], __ldg(v + c[u]));
      }
      for (; k < hi; k += 32) acc[0] = mac(acc[0], ld_stream(vals + k), __ldg(v + ld_stream(idx + k)));
      const double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      const double t = warp_sum(s);
      if (lane == 0) epi.line(r, t, pre);
    }
    return;
  }
  }
  b -= med_blocks;
  if constexpr ((Seg & 4) == 0) return;
  extern __shared__ double tile_smem[];
  double* sm = tile_smem + warp * kTileNnz;
  const int64_t nwarps = static_cast<int64_t>(A.tile_blocks) * kSpmvWarps;
  int64_t t = b * kSpmvWarps + warp;
  // Tile metadata (first line, lines | entries << 8, first entry) comes from
  // the host schedule, so the index/value stream of a tile does not wait for
  // its row pointers; the next tile's metadata is prefetched.
  int64_t n_r0 = 0, n_s0 = 0;
  int n_pack = 0;
  if (t < A.n_tiles) {
    n_r0 = A.tile_row0[t];
    n_pack = A.tile_rows[t];
    n_s0 = A.tile_nnz0[t];
  }
  for (; t < A.n_tiles; t += nwarps) {
    const int64_t r0 = n_r0, s0 = n_s0;
    const int cnt = n_pack & 0xff;
    const int len = n_pack >> 8;
    const int64_t tn = t + nwarps;
    if (tn < A.n_tiles) {
      n_r0 = A.tile_row0[tn];
      n_pack = A.tile_rows[tn];
      n_s0 = A.tile_nnz0[tn];
    }
    // index/value stream of the tile: independent of everything but s0
    int32_t ci[kTileNnz / 32];
    double av[kTileNnz / 32];
#pragma unroll
    for (int u = 0; u < kTileNnz / 32; ++u) {
      const int j = lane + 32 * u;
      if (j < len) {
        ci[u] = ld_stream(idx + s0 + j);
        av[u] = ld_stream(vals + s0 + j);
      }
    }
    // Line i = lane + 32q of the tile starts at rb[q]; it ends where line i+1
    // starts (lane+1's rb[q], or lane 0's rb[q+1] for lane 31), or at s1.
    int64_t rb[kTileRowsPerLane];
    typename Epi::Pre pre[kTileRowsPerLane];
#pragma unroll
    for (int q = 0; q < kTileRowsPerLane; ++q) {
      const int i = lane + 32 * q;
      rb[q] = i < cnt ? static_cast<int64_t>(start[r0 + i]) : 0;
      // epilogue operands do not depend on the products either
      if (i < cnt) pre[q] = epi.load(r0 + i);
    }
    const int64_t s1 = s0 + len;
#pragma unroll
    for (int u = 0; u < kTileNnz / 32; ++u) {
      const int j = lane + 32 * u;
      if (j < len) sm[j] = av[u] * __ldg(v + ci[u]);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kTileRowsPerLane; ++q) {
      const int i = lane + 32 * q;
      const int64_t next_same = __shfl_down_sync(0xffffffffu, rb[q], 1);
      const int64_t next_wrap =
          __shfl_sync(0xffffffffu, q + 1 < kTileRowsPerLane ? rb[q + 1 < kTileRowsPerLane ? q + 1 : q] : 0, 0);
      if (i < cnt) {
        const int64_t end = (i + 1 < cnt) ? (lane < 31 ? next_same : next_wrap) : s1;
        double acc = 0.0;
        for (int j = static_cast<int>(rb[q] - s0); j < static_cast<int>(end - s0); ++j) acc += sm[j];
        epi.line(r0 + i, acc, pre[q]);
      }
    }
    __syncwarp();
  }
}

// Dispatch helper: calls F::template go<P, Seg>() for the row-pointer width
// and the segment mask of the layout.
template <class P, class F>
inline int dispatch_seg(int seg, F&& f) {
  switch (seg) {
    case 1: return f.template go<P, 1>();
    case 2: return f.template go<P, 2>();
    case 3: return f.template go<P, 3>();
    case 4: return f.template go<P, 4>();
    case 5: return f.template go<P, 5>();
    case 6: return f.template go<P, 6>();
    default: return f.template go<P, 7>();
  }
}

template <class F>
inline int dispatch_p(const pdlpk_csr& A, F&& f) {
  if (A.wide) return dispatch_seg<int64_t>(seg_mask(A), f);
  return dispatch_seg<int32_t>(seg_mask(A), f);
}

}  // namespace pdlp
