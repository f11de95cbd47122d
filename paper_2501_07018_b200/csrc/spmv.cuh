// Load-balanced CSR SpMV skeleton with a fused per-line epilogue.
//
// One launch covers up to two segments of CTAs (schedule built once per
// solve from the line lengths, see solver.cpp build_schedule):
//   [0, ceil(n_wchunks/8))    one warp per line of kShortMax < len <=
//                             PDLPK_WARP_LINE_MAX entries (8 independent
//                             accumulator chains per lane)
//   [.., + n_cta_chunks)      one CTA per chunk (<= kChunk entries) of a
//                             longer line, a 256-entry slice per warp, warp
//                             sums added in warp order; the last-arriving CTA
//                             of a multi-chunk line sums the chunk partials in
//                             chunk order (deterministic) and runs the
//                             epilogue, whose contributions go to the line's
//                             fixed slot (line_acc)
//   [.., + n_tiles)           direct tiles (layouts of very short lines, e.g.
//                             C1's two-entry columns): one CTA per run of
//                             <= kDirectRows consecutive short lines, one
//                             thread per line summing it in storage order;
//                             no staging, full occupancy hides the
//                             pointer -> index -> gather chain
//   [.., + tile_blocks)       staged tiles of consecutive short lines
//                             (len <= kShortMax; <= kTileRows lines and
//                             <= kTileNnz entries per tile), grid-stride
// Skewed (power-law) line lengths thus cost the same as uniform ones.
//
// Tiles are fed by the TMA engine: an elected thread bulk-copies the tile's
// contiguous streams — column indices, values, row pointers and the
// epilogue's per-line operands — into a multi-stage shared-memory ring
// (cp.async.bulk, completion on an mbarrier), kStages tiles ahead of the
// consumers.  The CTA then forms the rounded products value*x[index] (the
// only dependent global access is the gather), and each thread sums one
// line's products in storage order.  Because every product is rounded on its
// own and added in storage order starting from 0.0, a tiled line's sum is
// bit-identical to the reference's `acc += value * x[idx]`
// (kernels.hpp:30-59).
//
// Each line's sum is produced by exactly one thread/warp/CTA with a fixed
// order, so results are deterministic run to run.  The epilogue functor sees
// (line, sum, operands) once per line and accumulates its own partials.
#pragma once

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace pdlp {

#ifndef PDLPK_SPMV_THREADS
#define PDLPK_SPMV_THREADS 256
#endif
constexpr int kSpmvThreads = PDLPK_SPMV_THREADS;
constexpr int kSpmvWarps = kSpmvThreads / 32;
constexpr int kShortMax = PDLPK_SHORT_MAX;  // longest tiled line
constexpr int kChunk = PDLPK_CHUNK;         // entries per warp chunk of a long line
constexpr int kTileNnz = PDLPK_TILE_NNZ;    // entries per CTA tile
constexpr int kTileRows = PDLPK_TILE_ROWS;  // lines per CTA tile
constexpr int kMaxStaged = 4;               // epilogue operand streams per line (at most)
constexpr int kDefaultStaged = 3;           // what a layout's stage reserves unless told otherwise
constexpr int kConsumerWarps = kSpmvWarps - 1;  // warp 0 produces
// lines per consumer lane: a consumer warp owns 32 * kLinesPerLane lines of a
// tile, lane l taking lines l, l + 32, ... (stores stay coalesced)
constexpr int kLinesPerLane = (kTileRows + 32 * kConsumerWarps - 1) / (32 * kConsumerWarps);
static_assert(kTileRows <= 32 * kConsumerWarps * kLinesPerLane, "tile lines per consumer warp");

__host__ __device__ constexpr size_t align16(size_t v) { return (v + 15) & ~size_t(15); }
// Stage buffer: [indices | values | row pointers | staged operands...] for a
// tile of <= L lines and <= E entries.  Every ring stage has the bytes of the
// default shape (kTileRows, kTileNnz); a layout picks its own (L, E) inside
// that budget from its line lengths (solver.cpp build_schedule): C1's
// two-entry columns use 672 x 1344, C2's ~27-entry rows ~100 x 2900, so both
// fill their stages.
struct StageLayout {
  uint32_t val, ptr, epi, epi_stride, bytes;
};
__host__ __device__ constexpr StageLayout stage_layout(int L, int E, int ns = kDefaultStaged) {
  return StageLayout{
      static_cast<uint32_t>(align16(sizeof(int32_t) * E + 32)),
      static_cast<uint32_t>(align16(sizeof(int32_t) * E + 32) + align16(sizeof(double) * E + 32)),
      static_cast<uint32_t>(align16(sizeof(int32_t) * E + 32) + align16(sizeof(double) * E + 32) +
                            align16(sizeof(int64_t) * (L + 1) + 32)),
      static_cast<uint32_t>(align16(sizeof(double) * L + 32)),
      static_cast<uint32_t>(align16(sizeof(int32_t) * E + 32) + align16(sizeof(double) * E + 32) +
                            align16(sizeof(int64_t) * (L + 1) + 32) +
                            ns * align16(sizeof(double) * L + 32))};
}
// Largest entry count that fits a stage of `budget` bytes next to L lines.
__host__ __device__ inline int stage_nnz_for(int L, size_t budget, int ns = kDefaultStaged) {
  int lo = 32, hi = 1 << 18;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (stage_layout(L, mid, ns).bytes <= budget) lo = mid; else hi = mid - 1;
  }
  return lo;
}
constexpr int kStages = PDLPK_TILE_STAGES;  // ring depth: tiles in flight per CTA
// What the consumers of a stage need about its tile, written by the producer
// lane (which computes it anyway for the bulk copies) before its arrive on
// full[stage]: the consumers read 32 bytes instead of re-deriving the tile's
// metadata and six window shifts per warp.
struct TileHdr {
  int64_t r0, s0;    // first line, first entry
  int32_t cnt;       // lines
  uint32_t shifts;   // 4-bit byte shifts: idx, val, ptr, staged operands 0..2
  int32_t per;       // lines per consumer warp
  int32_t pad;
};
// Ring header: full/empty mbarriers, then one TileHdr per stage (128-byte
// aligned so every stage buffer stays aligned for the bulk copies).
constexpr size_t kRingHeader = (2 * 8 * kStages + sizeof(TileHdr) * kStages + 127) / 128 * 128;
// Dynamic shared memory of a layout's staged ring (its stage size is chosen
// per layout, see solver.cpp build_schedule).
__host__ __device__ inline size_t ring_smem(const pdlpk_csr& A) {
  return kRingHeader + kStages * static_cast<size_t>(A.tile_stage_bytes);
}

// acc + a*b with the product rounded separately (the TU is built with
// -fmad=false): per-term rounding identical to the reference.  No cost: the
// pass is HBM-bound.
__device__ __forceinline__ double mac(double acc, double a, double b) { return acc + a * b; }

constexpr int kDirectRows = kSpmvThreads;  // lines per direct tile
#ifndef PDLPK_TILE_GATHER
#define PDLPK_TILE_GATHER 4 /* gathers in flight per consumer lane */
#endif
constexpr int kTileGather = PDLPK_TILE_GATHER;

// ------------------------------------------------------ segmented spans ---
// A warp walks one span at a time (grid-stride over spans).  Line runs: steps
// of 256 entries starting on 8-entry boundaries; lane l holds entries
// [base + 8l, base + 8l + 8) (vector loads of indices and values, 8 gathers
// in flight), sums the line segments inside its 8 entries in storage order,
// and a segmented scan across the lanes joins segments that cross lanes; a
// carry joins steps.  The lane holding a line's last entry runs the
// epilogue (the operands of the step's lines are warmed in L2 first).  Lines
// longer than a span are cut into chunks summed by lane chains + a warp tree
// and combined in chunk order by the last-arriving chunk (deterministic).
// Every line sum has one fixed association, so results are deterministic run
// to run; only lines that cross lanes are not summed in storage order.
__device__ __forceinline__ int warp_excl_scan_i(int v, int lane) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  return x - v;
}

#ifndef PDLPK_SEG_PREFETCH
#define PDLPK_SEG_PREFETCH 0 /* warm a step's epilogue operands in L2 (measured: 18 us slower) */
#endif
#ifndef PDLPK_SEG_PIPELINE
#define PDLPK_SEG_PIPELINE 0 /* software-pipelined stream loads (one step ahead) */
#endif
#ifndef PDLPK_SEG_GATHER_KEEP
#define PDLPK_SEG_GATHER_KEEP 0 /* L2 evict_last hint on the gathers */
#endif
#ifndef PDLPK_SEG_EVICT_FIRST
#define PDLPK_SEG_EVICT_FIRST 1 /* L2 evict_first hint on the spans' index/value streams */
#endif
template <class Epi>
__device__ __forceinline__ void seg_spans(const pdlpk_csr& A, const double* __restrict__ vals,
                                          const double* __restrict__ v, Epi& epi) {
  const int32_t* __restrict__ idx = A.index;
#if PDLPK_SEG_EVICT_FIRST
  const uint64_t pol = l2_first_policy();
#define SEG_LD(p) ld_stream_ef(p, pol)
#else
#define SEG_LD(p) ld_stream(p)
#endif
#if PDLPK_SEG_GATHER_KEEP
  const uint64_t gpol = l2_last_policy();
#define SEG_G(p) ld_gather_pol(p, gpol)
#else
#define SEG_G(p) __ldg(p)
#endif
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t it = gw; it < A.n_seg_spans; it += nw) {
    const int4 d = A.seg_spans[it];
    const int64_t e0 = static_cast<int64_t>(static_cast<uint32_t>(d.z)) |
                       (static_cast<int64_t>(A.seg_aux[it].w) << 32);
    const int64_t e1 = e0 + d.w;
    if (d.y < 0) {
      // chunk c of a long line (or an empty line)
      double acc = 0.0;
      for (int64_t base = e0 & ~int64_t(7); base < e1; base += 256) {
        const int64_t k0 = base + 8 * lane;
        if (k0 + 8 > e0 && k0 < e1) {
          const int4 i0 = SEG_LD(reinterpret_cast<const int4*>(idx + k0));
          const int4 i1 = SEG_LD(reinterpret_cast<const int4*>(idx + k0 + 4));
          const int ci[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
          double a[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 t = SEG_LD(reinterpret_cast<const double2*>(vals + k0) + q);
            a[2 * q] = t.x;
            a[2 * q + 1] = t.y;
          }
          double g[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) g[u] = (k0 + u >= e0 && k0 + u < e1) ? SEG_G(v + ci[u]) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (k0 + u >= e0 && k0 + u < e1) acc = mac(acc, a[u], g[u]);
          }
        }
      }
      const double t = warp_sum(acc);
      if (lane == 0) {
        const int4 x = A.seg_aux[it];
        const int c = -1 - d.y, nch = x.y;
        if (nch == 1) {
          const typename Epi::Pre pre = epi.load(d.x);
          epi.line(d.x, epi.init(pre) + t, pre);
        } else {
          A.chunk_part[x.x + c] = t;
          __threadfence();
          const unsigned arrived = atomicAdd(A.chunk_cnt + x.x, 1u);
          if (arrived == static_cast<unsigned>(nch - 1)) {
            __threadfence();
            double tot = 0.0;
            for (int q = 0; q < nch; ++q) tot += __ldcg(A.chunk_part + x.x + q);
            A.chunk_cnt[x.x] = 0;
            Epi solo = epi;
            solo.reset_acc();
            const typename Epi::Pre pre = solo.load(d.x);
            solo.line(d.x, solo.init(pre) + tot, pre);
            solo.export_acc(A.line_acc + static_cast<int64_t>(x.z) * PDLPK_LINE_ACC);
          }
        }
      }
      continue;
    }
    int64_t rc = d.x;
    double carry = 0.0;
    int64_t sid = A.seg_step0[it];
#if PDLPK_SEG_PIPELINE
    // the next step's index / value / mask loads are issued before this
    // step's gathers: the stream latency overlaps the gather round trip
    int4 ni0 = make_int4(0, 0, 0, 0), ni1 = make_int4(0, 0, 0, 0);
    double2 nv[4];
    uint32_t nmw = 0u;
    auto fetch = [&](int64_t b, int64_t sidx) {
      const int64_t kk = b + 8 * lane;
      nmw = lane < 16 ? __ldg(A.seg_masks + sidx * 16 + lane) : 0u;
      if (kk + 8 > e0 && kk < e1) {
        ni0 = SEG_LD(reinterpret_cast<const int4*>(idx + kk));
        ni1 = SEG_LD(reinterpret_cast<const int4*>(idx + kk + 4));
#pragma unroll
        for (int q = 0; q < 4; ++q) nv[q] = SEG_LD(reinterpret_cast<const double2*>(vals + kk) + q);
      }
    };
    fetch(e0 & ~int64_t(7), sid);
#endif
    for (int64_t base = e0 & ~int64_t(7); base < e1; base += 256, ++sid) {
      const int64_t k0 = base + 8 * lane;
      double p[8];
#if PDLPK_SEG_PIPELINE
      const uint32_t mw = nmw;
      const int4 i0 = ni0, i1 = ni1;
      double a8[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a8[2 * q] = nv[q].x;
        a8[2 * q + 1] = nv[q].y;
      }
      if (base + 256 < e1) fetch(base + 256, sid + 1);
      if (k0 + 8 > e0 && k0 < e1) {
        const int ci[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          p[u] = (k0 + u >= e0 && k0 + u < e1) ? a8[u] * SEG_G(v + ci[u]) : 0.0;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = 0.0;
      }
#else
      const uint32_t mw = lane < 16 ? __ldg(A.seg_masks + sid * 16 + lane) : 0u;
      if (k0 + 8 > e0 && k0 < e1) {
        const int4 i0 = SEG_LD(reinterpret_cast<const int4*>(idx + k0));
        const int4 i1 = SEG_LD(reinterpret_cast<const int4*>(idx + k0 + 4));
        const int ci[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 t = SEG_LD(reinterpret_cast<const double2*>(vals + k0) + q);
          p[2 * q] = t.x;
          p[2 * q + 1] = t.y;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          p[u] = (k0 + u >= e0 && k0 + u < e1) ? p[u] * SEG_G(v + ci[u]) : 0.0;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = 0.0;
      }
#endif
      const uint32_t hw = __shfl_sync(0xffffffffu, mw, lane >> 2);
      const uint32_t ew = __shfl_sync(0xffffffffu, mw, 8 + (lane >> 2));
      const uint32_t hb = (hw >> (8 * (lane & 3))) & 0xffu, eb = (ew >> (8 * (lane & 3))) & 0xffu;
      const int nend_lane = __popc(eb);
      const int ends_before = warp_excl_scan_i(nend_lane, lane);
      const int nend = __shfl_sync(0xffffffffu, ends_before + nend_lane, 31);
#if PDLPK_SEG_PREFETCH
      for (int j = lane; j < nend; j += 32) epi.prefetch(rc + j);
#endif
      // the segment open at the lane's end, then the segmented scan of those
      // across lanes: what flows into each lane
      double tail = 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) tail = ((hb >> u) & 1u) ? p[u] : tail + p[u];
      const unsigned hmask = __ballot_sync(0xffffffffu, hb != 0u);
      double inc = tail;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, inc, o);
        const unsigned win = lane >= o ? (((2u << lane) - 1u) & ~((1u << (lane - o + 1)) - 1u)) : 0u;
        if (lane >= o && (hmask & win) == 0u) inc += t;
      }
      double into = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) into = 0.0;
      if ((hmask & ((1u << lane) - 1u)) == 0u) into += carry;
      double run = into;
      int64_t line = rc + ends_before;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        run = ((hb >> u) & 1u) ? p[u] : run + p[u];
        if ((eb >> u) & 1u) {
          const typename Epi::Pre pre = epi.load(line);
          epi.line(line, epi.init(pre) + run, pre);
          ++line;
        }
      }
      carry = __shfl_sync(0xffffffffu, run, 31);
      if ((__shfl_sync(0xffffffffu, eb, 31) >> 7) & 1u) carry = 0.0;
      rc += nend;
    }
  }
#undef SEG_LD
#undef SEG_G
}

// Segment mask of a layout: 1 chunks, 2 direct tiles, 4 staged tiles.
// Kernels are instantiated per mask so each pass only pays the registers and
// shared memory of the paths it runs.  The staged tile segment is kept when
// nothing else exists so the grid is never empty (the column pass's last CTA
// makes the step decision).
__host__ __device__ inline int seg_mask(const pdlpk_csr& A) {
  if (A.seg_mode) return 16;
  int s = A.n_chunks > A.n_cta_chunks ? 1 : 0;
  if (A.n_cta_chunks > 0) s |= 8;
  if (A.n_tiles > 0) s |= A.tile_direct ? 2 : 4;
  if (s == 0) s = 4;
  return s;
}

#ifndef PDLPK_CHUNK_MIN_BLOCKS
#define PDLPK_CHUNK_MIN_BLOCKS 4 /* CTAs/SM the chunk-only kernels are compiled for */
#endif
#ifndef PDLPK_TILE_MIN_BLOCKS
#define PDLPK_TILE_MIN_BLOCKS 4 /* CTAs/SM the staged-tile kernels are compiled for */
#endif
#ifndef PDLPK_SEG_MIN_BLOCKS
#define PDLPK_SEG_MIN_BLOCKS 4 /* CTAs/SM the segmented-span kernels are compiled for */
#endif
__host__ __device__ constexpr int spmv_min_blocks(int seg) {
  return seg == 16 ? PDLPK_SEG_MIN_BLOCKS
                   : (seg == 2 ? 5 : (seg == 1 ? PDLPK_CHUNK_MIN_BLOCKS : ((seg & 4) ? PDLPK_TILE_MIN_BLOCKS : 4)));
}

// Chunk segments are grid-stride with a bounded number of CTAs: a pass pays
// its per-CTA partials (block reductions, the decision's combine) once per
// CTA, so millions of short-lived CTAs (C2's 33..2048-entry rows) would cost
// more than the products.
constexpr int64_t kMaxWarpChunkBlocks = 148 * 8;
constexpr int64_t kMaxCtaChunkBlocks = 148 * 4;

__host__ __device__ inline int64_t warp_chunk_blocks(const pdlpk_csr& A) {
  const int64_t b = (A.n_chunks - A.n_cta_chunks + kSpmvWarps - 1) / kSpmvWarps;
  return b < kMaxWarpChunkBlocks ? b : kMaxWarpChunkBlocks;
}

__host__ __device__ inline int64_t cta_chunk_blocks(const pdlpk_csr& A) {
  return A.n_cta_chunks < kMaxCtaChunkBlocks ? A.n_cta_chunks : kMaxCtaChunkBlocks;
}

__host__ __device__ inline int64_t sched_blocks(const pdlpk_csr& A) {
  if (A.seg_mode) return A.tile_blocks;  // persistent warps over the spans
  const int s = seg_mask(A);
  return warp_chunk_blocks(A) + cta_chunk_blocks(A) + ((s & 6) ? A.tile_blocks : 0);
}

__host__ __device__ inline size_t spmv_smem(const pdlpk_csr& A, int seg) {
  return (seg & 4) ? ring_smem(A) : 0;
}

// Opt a kernel into more than 48 KB of dynamic shared memory (staged rings
// above that).  Always the device maximum, never the launch's own size:
// layouts have different rings, and with ranks as threads (ThreadComm) a
// smaller value set by one rank would invalidate another rank's launch.  The
// cap does not change occupancy (the launch's actual size does).
constexpr int kMaxDynSmem = 160 * 1024;  // rings stay far below; leaves room for static smem
template <class Kernel>
inline void allow_smem(Kernel k, size_t smem) {
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
  }
}

// 16-byte-aligned window of elements [first, first + count) of a global array.
struct Win {
  const char* src;
  uint32_t bytes;
  uint32_t shift;  // byte offset of element `first` inside the window
};

__device__ __forceinline__ Win win(const void* base, int64_t first, int64_t count, int esz) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(base) + static_cast<uintptr_t>(first) * esz;
  const uintptr_t hi = lo + static_cast<uintptr_t>(count) * esz;
  const uintptr_t alo = lo & ~uintptr_t(15);
  const uintptr_t ahi = (hi + 15) & ~uintptr_t(15);
  return Win{reinterpret_cast<const char*>(alo), count > 0 ? static_cast<uint32_t>(ahi - alo) : 0u,
             static_cast<uint32_t>(lo - alo)};
}

// Entries [k0, hi) stepping 32 (one lane's share of a warp's range), in
// predicated batches of 8 independent loads then 8 gathers; acc[u] takes
// every 8th of the lane's entries.
#ifndef PDLPK_BATCH
#define PDLPK_BATCH 8 /* independent loads per lane per batch (multiple of 8) */
#endif
constexpr int kBatch = PDLPK_BATCH;

#ifndef PDLPK_IDX_PREFETCH
#define PDLPK_IDX_PREFETCH 1
#endif

__device__ __forceinline__ void warp_batches(const int32_t* __restrict__ idx,
                                             const double* __restrict__ vals,
                                             const double* __restrict__ v, int64_t k0, int64_t hi,
                                             double (&acc)[8]) {
#if PDLPK_IDX_PREFETCH
  // The dependent chain is index -> gather; the values are only needed by
  // the multiply.  So each batch loads its values and the NEXT batch's
  // indices while its gathers (indices loaded one batch earlier) resolve:
  // one memory round trip per batch instead of two.
  int32_t ci[kBatch];
#pragma unroll
  for (int u = 0; u < kBatch; ++u) {
    const int64_t k = k0 + u * 32;
    if (k < hi) ci[u] = ld_stream(idx + k);
  }
  for (int64_t base = k0; base < hi; base += kBatch * 32) {
    const int64_t nb = base + kBatch * 32;
    double a[kBatch];
    int32_t cn[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      if (base + u * 32 < hi) a[u] = ld_stream(vals + base + u * 32);
      if (nb + u * 32 < hi) cn[u] = ld_stream(idx + nb + u * 32);
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      if (base + u * 32 < hi) acc[u & 3] = mac(acc[u & 3], a[u], __ldg(v + ci[u]));
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) ci[u] = cn[u];
  }
#else
  for (int64_t base = k0; base < hi; base += kBatch * 32) {
    int32_t ci[kBatch];
    double a[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int64_t k = base + u * 32;
      if (k < hi) {
        ci[u] = ld_stream(idx + k);
        a[u] = ld_stream(vals + k);
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      if (base + u * 32 < hi) acc[u & 7] = mac(acc[u & 7], a[u], __ldg(v + ci[u]));
    }
  }
#endif
}

struct TileMeta {
  int64_t r0, s0;
  int cnt, len;
};

__device__ __forceinline__ TileMeta tile_meta(const pdlpk_csr& A, int64_t t) {
  const int pack = A.tile_rows[t];
  return TileMeta{A.tile_row0[t], A.tile_nnz0[t], pack & 0xfff, pack >> 12};
}

template <class P, int Seg, class Epi>
__device__ __forceinline__ void sched_spmv(const pdlpk_csr& A, const double* __restrict__ vals,
                                           const double* __restrict__ v, Epi& epi) {
  const P* __restrict__ start = static_cast<const P*>(A.start);
  const int32_t* __restrict__ idx = A.index;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  int64_t b = blockIdx.x;
  if constexpr ((Seg & 16) != 0) {
    seg_spans(A, vals, v, epi);
    return;
  }
  if constexpr ((Seg & 1) != 0) {
    const int64_t chunk_blocks = warp_chunk_blocks(A);
    if (b < chunk_blocks) {
      // one warp per medium line (a warp chunk is always a whole line)
      const int64_t nw = A.n_chunks - A.n_cta_chunks;
      for (int64_t c = b * kSpmvWarps + warp; c < nw; c += chunk_blocks * kSpmvWarps) {
        const int64_t r = A.chunk_row[c];
        const int64_t lo = A.chunk_beg[c];
        const int64_t hi = lo + A.chunk_len[c];
        typename Epi::Pre pre{};
        if (lane == 0) pre = epi.load(r);
        // predicated batches of 8 entries per lane: independent loads, then
        // their gathers
        double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        warp_batches(idx, vals, v, lo + lane, hi, acc);
        const double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        const double t = warp_sum(s);
        if (lane == 0) epi.line(r, epi.init(pre) + t, pre);
      }
      return;
    }
    b -= chunk_blocks;
  }
  if constexpr ((Seg & 8) != 0) {
    const int64_t cblocks = cta_chunk_blocks(A);
    if (b < cblocks) {
      __shared__ double wsum[kSpmvWarps];
      for (int64_t cc = b; cc < A.n_cta_chunks; cc += cblocks) {
      // One CTA per chunk of <= kChunk entries: warp w takes one slice of
      // <= 256 entries (a single batch of independent loads), the 8 warp
      // sums are added in warp order, thread 0 runs the epilogue or the
      // ordered multi-chunk combine.  C1's 2,000-entry rows: one round trip
      // per row instead of eight per warp.
      const int64_t c = (A.n_chunks - A.n_cta_chunks) + cc;
      const int64_t r = A.chunk_row[c];
      const int64_t lo = A.chunk_beg[c];
      const int64_t hi = lo + A.chunk_len[c];
      const int pos = A.chunk_pos[c];
      const int nch = pos >> 16;
      const int64_t per = (((hi - lo) + kSpmvWarps - 1) / kSpmvWarps + 31) & ~int64_t(31);
      const int64_t wlo = lo + warp * per;
      const int64_t whi = wlo + per < hi ? wlo + per : hi;
      double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      warp_batches(idx, vals, v, wlo + lane, whi, acc);
      const double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      const double t = warp_sum(s);
      if (lane == 0) wsum[warp] = t;
      __syncthreads();
      if (threadIdx.x == 0) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kSpmvWarps; ++w) sum += wsum[w];
        if (nch == 1) {
          const typename Epi::Pre pre = epi.load(r);
          epi.line(r, epi.init(pre) + sum, pre);
        } else {
          const int64_t c0 = c - (pos & 0xffff);
          A.chunk_part[c] = sum;
          __threadfence();
          const unsigned arrived = atomicAdd(A.chunk_cnt + c0, 1u);
          if (arrived == static_cast<unsigned>(nch - 1)) {
            __threadfence();
            double tot = 0.0;
            for (int q = 0; q < nch; ++q) tot += __ldcg(A.chunk_part + c0 + q);
            A.chunk_cnt[c0] = 0;
            Epi solo = epi;
            solo.reset_acc();
            const typename Epi::Pre pre = solo.load(r);
            solo.line(r, solo.init(pre) + tot, pre);
            solo.export_acc(A.line_acc + static_cast<int64_t>(A.chunk_slot[c]) * PDLPK_LINE_ACC);
          }
        }
      }
      __syncthreads();  // wsum is rewritten by the next chunk
      }
      return;
    }
    b -= cblocks;
  }
  if constexpr ((Seg & 2) != 0) {
    if (b < A.tile_blocks) {
      // grid-stride over the tiles: the pass's per-CTA partials and
      // decision ticket are paid once per CTA, not once per tile
      for (int64_t t = b; t < A.n_tiles; t += A.tile_blocks) {
      const TileMeta tm = tile_meta(A, t);
      if (static_cast<int>(threadIdx.x) < tm.cnt) {
        const int64_t r = tm.r0 + threadIdx.x;
        const typename Epi::Pre pre = epi.load(r);
        const int64_t a = start[r], e = start[r + 1];
        // predicated pairs: independent loads, then the gathers, then the
        // products added in storage order (bit-identical line sums)
        double acc = epi.init(pre);
        for (int64_t k = a; k < e; k += 2) {
          const bool two = k + 1 < e;
          const int32_t c0 = ld_stream(idx + k);
          const int32_t c1 = two ? ld_stream(idx + k + 1) : c0;
          const double a0 = ld_stream(vals + k);
          const double a1 = two ? ld_stream(vals + k + 1) : 0.0;
          const double g0 = __ldg(v + c0);
          const double g1 = __ldg(v + c1);
          acc = mac(acc, a0, g0);
          if (two) acc = mac(acc, a1, g1);
        }
        epi.line(r, acc, pre);
      }
      }
      return;
    }
    b -= A.tile_blocks;
  }
  if constexpr ((Seg & 4) != 0) {
    // Warp-specialized ring: warp 0 produces (one lane issues the bulk
    // copies of a whole tile), warps 1..kConsumerWarps consume, each owning
    // 32 consecutive lines of the tile.  full[s] completes on the copies'
    // transaction bytes, empty[s] on one arrive per consumer warp; no CTA
    // barrier inside the loop.
    extern __shared__ __align__(128) unsigned char ring[];
    uint64_t* full = reinterpret_cast<uint64_t*>(ring);
    uint64_t* empty = full + kStages;
    TileHdr* hdr = reinterpret_cast<TileHdr*>(ring + 2 * 8 * kStages);
    unsigned char* stage0 = ring + kRingHeader;
    const int64_t tb = A.tile_blocks;
    const StageLayout sl = stage_layout(A.tile_lines_cap, A.tile_nnz_cap);
    const size_t stage_bytes = static_cast<size_t>(A.tile_stage_bytes);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < kStages; ++q) {
        mbar_init(&full[q], 1);
        mbar_init(&empty[q], kConsumerWarps);
      }
      mbar_fence_init();
    }
    __syncthreads();
    if (warp == 0) {
      if (lane == 0) {
        int i = 0;
        for (int64_t t = b; t < A.n_tiles; t += tb, ++i) {
          const int stage = i % kStages;
          if (i >= kStages) mbar_wait(&empty[stage], ((i / kStages) + 1) & 1);
          const TileMeta tm = tile_meta(A, t);
          unsigned char* buf = stage0 + stage * stage_bytes;
          const Win wi = win(idx, tm.s0, tm.len, 4);
          const Win wv = win(vals, tm.s0, tm.len, 8);
          const Win wp = win(start, tm.r0, tm.cnt + 1, static_cast<int>(sizeof(P)));
          uint32_t total = wi.bytes + wv.bytes + wp.bytes;
          uint32_t shifts = wi.shift | (wv.shift << 4) | (wp.shift << 8);
          Win we[kMaxStaged];
#pragma unroll
          for (int q = 0; q < Epi::kStaged; ++q) {
            we[q] = win(epi.staged_src(q), tm.r0, tm.cnt, 8);
            total += we[q].bytes;
            shifts |= we[q].shift << (12 + 4 * q);
          }
          TileHdr h;
          h.r0 = tm.r0;
          h.s0 = tm.s0;
          h.cnt = tm.cnt;
          h.shifts = shifts;
          h.per = (tm.cnt + kConsumerWarps - 1) / kConsumerWarps;
          h.pad = 0;
          hdr[stage] = h;  // released by the arrive below
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full[stage], total);
#if PDLPK_MATRIX_EVICT_FIRST
          const uint64_t pol = l2_evict_first_policy();
          if (wi.bytes) bulk_g2s_hint(buf, wi.src, wi.bytes, &full[stage], pol);
          if (wv.bytes) bulk_g2s_hint(buf + sl.val, wv.src, wv.bytes, &full[stage], pol);
          if (wp.bytes) bulk_g2s_hint(buf + sl.ptr, wp.src, wp.bytes, &full[stage], pol);
#else
          if (wi.bytes) bulk_g2s(buf, wi.src, wi.bytes, &full[stage]);
          if (wv.bytes) bulk_g2s(buf + sl.val, wv.src, wv.bytes, &full[stage]);
          if (wp.bytes) bulk_g2s(buf + sl.ptr, wp.src, wp.bytes, &full[stage]);
#endif
#pragma unroll
          for (int q = 0; q < Epi::kStaged; ++q) {
            if (we[q].bytes) {
#if PDLPK_MATRIX_EVICT_FIRST
              if (!epi.staged_reused(q)) {
                bulk_g2s_hint(buf + sl.epi + q * sl.epi_stride, we[q].src, we[q].bytes,
                              &full[stage], pol);
                continue;
              }
#endif
              bulk_g2s(buf + sl.epi + q * sl.epi_stride, we[q].src, we[q].bytes, &full[stage]);
            }
          }
        }
      }
    } else {
      const int cw = warp - 1;  // consumer warp: lines [per cw, per cw + per) of each tile
      int i = 0;
      for (int64_t t = b; t < A.n_tiles; t += tb, ++i) {
        const int stage = i % kStages;
        unsigned char* buf = stage0 + stage * stage_bytes;
        mbar_wait(&full[stage], (i / kStages) & 1);
        const TileHdr h = hdr[stage];
        const TileMeta tm{h.r0, h.s0, h.cnt, 0};
        const uint32_t sh = h.shifts;
        const int32_t* s_idx = reinterpret_cast<const int32_t*>(buf + (sh & 15u));
        double* s_val = reinterpret_cast<double*>(buf + sl.val + ((sh >> 4) & 15u));
        const P* s_ptr = reinterpret_cast<const P*>(buf + sl.ptr + ((sh >> 8) & 15u));
        const double* s_epi[kMaxStaged];
#pragma unroll
        for (int q = 0; q < Epi::kStaged; ++q) {
          s_epi[q] = reinterpret_cast<const double*>(buf + sl.epi + q * sl.epi_stride +
                                                     ((sh >> (12 + 4 * q)) & 15u));
        }
        // the tile's lines split evenly over the consumer warps (a tile of
        // 20-32-entry lines holds only ~45 lines: fixed 96-line ranges would
        // leave six warps idle)
        const int per = h.per;
        const int l0 = per * cw;
        if (l0 < tm.cnt) {
          const int l1 = l0 + per < tm.cnt ? l0 + per : tm.cnt;
          const int e0 = static_cast<int>(static_cast<int64_t>(s_ptr[l0]) - tm.s0);
          const int e1 = static_cast<int>(static_cast<int64_t>(s_ptr[l1]) - tm.s0);
          // this warp's products in place (the gather is the only global
          // access): batches of kTileGather per lane keep that many gathers
          // in flight
          for (int j0 = e0 + lane; j0 < e1; j0 += kTileGather * 32) {
            int32_t ci[kTileGather];
            double g[kTileGather];
#pragma unroll
            for (int u = 0; u < kTileGather; ++u) {
              if (j0 + 32 * u < e1) ci[u] = s_idx[j0 + 32 * u];
            }
#pragma unroll
            for (int u = 0; u < kTileGather; ++u) {
              if (j0 + 32 * u < e1) g[u] = __ldg(v + ci[u]);
            }
#pragma unroll
            for (int u = 0; u < kTileGather; ++u) {
              if (j0 + 32 * u < e1) s_val[j0 + 32 * u] = s_val[j0 + 32 * u] * g[u];
            }
          }
          __syncwarp();
#pragma unroll
          for (int q = 0; q < kLinesPerLane; ++q) {
            const int li = l0 + lane + 32 * q;
            if (li < l1) {
              const int a = static_cast<int>(static_cast<int64_t>(s_ptr[li]) - tm.s0);
              const int e = static_cast<int>(static_cast<int64_t>(s_ptr[li + 1]) - tm.s0);
              const typename Epi::Pre pre = epi.from_stage(s_epi, li);
              double acc = epi.init(pre);  // 0, or the line's carried partial sum
              for (int j = a; j < e; ++j) acc += s_val[j];
              epi.line(tm.r0 + li, acc, pre);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
      }
    }
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
    case 8: return f.template go<P, 8>();
    case 9: return f.template go<P, 9>();
    case 12: return f.template go<P, 12>();
    case 16: return f.template go<P, 16>();
    default: return f.template go<P, 13>();  // (direct tiles never mix with CTA chunks)
  }
}

template <class F>
inline int dispatch_p(const pdlpk_csr& A, F&& f) {
  if (A.wide) return dispatch_seg<int64_t>(seg_mask(A), f);
  return dispatch_seg<int32_t>(seg_mask(A), f);
}

}  // namespace pdlp
