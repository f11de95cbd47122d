// Generic multi-value reductions in the three orders of kernels.h:
//   TREE  — grid-stride per-thread chains, fixed block tree, per-CTA
//           partials, fixed final tree (perf mode; deterministic)
//   SEQ   — one chain in index order (the reference's plain loops)
//   SHARD — make_shard_plan(dim, 1, S) chains, ascending combine
//           (kernels.hpp:69-97)
// A functor f(i, v[K]) -> bitmask of the values that coordinate i
// contributes; bit k of maxmask selects max (std::max semantics) instead of
// sum for value k.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace pdlp {

constexpr int kRedThreads = 256;

// Row-sharded solves: reductions launched while a log is set on this host
// thread record where their K values went (pdlpk_set_red_log, kernels.h).
inline thread_local pdlpk_red_log* g_red_log = nullptr;

inline void red_log_record(double* out, int k, unsigned maxmask) {
  pdlpk_red_log* L = g_red_log;
  if (L == nullptr) return;
  if (L->count < 48) {
    L->k[L->count] = k;
    L->maxmask[L->count] = maxmask;
    L->out[L->count] = out;
  }
  ++L->count;  // > 48: the engine reports an overflow
}
constexpr int kRedMaxBlocks = 148 * 8;

template <int K>
__device__ __forceinline__ void red_accum(double* acc, const double* v, unsigned use,
                                          unsigned maxmask) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if ((use >> k) & 1u) acc[k] = ((maxmask >> k) & 1u) ? max_keep(acc[k], v[k]) : acc[k] + v[k];
  }
}

template <int K, class F>
__global__ void red_seq_kernel(F f, int64_t n, unsigned maxmask, double* out) {
  pdl_wait_cadence();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double v[K];
    const unsigned use = f(i, v);
    red_accum<K>(acc, v, use, maxmask);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = acc[k];
}

template <int K, class F>
__global__ void red_shard_kernel(F f, int64_t n, int S, unsigned maxmask, double* part) {
  pdl_wait_cadence();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const int64_t base = n / S, rem = n % S;
  const int64_t lo = s * base + (s < rem ? s : rem);
  const int64_t hi = lo + base + (s < rem ? 1 : 0);
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  for (int64_t i = lo; i < hi; ++i) {
    double v[K];
    const unsigned use = f(i, v);
    red_accum<K>(acc, v, use, maxmask);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) part[k * S + s] = acc[k];
}

template <int K>
__global__ void red_shard_final(const double* part, int S, unsigned maxmask, double* out) {
  pdl_wait_cadence();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = 0.0;
    for (int s = 0; s < S; ++s) {
      t = ((maxmask >> k) & 1u) ? max_keep(t, part[k * S + s]) : t + part[k * S + s];
    }
    out[k] = t;
  }
}

template <int K, class F>
__global__ void __launch_bounds__(kRedThreads) red_tree_kernel(F f, int64_t n, unsigned maxmask,
                                                               double* part) {
  pdl_wait_cadence();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    double v[K];
    const unsigned use = f(i, v);
    red_accum<K>(acc, v, use, maxmask);
  }
  __shared__ double sm[32];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double r = ((maxmask >> k) & 1u) ? block_max(acc[k], sm) : block_sum(acc[k], sm);
    if (threadIdx.x == 0) part[k * gridDim.x + blockIdx.x] = r;
    __syncthreads();
  }
}

template <int K>
__global__ void __launch_bounds__(kRedThreads) red_tree_final(const double* part, int G,
                                                              unsigned maxmask, double* out) {
  pdl_wait_cadence();
  __shared__ double sm[32];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool mx = (maxmask >> k) & 1u;
    double a = 0.0;
    for (int b = threadIdx.x; b < G; b += blockDim.x) {
      a = mx ? max_keep(a, part[k * G + b]) : a + part[k * G + b];
    }
    const double r = mx ? block_max(a, sm) : block_sum(a, sm);
    if (threadIdx.x == 0) out[k] = r;
    __syncthreads();
  }
}

inline int red_tree_blocks(int64_t n) {
  int64_t b = (n + kRedThreads - 1) / kRedThreads;
  if (b > kRedMaxBlocks) b = kRedMaxBlocks;
  return b < 1 ? 1 : static_cast<int>(b);
}

// order: PDLPK_RED_*; scratch needs K * max(kRedMaxBlocks, S) doubles.
template <int K, class F>
inline int multi_reduce(F f, int64_t n, int order, int shards, unsigned maxmask,
                        double* scratch, double* out, cudaStream_t s) {
  if (order == PDLPK_RED_SEQ) {
    launch_pdl(PDLPK_PDL_CADENCE, red_seq_kernel<K, F>, 1, 1, 0, s, f, n, maxmask, out);
  } else if (order == PDLPK_RED_SHARD) {
    launch_pdl(PDLPK_PDL_CADENCE, red_shard_kernel<K, F>, static_cast<unsigned>((shards + 127) / 128), 128, 0, s,
               f, n, shards, maxmask, scratch);
    launch_pdl(PDLPK_PDL_CADENCE, red_shard_final<K>, 1, 1, 0, s, static_cast<const double*>(scratch), shards,
               maxmask, out);
  } else {
    const int g = red_tree_blocks(n);
    launch_pdl(PDLPK_PDL_CADENCE, red_tree_kernel<K, F>, static_cast<unsigned>(g), kRedThreads, 0, s, f, n,
               maxmask, scratch);
    launch_pdl(PDLPK_PDL_CADENCE, red_tree_final<K>, 1, kRedThreads, 0, s, static_cast<const double*>(scratch), g,
               maxmask, out);
  }
  red_log_record(out, K, maxmask);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace pdlp
