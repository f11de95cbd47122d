// Exact normalized duality gap on device (reference
// proj/include/pdhglp/restarts.hpp:107-220), in two launches around one host
// read of the event count:
//
//   prepare  1. lam -> inf masses b_inf, c_inf (SEQ order in parity mode)
//            2. breakpoint events: <= 1 per primal coordinate (slot i), <= 2
//               per dual coordinate (slots n+2j, n+2j+1) — slot order is the
//               reference's push order — flagged and compacted with an
//               order-preserving select, so only real events go further
//   finish   3. stable radix sort of the E events by lambda, descending, on an
//               order-preserving uint64 key (decoded back to lambda exactly)
//            4. sweep to the first group with phi(lam) = C + B/lam^2 >= r^2:
//               parity — the reference's sequential loop on one thread;
//               perf   — exclusive scans of the event masses + parallel first hit
//            5. closed-form lambda*, candidate assembly (assemble_candidate
//               :73-101) and the gap value (gap_value_at :50-71), SEQ in parity.
//
// Parity caveat: std::sort is not stable, so events with EQUAL lambda may be
// visited in a different order than the reference's introsort puts them,
// which can change the last bit of the running masses.  Exact ties need
// bitwise-equal breakpoints; DESIGN.md records this.
//
// CUB (part of the CUDA toolkit) provides select/sort/scan; this is cadence
// work (2-3 evaluations per 64 steps), not the per-step hot loop.
// Translation unit compiled with -fmad=false (see common.cuh).

#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "kernels.h"
#include "reduce.cuh"

namespace pdlp {
namespace {

constexpr int kT = 256;

inline int ew_blocks(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  if (b > 148 * 8) b = 148 * 8;
  return b < 1 ? 1 : static_cast<int>(b);
}

#define GRID_STRIDE(i, n)                                                                   \
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)

struct GapScalars {
  double sums[2];  // b_inf, c_inf
  double lambda_star;
  double value;
  unsigned long long first;  // first crossing group index (perf)
  int num_events;            // compacted event count (select output)
  int num_high;              // window sort: events inside the window
  unsigned long long thresh; // (unused)
  // Sweep start: masses before the first sorted event (c, b) and the lambda
  // of the group before it (hi0).  Full sort: the lambda -> inf masses and
  // inf; window sort: plus every event above the window.
  double base[3];
  unsigned long long lo_key, hi_key;  // window [lo_key, hi_key]
  unsigned long long above_min;       // smallest key above the window
  unsigned long long above_count;     // events above the window
  double above[2];                    // their masses (c, b), tree order
  int est_ra, est_rb;                 // estimated window: sample ranks (rb < 0: to the bottom)
};

struct Work {
  uint8_t* flag;  // per slot
  double *lam, *dc, *di;  // per slot
  int32_t *sel;            // compacted slot ids (slot order)
  uint64_t *keys_in, *keys_out;
  int32_t* vals_out;
  double *cs, *bs;  // sorted masses (perf scans)
  int32_t* hsel;    // partial sort: slots of the selected (top) events
  uint64_t *samp_in, *samp_out;  // partial sort: key sample and its sort
  int32_t *sidx_in, *sidx_out;    // estimated window: sample ranks through the sort
  double *sdc, *sdi;              // ... and the sampled events' masses
  GapScalars* sc;
  void* cub_tmp;
  size_t cub_bytes;
};

__host__ __device__ inline size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

constexpr int kGapSample = 65536;  // keys sampled to place the partial-sort threshold

size_t cub_bytes_for(int64_t N) {
  size_t a = 0, b = 0, c = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, a, static_cast<uint64_t*>(nullptr),
                                            static_cast<uint64_t*>(nullptr),
                                            static_cast<int32_t*>(nullptr),
                                            static_cast<int32_t*>(nullptr), static_cast<int>(N));
  cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<double*>(nullptr),
                                static_cast<double*>(nullptr), static_cast<int>(N));
  cub::DeviceSelect::Flagged(nullptr, c, thrust::counting_iterator<int32_t>(0),
                             static_cast<uint8_t*>(nullptr), static_cast<int32_t*>(nullptr),
                             static_cast<int*>(nullptr), static_cast<int>(N));
  size_t d = 0, e = 0, f = 0;
  cub::DeviceSelect::Flagged(nullptr, d, static_cast<uint64_t*>(nullptr),
                             static_cast<uint8_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                             static_cast<int*>(nullptr), static_cast<int>(N));
  cub::DeviceRadixSort::SortKeysDescending(nullptr, e, static_cast<uint64_t*>(nullptr),
                                           static_cast<uint64_t*>(nullptr), kGapSample);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, f, static_cast<uint64_t*>(nullptr),
                                            static_cast<uint64_t*>(nullptr),
                                            static_cast<int32_t*>(nullptr),
                                            static_cast<int32_t*>(nullptr), kGapSample);
  return std::max(std::max(std::max(a, f), std::max(b, c)), std::max(d, e));
}

Work carve(void* base, int64_t n, int64_t m) {
  const int64_t N = n + 2 * m;
  char* p = static_cast<char*>(base);
  Work w;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += align_up(bytes);
    return r;
  };
  w.flag = reinterpret_cast<uint8_t*>(take(N));
  w.lam = reinterpret_cast<double*>(take(8 * N));
  w.dc = reinterpret_cast<double*>(take(8 * N));
  w.di = reinterpret_cast<double*>(take(8 * N));
  w.sel = reinterpret_cast<int32_t*>(take(4 * N));
  w.keys_in = reinterpret_cast<uint64_t*>(take(8 * N));
  w.keys_out = reinterpret_cast<uint64_t*>(take(8 * N));
  w.vals_out = reinterpret_cast<int32_t*>(take(4 * N));
  w.cs = reinterpret_cast<double*>(take(8 * N));
  w.bs = reinterpret_cast<double*>(take(8 * N));
  w.hsel = reinterpret_cast<int32_t*>(take(4 * N));
  w.samp_in = reinterpret_cast<uint64_t*>(take(8 * kGapSample));
  w.samp_out = reinterpret_cast<uint64_t*>(take(8 * kGapSample));
  w.sidx_in = reinterpret_cast<int32_t*>(take(4 * kGapSample));
  w.sidx_out = reinterpret_cast<int32_t*>(take(4 * kGapSample));
  w.sdc = reinterpret_cast<double*>(take(8 * kGapSample));
  w.sdi = reinterpret_cast<double*>(take(8 * kGapSample));
  w.sc = reinterpret_cast<GapScalars*>(take(sizeof(GapScalars)));
  w.cub_bytes = cub_bytes_for(N);
  w.cub_tmp = take(w.cub_bytes);
  return w;
}

// Order-preserving map double -> uint64 and its exact inverse.
__device__ __forceinline__ uint64_t order_key(double d) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

struct GapIn {
  const double *c, *lv, *uv, *lc, *uc;
  const double *x, *y, *ax, *aty;
  int64_t n, m;
  double omega;
  uint32_t uni;          // pdlpk_problem::uniform: scalar c / l_v / u_v
  double cu, lvu, uvu;
  __device__ __forceinline__ double cc(int64_t i) const { return (uni & 1u) ? cu : c[i]; }
  __device__ __forceinline__ double lo(int64_t i) const { return (uni & 2u) ? lvu : lv[i]; }
  __device__ __forceinline__ double hi(int64_t i) const { return (uni & 4u) ? uvu : uv[i]; }
};

// Per-coordinate logic of restarts.hpp:117-170: the b_inf / c_inf
// contributions (flags bit0 / bit1) and up to two events.
struct Coord {
  unsigned mass_use = 0;
  double b = 0.0, c = 0.0;
  int ne = 0;
  double lam0 = 0.0, dc0 = 0.0, di0 = 0.0, lam1 = 0.0, dc1 = 0.0, di1 = 0.0;
  // events are pushed in the reference's order; fixed slots keep them in
  // registers (a dynamically indexed array would live in local memory)
  __device__ __forceinline__ void push(double l, double c_, double d_) {
    if (ne == 0) {
      lam0 = l; dc0 = c_; di0 = d_;
    } else {
      lam1 = l; dc1 = c_; di1 = d_;
    }
    ++ne;
  }
};

__device__ __forceinline__ Coord gap_coord(const GapIn& g, int64_t t) {
  Coord o;
  const double omega = g.omega;
  if (t < g.n) {
    const int64_t i = t;
    const double gg = g.aty[i] - g.cc(i);
    if (gg == 0.0) return o;
    const double off = (gg > 0.0 ? g.hi(i) : g.lo(i)) - g.x[i];
    if (off == 0.0) return o;
    o.b = gg * gg / omega;
    o.mass_use |= 1u;
    if (finite_d(off)) {
      o.push(gg / (omega * off), omega * off * off, -gg * gg / omega);
    }
    return o;
  }
  const int64_t j = t - g.n;
  const double yj = g.y[j];
  const double bm = g.ax[j] - g.uc[j];
  const double bp = g.ax[j] - g.lc[j];
  const double im = yj * yj / omega;
  if (yj > 0.0) {
    if (bp <= 0.0) {
      if (bp < 0.0) {
        o.b = omega * bp * bp;
        o.mass_use |= 1u;
      }
      return o;
    }
    if (finite_d(bp)) {
      o.b = omega * bp * bp;
      o.mass_use |= 1u;
      o.push(omega * bp / yj, im, -omega * bp * bp);
    } else {
      o.c = im;
      o.mass_use |= 2u;
    }
    if (bm > 0.0) {
      o.push(omega * bm / yj, -im, omega * bm * bm);
    }
  } else if (yj < 0.0) {
    if (bm >= 0.0) {
      if (bm > 0.0) {
        o.b = omega * bm * bm;
        o.mass_use |= 1u;
      }
      return o;
    }
    if (finite_d(bm)) {
      o.b = omega * bm * bm;
      o.mass_use |= 1u;
      o.push(omega * bm / yj, im, -omega * bm * bm);
    } else {
      o.c = im;
      o.mass_use |= 2u;
    }
    if (bp < 0.0) {
      o.push(omega * bp / yj, -im, omega * bp * bp);
    }
  } else {
    if (bm > 0.0) {
      o.b = omega * bm * bm;
      o.mass_use |= 1u;
    } else if (bp < 0.0) {
      o.b = omega * bp * bp;
      o.mass_use |= 1u;
    }
  }
  return o;
}

// Breakpoint events of coordinate t into its slot(s).
__device__ __forceinline__ void write_events(const GapIn& g, const Work& w, int64_t t,
                                             const Coord& o) {
  const int64_t s0 = t < g.n ? t : g.n + 2 * (t - g.n);
  const int slots = t < g.n ? 1 : 2;
  for (int e = 0; e < slots; ++e) {
    const int64_t s = s0 + e;
    const bool valid = e < o.ne;
    w.flag[s] = valid ? 1 : 0;
    if (valid) {
      w.lam[s] = e == 0 ? o.lam0 : o.lam1;
      w.dc[s] = e == 0 ? o.dc0 : o.dc1;
      w.di[s] = e == 0 ? o.di0 : o.di1;
    }
  }
}

__global__ void events_kernel(GapIn g, Work w) {
  pdl_wait_cadence();
  GRID_STRIDE(t, g.n + g.m) write_events(g, w, t, gap_coord(g, t));
}

__global__ void keys_kernel(Work w, int64_t E) {
  pdl_wait_cadence();
  GRID_STRIDE(e, E) w.keys_in[e] = order_key(w.lam[w.sel[e]]);
}

__device__ double finish_lambda(double lambda_star) {
  if (!finite_d(lambda_star)) lambda_star = 1e300;
  if (lambda_star <= 0.0) lambda_star = 1e-300;
  return lambda_star;
}

// Reference sweep (restarts.hpp:175-212), one thread, sorted order.
__global__ void sweep_seq_kernel(Work w, int64_t E, const double* r_slot, double r_value) {
  pdl_wait_cadence();
  const double r = r_slot ? *r_slot : r_value;
  const double r2 = r * r;
  double c_sum = w.sc->sums[1];
  double b_sum = w.sc->sums[0];
  double hi = CUDART_INF;
  double ls = -1.0;
  int64_t idx = 0;
  while (idx < E) {
    const double lam = key_value(w.keys_out[idx]);
    const double phi_lo = c_sum + b_sum / (lam * lam);
    if (phi_lo >= r2) {
      if (b_sum > 0.0 && r2 > c_sum) {
        ls = sqrt(b_sum / (r2 - c_sum));
      } else {
        ls = lam;
      }
      ls = clampd(ls, lam, hi);
      break;
    }
    while (idx < E && key_value(w.keys_out[idx]) == lam) {
      const int32_t s = w.vals_out[idx];
      c_sum += w.dc[s];
      b_sum += w.di[s];
      ++idx;
    }
    hi = lam;
  }
  if (ls < 0.0) {
    if (b_sum > 0.0 && r2 > c_sum) {
      ls = sqrt(b_sum / (r2 - c_sum));
      ls = ls < hi ? ls : hi;  // std::min(ls, hi)
    } else if (b_sum > 0.0) {
      ls = hi;
    } else {
      ls = finite_d(hi) ? hi / 2.0 : 1.0;
    }
  }
  w.sc->lambda_star = finish_lambda(ls);
}

__global__ void gather_masses_kernel(Work w, int64_t E) {
  pdl_wait_cadence();
  GRID_STRIDE(idx, E) {
    const int32_t s = w.vals_out[idx];
    w.cs[idx] = w.dc[s];
    w.bs[idx] = w.di[s];
  }
}

__global__ void init_first_kernel(Work w) {
  pdl_wait_cadence();
  w.sc->first = ~0ull;
}

// Window sort: a strided sample of the keys places the window's bounds at
// depth fractions of the descending order.
__global__ void sample_keys_kernel(Work w, int64_t E) {
  pdl_wait_cadence();
  GRID_STRIDE(i, kGapSample) w.samp_in[i] = w.keys_in[(i * E) / kGapSample];
}
// Position of the first crossing as a fraction of all events (1 when none):
// the engine sizes the next partial sort from it.
__global__ void hit_fraction_kernel(Work w, int64_t E, double* out) {
  pdl_wait_cadence();
  const unsigned long long f = w.sc->first;
  *out = (f == ~0ull || E <= 0)
             ? 1.0
             : static_cast<double>(f + w.sc->above_count) / static_cast<double>(E);
}

__global__ void base_full_kernel(Work w) {
  pdl_wait_cadence();
  w.sc->base[0] = w.sc->sums[1];
  w.sc->base[1] = w.sc->sums[0];
  w.sc->base[2] = CUDART_INF;
  w.sc->above_count = 0;
}

// First evaluation of a (subproblem, query) -- no previous crossing depth to
// place a window: the strided sample carries its events' masses, is sorted,
// and one CTA scans it with the masses scaled by E / S to estimate where
// phi first reaches r^2; the window is the sample ranks around it.  A miss
// falls back to the full sort (gap_window returns 0), so the estimate only
// decides the cost, never the value.
__global__ void sample_masses_kernel(Work w, int64_t E) {
  pdl_wait_cadence();
  GRID_STRIDE(i, kGapSample) {
    const int64_t pos = (i * E) / kGapSample;
    const int32_t t = w.sel[pos];
    w.samp_in[i] = w.keys_in[pos];
    w.sidx_in[i] = static_cast<int32_t>(i);
    w.sdc[i] = w.dc[t];
    w.sdi[i] = w.di[t];
  }
}

// The sample's masses in sorted order (w.cs / w.bs are free until the window
// is selected), so the one-CTA scan below reads them with independent,
// pipelined loads instead of a dependent gather per sample rank.
__global__ void sorted_masses_kernel(Work w) {
  pdl_wait_cadence();
  GRID_STRIDE(j, kGapSample) {
    const int32_t q = w.sidx_out[j];
    w.cs[j] = w.sdc[q];
    w.bs[j] = w.sdi[q];
  }
}

constexpr int kEstThreads = 1024;
constexpr int kEstPer = kGapSample / kEstThreads;
__global__ void __launch_bounds__(kEstThreads) estimate_window_kernel(Work w, int64_t E, double r,
                                                                      int margin) {
  pdl_wait_cadence();
  const double scale = static_cast<double>(E) / kGapSample;
  const double r2 = r * r;
  const int j0 = threadIdx.x * kEstPer;
  double c = 0.0, b = 0.0;
#pragma unroll 16
  for (int j = j0; j < j0 + kEstPer; ++j) {
    c += w.cs[j];
    b += w.bs[j];
  }
  using Scan = cub::BlockScan<double, kEstThreads>;
  __shared__ typename Scan::TempStorage tmp;
  double cx, bx;
  Scan(tmp).ExclusiveSum(c, cx);
  __syncthreads();
  Scan(tmp).ExclusiveSum(b, bx);
  __shared__ int hit;
  if (threadIdx.x == 0) hit = kGapSample;
  __syncthreads();
  double cs = cx, bs = bx;  // sample masses above rank j
  const double s0 = w.sc->sums[0], s1 = w.sc->sums[1];
  int first = kGapSample;   // this thread's first rank with phi >= r^2 (no early exit: loads stay independent)
#pragma unroll 8
  for (int j = j0; j < j0 + kEstPer; ++j) {
    const double lam = key_value(w.samp_out[j]);
    const double phi = (s1 + scale * cs) + (s0 + scale * bs) / (lam * lam);
    if (phi >= r2 && first == kGapSample) first = j;
    cs += w.cs[j];
    bs += w.bs[j];
  }
  if (first < kGapSample) atomicMin(&hit, first);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int h = hit;
    w.sc->est_ra = h - margin > 0 ? h - margin : 0;
    w.sc->est_rb = h + margin < kGapSample - 1 ? h + margin : -1;
  }
}

__global__ void window_keys_est_kernel(Work w) {
  pdl_wait_cadence();
  const int ra = w.sc->est_ra, rb = w.sc->est_rb;
  w.sc->hi_key = ra > 0 ? w.samp_out[ra] : ~0ull;
  w.sc->lo_key = rb >= 0 ? w.samp_out[rb] : 0ull;
  w.sc->above_min = ~0ull;
  w.sc->above_count = 0;
}

// Window [lo_key, hi_key] between sample ranks ra (0: no events above) and rb.
__global__ void window_keys_kernel(Work w, int ra, int rb) {
  pdl_wait_cadence();
  w.sc->hi_key = ra > 0 ? w.samp_out[ra] : ~0ull;
  w.sc->lo_key = rb >= 0 ? w.samp_out[rb] : 0ull;  // rb < 0: down to the last event
  w.sc->above_min = ~0ull;
  w.sc->above_count = 0;
}

// Flags the window's events (whole tie groups: the window is a key range)
// and finds the smallest key and the count above it (exact integer work).
__global__ void __launch_bounds__(kT) window_flags_kernel(Work w, int64_t E) {
  pdl_wait_cadence();
  const uint64_t lo = w.sc->lo_key, hi = w.sc->hi_key;
  unsigned long long mn = ~0ull, cnt = 0;
  GRID_STRIDE(i, E) {
    const uint64_t k = w.keys_in[i];
    w.flag[i] = (k >= lo && k <= hi) ? 1 : 0;
    if (k > hi) {
      mn = k < mn ? k : mn;
      ++cnt;
    }
  }
  using BR = cub::BlockReduce<unsigned long long, kT>;
  __shared__ typename BR::TempStorage tmp;
  const unsigned long long bmn = BR(tmp).Reduce(mn, [](unsigned long long a, unsigned long long b) {
    return a < b ? a : b;
  });
  __syncthreads();
  const unsigned long long bcnt = BR(tmp).Sum(cnt);
  if (threadIdx.x == 0 && bcnt > 0) {
    atomicMin(&w.sc->above_min, bmn);
    atomicAdd(&w.sc->above_count, bcnt);
  }
}

__global__ void base_window_kernel(Work w) {
  pdl_wait_cadence();
  // nothing above (a top window): exactly the full sort's start
  const bool none = w.sc->above_count == 0;
  w.sc->base[0] = none ? w.sc->sums[1] : w.sc->sums[1] + w.sc->above[0];
  w.sc->base[1] = none ? w.sc->sums[0] : w.sc->sums[0] + w.sc->above[1];
  w.sc->base[2] = w.sc->above_count > 0 ? key_value(w.sc->above_min) : CUDART_INF;
}

// Parallel sweep: cs/bs hold exclusive prefix masses in sorted order.
__global__ void first_hit_kernel(Work w, int64_t E, const double* r_slot, double r_value) {
  pdl_wait_cadence();
  const double r = r_slot ? *r_slot : r_value;
  const double r2 = r * r;
  const double c0 = w.sc->base[0], b0 = w.sc->base[1];
  unsigned long long best = ~0ull;
  GRID_STRIDE(idx, E) {
    const uint64_t key = w.keys_out[idx];
    if (idx > 0 && w.keys_out[idx - 1] == key) continue;  // not a group head
    const double lam = key_value(key);
    const double c_sum = c0 + w.cs[idx];
    const double b_sum = b0 + w.bs[idx];
    if (c_sum + b_sum / (lam * lam) >= r2) {
      best = static_cast<unsigned long long>(idx);
      break;  // grid-stride order: this thread's later hits are larger
    }
  }
  // min over the CTA, then one atomic (the predicate holds for a suffix of
  // group heads, so per-hit atomics would serialize on one word)
  __shared__ unsigned long long sbest;
  if (threadIdx.x == 0) sbest = ~0ull;
  __syncthreads();
  if (best != ~0ull) atomicMin(&sbest, best);
  __syncthreads();
  if (threadIdx.x == 0 && sbest != ~0ull) atomicMin(&w.sc->first, sbest);
}

__global__ void finalize_perf_kernel(Work w, int64_t E, const double* r_slot, double r_value) {
  pdl_wait_cadence();
  const double r = r_slot ? *r_slot : r_value;
  const double r2 = r * r;
  const double c0 = w.sc->base[0], b0 = w.sc->base[1];
  double ls;
  const unsigned long long f = w.sc->first;
  if (f != ~0ull) {
    const int64_t idx = static_cast<int64_t>(f);
    const double lam = key_value(w.keys_out[idx]);
    const double hi = idx > 0 ? key_value(w.keys_out[idx - 1]) : w.sc->base[2];
    const double c_sum = c0 + w.cs[idx], b_sum = b0 + w.bs[idx];
    if (b_sum > 0.0 && r2 > c_sum) {
      ls = sqrt(b_sum / (r2 - c_sum));
    } else {
      ls = lam;
    }
    ls = clampd(ls, lam, hi);
  } else {
    // hi: the lambda of the last group above the sorted events (inf for a
    // full sort; the bracket's upper neighbour for the distributed gap)
    double c_sum = c0, b_sum = b0, hi = w.sc->base[2];
    if (E > 0) {
      c_sum = c0 + (w.cs[E - 1] + w.dc[w.vals_out[E - 1]]);
      b_sum = b0 + (w.bs[E - 1] + w.di[w.vals_out[E - 1]]);
      hi = key_value(w.keys_out[E - 1]);
    }
    if (b_sum > 0.0 && r2 > c_sum) {
      ls = sqrt(b_sum / (r2 - c_sum));
      ls = ls < hi ? ls : hi;
    } else if (b_sum > 0.0) {
      ls = hi;
    } else {
      ls = finite_d(hi) ? hi / 2.0 : 1.0;
    }
  }
  w.sc->lambda_star = finish_lambda(ls);
}

// Candidate coordinate (assemble_candidate, restarts.hpp:73-101).
__device__ __forceinline__ double cand_x(const GapIn& g, int64_t i, double lambda) {
  const double gg = g.aty[i] - g.cc(i);
  return clampd(g.x[i] + gg / (lambda * g.omega), g.lo(i), g.hi(i));
}

__device__ __forceinline__ double cand_y(const GapIn& g, int64_t j, double lambda) {
  const double nu = lambda / g.omega;
  const double bm = g.ax[j] - g.uc[j];
  const double bp = g.ax[j] - g.lc[j];
  const double t = nu * g.y[j];
  double v;
  if (t >= bp) {
    v = g.y[j] - bp / nu;
  } else if (t <= bm) {
    v = g.y[j] - bm / nu;
  } else {
    v = 0.0;
  }
  return cone_project(v, cone_of_bounds(g.lc[j], g.uc[j]));
}

// Coordinate t's term of gap_value_at (restarts.hpp:50-71): primal
// coordinates first, then the dual ones.
__device__ __forceinline__ double value_term(const GapIn& g, int64_t t, double lambda) {
  if (t < g.n) {
    const double xh = cand_x(g, t, lambda);
    return g.cc(t) * (g.x[t] - xh) + g.aty[t] * xh;
  }
  const int64_t j = t - g.n;
  const double yh = cand_y(g, j, lambda);
  const double yj = g.y[j];
  double d = -(yh * g.ax[j]);
  if (yh > 0.0) {
    d -= mul_zero_inf(-g.lc[j], yh);
  } else if (yh < 0.0) {
    d -= mul_zero_inf(-g.uc[j], yh);
  }
  if (yj > 0.0) {
    d += mul_zero_inf(-g.lc[j], yj);
  } else if (yj < 0.0) {
    d += mul_zero_inf(-g.uc[j], yj);
  }
  return d;
}

// gap_value_at (restarts.hpp:50-71) in the reference's exact order.
__global__ void value_seq_kernel(GapIn g, Work w, const double* r_slot, double r_value,
                                 double* out) {
  pdl_wait_cadence();
  const double r = r_slot ? *r_slot : r_value;
  if (!(r > 0.0)) {
    *out = 0.0;
    return;
  }
  const double lambda = w.sc->lambda_star;
  double value = 0.0;
  for (int64_t i = 0; i < g.n; ++i) {
    const double xh = cand_x(g, i, lambda);
    value += g.cc(i) * (g.x[i] - xh) + g.aty[i] * xh;
  }
  for (int64_t j = 0; j < g.m; ++j) {
    const double yh = cand_y(g, j, lambda);
    const double yj = g.y[j];
    value -= yh * g.ax[j];
    if (yh > 0.0) {
      value -= mul_zero_inf(-g.lc[j], yh);
    } else if (yh < 0.0) {
      value -= mul_zero_inf(-g.uc[j], yh);
    }
    if (yj > 0.0) {
      value += mul_zero_inf(-g.lc[j], yj);
    } else if (yj < 0.0) {
      value += mul_zero_inf(-g.uc[j], yj);
    }
  }
  *out = (value > 0.0) ? value / r : 0.0;
}

__global__ void value_finish_kernel(const double* sum, const double* r_slot, double r_value,
                                    double* out) {
  pdl_wait_cadence();
  const double r = r_slot ? *r_slot : r_value;
  const double value = *sum;
  *out = (r > 0.0 && value > 0.0) ? value / r : 0.0;
}

GapIn make_in(const pdlpk_problem* P, const double* x, const double* y, const double* ax,
              const double* aty, double omega) {
  return GapIn{P->c, P->lv, P->uv, P->lc, P->uc, x, y, ax, aty, P->n, P->m, omega,
               P->uniform, P->c_u, P->lv_u, P->uv_u};
}

}  // namespace
}  // namespace pdlp

using namespace pdlp;

extern "C" size_t pdlpk_gap_work_bytes(int64_t n, int64_t m) {
  const int64_t N = n + 2 * m;
  return align_up(N) + align_up(8 * N) * 3 + align_up(4 * N) + align_up(8 * N) * 2 +
         align_up(4 * N) + align_up(8 * N) * 2 + align_up(4 * N) + 2 * align_up(8 * kGapSample) +
         2 * align_up(4 * kGapSample) + 2 * align_up(8 * kGapSample) +
         align_up(sizeof(GapScalars)) + align_up(cub_bytes_for(N)) + 256;
}

extern "C" int pdlpk_gap_prepare(const pdlpk_problem* P, const double* x, const double* y,
                                 const double* ax, const double* aty, double omega,
                                 const pdlpk_red* red, void* work, int* count_out,
                                 cudaStream_t s) {
  const int64_t n = P->n, m = P->m, N = n + 2 * m;
  Work w = carve(work, n, m);
  const GapIn g = make_in(P, x, y, ax, aty, omega);
  int rc;
  if (red->parity) {
    // the lambda -> inf masses in the reference's order (one thread), then
    // the events in parallel
    auto fm = [g] __device__(int64_t t, double* v) -> unsigned {
      const Coord o = gap_coord(g, t);
      v[0] = o.b;
      v[1] = o.c;
      return o.mass_use;
    };
    rc = multi_reduce<2>(fm, n + m, PDLPK_RED_SEQ, red->shards, 0u, red->scratch, w.sc->sums, s);
    if (rc == 0 && N > 0) launch_pdl(PDLPK_PDL_CADENCE, events_kernel, static_cast<unsigned>(ew_blocks(n + m)), kT, 0, s, g, w);
  } else {
    // one pass: the tree reduction visits every coordinate once and writes
    // its events on the way
    auto fe = [g, w] __device__(int64_t t, double* v) -> unsigned {
      const Coord o = gap_coord(g, t);
      write_events(g, w, t, o);
      v[0] = o.b;
      v[1] = o.c;
      return o.mass_use;
    };
    rc = multi_reduce<2>(fe, n + m, PDLPK_RED_TREE, red->shards, 0u, red->scratch, w.sc->sums, s);
  }
  if (rc != 0) return rc;
  if (N > 0) {
    size_t bytes = w.cub_bytes;
    const cudaError_t e = cub::DeviceSelect::Flagged(w.cub_tmp, bytes, thrust::counting_iterator<int32_t>(0),
                                                     w.flag, w.sel, &w.sc->num_events,
                                                     static_cast<int>(N), s);
    if (e != cudaSuccess) return static_cast<int>(e);
  } else {
    cudaMemsetAsync(&w.sc->num_events, 0, sizeof(int), s);
  }
  if (count_out != nullptr) {
    cudaMemcpyAsync(count_out, &w.sc->num_events, sizeof(int), cudaMemcpyDeviceToDevice, s);
  }
  return static_cast<int>(cudaGetLastError());
}

thread_local int64_t g_window_stats[2] = {0, 0};  // windows tried, decided

// Perf mode, large E: sort only the events whose keys lie in a window
// [lo_key, hi_key] placed (from a strided key sample) at depth fractions
// [qa, qb] of the descending order.  Events above the window enter the sweep
// as summed masses (a deterministic tree reduction) and the lambda of their
// last group; the window is a key range, so tie groups are never split.  The
// sweep's predicate holds on a suffix of group heads, so a hit at a window
// head other than the first (or at the first one when nothing lies above)
// is the full sweep's first crossing; no hit in a window that reaches the
// last event (qb >= 1) means no crossing at all.  A hit at the first head
// with events above, or no hit above the bottom, returns 0 and the full sort
// runs.  Returns the window's event count when it decided.  Two host syncs
// (the window count, the hit).
// qa == -2: the estimated window (first evaluation, see estimate_window_kernel).
static int64_t gap_window(const Work& w, int64_t E, double qa, double qb, const pdlpk_red* red,
                          const double* r_slot, double r_value, cudaStream_t s) {
  const bool est = qa == -2.0;
  if (est && r_slot != nullptr) return 0;  // the estimate needs the radius on the host
  launch_pdl(PDLPK_PDL_CADENCE, keys_kernel, static_cast<unsigned>(ew_blocks(E)), kT, 0, s, w, E);
  size_t bytes = w.cub_bytes;
  int ra = 0, rb = -1;
  bool to_bottom = true;
  if (est) {
    launch_pdl(PDLPK_PDL_CADENCE, sample_masses_kernel, static_cast<unsigned>(ew_blocks(kGapSample)), kT, 0, s, w, E);
    if (cub::DeviceRadixSort::SortPairsDescending(w.cub_tmp, bytes, w.samp_in, w.samp_out, w.sidx_in,
                                                  w.sidx_out, kGapSample, 0, 64, s) != cudaSuccess) {
      return -1;
    }
    const int margin = static_cast<int>(0.05 * kGapSample);
    launch_pdl(PDLPK_PDL_CADENCE, sorted_masses_kernel, static_cast<unsigned>(ew_blocks(kGapSample)), kT, 0, s, w);
    estimate_window_kernel<<<1, kEstThreads, 0, s>>>(w, E, r_value, margin);
    // A deep estimate (or none) comes from a sample that missed a few heavy
    // breakpoints (C2: estimated depth >= 0.88 for crossings at 0.11-0.63):
    // go straight to the full sort instead of a window that would miss.
    int est_h[2] = {0, 0};
    cudaMemcpyAsync(est_h, &w.sc->est_ra, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
    if (est_h[1] < 0 || est_h[0] > (3 * kGapSample) / 4) return 0;
    launch_pdl(PDLPK_PDL_CADENCE, window_keys_est_kernel, static_cast<unsigned>(1), 1, 0, s, w);
    ra = est_h[0];
  } else {
    launch_pdl(PDLPK_PDL_CADENCE, sample_keys_kernel, static_cast<unsigned>(ew_blocks(kGapSample)), kT, 0, s, w, E);
    if (cub::DeviceRadixSort::SortKeysDescending(w.cub_tmp, bytes, w.samp_in, w.samp_out, kGapSample,
                                                 0, 64, s) != cudaSuccess) {
      return -1;
    }
    ra = qa <= 0.0 ? 0 : std::min(kGapSample - 1, static_cast<int>(qa * kGapSample));
    to_bottom = qb >= 1.0;
    rb = to_bottom ? -1 : std::min(kGapSample - 1, static_cast<int>(qb * kGapSample));
    launch_pdl(PDLPK_PDL_CADENCE, window_keys_kernel, static_cast<unsigned>(1), 1, 0, s, w, ra, rb);
  }
  launch_pdl(PDLPK_PDL_CADENCE, window_flags_kernel, static_cast<unsigned>(ew_blocks(E)), kT, 0, s, w, E);
  if (ra > 0) {
    const Work wc = w;
    auto fa = [wc] __device__(int64_t e, double* v) -> unsigned {
      if (wc.keys_in[e] <= wc.sc->hi_key) return 0u;
      const int32_t t = wc.sel[e];
      v[0] = wc.dc[t];
      v[1] = wc.di[t];
      return 3u;
    };
    if (multi_reduce<2>(fa, E, PDLPK_RED_TREE, red->shards, 0u, red->scratch, w.sc->above, s) != 0) {
      return -1;
    }
  } else {
    cudaMemsetAsync(w.sc->above, 0, sizeof(w.sc->above), s);
  }
  launch_pdl(PDLPK_PDL_CADENCE, base_window_kernel, static_cast<unsigned>(1), 1, 0, s, w);
  uint64_t* keys_h = reinterpret_cast<uint64_t*>(w.cs);
  bytes = w.cub_bytes;
  if (cub::DeviceSelect::Flagged(w.cub_tmp, bytes, w.keys_in, w.flag, keys_h, &w.sc->num_high,
                                 static_cast<int>(E), s) != cudaSuccess) {
    return -1;
  }
  bytes = w.cub_bytes;
  if (cub::DeviceSelect::Flagged(w.cub_tmp, bytes, w.sel, w.flag, w.hsel, &w.sc->num_high,
                                 static_cast<int>(E), s) != cudaSuccess) {
    return -1;
  }
  int eh = 0, est_rb = -1;
  cudaMemcpyAsync(&eh, &w.sc->num_high, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (est) cudaMemcpyAsync(&est_rb, &w.sc->est_rb, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
  if (est) to_bottom = est_rb < 0;
  if (eh <= 0 || eh >= E) return 0;
  bytes = w.cub_bytes;
  if (cub::DeviceRadixSort::SortPairsDescending(w.cub_tmp, bytes, keys_h, w.keys_out, w.hsel,
                                                w.vals_out, eh, 0, 64, s) != cudaSuccess) {
    return -1;
  }
  launch_pdl(PDLPK_PDL_CADENCE, gather_masses_kernel, static_cast<unsigned>(ew_blocks(eh)), kT, 0, s, w, eh);
  bytes = w.cub_bytes;
  cub::DeviceScan::ExclusiveSum(w.cub_tmp, bytes, w.cs, w.cs, eh, s);
  bytes = w.cub_bytes;
  cub::DeviceScan::ExclusiveSum(w.cub_tmp, bytes, w.bs, w.bs, eh, s);
  launch_pdl(PDLPK_PDL_CADENCE, init_first_kernel, static_cast<unsigned>(1), 1, 0, s, w);
  launch_pdl(PDLPK_PDL_CADENCE, first_hit_kernel, static_cast<unsigned>(ew_blocks(eh)), kT, 0, s, w, eh, r_slot, r_value);
  struct {
    unsigned long long first, above;
  } h{};
  cudaMemcpyAsync(&h.first, &w.sc->first, sizeof(h.first), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&h.above, &w.sc->above_count, sizeof(h.above), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
  static const bool dbg = std::getenv("PDLP_GAP_DEBUG") != nullptr;
  if (dbg && est) {
    int ra_h = 0;
    cudaMemcpy(&ra_h, &w.sc->est_ra, sizeof(int), cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "gap window est: ranks [%d, %d] of %d, window events %d, first %lld, above %llu\n",
                 ra_h, est_rb, kGapSample, eh, static_cast<long long>(h.first), h.above);
  }
  if (h.first == ~0ull) return to_bottom ? eh : 0;
  if (h.first == 0 && h.above > 0) return 0;
  return eh;
}

extern "C" void pdlpk_gap_window_stats(int64_t* tried, int64_t* decided) {
  *tried = g_window_stats[0];
  *decided = g_window_stats[1];
}

extern "C" int pdlpk_gap_finish(const pdlpk_problem* P, const double* x, const double* y,
                                const double* ax, const double* aty, double omega,
                                const double* r_slot, double r_value, int64_t E,
                                const pdlpk_red* red, void* work, double* gap_slot, double qa,
                                double qb, cudaStream_t s) {
  const int64_t n = P->n, m = P->m;
  Work w = carve(work, n, m);
  const GapIn g = make_in(P, x, y, ax, aty, omega);
  const bool parity = red->parity != 0;
  bool decided = false;
  int64_t E_fin = E;  // events the finalize reads (the window's when it decided)
  if (!parity && ((qa >= 0.0 && qb > qa && qb - qa < 0.5) || qa == -2.0) &&
      E > (int64_t(1) << 20)) {
    const int64_t pr = gap_window(w, E, qa, qb, red, r_slot, r_value, s);
    if (pr < 0) return static_cast<int>(cudaGetLastError());
    decided = pr > 0;
    if (decided) E_fin = pr;
    ++g_window_stats[0];
    if (decided) ++g_window_stats[1];
  }
  if (!decided) launch_pdl(PDLPK_PDL_CADENCE, base_full_kernel, static_cast<unsigned>(1), 1, 0, s, w);
  if (E > 0 && !decided) {
    launch_pdl(PDLPK_PDL_CADENCE, keys_kernel, static_cast<unsigned>(ew_blocks(E)), kT, 0, s, w, E);
    size_t bytes = w.cub_bytes;
    const cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(
        w.cub_tmp, bytes, w.keys_in, w.keys_out, w.sel, w.vals_out, static_cast<int>(E), 0, 64, s);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  if (parity) {
    launch_pdl(PDLPK_PDL_CADENCE, sweep_seq_kernel, static_cast<unsigned>(1), 1, 0, s, w, E, r_slot, r_value);
    launch_pdl(PDLPK_PDL_CADENCE, value_seq_kernel, static_cast<unsigned>(1), 1, 0, s, g, w, r_slot, r_value, gap_slot);
    return static_cast<int>(cudaGetLastError());
  }
  if (!decided) {
    if (E > 0) {
      launch_pdl(PDLPK_PDL_CADENCE, gather_masses_kernel, static_cast<unsigned>(ew_blocks(E)), kT, 0, s, w, E);
      size_t bytes = w.cub_bytes;
      cub::DeviceScan::ExclusiveSum(w.cub_tmp, bytes, w.cs, w.cs, static_cast<int>(E), s);
      bytes = w.cub_bytes;
      cub::DeviceScan::ExclusiveSum(w.cub_tmp, bytes, w.bs, w.bs, static_cast<int>(E), s);
    }
    launch_pdl(PDLPK_PDL_CADENCE, init_first_kernel, static_cast<unsigned>(1), 1, 0, s, w);
    if (E > 0) launch_pdl(PDLPK_PDL_CADENCE, first_hit_kernel, static_cast<unsigned>(ew_blocks(E)), kT, 0, s, w, E, r_slot, r_value);
  }
  // (a decided window: its crossing index, or the no-crossing branch over
  // the window's events with the masses above in base)
  launch_pdl(PDLPK_PDL_CADENCE, finalize_perf_kernel, static_cast<unsigned>(1), 1, 0, s, w, E_fin, r_slot, r_value);
  launch_pdl(PDLPK_PDL_CADENCE, hit_fraction_kernel, static_cast<unsigned>(1), 1, 0, s, w, E, gap_slot + 2);
  const double* lam_star = &w.sc->lambda_star;
  auto fv = [g, lam_star] __device__(int64_t t, double* v) -> unsigned {
    v[0] = value_term(g, t, *lam_star);
    return 1u;
  };
  const int rc = multi_reduce<1>(fv, n + m, PDLPK_RED_TREE, red->shards, 0u, red->scratch,
                                 &w.sc->value, s);
  if (rc != 0) return rc;
  launch_pdl(PDLPK_PDL_CADENCE, value_finish_kernel, static_cast<unsigned>(1), 1, 0, s, &w.sc->value, r_slot, r_value, gap_slot);
  return static_cast<int>(cudaGetLastError());
}

// ------------------------------------------- distributed gap ---
// Row-sharded solves: each rank holds only its own column block (x, A'y, c,
// bounds) and row block (y, A x, row bounds), so it builds the breakpoint
// events of those coordinates (pdlpk_gap_prepare on the local views).  The
// first crossing of the global descending order is located by a bracket
// search that the host drives (solver.cpp Engine::gap_dist): at a sampled
// key s every rank reduces, over its events inside the bracket, the masses
// strictly above s and at-or-above s (TREE order) and the count below s;
// the ranks' values are combined in rank order, phi(s) = C + B / lam(s)^2
// says which side of s the crossing lies on, and each rank compacts its
// bracket.  When the bracket is small its events are all-gathered, stably
// sorted (rank order breaks key ties identically on every rank) and swept
// with the single-GPU kernels, starting from the masses above the bracket.
// No rank ever holds another rank's vectors.

namespace pdlp {
namespace {

__global__ void gapd_stage_kernel(Work w, double* dst) {
  dst[0] = w.sc->sums[0];
  dst[1] = w.sc->sums[1];
  dst[2] = static_cast<double>(w.sc->num_events);
}

__global__ void gapd_sample_kernel(const uint64_t* keys, int64_t A, int S, double* out) {
  GRID_STRIDE(i, S) {
    const int64_t k = A >= S ? (i * A) / S : i;
    out[i] = __longlong_as_double(i < A ? static_cast<long long>(keys[k]) : 0ll);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[S] = static_cast<double>(A < S ? A : S);
}

__global__ void gapd_flag_kernel(Work w, const uint64_t* keys, int64_t A, uint64_t lo, uint64_t hi) {
  GRID_STRIDE(e, A) {
    const uint64_t k = keys[e];
    w.flag[e] = (k >= lo && k <= hi) ? 1 : 0;
  }
}

__global__ void gapd_pack_kernel(Work w, const uint64_t* keys, const int32_t* slots, int64_t A,
                                 int64_t K, double* dst) {
  GRID_STRIDE(e, K) {
    const bool v = e < A;
    dst[e] = __longlong_as_double(v ? static_cast<long long>(keys[e]) : 0ll);
    dst[K + e] = v ? w.dc[slots[e]] : 0.0;
    dst[2 * K + e] = v ? w.di[slots[e]] : 0.0;
  }
}

struct GapdOffsets {
  int world;
  int64_t K;
  int64_t off[PDLPK_GAPD_MAX_RANKS + 1];
};

// rank-ordered concatenation of the gathered brackets into slots 0..T-1
__global__ void gapd_unpack_kernel(Work f, const double* all, GapdOffsets o) {
  const int64_t T = o.off[o.world];
  GRID_STRIDE(t, T) {
    int r = 0;
    while (t >= o.off[r + 1]) ++r;
    const int64_t e = t - o.off[r];
    const double* blk = all + static_cast<int64_t>(r) * 3 * o.K;
    f.keys_in[t] = static_cast<uint64_t>(__double_as_longlong(blk[e]));
    f.dc[t] = blk[o.K + e];
    f.di[t] = blk[2 * o.K + e];
    f.sel[t] = static_cast<int32_t>(t);
  }
}

__global__ void gapd_base_kernel(Work f, double c0, double b0, double hi0) {
  f.sc->base[0] = c0;
  f.sc->base[1] = b0;
  f.sc->base[2] = hi0;
  f.sc->above_count = 0;
}

// The bracket's lowest group is known to cross (phi >= r^2 at its head, from
// the search's reductions): if the sweep's own sums (scan order) put it just
// below r^2, that group is the crossing.
__global__ void gapd_force_last_kernel(Work f, int64_t T) {
  if (f.sc->first != ~0ull || T <= 0) return;
  int64_t h = T - 1;
  const uint64_t k = f.keys_out[h];
  while (h > 0 && f.keys_out[h - 1] == k) --h;
  f.sc->first = static_cast<unsigned long long>(h);
}

}  // namespace
}  // namespace pdlp

extern "C" int pdlpk_gapd_lists(void* work, int64_t n, int64_t m, uint64_t** keys0, int32_t** slots0,
                                uint64_t** keys1, int32_t** slots1) {
  Work w = carve(work, n, m);
  *keys0 = w.keys_in;
  *slots0 = w.sel;
  *keys1 = w.keys_out;
  *slots1 = w.vals_out;
  return 0;
}

extern "C" int pdlpk_gapd_stage(void* work, int64_t n, int64_t m, double* dst, cudaStream_t s) {
  Work w = carve(work, n, m);
  gapd_stage_kernel<<<1, 1, 0, s>>>(w, dst);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_gapd_keys(void* work, int64_t n, int64_t m, int64_t E, cudaStream_t s) {
  Work w = carve(work, n, m);
  if (E > 0) keys_kernel<<<ew_blocks(E), kT, 0, s>>>(w, E);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_gapd_sample(const uint64_t* keys, int64_t A, int S, double* out, cudaStream_t s) {
  gapd_sample_kernel<<<ew_blocks(S), kT, 0, s>>>(keys, A, S, out);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_gapd_split(void* work, int64_t n, int64_t m, const uint64_t* keys,
                                const int32_t* slots, int64_t A, uint64_t s_key,
                                const pdlpk_red* red, double* out, cudaStream_t s) {
  const Work w = carve(work, n, m);
  auto f = [w, keys, slots, s_key] __device__(int64_t e, double* v) -> unsigned {
    const uint64_t k = keys[e];
    if (k < s_key) {
      v[4] = 1.0;
      return 16u;
    }
    const int32_t t = slots[e];
    const double dc = w.dc[t], di = w.di[t];
    v[2] = dc;
    v[3] = di;
    if (k == s_key) return 12u;
    v[0] = dc;
    v[1] = di;
    return 15u;
  };
  return multi_reduce<5>(f, A, PDLPK_RED_TREE, red->shards, 0u, red->scratch, out, s);
}

extern "C" int pdlpk_gapd_compact(void* work, int64_t n, int64_t m, const uint64_t* keys_in,
                                  const int32_t* slots_in, int64_t A, uint64_t lo, uint64_t hi,
                                  uint64_t* keys_out, int32_t* slots_out, cudaStream_t s) {
  Work w = carve(work, n, m);
  if (A <= 0) return 0;
  gapd_flag_kernel<<<ew_blocks(A), kT, 0, s>>>(w, keys_in, A, lo, hi);
  size_t bytes = w.cub_bytes;
  cudaError_t e = cub::DeviceSelect::Flagged(w.cub_tmp, bytes, keys_in, w.flag, keys_out,
                                             &w.sc->num_high, static_cast<int>(A), s);
  if (e != cudaSuccess) return static_cast<int>(e);
  bytes = w.cub_bytes;
  e = cub::DeviceSelect::Flagged(w.cub_tmp, bytes, slots_in, w.flag, slots_out, &w.sc->num_high,
                                 static_cast<int>(A), s);
  if (e != cudaSuccess) return static_cast<int>(e);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_gapd_pack(void* work, int64_t n, int64_t m, const uint64_t* keys,
                               const int32_t* slots, int64_t A, int64_t K, double* dst,
                               cudaStream_t s) {
  Work w = carve(work, n, m);
  if (K > 0) gapd_pack_kernel<<<ew_blocks(K), kT, 0, s>>>(w, keys, slots, A, K, dst);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_gap_lambda_star(void* work, int64_t n, int64_t m, double* dst, cudaStream_t s) {
  Work w = carve(work, n, m);
  return static_cast<int>(cudaMemcpyAsync(dst, &w.sc->lambda_star, sizeof(double),
                                          cudaMemcpyDeviceToDevice, s));
}

extern "C" size_t pdlpk_gapd_final_bytes(int64_t T) { return pdlpk_gap_work_bytes(T, 0); }

extern "C" int pdlpk_gapd_final(void* fwork, int64_t cap, const double* all, int world, int64_t K,
                                const int64_t* counts, double c0, double b0, double hi0,
                                int lower_bounded, double r, double** lambda_star, cudaStream_t s) {
  if (world < 1 || world > PDLPK_GAPD_MAX_RANKS) return static_cast<int>(cudaErrorInvalidValue);
  Work f = carve(fwork, cap, 0);
  GapdOffsets o{};
  o.world = world;
  o.K = K;
  o.off[0] = 0;
  for (int q = 0; q < world; ++q) o.off[q + 1] = o.off[q] + counts[q];
  const int64_t T = o.off[world];
  if (T > cap) return static_cast<int>(cudaErrorInvalidValue);
  gapd_base_kernel<<<1, 1, 0, s>>>(f, c0, b0, hi0);
  init_first_kernel<<<1, 1, 0, s>>>(f);
  if (T > 0) {
    gapd_unpack_kernel<<<ew_blocks(T), kT, 0, s>>>(f, all, o);
    size_t bytes = f.cub_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(f.cub_tmp, bytes, f.keys_in, f.keys_out,
                                                              f.sel, f.vals_out, static_cast<int>(T),
                                                              0, 64, s);
    if (e != cudaSuccess) return static_cast<int>(e);
    gather_masses_kernel<<<ew_blocks(T), kT, 0, s>>>(f, T);
    bytes = f.cub_bytes;
    cub::DeviceScan::ExclusiveSum(f.cub_tmp, bytes, f.cs, f.cs, static_cast<int>(T), s);
    bytes = f.cub_bytes;
    cub::DeviceScan::ExclusiveSum(f.cub_tmp, bytes, f.bs, f.bs, static_cast<int>(T), s);
    first_hit_kernel<<<ew_blocks(T), kT, 0, s>>>(f, T, nullptr, r);
    if (lower_bounded) gapd_force_last_kernel<<<1, 1, 0, s>>>(f, T);
  }
  finalize_perf_kernel<<<1, 1, 0, s>>>(f, T, nullptr, r);
  *lambda_star = &f.sc->lambda_star;
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_gapd_value(const pdlpk_problem* P, const double* x, const double* y,
                                const double* ax, const double* aty, double omega,
                                const double* lambda_star, const pdlpk_red* red, double* out,
                                cudaStream_t s) {
  const GapIn g = make_in(P, x, y, ax, aty, omega);
  auto fv = [g, lambda_star] __device__(int64_t t, double* v) -> unsigned {
    v[0] = value_term(g, t, *lambda_star);
    return 1u;
  };
  return multi_reduce<1>(fv, P->n + P->m, PDLPK_RED_TREE, red->shards, 0u, red->scratch, out, s);
}
