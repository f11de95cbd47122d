// The PDHG step attempt on device: pdhg_step_into + the adaptive step-size
// decision of the reference (proj/include/pdhglp/step.hpp:60-95, 126-193),
// with the deferred running-average update (step.hpp:209-216).
//
// PERF mode, three launches per attempt:
//   primal_pass   x' = clamp(x - tau (c - aty)), xbar = 2x' - x      (n, elementwise)
//                 [+ pending  sum_x += w x  of the previously accepted step]
//   row_pass      a_ext = K xbar (load-balanced CSR), fused dual update
//                 y' = yhat - sigma clamp(yhat/sigma, -u_c, -l_c), dy = y' - y,
//                 per-CTA partials of |dy|^2 and |y'|_inf
//                 [+ pending  sum_y += w y]
//   col_pass      aty' = aty + K^T dy (load-balanced CSR of K^T), per-CTA
//                 partials of |dx|^2, dy^T K dx and |x'|_inf; the last CTA
//                 combines all partials in a fixed order and runs the
//                 accept/reject rule, flipping the ping-pong buffers on
//                 acceptance.  No host round trip per attempt.
// PARITY mode reproduces the reference's arithmetic order bit for bit:
// thread-per-line sequential products, per-shard sequential reductions over
// make_shard_plan(dim, 1, S) and an ascending combine (kernels.hpp:69-97).
//
// Translation unit compiled with -fmad=false (see common.cuh).

#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "kernels.h"
#include "spmv.cuh"

namespace pdlp {
namespace {

constexpr int kEwThreads = 256;
#ifndef PDLPK_COL_SPLIT
#define PDLPK_COL_SPLIT 1 /* segmented-span column pass as product + elementwise epilogue */
#endif

inline int ew_blocks(int64_t n) {
  int64_t b = (n + kEwThreads - 1) / kEwThreads;
  if (b > 148 * 8) b = 148 * 8;
  return b < 1 ? 1 : static_cast<int>(b);
}

// ------------------------------------------------------------ primal pass ---
// Push = the all-gather of x-bar folded in (row-sharded solve): each x-bar
// pair is also stored into every peer's gathered vector over NVLink, so the
// transfer overlaps this HBM-bound pass; dst.p[rank] is null (local block
// is a.xbar itself).
template <bool Push>
__global__ void __launch_bounds__(kEwThreads) primal_pass(pdlpk_step_args a, pdlpk_peer_sum dst) {
  pdl_wait();
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const double eta = st->eta;
  if (!st->fixed && (!(eta > 0.0) || !finite_d(eta))) {  // step.hpp:166
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->status = 1;
      st->halt = 1;
    }
    return;
  }
  const double tau = eta / st->omega;
  const int cur = st->cur;
  const double* __restrict__ x = a.x[cur];
  const double* __restrict__ aty = a.aty[cur];
  double* __restrict__ xn = a.x[cur ^ 1];
  const double* __restrict__ c = a.P.c;
  const double* __restrict__ lv = a.P.lv;
  const double* __restrict__ uv = a.P.uv;
  double* __restrict__ xbar = a.xbar;
  const bool pend = st->avg_pending != 0;
  const double w = st->avg_w;
  double* __restrict__ sx = a.sum_x;
  const int64_t n = a.P.n;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // 128-bit accesses (every vector is a separate cudaMalloc, so 16B aligned);
  // c, l_v, u_v are read once per pass: streaming loads.
  const int64_t n2 = n >> 1;
#if PDLPK_XBAR_KEEP
  // keep x-bar (<= kXbarKeepBytes of it) in L2 for the row pass's gathers;
  // x' and the running sum are streamed out
  const float keep = fminf(1.0f, static_cast<float>(PDLPK_XBAR_KEEP_MB * 1048576.0 /
                                                    (8.0 * static_cast<double>(n > 0 ? n : 1))));
  const uint64_t pol = l2_keep_policy(keep);
#endif
  const double2* __restrict__ x2 = reinterpret_cast<const double2*>(x);
  const double2* __restrict__ a2 = reinterpret_cast<const double2*>(aty);
  const double2* __restrict__ c2 = reinterpret_cast<const double2*>(c);
  const double2* __restrict__ l2 = reinterpret_cast<const double2*>(lv);
  const double2* __restrict__ u2 = reinterpret_cast<const double2*>(uv);
  double2* __restrict__ xn2 = reinterpret_cast<double2*>(xn);
  double2* __restrict__ xb2 = reinterpret_cast<double2*>(xbar);
  double2* __restrict__ sx2 = reinterpret_cast<double2*>(sx);
  // bitwise-uniform vectors come from their scalar (no stream)
  const uint32_t uni = a.P.uniform;
  const double2 cu = make_double2(a.P.c_u, a.P.c_u), lu = make_double2(a.P.lv_u, a.P.lv_u),
                uu = make_double2(a.P.uv_u, a.P.uv_u);
  for (int64_t p = tid; p < n2; p += stride) {
    const double2 xi = x2[p], ai = a2[p];
    const double2 ci = (uni & 1u) ? cu : __ldcs(c2 + p);
    const double2 li = (uni & 2u) ? lu : __ldcs(l2 + p);
    const double2 ui = (uni & 4u) ? uu : __ldcs(u2 + p);
    double2 xp, xb;
    xp.x = clampd(xi.x - tau * (ci.x - ai.x), li.x, ui.x);
    xp.y = clampd(xi.y - tau * (ci.y - ai.y), li.y, ui.y);
    xb.x = 2.0 * xp.x - xi.x;
    xb.y = 2.0 * xp.y - xi.y;
#if PDLPK_XBAR_KEEP
#if PDLPK_XN_STREAM
    __stcs(xn2 + p, xp);
#else
    xn2[p] = xp;
#endif
    st_keep(xb2 + p, xb, pol);
#else
    xn2[p] = xp;
    xb2[p] = xb;
#endif
    if constexpr (Push) {
#pragma unroll
      for (int r = 0; r < PDLPK_MAX_PEERS; ++r) {
        if (r < dst.world && dst.p[r] != nullptr) {
          reinterpret_cast<double2*>(const_cast<double*>(dst.p[r]) + dst.offset)[p] = xb;
        }
      }
    }
    if (pend) {
      const double2 s = sx2[p];
      sx2[p] = make_double2(s.x + w * xi.x, s.y + w * xi.y);
    }
  }
  if ((n & 1) && tid == 0) {
    const int64_t i = n - 1;
    const double xi = x[i];
    const double ci = (uni & 1u) ? cu.x : c[i], li = (uni & 2u) ? lu.x : lv[i],
                 ui = (uni & 4u) ? uu.x : uv[i];
    const double xp = clampd(xi - tau * (ci - aty[i]), li, ui);
    xn[i] = xp;
    xbar[i] = 2.0 * xp - xi;
    if constexpr (Push) {
      for (int r = 0; r < dst.world; ++r) {
        if (dst.p[r] != nullptr) const_cast<double*>(dst.p[r])[dst.offset + i] = 2.0 * xp - xi;
      }
    }
    if (pend) sx[i] = sx[i] + w * xi;
  }
  pdl_trigger();
}

// ---------------------------------------------------------- decision rule ---
__device__ void decide(pdlpk_step_state* s, double dx2, double dy2, double curv, double infx,
                       double infy, const double* f_down, const double* f_up,
                       int64_t table_len) {
  s->attempts += 1;
  s->avg_pending = 0;
  s->dx2 = dx2;
  s->dy2 = dy2;
  s->curv = curv;
  s->inf_x = infx;
  s->inf_y = infy;
  const double eta = s->eta;
  if (s->fixed) {  // solver.hpp:477-491
    if (!finite_d(infx) || !finite_d(infy)) {
      s->status = 1;
      s->halt = 1;
      return;
    }
    s->cur ^= 1;
    s->k += 1;
    s->accepted += 1;
    s->eta_used = eta;
    s->avg_pending = 1;
    s->avg_w = eta;
    s->avg_weight += eta;
    s->avg_count += 1;
    if (s->k >= s->k_target) s->halt = 1;
    return;
  }
  const double omega = s->omega;
  const double movement = omega * dx2 + dy2 / omega;
  if (!finite_d(movement) || !finite_d(curv)) {  // step.hpp:175
    s->status = 1;
    s->halt = 1;
    return;
  }
  // step_size_limit (step.hpp:126-130)
  const double denom = 2.0 * fabs(curv);
  const double eta_bar = (denom > 0.0) ? movement / denom : CUDART_INF;
  s->eta_bar = eta_bar;
  if (finite_d(eta_bar)) s->min_eta_bar = (eta_bar < s->min_eta_bar) ? eta_bar : s->min_eta_bar;
  // next_step_size (step.hpp:136-141); factors from the host-libm table.
  const int64_t k = s->k;
  if (k >= table_len) {
    s->table_short = 1;
    s->status = 1;
    s->halt = 1;
    return;
  }
  const double down = f_down[k] * eta_bar;
  const double up = f_up[k] * eta;
  const double eta_next = (up < down) ? up : down;
  if (eta <= eta_bar) {
    s->cur ^= 1;
    s->eta = eta_next;
    s->k = k + 1;
    s->accepted += 1;
    s->eta_used = eta;
    s->attempt_in_step = 0;
    s->avg_pending = 1;
    s->avg_w = eta;
    s->avg_weight += eta;
    s->avg_count += 1;
    if (s->k >= s->k_target) s->halt = 1;
    return;
  }
  s->retries += 1;
  s->eta = eta_next;
  s->attempt_in_step += 1;
  if (s->attempt_in_step > s->max_retries) {  // step.hpp:165,192
    s->status = 1;
    s->halt = 1;
  }
}

// --------------------------------------------------------- perf row pass ---
// Carry = true: the last launch of a column-panel row pass -- the line sum
// starts from the partial sum the earlier panels carried (staged as a 4th
// operand).
template <bool Carry>
struct RowEpiT {
  const double* __restrict__ y;
  double* __restrict__ yn;
  double* __restrict__ dy;
  const double* __restrict__ lc;
  const double* __restrict__ uc;
  double* __restrict__ sy;
  double sigma, w;
  bool pend;
  uint64_t keep = 0;  // L2 evict_last policy for dy (gathered by the column pass)
  double* lp = nullptr;  // line_partials: per-line terms (part2[r], part2[m + r])
  int64_t lm = 0;
  double dy2 = 0.0, infy = 0.0;
  const double* __restrict__ carry = nullptr;
  struct Pre {
    double y, lc, uc, c;
  };
  __device__ __forceinline__ Pre load(int64_t r) const {
    return {y[r], lc[r], uc[r], Carry ? carry[r] : 0.0};
  }
  __device__ __forceinline__ double init(const Pre& p) const { return Carry ? p.c : 0.0; }
  __device__ __forceinline__ void prefetch(int64_t r) const {
    prefetch_l2(y + r);
    prefetch_l2(lc + r);
    prefetch_l2(uc + r);
  }
  // per-line operands the tile path stages with bulk copies
  static constexpr int kStaged = Carry ? 4 : 3;
  // y, l_c, u_c (and the carried sums): not read again before they would
  // leave L2 anyway
  __device__ __forceinline__ bool staged_reused(int) const { return false; }
  __device__ __forceinline__ const double* staged_src(int q) const {
    return q == 0 ? y : (q == 1 ? lc : (q == 2 ? uc : carry));
  }
  // accumulators of a multi-chunk line go to its fixed slot: [dy2, infy]
  __device__ __forceinline__ void reset_acc() { dy2 = 0.0; infy = 0.0; }
  __device__ __forceinline__ void export_acc(double* dst) const {
    dst[0] = dy2;
    dst[1] = infy;
  }
  __device__ __forceinline__ Pre from_stage(const double* const* s, int li) const {
    return {s[0][li], s[1][li], s[2][li], Carry ? s[3][li] : 0.0};
  }
  __device__ __forceinline__ void line(int64_t r, double acc, const Pre& p) {
    const double yr = p.y;
    const double yhat = yr - sigma * acc;
    const double proj = clampd(yhat / sigma, -p.uc, -p.lc);
    const double yp = yhat - sigma * proj;  // exact cancellation: no FMA (step.hpp:85)
    yn[r] = yp;
    const double d = yp - yr;
#if PDLPK_DY_KEEP
    st_keep(dy + r, d, keep);
#else
    dy[r] = d;
#endif
    if (pend) sy[r] = sy[r] + w * yr;
    if (lp != nullptr) {
      lp[r] = d * d;
      lp[lm + r] = fabs(yp);
      return;
    }
    dy2 += d * d;
    infy = max_keep(infy, fabs(yp));
  }
};
using RowEpi = RowEpiT<false>;

// Earlier launches of a column-panel row pass: the line's running sum goes
// to carry[r] (In: it starts from the previous panels' sum, staged).
template <bool In>
struct CarryEpi {
  double* __restrict__ carry;
  struct Pre {
    double c;
  };
  __device__ __forceinline__ Pre load(int64_t r) const { return {In ? carry[r] : 0.0}; }
  __device__ __forceinline__ double init(const Pre& p) const { return In ? p.c : 0.0; }
  __device__ __forceinline__ void prefetch(int64_t r) const {
    if (In) prefetch_l2(carry + r);
  }
  static constexpr int kStaged = In ? 1 : 0;
  __device__ __forceinline__ bool staged_reused(int) const { return false; }
  __device__ __forceinline__ const double* staged_src(int) const { return carry; }
  __device__ __forceinline__ void reset_acc() {}
  __device__ __forceinline__ void export_acc(double*) const {}
  __device__ __forceinline__ Pre from_stage(const double* const* s, int li) const {
    return {In ? s[0][li] : 0.0};
  }
  __device__ __forceinline__ void line(int64_t r, double acc, const Pre&) { carry[r] = acc; }
};

// Ph: 0 whole row pass; 1 / 2 first / middle column panel (carry out);
// 3 last column panel (carry in, dual update)
template <class P, int Seg, int Ph>
__global__ void __launch_bounds__(kSpmvThreads, spmv_min_blocks(Seg)) row_pass(pdlpk_step_args a) {
  pdl_wait();
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  if constexpr (Ph == 1 || Ph == 2) {
    CarryEpi<Ph == 2> ce{a.carry};
    sched_spmv<P, Seg>(a.P.K, a.P.K.value, a.xbar, ce);
    pdl_trigger();
    return;
  }
  const int cur = st->cur;
  RowEpiT<Ph == 3> e;
  e.carry = a.carry;
  e.y = a.y[cur];
  e.yn = a.y[cur ^ 1];
  e.dy = a.dy;
  e.lc = a.P.lc;
  e.uc = a.P.uc;
  e.sy = a.sum_y;
  e.sigma = st->eta * st->omega;
#if PDLPK_DY_KEEP
  e.keep = l2_keep_policy(fminf(1.0f, static_cast<float>(PDLPK_XBAR_KEEP_MB * 1048576.0 /
                                                         (8.0 * static_cast<double>(a.P.m > 0 ? a.P.m : 1)))));
#endif
  e.pend = st->avg_pending != 0;
  e.w = st->avg_w;
  if (a.line_partials) {
    e.lp = a.part2;
    e.lm = a.P.m;
  }
  sched_spmv<P, Seg>(a.P.K, a.P.K.value, a.xbar, e);
  pdl_trigger();
  if (a.line_partials) return;  // per-line terms already written
  __shared__ double red[32];
  const double s1 = block_sum(e.dy2, red);
  __syncthreads();
  const double s2 = block_max(e.infy, red);
  if (threadIdx.x == 0) {
    a.part2[blockIdx.x] = s1;
    a.part2[gridDim.x + blockIdx.x] = s2;
  }
}

// ------------------------------------------- sliced-ELL row pass (knob) ---
// PDLP_ROW_SELL=1: the row pass over the SELL-32 copy of the row layout
// (kernels.h pdlpk_step_args::sell).  One warp per slice of 32 rows, lane =
// row; index and value loads are coalesced straight from global memory, each
// lane adds its row's products in storage order (the sums of the tile path's
// storage-order lines), the dual update runs in the same lane.
#ifndef PDLPK_SELL_UNROLL
#define PDLPK_SELL_UNROLL 8
#endif
#ifndef PDLPK_SELL_MINB
#define PDLPK_SELL_MINB 4
#endif
constexpr int kSellUnroll = PDLPK_SELL_UNROLL;
template <class P>
__global__ void __launch_bounds__(kSpmvThreads, PDLPK_SELL_MINB) row_pass_sell(pdlpk_step_args a) {
  pdl_wait();
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const int cur = st->cur;
  RowEpiT<false> e;
  e.y = a.y[cur];
  e.yn = a.y[cur ^ 1];
  e.dy = a.dy;
  e.lc = a.P.lc;
  e.uc = a.P.uc;
  e.sy = a.sum_y;
  e.sigma = st->eta * st->omega;
  e.pend = st->avg_pending != 0;
  e.w = st->avg_w;
  if (a.line_partials) {
    e.lp = a.part2;
    e.lm = a.P.m;
  }
  const P* __restrict__ start = static_cast<const P*>(a.P.K.start);
  const double* __restrict__ v = a.xbar;
  const int64_t m = a.P.K.dim;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t g = w0; g < a.sell.ng; g += nw) {
    const int64_t r = g * 32 + lane;
    const bool live = r < m;
    const int32_t n = live ? static_cast<int32_t>(start[r + 1] - start[r]) : 0;
    const int64_t o = a.sell.off[g];
    const int32_t w = static_cast<int32_t>((a.sell.off[g + 1] - o) >> 5);
    RowEpiT<false>::Pre pre{};
    if (live) pre = e.load(r);
    const int32_t* __restrict__ pi = a.sell.sidx + o + lane;
    const double* __restrict__ pv = a.sell.sval + o + lane;
    double acc = 0.0;
    for (int32_t k = 0; k < w; k += kSellUnroll) {
      int32_t c[kSellUnroll];
      double x[kSellUnroll], t[kSellUnroll];
#pragma unroll
      for (int u = 0; u < kSellUnroll; ++u) {
        const bool on = k + u < n;
        c[u] = on ? ld_stream(pi + 32 * (k + u)) : 0;
        x[u] = on ? ld_stream(pv + 32 * (k + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kSellUnroll; ++u) t[u] = (k + u < n) ? __ldg(v + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < kSellUnroll; ++u) {
        if (k + u < n) acc = mac(acc, x[u], t[u]);
      }
    }
    if (live) e.line(r, acc, pre);
  }
  pdl_trigger();
  if (a.line_partials) return;
  __shared__ double red[32];
  const double s1 = block_sum(e.dy2, red);
  __syncthreads();
  const double s2 = block_max(e.infy, red);
  if (threadIdx.x == 0) {
    a.part2[blockIdx.x] = s1;
    a.part2[gridDim.x + blockIdx.x] = s2;
  }
}

// SELL build: 32 x the longest line of each slice, and the scatter of the
// row layout's entries to their slots (padding slots are never read).
template <class P>
__global__ void sell_width_kernel(const P* __restrict__ start, int64_t m, int64_t ng,
                                  int64_t* __restrict__ w32) {
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < ng;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t w = 0;
    for (int l = 0; l < 32; ++l) {
      const int64_t r = g * 32 + l;
      if (r < m) {
        const int64_t len = static_cast<int64_t>(start[r + 1] - start[r]);
        w = len > w ? len : w;
      }
    }
    w32[g] = 32 * w;
  }
}
template <class P>
__global__ void sell_fill_kernel(const P* __restrict__ start, const int32_t* __restrict__ idx,
                                 const double* __restrict__ val, int64_t m,
                                 const int64_t* __restrict__ off, int32_t* __restrict__ sidx,
                                 double* __restrict__ sval) {
  // one warp per row: coalesced reads of the row, 128-byte-strided writes
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w0; r < m; r += nw) {
    const int64_t b = static_cast<int64_t>(start[r]), e = static_cast<int64_t>(start[r + 1]);
    const int64_t base = off[r >> 5] + (r & 31);
    for (int64_t k = b + lane; k < e; k += 32) {
      sidx[base + 32 * (k - b)] = idx[k];
      sval[base + 32 * (k - b)] = val[k];
    }
  }
}

// ------------------------------------------------------ perf column pass ---
struct ColEpi {
  const double* __restrict__ aty;
  double* __restrict__ atyn;
  const double* __restrict__ x;
  const double* __restrict__ xn;
  double dx2 = 0.0, curv = 0.0, infx = 0.0;
  struct Pre {
    double aty, x, xn;
  };
  __device__ __forceinline__ Pre load(int64_t i) const { return {aty[i], x[i], xn[i]}; }
  __device__ __forceinline__ double init(const Pre&) const { return 0.0; }
  __device__ __forceinline__ void prefetch(int64_t i) const {
    prefetch_l2(aty + i);
    prefetch_l2(x + i);
    prefetch_l2(xn + i);
  }
  static constexpr int kStaged = 3;
  // aty and x are dead after this pass; x' is the next primal pass's x
  __device__ __forceinline__ bool staged_reused(int q) const { return q == 2; }
  __device__ __forceinline__ const double* staged_src(int q) const {
    return q == 0 ? aty : (q == 1 ? x : xn);
  }
  // [dx2, curv, infx] of a multi-chunk line
  __device__ __forceinline__ void reset_acc() { dx2 = 0.0; curv = 0.0; infx = 0.0; }
  __device__ __forceinline__ void export_acc(double* dst) const {
    dst[0] = dx2;
    dst[1] = curv;
    dst[2] = infx;
  }
  __device__ __forceinline__ Pre from_stage(const double* const* s, int li) const {
    return {s[0][li], s[1][li], s[2][li]};
  }
  __device__ __forceinline__ void line(int64_t i, double d, const Pre& p) {
    atyn[i] = p.aty + d;
    const double dxi = p.xn - p.x;
    dx2 += dxi * dxi;
    curv += d * dxi;
    infx = max_keep(infx, fabs(p.xn));
  }
};

// The column pass's tail: this CTA's partials of |dx|^2, dy'K dx and |x'|
// into part3; with Decide, the last CTA combines every partial in a fixed
// order and runs the accept/reject rule.  kt_slots: add the fixed slots of
// K^T's multi-chunk lines (their epilogue terms live there).
template <bool Decide>
__device__ __forceinline__ void col_tail(const pdlpk_step_args& a, const ColEpi& e, bool kt_slots) {
  pdlpk_step_state* st = a.state;
  __shared__ double red[32];
  __shared__ bool last;
  const double s1 = block_sum(e.dx2, red);
  __syncthreads();
  const double s2 = block_sum(e.curv, red);
  __syncthreads();
  const double s3 = block_max(e.infx, red);
  const int64_t g3 = gridDim.x;
  if (threadIdx.x == 0) {
    a.part3[blockIdx.x] = s1;
    a.part3[g3 + blockIdx.x] = s2;
    a.part3[2 * g3 + blockIdx.x] = s3;
  }
  if (!Decide) return;  // row-sharded: the host combines ranks first
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(&st->ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // Last CTA: combine every partial in a fixed order, then decide.
  double dy2 = 0.0, infy = 0.0, dx2 = 0.0, curv = 0.0, infx = 0.0;
  if (a.line_partials) {
    // per-line terms, grouped by line index into blocks of 8 summed as an
    // 8-warp CTA's block_sum adds one line per warp -- the grouping the
    // per-CTA partials had when every warp took one line in order -- then
    // strided over the blocks like the CTA partials: independent of the
    // SpMV schedule
    const int64_t m = a.P.m, nb8 = (m + 7) / 8;
    for (int64_t b = threadIdx.x; b < nb8; b += blockDim.x) {
      double v[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int64_t r = 8 * b + w;
        v[w] = r < m ? __ldcg(a.part2 + r) : 0.0;
        if (r < m) infy = max_keep(infy, __ldcg(a.part2 + m + r));
      }
      dy2 += ((v[0] + v[4]) + (v[2] + v[6])) + ((v[1] + v[5]) + (v[3] + v[7]));
    }
  } else {
    const int64_t g2 = sched_blocks(a.P.K);
    for (int64_t b = threadIdx.x; b < g2; b += blockDim.x) {
      dy2 += __ldcg(a.part2 + b);
      infy = max_keep(infy, __ldcg(a.part2 + g2 + b));
    }
  }
  for (int64_t b = threadIdx.x; b < g3; b += blockDim.x) {
    dx2 += __ldcg(a.part3 + b);
    curv += __ldcg(a.part3 + g3 + b);
    infx = max_keep(infx, __ldcg(a.part3 + 2 * g3 + b));
  }
  // then the fixed slots of multi-chunk lines (spmv.cuh), in slot order
  for (int64_t q = threadIdx.x; q < a.P.K.n_multi; q += blockDim.x) {
    const double* sl = a.P.K.line_acc + q * PDLPK_LINE_ACC;
    dy2 += __ldcg(sl);
    infy = max_keep(infy, __ldcg(sl + 1));
  }
  if (kt_slots) {
    for (int64_t q = threadIdx.x; q < a.P.KT.n_multi; q += blockDim.x) {
      const double* sl = a.P.KT.line_acc + q * PDLPK_LINE_ACC;
      dx2 += __ldcg(sl);
      curv += __ldcg(sl + 1);
      infx = max_keep(infx, __ldcg(sl + 2));
    }
  }
  dy2 = block_sum(dy2, red);
  __syncthreads();
  infy = block_max(infy, red);
  __syncthreads();
  dx2 = block_sum(dx2, red);
  __syncthreads();
  curv = block_sum(curv, red);
  __syncthreads();
  infx = block_max(infx, red);
  if (threadIdx.x == 0) {
    st->ticket = 0;
    decide(st, dx2, dy2, curv, infx, infy, a.f_down, a.f_up, a.table_len);
  }
}

template <class P, int Seg, bool Decide>
__global__ void __launch_bounds__(kSpmvThreads, spmv_min_blocks(Seg)) col_pass(pdlpk_step_args a) {
  pdl_wait();
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const int cur = st->cur;
  ColEpi e;
  e.aty = a.aty[cur];
  e.atyn = a.aty[cur ^ 1];
  e.x = a.x[cur];
  e.xn = a.x[cur ^ 1];
  sched_spmv<P, Seg>(a.P.KT, a.P.KT.value, a.dy, e);
  pdl_trigger();
  col_tail<Decide>(a, e, true);
}

// Split column pass (segmented-span layouts): the product alone writes
// d = K^T dy to aty_diff (one 8-byte store per line instead of the
// epilogue's three loads and a store at scattered lanes), then a coalesced
// elementwise pass runs the epilogue and the decision.
struct DiffEpi {
  double* __restrict__ out;
  struct Pre {};
  __device__ __forceinline__ Pre load(int64_t) const { return {}; }
  __device__ __forceinline__ double init(const Pre&) const { return 0.0; }
  __device__ __forceinline__ void prefetch(int64_t) const {}
  static constexpr int kStaged = 0;
  __device__ __forceinline__ const double* staged_src(int) const { return nullptr; }
  __device__ __forceinline__ bool staged_reused(int) const { return false; }
  __device__ __forceinline__ Pre from_stage(const double* const*, int) const { return {}; }
  __device__ __forceinline__ void reset_acc() {}
  __device__ __forceinline__ void export_acc(double*) const {}
  __device__ __forceinline__ void line(int64_t r, double acc, const Pre&) { out[r] = acc; }
};

template <class P, int Seg>
__global__ void __launch_bounds__(kSpmvThreads, spmv_min_blocks(Seg)) col_product(pdlpk_step_args a) {
  pdl_wait();
  if (a.state->halt) return;
  DiffEpi e{a.aty_diff};
  sched_spmv<P, Seg>(a.P.KT, a.P.KT.value, a.dy, e);
  pdl_trigger();
}

__global__ void __launch_bounds__(kEwThreads) col_epi_decide(pdlpk_step_args a) {
  pdl_wait();
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const int cur = st->cur;
  ColEpi e;
  e.aty = a.aty[cur];
  e.atyn = a.aty[cur ^ 1];
  e.x = a.x[cur];
  e.xn = a.x[cur ^ 1];
  const int64_t n = a.P.n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    e.line(i, __ldcs(a.aty_diff + i), {__ldcs(e.aty + i), __ldcs(e.x + i), e.xn[i]});
  }
  pdl_trigger();
  col_tail<true>(a, e, false);
}

// ------------------------------------------------------------ parity path ---
template <class P>
__global__ void __launch_bounds__(kEwThreads) parity_row_pass(pdlpk_step_args a) {
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const int cur = st->cur;
  const double* __restrict__ y = a.y[cur];
  double* __restrict__ yn = a.y[cur ^ 1];
  const double sigma = st->eta * st->omega;
  const bool pend = st->avg_pending != 0;
  const double w = st->avg_w;
  const P* __restrict__ start = static_cast<const P*>(a.P.K.start);
  const int32_t* __restrict__ idx = a.P.K.index;
  const double* __restrict__ val = a.P.K.value;
  const double* __restrict__ xbar = a.xbar;
  const int64_t m = a.P.m;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < m;
       r += stride) {
    double acc = 0.0;
    for (int64_t k = start[r]; k < start[r + 1]; ++k) acc = acc + val[k] * xbar[idx[k]];
    const double yr = y[r];
    const double yhat = yr - sigma * acc;
    const double proj = clampd(yhat / sigma, -a.P.uc[r], -a.P.lc[r]);
    const double yp = yhat - sigma * proj;
    yn[r] = yp;
    a.dy[r] = yp - yr;
    if (pend) a.sum_y[r] = a.sum_y[r] + w * yr;
  }
}

template <class P>
__global__ void __launch_bounds__(kEwThreads) parity_col_pass(pdlpk_step_args a) {
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const int cur = st->cur;
  const double* __restrict__ aty = a.aty[cur];
  double* __restrict__ atyn = a.aty[cur ^ 1];
  const P* __restrict__ start = static_cast<const P*>(a.P.KT.start);
  const int32_t* __restrict__ idx = a.P.KT.index;
  const double* __restrict__ val = a.P.KT.value;
  const double* __restrict__ dy = a.dy;
  const int64_t n = a.P.n;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    double acc = 0.0;
    for (int64_t k = start[i]; k < start[i + 1]; ++k) acc = acc + val[k] * dy[idx[k]];
    a.aty_diff[i] = acc;
    atyn[i] = aty[i] + acc;
  }
}

__device__ __forceinline__ void shard_range(int64_t dim, int s, int S, int64_t& lo, int64_t& hi) {
  const int64_t base = dim / S, rem = dim % S;
  lo = s * base + (s < rem ? s : rem);
  hi = lo + base + (s < rem ? 1 : 0);
}

// One thread per shard: x-plan shards [0,S) and y-plan shards [S,2S).
__global__ void parity_shard_reduce(pdlpk_step_args a) {
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const int S = a.shards;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * S) return;
  const int cur = st->cur;
  double* part = a.shard_part;
  int64_t lo, hi;
  if (t < S) {
    const double* x = a.x[cur];
    const double* xn = a.x[cur ^ 1];
    shard_range(a.P.n, t, S, lo, hi);
    double dx2 = 0.0, curv = 0.0, infx = 0.0;
    for (int64_t i = lo; i < hi; ++i) {
      const double d = xn[i] - x[i];
      dx2 += d * d;
    }
    for (int64_t i = lo; i < hi; ++i) curv += a.aty_diff[i] * (xn[i] - x[i]);
    if (st->fixed) {
      for (int64_t i = lo; i < hi; ++i) infx = max_keep(infx, fabs(xn[i]));
    }
    part[t] = dx2;
    part[S + t] = curv;
    part[2 * S + t] = infx;
  } else {
    const int s = t - S;
    const double* yn = a.y[cur ^ 1];
    shard_range(a.P.m, s, S, lo, hi);
    double dy2 = 0.0, infy = 0.0;
    for (int64_t j = lo; j < hi; ++j) {
      const double d = a.dy[j];
      dy2 += d * d;
    }
    if (st->fixed) {
      for (int64_t j = lo; j < hi; ++j) infy = max_keep(infy, fabs(yn[j]));
    }
    part[3 * S + s] = dy2;
    part[4 * S + s] = infy;
  }
}

__global__ void parity_decide(pdlpk_step_args a) {
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const int S = a.shards;
  const double* part = a.shard_part;
  double dx2 = 0.0, curv = 0.0, infx = 0.0, dy2 = 0.0, infy = 0.0;
  for (int s = 0; s < S; ++s) dx2 += part[s];
  for (int s = 0; s < S; ++s) curv += part[S + s];
  for (int s = 0; s < S; ++s) infx = max_keep(infx, part[2 * S + s]);
  for (int s = 0; s < S; ++s) dy2 += part[3 * S + s];
  for (int s = 0; s < S; ++s) infy = max_keep(infy, part[4 * S + s]);
  decide(st, dx2, dy2, curv, infx, infy, a.f_down, a.f_up, a.table_len);
}

// ---------------------------------------------------------- bookkeeping ---
__global__ void arm_kernel(pdlpk_step_state* st, int64_t k_target) {
  st->k_target = k_target;
  st->halt = (st->status != 0 || st->k >= k_target) ? 1 : 0;
}

__global__ void __launch_bounds__(kEwThreads) flush_average_kernel(pdlpk_step_args a) {
  const pdlpk_step_state* st = a.state;
  if (!st->avg_pending) return;
  const int cur = st->cur;
  const double w = st->avg_w;
  const double* x = a.x[cur];
  const double* y = a.y[cur];
  const int64_t n = a.P.n, m = a.P.m;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n + m;
       i += stride) {
    if (i < n) {
      a.sum_x[i] = a.sum_x[i] + w * x[i];
    } else {
      const int64_t j = i - n;
      a.sum_y[j] = a.sum_y[j] + w * y[j];
    }
  }
}

__global__ void clear_pending_kernel(pdlpk_step_state* st) { st->avg_pending = 0; }

struct LaunchRowCol {
  const pdlpk_step_args* a;
  cudaStream_t s;
  bool row;
  bool decide_here = true;
  bool pdl = false;
  template <class P, int Seg>
  int go() {
    const pdlpk_csr& A = row ? a->P.K : a->P.KT;
    const int64_t g = sched_blocks(A);
    if (g <= 0) return 0;
    const size_t smem = spmv_smem(A, Seg);
    const unsigned gu = static_cast<unsigned>(g);
    if (row) {
      switch (a->panel_phase) {
        case 1:
          allow_smem(row_pass<P, Seg, 1>, smem);
          launch_pdl(pdl, row_pass<P, Seg, 1>, gu, kSpmvThreads, smem, s, *a);
          break;
        case 2:
          allow_smem(row_pass<P, Seg, 2>, smem);
          launch_pdl(pdl, row_pass<P, Seg, 2>, gu, kSpmvThreads, smem, s, *a);
          break;
        case 3:
          allow_smem(row_pass<P, Seg, 3>, smem);
          launch_pdl(pdl, row_pass<P, Seg, 3>, gu, kSpmvThreads, smem, s, *a);
          break;
        default:
          allow_smem(row_pass<P, Seg, 0>, smem);
          launch_pdl(pdl, row_pass<P, Seg, 0>, gu, kSpmvThreads, smem, s, *a);
      }
    } else {
      if (decide_here && ((PDLPK_COL_SPLIT && A.seg_mode) || A.col_split)) {
        allow_smem(col_product<P, Seg>, smem);
        launch_pdl(pdl, col_product<P, Seg>, gu, kSpmvThreads, smem, s, *a);
        launch_pdl(pdl, col_epi_decide, static_cast<unsigned>(ew_blocks(a->P.n)), kEwThreads,
                   static_cast<size_t>(0), s, *a);
      } else if (decide_here) {
        allow_smem(col_pass<P, Seg, true>, smem);
        launch_pdl(pdl, col_pass<P, Seg, true>, gu, kSpmvThreads, smem, s, *a);
      } else {
        allow_smem(col_pass<P, Seg, false>, smem);
        launch_pdl(pdl, col_pass<P, Seg, false>, gu, kSpmvThreads, smem, s, *a);
      }
    }
    return 0;
  }
};

// ------------------------------------------------- row-sharded attempt ---
// Epilogues over reduce-scattered line sums (the layout's lines live on
// other ranks' partial products), and the cross-rank decision.
// Line sum i: acc[i], or the rank-ordered sum of the peers' partials.  The
// loads are independent (one per rank, issued together) so the NVLink
// latency of the remote reads overlaps.
__device__ __forceinline__ double peer_value(const pdlpk_peer_sum& ps, const double* acc, int64_t i) {
  if (ps.world == 0) return acc[i];
  double v[PDLPK_MAX_PEERS];
#pragma unroll
  for (int r = 0; r < PDLPK_MAX_PEERS; ++r) {
    if (r < ps.world) v[r] = __ldcg(ps.p[r] + ps.offset + i);
  }
  double t = v[0];
#pragma unroll
  for (int r = 1; r < PDLPK_MAX_PEERS; ++r) {
    if (r < ps.world) t += v[r];
  }
  return t;
}

__global__ void __launch_bounds__(kEwThreads) row_epi_kernel(pdlpk_step_args a, const double* acc,
                                                            pdlpk_peer_sum ps) {
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const int cur = st->cur;
  RowEpi e;
  e.y = a.y[cur];
  e.yn = a.y[cur ^ 1];
  e.dy = a.dy;
  e.lc = a.P.lc;
  e.uc = a.P.uc;
  e.sy = a.sum_y;
  e.sigma = st->eta * st->omega;
#if PDLPK_DY_KEEP
  e.keep = l2_keep_policy(fminf(1.0f, static_cast<float>(PDLPK_XBAR_KEEP_MB * 1048576.0 /
                                                         (8.0 * static_cast<double>(a.P.m > 0 ? a.P.m : 1)))));
#endif
  e.pend = st->avg_pending != 0;
  e.w = st->avg_w;
  const int64_t m = a.P.m;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    e.line(r, peer_value(ps, acc, r), e.load(r));
  }
  __shared__ double red[32];
  const double s1 = block_sum(e.dy2, red);
  __syncthreads();
  const double s2 = block_max(e.infy, red);
  if (threadIdx.x == 0) {
    a.part2[blockIdx.x] = s1;
    a.part2[gridDim.x + blockIdx.x] = s2;
  }
}

__global__ void __launch_bounds__(kEwThreads) col_epi_kernel(pdlpk_step_args a, const double* d,
                                                            pdlpk_peer_sum ps) {
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  const int cur = st->cur;
  ColEpi e;
  e.aty = a.aty[cur];
  e.atyn = a.aty[cur ^ 1];
  e.x = a.x[cur];
  e.xn = a.x[cur ^ 1];
  const int64_t n = a.P.n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    e.line(i, peer_value(ps, d, i), e.load(i));
  }
  __shared__ double red[32];
  const double s1 = block_sum(e.dx2, red);
  __syncthreads();
  const double s2 = block_sum(e.curv, red);
  __syncthreads();
  const double s3 = block_max(e.infx, red);
  const int64_t g3 = gridDim.x;
  if (threadIdx.x == 0) {
    a.part3[blockIdx.x] = s1;
    a.part3[g3 + blockIdx.x] = s2;
    a.part3[2 * g3 + blockIdx.x] = s3;
  }
}

// This rank's totals, combined exactly like col_pass's last CTA.
__global__ void __launch_bounds__(kEwThreads) dist_totals_kernel(pdlpk_step_args a, int64_t g2,
                                                                 int64_t g3, int k_acc, int kt_acc,
                                                                 double* out) {
  if (a.state->halt) return;
  __shared__ double red[32];
  double dy2 = 0.0, infy = 0.0, dx2 = 0.0, curv = 0.0, infx = 0.0;
  for (int64_t b = threadIdx.x; b < g2; b += blockDim.x) {
    dy2 += a.part2[b];
    infy = max_keep(infy, a.part2[g2 + b]);
  }
  for (int64_t b = threadIdx.x; b < g3; b += blockDim.x) {
    dx2 += a.part3[b];
    curv += a.part3[g3 + b];
    infx = max_keep(infx, a.part3[2 * g3 + b]);
  }
  if (k_acc) {
    for (int64_t q = threadIdx.x; q < a.P.K.n_multi; q += blockDim.x) {
      const double* s = a.P.K.line_acc + q * PDLPK_LINE_ACC;
      dy2 += s[0];
      infy = max_keep(infy, s[1]);
    }
  }
  if (kt_acc) {
    for (int64_t q = threadIdx.x; q < a.P.KT.n_multi; q += blockDim.x) {
      const double* s = a.P.KT.line_acc + q * PDLPK_LINE_ACC;
      dx2 += s[0];
      curv += s[1];
      infx = max_keep(infx, s[2]);
    }
  }
  dy2 = block_sum(dy2, red);
  __syncthreads();
  infy = block_max(infy, red);
  __syncthreads();
  dx2 = block_sum(dx2, red);
  __syncthreads();
  curv = block_sum(curv, red);
  __syncthreads();
  infx = block_max(infx, red);
  if (threadIdx.x == 0) {
    out[0] = dy2;
    out[1] = infy;
    out[2] = dx2;
    out[3] = curv;
    out[4] = infx;
    out[5] = out[6] = out[7] = 0.0;
  }
}

// All ranks run this on identical gathered totals, in rank order: the
// controllers stay bitwise identical without another exchange.
__global__ void dist_decide_kernel(pdlpk_step_args a, const double* all, int world) {
  pdlpk_step_state* st = a.state;
  if (st->halt) return;
  double dy2 = 0.0, infy = 0.0, dx2 = 0.0, curv = 0.0, infx = 0.0;
  for (int r = 0; r < world; ++r) {
    const double* t = all + 8 * r;
    dy2 += t[0];
    infy = max_keep(infy, t[1]);
    dx2 += t[2];
    curv += t[3];
    infx = max_keep(infx, t[4]);
  }
  decide(st, dx2, dy2, curv, infx, infy, a.f_down, a.f_up, a.table_len);
}

}  // namespace
}  // namespace pdlp

using namespace pdlp;

extern "C" int64_t pdlpk_step_partials(const pdlpk_problem* P) {
  const int64_t g2 = sched_blocks(P->K), g3 = sched_blocks(P->KT);
  int64_t need = 2 * g2 > 3 * g3 ? 2 * g2 : 3 * g3;
  const int64_t ge = 3 * static_cast<int64_t>(ew_blocks(P->n));  // split column pass
  if ((P->KT.seg_mode || P->KT.col_split) && ge > need) need = ge;
  if (P->m <= PDLPK_LINE_PARTIALS_MAX && 2 * P->m > need) need = 2 * P->m;  // line_partials
  return need + 64;
}

extern "C" int pdlpk_sell_plan(const pdlpk_csr* K, int64_t* w32, int64_t* off, void* tmp,
                               size_t* tmp_bytes, cudaStream_t s) {
  const int64_t ng = (K->dim + 31) / 32;
  if (tmp == nullptr) {
    *tmp_bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, *tmp_bytes, w32, off + 1, static_cast<int>(ng), s);
    return static_cast<int>(cudaGetLastError());
  }
  if (ng <= 0) return 0;
  const unsigned g = static_cast<unsigned>(std::min<int64_t>((ng + 255) / 256, 148 * 8));
  if (K->wide) {
    sell_width_kernel<<<g, 256, 0, s>>>(static_cast<const int64_t*>(K->start), K->dim, ng, w32);
  } else {
    sell_width_kernel<<<g, 256, 0, s>>>(static_cast<const int32_t*>(K->start), K->dim, ng, w32);
  }
  cudaMemsetAsync(off, 0, sizeof(int64_t), s);
  size_t bytes = *tmp_bytes;
  cub::DeviceScan::InclusiveSum(tmp, bytes, w32, off + 1, static_cast<int>(ng), s);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_sell_fill(const pdlpk_csr* K, const int64_t* off, int32_t* sidx, double* sval,
                               cudaStream_t s) {
  if (K->dim <= 0) return 0;
  const unsigned g = 148 * 16;
  if (K->wide) {
    sell_fill_kernel<<<g, 256, 0, s>>>(static_cast<const int64_t*>(K->start), K->index, K->value,
                                       K->dim, off, sidx, sval);
  } else {
    sell_fill_kernel<<<g, 256, 0, s>>>(static_cast<const int32_t*>(K->start), K->index, K->value,
                                       K->dim, off, sidx, sval);
  }
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_arm(pdlpk_step_state* st, int64_t k_target, cudaStream_t s) {
  arm_kernel<<<1, 1, 0, s>>>(st, k_target);
  return static_cast<int>(cudaGetLastError());
}

// The row pass: one launch, or one per column panel (carry chained).  The
// returned args are the column pass's: with panels its decision reads the
// last panel launch's partials, so P.K is that layout.
static pdlpk_step_args launch_row(const pdlpk_step_args* a, cudaStream_t s, bool pdl) {
  if (a->sell.off != nullptr) {
    const unsigned g = static_cast<unsigned>(a->sell.blocks);
    if (a->P.K.wide) {
      launch_pdl(pdl, row_pass_sell<int64_t>, g, kSpmvThreads, static_cast<size_t>(0), s, *a);
    } else {
      launch_pdl(pdl, row_pass_sell<int32_t>, g, kSpmvThreads, static_cast<size_t>(0), s, *a);
    }
    // the decision reads this pass's per-CTA partials: a layout view that
    // only says how many there are (sched_blocks) and has no line slots
    pdlpk_step_args b = *a;
    b.P.K.seg_mode = 1;
    b.P.K.tile_blocks = a->sell.blocks;
    b.P.K.n_multi = 0;
    return b;
  }
  if (a->n_row_panels < 2 || a->row_panels == nullptr) {
    dispatch_p(a->P.K, LaunchRowCol{a, s, true, true, pdl});
    return *a;
  }
  pdlpk_step_args b = *a;
  const int np = a->n_row_panels;
  for (int q = 0; q < np; ++q) {
    b.P.K = a->row_panels[q];
    b.panel_phase = q == 0 ? 1 : (q == np - 1 ? 3 : 2);
    dispatch_p(b.P.K, LaunchRowCol{&b, s, true, true, pdl});
  }
  b.panel_phase = 0;
  return b;
}

// PDLP_DY_PERSIST=1 (measurement knob, perf mode): the column pass's gathers
// of dy go through a persisting L2 access-policy window (dy stays resident
// while the matrix streams pass with evict_first).
static bool dy_persist_on(const pdlpk_step_args* a) {
  static const int on = [] {
    const char* e = std::getenv("PDLP_DY_PERSIST");
    return e != nullptr && e[0] == '1' ? 1 : 0;
  }();
  if (!on || a->dy == nullptr || a->P.m <= 0) return false;
  static int limit_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (limit_dev != dev) {
    size_t want = static_cast<size_t>(a->P.m) * 8;
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    cudaGetLastError();
    limit_dev = dev;
  }
  return true;
}

static void dy_window(cudaStream_t s, const pdlpk_step_args* a, bool set) {
  cudaStreamAttrValue v{};
  if (set) {
    v.accessPolicyWindow.base_ptr = const_cast<double*>(a->dy);
    v.accessPolicyWindow.num_bytes = static_cast<size_t>(a->P.m) * 8;
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  } else {
    v.accessPolicyWindow.num_bytes = 0;
  }
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();
}

extern "C" int pdlpk_attempt(const pdlpk_step_args* a, cudaStream_t s) {
  const bool pdl = a->mode == 0;  // perf mode: the three kernels chain with PDL
  launch_pdl(pdl, primal_pass<false>, static_cast<unsigned>(ew_blocks(a->P.n)), kEwThreads, 0, s,
              *a, pdlpk_peer_sum{});
  if (a->mode == 0) {
    // Degenerate shapes (an empty side) still need the decision, which the
    // column pass performs: it always has >= 1 CTA (short_blocks >= 1).
    const pdlpk_step_args c = launch_row(a, s, true);
    const bool persist = dy_persist_on(a);
    if (persist) dy_window(s, a, true);
    dispatch_p(c.P.KT, LaunchRowCol{&c, s, false, true, true});
    if (persist) dy_window(s, a, false);
  } else {
    const int gm = ew_blocks(a->P.m), gn = ew_blocks(a->P.n);
    if (a->P.K.wide) {
      parity_row_pass<int64_t><<<gm, kEwThreads, 0, s>>>(*a);
      parity_col_pass<int64_t><<<gn, kEwThreads, 0, s>>>(*a);
    } else {
      parity_row_pass<int32_t><<<gm, kEwThreads, 0, s>>>(*a);
      parity_col_pass<int32_t><<<gn, kEwThreads, 0, s>>>(*a);
    }
    const int t = 2 * a->shards;
    parity_shard_reduce<<<(t + 127) / 128, 128, 0, s>>>(*a);
    parity_decide<<<1, 1, 0, s>>>(*a);
  }
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_attempt_timed(const pdlpk_step_args* a, cudaEvent_t* ev, cudaStream_t s) {
  cudaEventRecord(ev[0], s);
  primal_pass<false><<<ew_blocks(a->P.n), kEwThreads, 0, s>>>(*a, pdlpk_peer_sum{});
  cudaEventRecord(ev[1], s);
  if (a->mode == 0) {
    const pdlpk_step_args c = launch_row(a, s, false);
    cudaEventRecord(ev[2], s);
    const bool persist = dy_persist_on(a);
    if (persist) dy_window(s, a, true);
    dispatch_p(c.P.KT, LaunchRowCol{&c, s, false});
    if (persist) dy_window(s, a, false);
  } else {
    const int gm = ew_blocks(a->P.m), gn = ew_blocks(a->P.n);
    if (a->P.K.wide) {
      parity_row_pass<int64_t><<<gm, kEwThreads, 0, s>>>(*a);
      cudaEventRecord(ev[2], s);
      parity_col_pass<int64_t><<<gn, kEwThreads, 0, s>>>(*a);
    } else {
      parity_row_pass<int32_t><<<gm, kEwThreads, 0, s>>>(*a);
      cudaEventRecord(ev[2], s);
      parity_col_pass<int32_t><<<gn, kEwThreads, 0, s>>>(*a);
    }
    const int t = 2 * a->shards;
    parity_shard_reduce<<<(t + 127) / 128, 128, 0, s>>>(*a);
    parity_decide<<<1, 1, 0, s>>>(*a);
  }
  cudaEventRecord(ev[3], s);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_flush_average(const pdlpk_step_args* a, cudaStream_t s) {
  flush_average_kernel<<<ew_blocks(a->P.n + a->P.m), kEwThreads, 0, s>>>(*a);
  clear_pending_kernel<<<1, 1, 0, s>>>(a->state);
  return static_cast<int>(cudaGetLastError());
}

// ------------------------------------------------- row-sharded attempt ---
extern "C" int64_t pdlpk_dist_ew_grid(int64_t n) { return ew_blocks(n); }

extern "C" int64_t pdlpk_dist_sched_grid(const pdlpk_csr* A) { return sched_blocks(*A); }

extern "C" int pdlpk_dist_primal(const pdlpk_step_args* a, cudaStream_t s) {
  primal_pass<false><<<ew_blocks(a->P.n), kEwThreads, 0, s>>>(*a, pdlpk_peer_sum{});
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_dist_primal_push(const pdlpk_step_args* a, const pdlpk_peer_sum* dst,
                                      cudaStream_t s) {
  primal_pass<true><<<ew_blocks(a->P.n), kEwThreads, 0, s>>>(*a, *dst);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_dist_row_fused(const pdlpk_step_args* a, cudaStream_t s) {
  dispatch_p(a->P.K, LaunchRowCol{a, s, true});
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_dist_row_epi(const pdlpk_step_args* a, const double* acc, cudaStream_t s) {
  pdlpk_peer_sum none{};
  row_epi_kernel<<<ew_blocks(a->P.m), kEwThreads, 0, s>>>(*a, acc, none);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_dist_row_epi_peers(const pdlpk_step_args* a, const pdlpk_peer_sum* ps,
                                        cudaStream_t s) {
  row_epi_kernel<<<ew_blocks(a->P.m), kEwThreads, 0, s>>>(*a, nullptr, *ps);
  return static_cast<int>(cudaGetLastError());
}

__global__ void __launch_bounds__(kEwThreads) peer_reduce_kernel(double* out, pdlpk_peer_sum ps,
                                                                int64_t count) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    out[i] = peer_value(ps, nullptr, i);
  }
}

extern "C" int pdlpk_peer_reduce(double* out, const pdlpk_peer_sum* ps, int64_t count,
                                 cudaStream_t s) {
  if (count <= 0) return 0;
  peer_reduce_kernel<<<ew_blocks(count), kEwThreads, 0, s>>>(out, *ps, count);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_dist_col_fused(const pdlpk_step_args* a, cudaStream_t s) {
  dispatch_p(a->P.KT, LaunchRowCol{a, s, false, false});
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_dist_col_epi(const pdlpk_step_args* a, const double* d, cudaStream_t s) {
  pdlpk_peer_sum none{};
  col_epi_kernel<<<ew_blocks(a->P.n), kEwThreads, 0, s>>>(*a, d, none);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_dist_col_epi_peers(const pdlpk_step_args* a, const pdlpk_peer_sum* ps,
                                        cudaStream_t s) {
  col_epi_kernel<<<ew_blocks(a->P.n), kEwThreads, 0, s>>>(*a, nullptr, *ps);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_dist_totals(const pdlpk_step_args* a, int64_t g2, int64_t g3, int32_t k_acc,
                                 int32_t kt_acc, double* out8, cudaStream_t s) {
  dist_totals_kernel<<<1, kEwThreads, 0, s>>>(*a, g2, g3, k_acc, kt_acc, out8);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_dist_decide(const pdlpk_step_args* a, const double* all8, int32_t world,
                                 cudaStream_t s) {
  dist_decide_kernel<<<1, 1, 0, s>>>(*a, all8, world);
  return static_cast<int>(cudaGetLastError());
}

// CTAs of the staged-tile kernels that are resident at once (the tile
// segment is grid-stride: a second wave of CTAs would start its tiles late).
extern "C" int64_t pdlpk_tile_resident_ctas(int32_t stage_bytes) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = kRingHeader + kStages * static_cast<size_t>(stage_bytes);
  allow_smem(col_pass<int32_t, 4, true>, smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, col_pass<int32_t, 4, true>,
                                                    kSpmvThreads, smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  return static_cast<int64_t>(sms) * per_sm;
}

// CTAs of the segmented-span kernels resident at once (their grid: each warp
// walks spans grid-stride).
extern "C" int64_t pdlpk_seg_resident_ctas(void) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, col_pass<int32_t, 16, true>,
                                                    kSpmvThreads, 0) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  return static_cast<int64_t>(sms) * per_sm;
}
