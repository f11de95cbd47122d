// Host C++ driver of the B200 PDLP solver and the public C-ABI (pdlp_b200.h).
//
// This is a restatement of the reference driver
//   solve            proj/include/pdhglp/solver.hpp:535-608
//   run_inner        solver.hpp:350-531  (64-step cadence, restarts, rays, polish gate)
//   screen_and_verify / capture_current / detect_rays / attempt_polish
//                    solver.hpp:207-348
// in which every O(n), O(m) or O(nnz) operation is a device kernel reached
// through the thin internal C-ABI of kernels.h.  The host holds only scalars
// (step controller mirror, restart metrics, omega) and makes the branchy
// decisions on them with the reference's exact formulas; vectors live in HBM
// for the whole solve and come back once, at the end.  There is no CPU
// fallback: without a usable device every entry point fails with
// PDLP_ERR_CUDA.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <exception>
#include <thread>
#include <vector>

#include "device.hpp"
#include "comm.hpp"
#include "host_stage.hpp"
#include "shard.hpp"
#include "kernels.h"
#include "pdlp_b200.h"

namespace pdlp_host {

constexpr double kInf = std::numeric_limits<double>::infinity();
using Clock = std::chrono::steady_clock;

thread_local std::string g_last_error;

struct InvalidProblem : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// ------------------------------------------------------------- host types ---
struct Summary {  // ResidualSummary, residuals.hpp:66-73
  double primal = kInf, dual = kInf, pobj = 0.0, dobj = 0.0, abs_gap = kInf, rel_gap = kInf;
};

// finish_summary (residuals.hpp:98-114)
Summary finish_summary(double primal_inf, double dual_inf, double pobj, double dobj) {
  Summary s;
  s.primal = primal_inf;
  s.dual = dual_inf;
  s.pobj = pobj;
  s.dobj = dobj;
  if (!std::isfinite(dobj)) return s;
  s.abs_gap = std::abs(pobj - dobj);
  const double denom = std::max(std::abs(pobj), std::abs(dobj));
  s.rel_gap = s.abs_gap == 0.0 ? 0.0 : s.abs_gap / denom;
  return s;
}

struct Tol {
  double eps_primal = 1e-8, eps_dual = 1e-8, eps_rel_gap = 1e-2;
};

bool check_termination(const Summary& s, const Tol& t) {  // residuals.hpp:193-196
  return s.primal <= t.eps_primal && s.dual <= t.eps_dual && s.rel_gap <= t.eps_rel_gap;
}

enum Status { kOptimal = 0, kPrimalInf, kDualInf, kIterLimit, kTimeLimit, kNumErr };

const char* status_name(int s) {  // solver.hpp:44-54
  switch (s) {
    case kOptimal: return "optimal";
    case kPrimalInf: return "primal_infeasible";
    case kDualInf: return "dual_infeasible";
    case kIterLimit: return "iteration_limit";
    case kTimeLimit: return "time_limit";
    default: return "numerical_error";
  }
}

enum Reason { kNone = 0, kSufficient, kStalled, kArtificial };
const char* reason_name(int r) {
  switch (r) {
    case kSufficient: return "sufficient";
    case kStalled: return "stalled";
    case kArtificial: return "artificial";
    default: return "none";
  }
}

struct Thresholds {
  double sufficient = 0.1, necessary = 0.9, artificial = 0.5;
};

// should_restart (restarts.hpp:257-271)
int should_restart(double cand, double mu_last, double prev_mu, int64_t since, int64_t total,
                   const Thresholds& th) {
  if (std::isfinite(mu_last)) {
    if (cand <= th.sufficient * mu_last) return kSufficient;
    if (cand <= th.necessary * mu_last && cand > prev_mu) return kStalled;
  }
  if (static_cast<double>(since) >= th.artificial * static_cast<double>(total)) return kArtificial;
  return kNone;
}

// update_primal_weight (restarts.hpp:298-303)
double update_primal_weight(double dx, double dy, double omega_prev) {
  const double theta = 0.5, eps_zero = 1e-12;
  if (!(dx > eps_zero) || !(dy > eps_zero)) return omega_prev;
  return std::exp(theta * std::log(dy / dx) + (1.0 - theta) * std::log(omega_prev));
}

// --------------------------------------------------------- device problem ---
struct DevLayout {
  DevBuf<int32_t> start32;
  DevBuf<int64_t> start64;
  DevBuf<int32_t> index;
  DevBuf<double> value, value_orig;
  DevBuf<int32_t> tile_row0, tile_rows, chunk_row, chunk_len, chunk_pos, chunk_slot;
  DevBuf<int64_t> tile_nnz0, chunk_beg;
  DevBuf<double> chunk_part, line_acc;
  DevBuf<unsigned> chunk_cnt;
  DevBuf<int4> seg_spans, seg_aux;
  DevBuf<int32_t> seg_step0;
  DevBuf<uint32_t> seg_masks;
  pdlpk_csr view{};
};

template <class T>
void upload_list(const std::vector<T>& h, DevBuf<T>& d) {
  d.alloc(h.size());
  // on the allocation stream: pool memory is stream-ordered
  if (!h.empty()) {
    PDLP_CK(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice,
                            g_alloc_stream));
    PDLP_CK(cudaStreamSynchronize(g_alloc_stream));
  }
}

// Perf-mode schedule (spmv.cuh), the analysis phase of the SpMV: lines of
// <= PDLPK_SHORT_MAX entries are packed into tiles of consecutive lines, longer
// lines into warp chunks.  Tiles are staged through the TMA ring
// (<= PDLPK_TILE_ROWS lines, <= PDLPK_TILE_NNZ entries).  PDLP_TILES=direct
// selects direct tiles instead (thread per line, <= 256 lines, no staging);
// on C1's two-entry columns they measured 86 us against 75 us staged, so
// they are opt-in.  O(lines) host pass over the row pointer.
bool direct_tiles(const int64_t* start, int64_t dim) {
  const char* env = std::getenv("PDLP_TILES");
  if (env == nullptr || std::strcmp(env, "direct") != 0) return false;
  for (int64_t r = 0; r < dim; ++r) {  // kernels never mix direct tiles and CTA chunks
    if (start[r + 1] - start[r] > PDLPK_WARP_LINE_MAX) return false;
  }
  return true;
}

// Set around the row layout's upload (Engine::load_parts).
thread_local bool g_interleave_warp_lines = false;
// The row layout of a solve whose warp lines may be interleaved (whether or
// not PDLP_NO_INTERLEAVE turns it off): column passes over it (the dual
// polishing subproblem) take the split form in both cases.
thread_local bool g_col_split_layout = false;

// Distributed-gap counters (pdlp_gap_dist_stats): evaluations, bisection
// rounds, events swept after the search, and -- with PDLP_GAPD_CHECK=1 --
// the largest relative difference from the gathered evaluation.
struct GapDistStats {
  std::mutex mu;
  int64_t evals = 0, rounds = 0, final_events = 0, checked = 0;
  double max_rel = 0.0, max_rel_lambda = 0.0;
};
GapDistStats& gapd_stats() {
  static GapDistStats g;
  return g;
}


// Line segments of a schedule build: [lo, hi) line ranges built by host
// threads (fixed boundaries, so the schedule is deterministic) and joined in
// line order.  A tile never spans a segment boundary.
struct SchedPart {
  std::vector<int32_t> t0, tc, ck_row, ck_len, ck_pos, ck_slot;
  std::vector<int64_t> tn, ck_beg;
  std::vector<int32_t> cc_row, cc_len, cc_pos, cc_slot;
  std::vector<int64_t> cc_beg;
  int64_t n_multi = 0;
  int64_t short_lines = 0, short_nnz = 0;
};

template <class F>
void for_segments(int64_t dim, int parts, F&& f) {
  if (parts <= 1) {
    f(0, 0, dim);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(static_cast<size_t>(parts));
  for (int q = 0; q < parts; ++q) {
    th.emplace_back([&, q] {
      try {
        f(q, dim * q / parts, dim * (q + 1) / parts);
      } catch (...) {
        err[q] = std::current_exception();
      }
    });
  }
  for (auto& t : th) t.join();
  for (auto& e : err) {
    if (e) std::rethrow_exception(e);
  }
}

void build_schedule(const int64_t* start, int64_t dim, DevLayout& L,
                    int64_t short_max = PDLPK_SHORT_MAX, int32_t budget = 0, int32_t staged = -1) {
  if (budget <= 0) budget = pdlpk_stage_budget(PDLPK_TILE_NNZ);
  int parts = static_cast<int>(std::clamp<int64_t>(
      dim / (int64_t(1) << 18), 1, std::max(1u, std::min(16u, std::thread::hardware_concurrency()))));
  if (const char* e = std::getenv("PDLP_SCHED_THREADS")) parts = std::max(1, std::atoi(e));
  std::vector<SchedPart> seg(static_cast<size_t>(parts));
  const bool direct = direct_tiles(start, dim);
  int32_t shape_lines = PDLPK_TILE_ROWS, shape_nnz = PDLPK_TILE_NNZ, stage_bytes = budget;
  if (!direct) {
    for_segments(dim, parts, [&](int q, int64_t lo, int64_t hi) {
      int64_t sl = 0, sn = 0;
      for (int64_t r = lo; r < hi; ++r) {
        const int64_t len = start[r + 1] - start[r];
        if (len <= short_max) {
          ++sl;
          sn += len;
        }
      }
      seg[q].short_lines = sl;
      seg[q].short_nnz = sn;
    });
    int64_t short_lines = 0, short_nnz = 0;
    for (const SchedPart& g : seg) {
      short_lines += g.short_lines;
      short_nnz += g.short_nnz;
    }
    const double avg = short_lines > 0 ? static_cast<double>(short_nnz) / short_lines : 1.0;
    pdlpk_tile_shape(avg, budget, &shape_lines, &shape_nnz, &stage_bytes, staged);
  }
  const int64_t tile_rows = direct ? 256 : shape_lines;
  const int64_t tile_nnz = direct ? 256 * PDLPK_SHORT_MAX : shape_nnz;
  if (direct) short_max = PDLPK_SHORT_MAX;
  // a tiled line must fit one stage on its own (longer ones go to warp lines)
  short_max = std::min<int64_t>(short_max, tile_nnz);
  // Segment boundaries on multiples of the tile's line count (uniform
  // layouts then re-synchronize at once, see the splice below).
  std::vector<int64_t> bnd(static_cast<size_t>(parts) + 1);
  for (int q = 0; q <= parts; ++q) {
    const int64_t raw = dim * q / parts;
    bnd[q] = q == parts ? dim : std::min<int64_t>(dim, raw / tile_rows * tile_rows);
  }
  // open tile of the greedy tiling: lines [r0, r0 + rows) with nnz entries
  struct Open {
    int64_t r0 = -1, rows = 0, nnz = 0;
  };
  std::vector<Open> tail(static_cast<size_t>(parts));
  for_segments(dim, parts, [&](int q, int64_t, int64_t) {
    const int64_t lo = bnd[q], hi = bnd[q + 1];
    SchedPart& g = seg[q];
    Open o;
    auto close = [&] {
      if (o.rows > 0) {
        g.t0.push_back(static_cast<int32_t>(o.r0));
        g.tc.push_back(static_cast<int32_t>(o.rows | (o.nnz << 12)));
        g.tn.push_back(start[o.r0]);
      }
      o = Open{};
    };
    for (int64_t r = lo; r < hi; ++r) {
      const int64_t len = start[r + 1] - start[r];
      if (len > short_max && len <= PDLPK_WARP_LINE_MAX) {
        // a medium line: one warp
        close();
        g.ck_row.push_back(static_cast<int32_t>(r));
        g.ck_beg.push_back(start[r]);
        g.ck_len.push_back(static_cast<int32_t>(len));
        g.ck_pos.push_back(static_cast<int32_t>(1 << 16));
        g.ck_slot.push_back(-1);
        continue;
      }
      if (len > PDLPK_WARP_LINE_MAX) {
        // a long line: consecutive CTA chunks of <= PDLPK_CHUNK entries
        // (multi-chunk slots numbered per segment, offset when joined)
        close();
        int64_t nch = (len + PDLPK_CHUNK - 1) / PDLPK_CHUNK;
        const int64_t per = (len + nch - 1) / nch;  // balanced chunk length
        nch = (len + per - 1) / per;
        if (nch > 0xffff) throw std::runtime_error("line too long for the chunk schedule");
        const int32_t slot = nch > 1 ? static_cast<int32_t>(g.n_multi++) : -1;
        for (int64_t c = 0; c < nch; ++c) {
          const int64_t b = start[r] + c * per;
          g.cc_row.push_back(static_cast<int32_t>(r));
          g.cc_beg.push_back(b);
          g.cc_len.push_back(static_cast<int32_t>(std::min(per, start[r + 1] - b)));
          g.cc_pos.push_back(static_cast<int32_t>(c | (nch << 16)));
          g.cc_slot.push_back(slot);
        }
        continue;
      }
      if (o.rows == tile_rows || o.nnz + len > tile_nnz) close();
      if (o.rows == 0) o.r0 = r;
      ++o.rows;
      o.nnz += len;
    }
    tail[q] = o;  // left open: the next segment may extend it
  });
  // Splice the speculative tilings into exactly the sequential greedy one:
  // the open tile carried out of segment q-1 is extended through segment q
  // until the greedy starts a tile where segment q's own run started one (or
  // a non-tiled line closes both); from there segment q's tiles are exact.
  std::vector<int32_t> t0, tc;
  std::vector<int64_t> tn;
  {
    Open carry;
    auto emit = [&](const Open& o) {
      if (o.rows > 0) {
        t0.push_back(static_cast<int32_t>(o.r0));
        tc.push_back(static_cast<int32_t>(o.rows | (o.nnz << 12)));
        tn.push_back(start[o.r0]);
      }
    };
    for (int q = 0; q < parts; ++q) {
      const SchedPart& g = seg[q];
      const int64_t lo = bnd[q], hi = bnd[q + 1];
      size_t k = 0;  // first speculative tile of segment q not yet replaced
      bool synced = carry.rows == 0;
      for (int64_t r = lo; r < hi && !synced; ++r) {
        const int64_t len = start[r + 1] - start[r];
        if (len > short_max) {  // a chunked line closes the tile in both runs
          emit(carry);
          carry = Open{};
          while (k < g.t0.size() && g.t0[k] <= r) ++k;
          synced = true;
          break;
        }
        if (carry.rows == tile_rows || carry.nnz + len > tile_nnz) {
          emit(carry);
          carry = Open{};
          while (k < g.t0.size() && g.t0[k] < r) ++k;
          if (k < g.t0.size() && g.t0[k] == r) {  // both runs start a tile at r
            synced = true;
            break;
          }
        }
        if (carry.rows == 0) carry.r0 = r;
        ++carry.rows;
        carry.nnz += len;
      }
      if (!synced) continue;  // the carry spans the whole segment
      for (; k < g.t0.size(); ++k) {
        t0.push_back(g.t0[k]);
        tc.push_back(g.tc[k]);
        tn.push_back(g.tn[k]);
      }
      carry = tail[q];
    }
    emit(carry);
  }
  // join in line order: warp chunks, then every CTA chunk
  std::vector<int32_t> ck_row, ck_len, ck_pos, ck_slot;
  std::vector<int64_t> ck_beg;
  std::vector<int32_t> cc_row, cc_len, cc_pos, cc_slot;
  std::vector<int64_t> cc_beg;
  int64_t n_multi = 0;
  auto append = [](auto& dst, const auto& src) { dst.insert(dst.end(), src.begin(), src.end()); };
  for (SchedPart& g : seg) {
    append(ck_row, g.ck_row);
    append(ck_beg, g.ck_beg);
    append(ck_len, g.ck_len);
    append(ck_pos, g.ck_pos);
    append(ck_slot, g.ck_slot);
    append(cc_row, g.cc_row);
    append(cc_beg, g.cc_beg);
    append(cc_len, g.cc_len);
    append(cc_pos, g.cc_pos);
    for (int32_t sl : g.cc_slot) cc_slot.push_back(sl < 0 ? sl : static_cast<int32_t>(sl + n_multi));
    n_multi += g.n_multi;
  }
  if (g_interleave_warp_lines && ck_row.size() > 1) {
    // warp lines in the order 0, h, 1, h+1, ... (h = half): a layout whose
    // slow lines cluster (C1's strided demand rows) spreads them over the
    // CTAs and SMs.  Only for the row layout when the row pass writes
    // per-line partials (step_args().line_partials): the step's reductions
    // then do not depend on the order, so neither do the iterates.
    const size_t nw = ck_row.size(), h = (nw + 1) / 2;
    auto perm = [&](auto& v) {
      auto w = v;
      for (size_t c = 0; c < nw; ++c) v[c] = w[(c & 1) ? h + c / 2 : c / 2];
    };
    if (nw % 2 == 0) {
      perm(ck_row);
      perm(ck_beg);
      perm(ck_len);
      perm(ck_pos);
      perm(ck_slot);
    }
  }
  const int64_t n_cta_chunks = static_cast<int64_t>(cc_row.size());
  ck_row.insert(ck_row.end(), cc_row.begin(), cc_row.end());
  ck_beg.insert(ck_beg.end(), cc_beg.begin(), cc_beg.end());
  ck_len.insert(ck_len.end(), cc_len.begin(), cc_len.end());
  ck_pos.insert(ck_pos.end(), cc_pos.begin(), cc_pos.end());
  ck_slot.insert(ck_slot.end(), cc_slot.begin(), cc_slot.end());
  upload_list(t0, L.tile_row0);
  upload_list(tc, L.tile_rows);
  upload_list(tn, L.tile_nnz0);
  upload_list(ck_row, L.chunk_row);
  upload_list(ck_beg, L.chunk_beg);
  upload_list(ck_len, L.chunk_len);
  upload_list(ck_pos, L.chunk_pos);
  upload_list(ck_slot, L.chunk_slot);
  const int64_t n_chunks = static_cast<int64_t>(ck_row.size());
  L.chunk_part.alloc(n_chunks);
  L.chunk_cnt.alloc(n_chunks);
  if (n_chunks > 0) {
    PDLP_CK(cudaMemsetAsync(L.chunk_cnt.get(), 0, n_chunks * sizeof(unsigned), g_alloc_stream));
  }
  L.line_acc.alloc(n_multi * PDLPK_LINE_ACC);
  const int64_t n_tiles = static_cast<int64_t>(t0.size());
  // ~41 KB staging ring per CTA -> 5 CTAs per SM; each CTA walks its tiles
  // grid-stride with a kStages-deep bulk-copy prefetch.
  // staged tiles: exactly the resident CTAs (one wave, each walks its tiles
  // grid-stride); direct tiles have no ring and run 4 waves of 5 per SM
  int64_t tb = n_tiles;
  tb = std::min<int64_t>(tb, direct ? 148 * 5 * 4 : pdlpk_tile_resident_ctas(stage_bytes));
  tb = std::max<int64_t>(tb, 1);  // the column pass's last CTA decides, so never empty
  L.view.chunk_row = L.chunk_row.get();
  L.view.chunk_beg = L.chunk_beg.get();
  L.view.chunk_len = L.chunk_len.get();
  L.view.chunk_pos = L.chunk_pos.get();
  L.view.chunk_slot = L.chunk_slot.get();
  L.view.n_chunks = n_chunks;
  L.view.n_cta_chunks = n_cta_chunks;
  L.view.n_multi = n_multi;
  L.view.chunk_part = L.chunk_part.get();
  L.view.chunk_cnt = L.chunk_cnt.get();
  L.view.line_acc = L.line_acc.get();
  L.view.tile_row0 = L.tile_row0.get();
  L.view.tile_rows = L.tile_rows.get();
  L.view.tile_nnz0 = L.tile_nnz0.get();
  L.view.n_tiles = n_tiles;
  L.view.tile_direct = direct ? 1 : 0;
  L.view.seg_mode = 0;
  L.view.col_split = g_col_split_layout ? 1 : 0;
  L.view.tile_lines_cap = static_cast<int32_t>(tile_rows);
  L.view.tile_nnz_cap = static_cast<int32_t>(tile_nnz);
  L.view.tile_stage_bytes = stage_bytes;
  L.view.tile_blocks = static_cast<int32_t>(tb);
}

// Tile line threshold per layout.  Which lines are cheaper in staged tiles
// than one warp each depends on the whole length distribution (C2's ~33-entry
// rows: 64 is best, 3.5 vs 4.0 ms at 256; its power-law columns: 256 is best,
// 2.8 vs 3.5 ms at 64), so a large layout times one product per candidate at
// setup and keeps the fastest; small layouts use 64.
// PDLP_SHORT_MAX=<n> forces a threshold.
// start[0] == 0, non-decreasing, start[dim] == nnz (what the schedule build
// relies on; the device validation reports the reference's message).
bool starts_valid(const int64_t* start, int64_t dim, int64_t nnz) {
  if (start[0] != 0 || start[dim] != nnz) return false;
  const int parts = static_cast<int>(std::clamp<int64_t>(dim / (int64_t(1) << 18), 1, 16));
  std::vector<uint8_t> ok(static_cast<size_t>(parts), 1);
  for_segments(dim, parts, [&](int q, int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      if (start[r + 1] < start[r]) {
        ok[q] = 0;
        return;
      }
    }
  });
  return std::all_of(ok.begin(), ok.end(), [](uint8_t v) { return v != 0; });
}

// Segmented-span schedule (spmv.cuh seg_spans): runs of whole lines of at
// most `span` entries, longer lines cut into chunks, empty lines as empty
// chunks; per 256-entry step of a run, 8 line-start and 8 line-end words.
void build_seg_schedule(const int64_t* start, int64_t dim, DevLayout& L, int64_t span) {
  std::vector<int4> spans, aux;
  std::vector<int32_t> step0;
  int64_t parts = 0, n_multi = 0, steps = 0;
  int64_t r0 = -1, nl = 0, nz = 0;
  auto push = [&](int64_t r, int64_t y, int64_t e0, int64_t len, int32_t ax, int32_t ay, int32_t az) {
    spans.push_back(make_int4(static_cast<int32_t>(r), static_cast<int32_t>(y),
                              static_cast<int32_t>(static_cast<uint32_t>(e0 & 0xffffffff)),
                              static_cast<int32_t>(len)));
    aux.push_back(make_int4(ax, ay, az, static_cast<int32_t>(e0 >> 32)));
    if (y > 0) {
      step0.push_back(static_cast<int32_t>(steps));
      steps += (e0 + len - (e0 & ~int64_t(7)) + 255) / 256;
    } else {
      step0.push_back(0);
    }
  };
  auto close = [&] {
    if (nl > 0) push(r0, nl, start[r0], nz, 0, 0, -1);
    nl = 0;
    nz = 0;
  };
  for (int64_t r = 0; r < dim; ++r) {
    const int64_t len = start[r + 1] - start[r];
    if (len == 0) {  // the epilogue still runs (sum 0)
      close();
      push(r, -1, start[r], 0, 0, 1, -1);
      continue;
    }
    if (len > span) {
      close();
      const int64_t nch = (len + span - 1) / span;
      const int32_t ms = static_cast<int32_t>(n_multi++);
      for (int64_t c = 0; c < nch; ++c) {
        const int64_t b = start[r] + c * span;
        push(r, -1 - c, b, std::min(span, start[r + 1] - b), static_cast<int32_t>(parts),
             static_cast<int32_t>(nch), ms);
      }
      parts += nch;
      continue;
    }
    if (nz + len > span || nl >= (int64_t(1) << 30)) close();
    if (nl == 0) r0 = r;
    ++nl;
    nz += len;
  }
  close();
  std::vector<uint32_t> masks(static_cast<size_t>(steps) * 16 + 16, 0u);
  // spans own disjoint step ranges of the mask array: threads over spans
  const int64_t nsp = static_cast<int64_t>(spans.size());
  for_segments(nsp, static_cast<int>(std::clamp<int64_t>(nsp / 4096, 1, 16)),
               [&](int, int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      const int4 d = spans[static_cast<size_t>(i)];
      if (d.y <= 0) continue;
      const int64_t e0 = static_cast<int64_t>(static_cast<uint32_t>(d.z)) |
                         (static_cast<int64_t>(aux[static_cast<size_t>(i)].w) << 32);
      const int64_t b0 = e0 & ~int64_t(7);
      const int64_t s0 = step0[static_cast<size_t>(i)];
      for (int64_t r = d.x; r < static_cast<int64_t>(d.x) + d.y; ++r) {
        const int64_t oh = start[r] - b0, oe = start[r + 1] - 1 - b0;
        masks[static_cast<size_t>((s0 + oh / 256) * 16 + (oh % 256) / 32)] |= 1u << (oh % 32);
        masks[static_cast<size_t>((s0 + oe / 256) * 16 + 8 + (oe % 256) / 32)] |= 1u << (oe % 32);
      }
    }
  });
  upload_list(spans, L.seg_spans);
  upload_list(aux, L.seg_aux);
  upload_list(step0, L.seg_step0);
  upload_list(masks, L.seg_masks);
  L.chunk_part.alloc(parts);
  L.chunk_cnt.alloc(parts);
  if (parts > 0) {
    PDLP_CK(cudaMemsetAsync(L.chunk_cnt.get(), 0, parts * sizeof(unsigned), g_alloc_stream));
    PDLP_CK(cudaStreamSynchronize(g_alloc_stream));
  }
  L.line_acc.alloc(n_multi * PDLPK_LINE_ACC);
  L.view.seg_mode = 1;
  L.view.seg_spans = L.seg_spans.get();
  L.view.seg_aux = L.seg_aux.get();
  L.view.seg_step0 = L.seg_step0.get();
  L.view.seg_masks = L.seg_masks.get();
  L.view.n_seg_spans = static_cast<int64_t>(spans.size());
  L.view.n_chunks = parts;  // partial slots (sizes the side stream's scratch)
  L.view.n_cta_chunks = 0;
  L.view.n_multi = n_multi;
  L.view.chunk_part = L.chunk_part.get();
  L.view.chunk_cnt = L.chunk_cnt.get();
  L.view.line_acc = L.line_acc.get();
  L.view.n_tiles = 0;
  L.view.tile_direct = 0;
  L.view.tile_blocks = static_cast<int32_t>(std::max<int64_t>(1, pdlpk_seg_resident_ctas()));
}

// Schedule choice per layout, a function of the line lengths only (so the
// perf-mode iterates do not depend on timing noise):
//  * skewed layouts of >= 16M entries (a tenth of the entries in lines over
//    256, or a line 16x the mean): segmented spans of 2,048 entries;
//  * otherwise staged tiles of lines <= 64 entries (<= 256 when a third of
//    the entries sit in longer lines), a 2,016-entry stage budget for
//    layouts of >= 16M entries.
// PDLP_SEG=0/1 and PDLP_SHORT_MAX=<n> override (measurements).
int64_t autotune_schedule(const int64_t* start, int64_t dim, int64_t /*operand_len*/, DevLayout& L,
                          cudaStream_t /*s*/, const unsigned* /*bad*/) {
  if (!starts_valid(start, dim, L.view.nnz)) {
    build_schedule(start, 0, L, PDLPK_SHORT_MAX);  // empty: validation throws before use
    return PDLPK_SHORT_MAX;
  }
  const int64_t nnz = L.view.nnz;
  int64_t over64 = 0, over256 = 0, maxlen = 0, empty = 0;
  for (int64_t r = 0; r < dim; ++r) {
    const int64_t len = start[r + 1] - start[r];
    if (len > 64) over64 += len;
    if (len > 256) over256 += len;
    if (len == 0) ++empty;
    maxlen = std::max(maxlen, len);
  }
  // a heavy tail (lines beyond a warp line's 2,048 entries and a tenth of the
  // entries in lines > 256: C2's power-law columns), and few empty lines
  // (each is a span of its own).  Bimodal layouts such as C3's rows (2 and
  // 1,000 entries) stay on tiles + warp lines.
  bool seg = nnz >= (int64_t(16) << 20) && !L.view.tile_direct && maxlen > PDLPK_WARP_LINE_MAX &&
             10 * over256 >= nnz && 100 * empty < dim;
  if (const char* e = std::getenv("PDLP_SEG")) seg = e[0] == '1';
  if (seg) {
    const char* es = std::getenv("PDLP_SEG_SPAN");
    build_seg_schedule(start, dim, L, es != nullptr && std::atoi(es) >= 64 ? std::atoi(es) : 2048);
    return -1;
  }
  const char* env = std::getenv("PDLP_SHORT_MAX");
  if (env != nullptr && std::atoi(env) > 0) {
    const int64_t t = std::atoi(env);
    build_schedule(start, dim, L, t);
    return t;
  }
  const int64_t t = 3 * over64 >= nnz ? 256 : 64;
  // stage budget: the C1 sweep's 896-entry default for very short lines
  // (C1's 2-entry columns, C3's 2-4-entry rows and columns); 2,016 entries
  // for large layouts of longer short lines (C2's ~33-entry rows)
  int64_t short_lines = 0, short_nnz = 0;
  for (int64_t r = 0; r < dim; ++r) {
    const int64_t len = start[r + 1] - start[r];
    if (len <= t) {
      ++short_lines;
      short_nnz += len;
    }
  }
  int32_t budget = (nnz >= (int64_t(16) << 20) && short_nnz >= 16 * short_lines)
                       ? pdlpk_stage_budget(2016) : 0;
  if (const char* eb = std::getenv("PDLP_STAGE_BUDGET")) budget = pdlpk_stage_budget(std::atoi(eb));
  build_schedule(start, dim, L, t, budget);
  return t;
}

// Uploads one orientation; the raw int64 row pointers and indices are checked
// on device before the int32 conversion (bad: device flag word, see
// k_valid.cu).  bound = the secondary dimension.
// A process-wide stream per device for schedule uploads built off the main
// thread (never destroyed: the schedule buffers free on it).
cudaStream_t schedule_stream() {
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  int dev = 0;
  PDLP_CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  cudaStream_t& st = streams[dev];
  if (st == nullptr) PDLP_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  return st;
}

void upload_layout(const pdlp_csr_view& v, int64_t bound, unsigned* bad, DevLayout& L,
                   cudaStream_t s) {
  const int64_t dim = v.primary_dim, nnz = v.nnz;
  const bool wide = nnz >= (int64_t(1) << 31) - 1;
  L.view.dim = dim;
  L.view.nnz = nnz;
  L.view.wide = wide ? 1 : 0;
  // The schedule (a host pass over the line starts plus small uploads) is
  // built on a second host thread while this one stages the layout's arrays.
  const auto ts = std::chrono::steady_clock::now();
  std::exception_ptr sched_err;
  int dev = 0;
  PDLP_CK(cudaGetDevice(&dev));
  const bool interleave = g_interleave_warp_lines, col_split = g_col_split_layout;
  const cudaStream_t ss = schedule_stream();
  std::thread sched([&, dev, interleave, col_split, ss] {
    try {
      PDLP_CK(cudaSetDevice(dev));
      AllocStreamScope scope(ss);
      g_interleave_warp_lines = interleave;
      g_col_split_layout = col_split;
      autotune_schedule(v.start, dim, bound, L, ss, bad);
      PDLP_CK(cudaStreamSynchronize(ss));
    } catch (...) {
      sched_err = std::current_exception();
    }
  });
  struct JoinOnExit {
    std::thread& t;
    ~JoinOnExit() {
      if (t.joinable()) t.join();
    }
  } join_guard{sched};
  // start: 64-bit for wide layouts, else narrowed to 32 bits on the host
  // (saturating, so the range checks below still see a bad value)
  if (wide) {
    L.start64.alloc(dim + 1);
    stage_h2d(L.start64.get(), v.start, (dim + 1) * 8, s);
    PDLP_LAUNCH(pdlpk_validate_raw_layout(L.start64.get(), dim, nullptr, 0, nnz, bound, bad, s));
  } else {
    L.start32.alloc(dim + 1);
    stage_h2d_narrow(L.start32.get(), v.start, static_cast<size_t>(dim + 1), s);
    PDLP_LAUNCH(pdlpk_validate_raw_layout32(L.start32.get(), dim, nullptr, 0, nnz, bound, bad, s));
  }
  // index: always 32 bits on device (bound < 2^31)
  L.index.alloc(nnz);
  if (nnz > 0) {
    stage_h2d_narrow(L.index.get(), v.index, static_cast<size_t>(nnz), s);
    PDLP_LAUNCH(pdlpk_validate_raw_layout32(nullptr, 0, L.index.get(), nnz, nnz, bound, bad, s));
  }
  L.value_orig.alloc(nnz);
  L.value.alloc(nnz);
  if (nnz > 0) {
    stage_h2d(L.value_orig.get(), v.value, nnz * 8, s);
    PDLP_CK(cudaMemcpyAsync(L.value.get(), L.value_orig.get(), nnz * 8, cudaMemcpyDeviceToDevice, s));
  }
  sched.join();
  if (sched_err) std::rethrow_exception(sched_err);
  L.view.start = wide ? static_cast<const void*>(L.start64.get())
                      : static_cast<const void*>(L.start32.get());
  L.view.index = L.index.get();
  L.view.value = L.value.get();
  L.view.value_orig = L.value_orig.get();
  if (std::getenv("PDLP_TIMING") != nullptr) {
    PDLP_CK(cudaStreamSynchronize(s));
    std::fprintf(stderr, "phase=setup event=layout lines=%lld nnz=%lld seconds=%.4f\n",
                 static_cast<long long>(dim), static_cast<long long>(nnz),
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count());
  }
}

DevBuf<double> upload_vec(const double* h, int64_t n, cudaStream_t s) {
  DevBuf<double> d(n);
  if (n > 0) stage_h2d(d.get(), h, n * 8, s);
  return d;
}

DevBuf<double> dev_fill(int64_t n, double v, cudaStream_t s) {
  DevBuf<double> d(n);
  PDLP_LAUNCH(pdlpk_fill(d.get(), v, n, s));
  return d;
}

void dev_copy(double* dst, const double* src, int64_t n, cudaStream_t s) {
  if (n > 0) PDLP_CK(cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToDevice, s));
}

void dev_zero(double* dst, int64_t n, cudaStream_t s) {
  if (n > 0) PDLP_CK(cudaMemsetAsync(dst, 0, n * 8, s));
}

struct DevProblem {
  int64_t m = 0, n = 0;
  DevLayout row, col;
  DevBuf<double> c, lc, uc, lv, uv;            // scaled (in place)
  DevBuf<double> c_o, lc_o, uc_o, lv_o, uv_o;  // original
  DevBuf<double> row_scale, col_scale;

  uint32_t uniform = 0;  // pdlpk_problem::uniform of the scaled c, l_v, u_v
  double c_u = 0.0, lv_u = 0.0, uv_u = 0.0;
  pdlpk_problem view() const {
    pdlpk_problem P{};
    P.m = m;
    P.n = n;
    P.uniform = uniform;
    P.c_u = c_u;
    P.lv_u = lv_u;
    P.uv_u = uv_u;
    P.K = row.view;
    P.KT = col.view;
    P.c = c.get();
    P.lc = lc.get();
    P.uc = uc.get();
    P.lv = lv.get();
    P.uv = uv.get();
    P.c_o = c_o.get();
    P.lc_o = lc_o.get();
    P.uc_o = uc_o.get();
    P.lv_o = lv_o.get();
    P.uv_o = uv_o.get();
    P.row_scale = row_scale.get();
    P.col_scale = col_scale.get();
    return P;
  }
};

// Problem validation (problem.hpp:119-154, sparse.hpp:118-133) runs on device
// inside Engine::load (k_valid.cu); the host never walks the matrix.
[[noreturn]] void invalid(const char* msg, int64_t idx) {
  throw InvalidProblem(std::string("invalid problem: ") + msg + " (index " + std::to_string(idx) + ")");
}

// ------------------------------------------------------------ inner state ---
struct Cert {
  bool have = false;
  int kind = 0;
  DevBuf<double> ray_x, ray_y, ray_r;
  double residual = kInf, objective = 0.0;
  std::string source;
};

struct Inner {  // InnerState (solver.hpp:135-193), vectors on device
  int64_t n = 0, m = 0;
  DevBuf<double> x[2], y[2], aty[2];
  DevBuf<double> xbar, dy, aty_diff, sum_x, sum_y;
  DevBuf<double> ref_x, ref_y, ax_cur, avg_x, avg_y, ax_avg, aty_avg, diff_x, diff_y, rc_a, rc_b;
  DevBuf<double> sol_x, sol_y, sol_r, tmp_x, tmp_y, tmp_r, ray_n, ray_m, prod_n, prod_m;
  DevBuf<double> ray_y[3], rhat[3];  // per ray candidate (batched cadence)
  DevBuf<pdlpk_step_state> state;
  DevBuf<double> part2, part3, shard_part;
  DevBuf<double> pbuf, dloc, tot_all;  // sharded attempts (partial product, RS output, totals)
  pdlpk_step_state hs{};  // host mirror of the controller

  // Host scalars of InnerState
  double omega = 1.0;
  double last_eta = 0.0;
  double mu_last = kInf, prev_candidate_mu = kInf;
  int64_t k_last_restart = 0, restarts = 0;
  int64_t next_polish_trigger = 100, polish_iterations = 0;
  Summary sol_summary;
  bool have_sol = false;
  std::string detail;
  Cert cert;

  // full > 0 (sharded): x-bar and dy double as the gathered column-side
  // buffers of `full` entries; block = the column block, world = ranks.
  void allocate(int64_t cols, int64_t rows, int64_t partials, int shards, int64_t full = 0,
                int64_t block = 0, int world = 1) {
    n = cols;
    m = rows;
    for (int b = 0; b < 2; ++b) {
      x[b].alloc(n);
      y[b].alloc(m);
      aty[b].alloc(n);
    }
    for (DevBuf<double>* v : {&xbar, &aty_diff, &sum_x, &ref_x, &avg_x, &aty_avg, &diff_x, &rc_a,
                              &rc_b, &sol_x, &sol_r, &tmp_x, &tmp_r, &ray_n, &prod_n}) {
      v->alloc(n);
    }
    for (DevBuf<double>* v :
         {&dy, &sum_y, &ref_y, &ax_cur, &avg_y, &ax_avg, &diff_y, &sol_y, &tmp_y, &ray_m, &prod_m}) {
      v->alloc(m);
    }
    for (int q = 0; q < 3; ++q) {
      ray_y[q].alloc(m);
      rhat[q].alloc(n);
    }
    cert.ray_x.alloc(n);
    cert.ray_y.alloc(m);
    cert.ray_r.alloc(n);
    state.alloc(1);
    part2.alloc(partials);
    part3.alloc(partials);
    shard_part.alloc(5 * std::max(shards, 1));
    if (full > 0) {
      xbar.alloc(std::max(n, full));
      dy.alloc(std::max(m, full));
      pbuf.alloc(full);
      dloc.alloc(std::max<int64_t>(block, 1));
      tot_all.alloc(8 * static_cast<int64_t>(world));
      PDLP_CK(cudaMemsetAsync(pbuf.get(), 0, full * sizeof(double), g_alloc_stream));
    }
  }
  int cur() const { return hs.cur; }
  int64_t k() const { return hs.k; }
  // k at which the cadence last computed ax_cur = K x[cur] and aty[cur] =
  // K' y[cur] afresh (-1: not current)
  int64_t fresh_products_k = -1;
};

struct InnerCfg {  // InnerConfig (solver.hpp:114-133)
  Tol tol;
  bool feasibility_only = false;
  int rc_mode = 0;  // 0 Natural, 1 BoundRobust
  int64_t budget = 0;
  Clock::time_point deadline = Clock::time_point::max();
  bool enable_restarts = true;
  bool detect_infeasibility = true;
  bool enable_polish = false;
  double eps_ray = 1e-12;
  int64_t check_interval = 64;
  Thresholds th;
  std::optional<double> fixed_eta;
  bool allow_omega_updates = true;
  pdlp_observer_fn observer = nullptr;
  void* observer_user = nullptr;
  bool logging = false;
  const char* tag = "main";
  // sharded solves: the whole-problem view the gap runs on, and whether the
  // problem is the swapped (dual polishing) one
  const pdlpk_problem* full = nullptr;
  bool swapped = false;
};

// Pinned host words the cadence reads back, one set per host thread and kept
// for its lifetime: a cudaMallocHost / cudaFreeHost pair per solve costs up
// to tens of milliseconds of driver time (cudaFreeHost synchronizes).
struct PinnedScratch {
  double* slots = nullptr;  // 64
  int* islots = nullptr;    // 8
  PinnedScratch() {
    PDLP_CK(cudaMallocHost(&slots, 64 * sizeof(double)));
    PDLP_CK(cudaMallocHost(&islots, 8 * sizeof(int)));
  }
  ~PinnedScratch() {
    cudaFreeHost(slots);
    cudaFreeHost(islots);
  }
};

PinnedScratch& pinned_scratch() {
  thread_local PinnedScratch p;
  return p;
}

// ------------------------------------------------------------------ engine ---
class Engine {
 public:
  // comm != nullptr: one rank of a row-sharded solve; this
  // engine then holds rows [r0,r1) of A in both layouts and the column
  // block [c0,c1), and every product / reduction crosses ranks.
  // shard != nullptr (with comm): this rank's shard as the caller built it
  // (shard-local ingest, pdlp_solve_sharded_local); p is then unused.
  Engine(const pdlp_problem_view* p, const pdlp_options& o, Comm* comm = nullptr,
         const pdlp_shard_view* shard = nullptr)
      : opt_(o), comm_(comm), shard_in_(shard) {
    parity_ = o.mode == PDLP_MODE_PARITY;
    shards_ = std::max(1, o.threads) * std::max(1, o.shards_per_thread);
    PDLP_CK(cudaSetDevice(o.device));
    stream_ = std::make_unique<Stream>();
    retain_pool_memory(o.device);
    alloc_scope_ = std::make_unique<AllocStreamScope>(stream_->get());
    if (comm_ != nullptr) {
      red_log_.count = 0;
      pdlpk_set_red_log(&red_log_);
    }
    load(p);
  }

  cudaStream_t s() const { return stream_->get(); }
  const DevProblem& problem() const { return prob_; }
  bool parity() const { return parity_; }

  // ---- setup -------------------------------------------------------------
  void load(const pdlp_problem_view* p) {
    NvtxRange nvtx("pdlp:upload");
    const auto t0 = Clock::now();
    if (comm_ == nullptr) {
      m_glob_ = p->rows;
      n_glob_ = p->cols;
      if (m_glob_ < 0 || n_glob_ < 0 || p->by_row.primary_dim != m_glob_ ||
          p->by_col.primary_dim != n_glob_ || p->by_row.nnz != p->by_col.nnz || p->by_row.nnz < 0) {
        invalid("row/column layouts disagree", -1);
      }
      load_parts(p->by_row, p->by_col, p->rows, p->cols, p->objective, p->con_lower,
                 p->con_upper, p->var_lower, p->var_upper, 0, 0, 0);
    } else {
      // Every rank sees the whole problem, so structural errors throw on
      // every rank alike before any collective.  (Shard-local ingest: each
      // rank passes its own shard; the plan was checked against
      // pdlp_shard_plan_for by the entry point.)
      ShardData sh;
      if (shard_in_ == nullptr) {
        extract_shard(*p, comm_->rank(), comm_->world(), auto_cut(p->rows, p->cols), sh);
      }
      const pdlp_shard_view& v = shard_in_ != nullptr ? *shard_in_ : sh.view;
      flag_.alloc(8);
      plan_ = v.plan;
      m_glob_ = plan_.rows;
      n_glob_ = plan_.cols;
      shard_rows_ = &v.rows;
      shard_row_entry_offset_ = v.row_entry_offset;
      load_parts(v.rows, v.cols, plan_.row_end - plan_.row_begin, plan_.col_end - plan_.col_begin,
                 v.objective, v.con_lower, v.con_upper, v.var_lower, v.var_upper, plan_.row_begin,
                 plan_.col_begin, v.entry_offset);
      shard_rows_ = nullptr;
      // the row cut gathers x-bar (K_g) and reduce-scatters K_g^T's partial
      // output; the column cut reduce-scatters K_g's partial row sums and
      // gathers dy (K_g^T)
      prob_.row.view.dist_kind = cols_cut() ? PDLPK_DIST_PARTIAL : PDLPK_DIST_GATHER;
      prob_.col.view.dist_kind = cols_cut() ? PDLPK_DIST_GATHER : PDLPK_DIST_PARTIAL;
      gbuf_.alloc(xch_full());
      pbuf_.alloc(xch_full());
      dev_zero(gbuf_.get(), xch_full(), s());
      dev_zero(pbuf_.get(), xch_full(), s());
      const char* pe = std::getenv("PDLP_PEER_RS");
      const int w = comm_->world();
      if (w > 1 && w <= PDLPK_MAX_PEERS && !(pe != nullptr && pe[0] == '0')) {
        peer_pbuf_ = comm_->alloc_peer_buffer(static_cast<size_t>(xch_full()));
        peer_gather_ = comm_->alloc_peer_buffer(static_cast<size_t>(xch_full()));
        dev_zero(peer_pbuf_, xch_full(), s());
        dev_zero(peer_gather_, xch_full(), s());
        const std::vector<double*> ptrs = comm_->peer_pointers(peer_pbuf_, s());
        const std::vector<double*> gptrs = comm_->peer_pointers(peer_gather_, s());
        // every rank must take the same path: fall back together if any
        // rank could not map its peers
        if (any_rank(ptrs.empty() || gptrs.empty())) {
          PDLP_CK(cudaStreamSynchronize(s()));
          comm_->free_peer_buffer(peer_pbuf_);
          comm_->free_peer_buffer(peer_gather_);
          peer_pbuf_ = peer_gather_ = nullptr;
          if (opt_.logging && comm_->rank() == 0) {
            std::fprintf(stderr, "phase=setup event=peer_exchange_unavailable fallback=nccl\n");
          }
        } else {
          const int rank = comm_->rank();
          peers_.world = push_.world = w;
          peers_.offset = push_.offset = xch_block() * rank;
          for (int r = 0; r < w; ++r) {
            peers_.p[r] = ptrs[r];
            push_.p[r] = r == rank ? nullptr : gptrs[r];
          }
          if (opt_.logging && rank == 0) {
            std::fprintf(stderr, "phase=setup event=peer_exchange world=%d\n", w);
          }
        }
      }
      slots_all_.alloc(static_cast<size_t>(kSlots) * comm_->world());
      PDLP_CK(cudaStreamSynchronize(s()));
    }
    upload_seconds_ = std::chrono::duration<double>(Clock::now() - t0).count();
  }

  // Uploads and validates the engine's part: m rows, n columns of the primal
  // block; the row layout's entries index n_glob_ columns and the column
  // layout has n_glob_ lines.  r0 / c0 / e0 shift reported indices to the
  // whole problem's numbering.
  void load_parts(const pdlp_csr_view& by_row, const pdlp_csr_view& by_col, int64_t m, int64_t n,
                  const double* objective, const double* con_lower, const double* con_upper,
                  const double* var_lower, const double* var_upper, int64_t r0, int64_t c0,
                  int64_t e0) {
    prob_.m = m;
    prob_.n = n;
    static const bool timing = std::getenv("PDLP_TIMING") != nullptr;
    auto lap = [&, t = Clock::now()]() mutable {
      if (timing) PDLP_CK(cudaStreamSynchronize(s()));
      const auto now = Clock::now();
      const double d = std::chrono::duration<double>(now - t).count();
      t = now;
      return d;
    };
    DevBuf<unsigned long long> keys(4);
    DevBuf<unsigned> bad(1);
    PDLP_CK(cudaMemsetAsync(bad.get(), 0, sizeof(unsigned), s()));
    {
      const char* e = std::getenv("PDLP_NO_INTERLEAVE");
      g_col_split_layout = comm_ == nullptr && m <= PDLPK_LINE_PARTIALS_MAX && line_partials_on_;
      g_interleave_warp_lines = g_col_split_layout && !(e != nullptr && e[0] == '1');
    }
    // index bounds: the row layout indexes columns (all n, or the block's
    // under the column cut), the column layout rows (the block's under the
    // row cut, all m under the column cut)
    const bool cc = comm_ != nullptr && cols_cut();
    upload_layout(by_row, cc ? n : n_glob_, bad.get(), prob_.row, s());
    g_interleave_warp_lines = false;
    g_col_split_layout = false;
    // the multi-product span schedule of the row layout: built on a second
    // host thread while the column layout uploads
    std::exception_ptr multi_err;
    std::thread multi_thread([&, dev = opt_.device] {
      try {
        PDLP_CK(cudaSetDevice(dev));
        AllocStreamScope scope(schedule_stream());
        build_multi_row(by_row);
        PDLP_CK(cudaStreamSynchronize(schedule_stream()));
      } catch (...) {
        multi_err = std::current_exception();
      }
    });
    struct JoinOnExit {
      std::thread& t;
      ~JoinOnExit() {
        if (t.joinable()) t.join();
      }
    } multi_guard{multi_thread};
    start_panel_plan(by_row, n_glob_);
    const double t_row = lap();
    upload_layout(by_col, cc ? m_glob_ : m, bad.get(), prob_.col, s());
    multi_thread.join();
    if (multi_err) std::rethrow_exception(multi_err);
    const double t_col = lap();
    prob_.c_o = upload_vec(objective, n, s());
    prob_.lc_o = upload_vec(con_lower, m, s());
    prob_.uc_o = upload_vec(con_upper, m, s());
    prob_.lv_o = upload_vec(var_lower, n, s());
    prob_.uv_o = upload_vec(var_upper, n, s());
    const double t_vec = lap();
    // validate (problem.hpp:119-154) on device, first failure in the
    // reference's order; layouts_consistent last.
    PDLP_LAUNCH(pdlpk_validate_vectors(prob_.c_o.get(), prob_.lv_o.get(), prob_.uv_o.get(), n,
                                       prob_.lc_o.get(), prob_.uc_o.get(), m,
                                       prob_.row.value_orig.get(), prob_.row.view.nnz, keys.get(), s()));
    {
      unsigned long long hk[4];
      unsigned hb = 0;
      PDLP_CK(cudaMemcpyAsync(hk, keys.get(), sizeof(hk), cudaMemcpyDeviceToHost, s()));
      PDLP_CK(cudaMemcpyAsync(&hb, bad.get(), sizeof(hb), cudaMemcpyDeviceToHost, s()));
      PDLP_CK(cudaStreamSynchronize(s()));
      if (comm_ != nullptr) {
        if (cc && hk[3] != ~0ull) hk[3] = col_cut_entry(hk[3]);
        combine_validation(hk, hb, r0, c0, cc ? 0 : e0);
      }
      static const char* var_msg[] = {"", "variable bound is NaN", "variable lower bound is +inf",
                                      "variable upper bound is -inf", "variable bounds crossed"};
      static const char* con_msg[] = {"", "constraint bound is NaN",
                                      "constraint lower bound is +inf",
                                      "constraint upper bound is -inf", "constraint bounds crossed"};
      const unsigned long long none = ~0ull;
      if (hk[0] != none) invalid("objective entry not finite", static_cast<int64_t>(hk[0] >> 3));
      if (hk[1] != none) invalid(var_msg[hk[1] & 7], static_cast<int64_t>(hk[1] >> 3));
      if (hk[2] != none) invalid(con_msg[hk[2] & 7], static_cast<int64_t>(hk[2] >> 3));
      if (hk[3] != none) invalid("matrix entry not finite", static_cast<int64_t>(hk[3] >> 3));
      if (hb != 0) invalid("row/column layouts disagree", -1);
    }
    const double t_valid = lap();
    {
      const int64_t nnz = prob_.row.view.nnz;
      row_of_.alloc(nnz);
      col_of_.alloc(nnz);
      const size_t work_bytes = pdlpk_line_of_work_bytes(nnz);
      DevBuf<char> work(work_bytes);
      PDLP_LAUNCH(pdlpk_line_of(&prob_.row.view, row_of_.get(), work.get(), work_bytes, s()));
      PDLP_LAUNCH(pdlpk_line_of(&prob_.col.view, col_of_.get(), work.get(), work_bytes, s()));
      DevBuf<int> row_count(std::max<int64_t>(prob_.row.view.dim, 1));
      PDLP_LAUNCH(pdlpk_validate_consistency(&prob_.row.view, row_of_.get(), &prob_.col.view,
                                             col_of_.get(), row_count.get(), bad.get(), s()));
      unsigned hb = 0;
      PDLP_CK(cudaMemcpyAsync(&hb, bad.get(), sizeof(hb), cudaMemcpyDeviceToHost, s()));
      PDLP_CK(cudaStreamSynchronize(s()));
      if (comm_ != nullptr) hb = any_rank(hb != 0) ? 1u : 0u;
      if (hb != 0) invalid("row/column layouts disagree", -1);
    }
    const double t_cons = lap();
    prob_.c.alloc(n);
    prob_.lc.alloc(m);
    prob_.uc.alloc(m);
    prob_.lv.alloc(n);
    prob_.uv.alloc(n);
    dev_copy(prob_.c.get(), prob_.c_o.get(), n, s());
    dev_copy(prob_.lc.get(), prob_.lc_o.get(), m, s());
    dev_copy(prob_.uc.get(), prob_.uc_o.get(), m, s());
    dev_copy(prob_.lv.get(), prob_.lv_o.get(), n, s());
    dev_copy(prob_.uv.get(), prob_.uv_o.get(), n, s());
    prob_.row_scale = dev_fill(m, 1.0, s());
    prob_.col_scale = dev_fill(n, 1.0, s());
    slots_.alloc(kSlots);
    host_slots_ = pinned_scratch().slots;
    red_scratch_.alloc(std::max<int64_t>(pdlpk_red_scratch_doubles(), 8 * int64_t(shards_) + 64));
    // the gap runs on whole vectors (gathered when sharded)
    // Two buffers let both gap queries of a cadence share one sync; above
    // 1 GB each (C4-shard sizes: 24 GB) one buffer is reused query by query.
    {
      // whole-problem events on one GPU (and for the gathered evaluation);
      // a sharded solve's distributed gap only holds the rank's blocks
      const int64_t gn = gap_whole() ? n_glob_ : n, gm = gap_whole() ? m_glob_ : m;
      const size_t gw = std::max(pdlpk_gap_work_bytes(gn, gm), pdlpk_gap_work_bytes(gm, gn));
      gap_shared_ = gw > (size_t(1) << 30);
      gap_work_[0].alloc(gw);
      if (!gap_shared_) gap_work_[1].alloc(gw);
    }
    islots_.alloc(8);
    host_islots_ = pinned_scratch().islots;
    zeros_n_.alloc(n);
    zeros_m_.alloc(m);
    dev_zero(zeros_n_.get(), n, s());
    dev_zero(zeros_m_.get(), m, s());
    PDLP_CK(cudaStreamSynchronize(s()));
    if (timing) {
      double sw = 0.0, sc = 0.0, smb = 0.0;
      stage_report(&sw, &sc, &smb);
      std::fprintf(stderr,
                   "phase=setup event=load row_layout=%.4f col_layout=%.4f vectors=%.4f "
                   "validate=%.4f consistency=%.4f rest=%.4f staged_mb=%.1f slot_wait=%.4f "
                   "host_copy=%.4f\n",
                   t_row, t_col, t_vec, t_valid, t_cons, lap(), smb, sw, sc);
    }
  }

  ~Engine() {
    if (panel_thread_.t.joinable()) panel_thread_.t.join();
    cudaStreamSynchronize(s());  // buffers on other streams (panels) free unordered with s()
    if (comm_ != nullptr) pdlpk_set_red_log(nullptr);
    if (peer_pbuf_ != nullptr) {
      cudaStreamSynchronize(s());
      comm_->free_peer_buffer(peer_pbuf_);
      comm_->free_peer_buffer(peer_gather_);
    }
    alloc_scope_.reset();  // members free on their own allocation stream
    for (cudaEvent_t e : prof_ev_) cudaEventDestroy(e);
  }

  void ensure_prof_events(int64_t attempts) {
    while (static_cast<int64_t>(prof_ev_.size()) < 4 * attempts) {
      cudaEvent_t e;
      PDLP_CK(cudaEventCreate(&e));
      prof_ev_.push_back(e);
    }
  }

  // Timed region of the main loop (bench): opens once k >= warmup.
  void maybe_start_timer(const Inner& D) {
    if (timing_started_ || &D != &main_ || D.k() < timing_warmup_) return;
    timing_started_ = true;
    timed_k0_ = D.k();
    timed_att0_ = D.hs.attempts;
    timed_begin_.record(s());
  }

  pdlpk_red red() const {
    pdlpk_red r{};
    r.order = parity_ ? PDLPK_RED_SEQ : PDLPK_RED_TREE;
    r.shards = shards_;
    r.parity = parity_ ? 1 : 0;
    r.scratch = red_scratch_.get();
    return r;
  }

  // ---- row-sharded plumbing (comm_ != nullptr) ---------------------------
  bool dist() const { return comm_ != nullptr; }
  int64_t full_cols() const { return plan_.col_block * comm_->world(); }
  // The dimension a sharded attempt exchanges: columns for the row cut
  // (x-bar gathered, K^T's output reduce-scattered), rows for the column cut
  // (K's output reduce-scattered, dy gathered).  The dual polishing
  // subproblem swaps the layouts' roles and exchanges the same dimension.
  bool cols_cut() const { return plan_.cut == PDLP_CUT_COLS; }
  int64_t xch_block() const { return cols_cut() ? plan_.row_block : plan_.col_block; }
  int64_t xch_full() const { return xch_block() * comm_->world(); }
  int64_t xch_local() const {
    return cols_cut() ? plan_.row_end - plan_.row_begin : plan_.col_end - plan_.col_begin;
  }
  int64_t full_rows() const { return plan_.row_block * comm_->world(); }
  int64_t full_len() const { return std::max<int64_t>(std::max(full_cols(), full_rows()), 1); }

  // The same verdict on every rank: true iff `flag` holds on any rank.
  bool any_rank(bool flag) {
    double v = flag ? 1.0 : 0.0;
    PDLP_CK(cudaStreamSynchronize(s()));
    PDLP_CK(cudaMemcpyAsync(flag_.get(), &v, sizeof(double), cudaMemcpyHostToDevice, s()));
    comm_->allreduce(flag_.get(), 1, true, s());
    PDLP_CK(cudaMemcpyAsync(&v, flag_.get(), sizeof(double), cudaMemcpyDeviceToHost, s()));
    PDLP_CK(cudaStreamSynchronize(s()));
    return v > 0.5;
  }

  // First failure per validation category over all ranks, in whole-problem
  // numbering (keys are index << 3 | code, see k_valid.cu).
  void combine_validation(unsigned long long hk[4], unsigned& hb, int64_t r0, int64_t c0,
                          int64_t e0) {
    const unsigned long long none = ~0ull;
    const int64_t off[4] = {c0, c0, r0, e0};
    double v[5];
    for (int q = 0; q < 4; ++q) {
      if (hk[q] == none) {
        v[q] = -kInf;
      } else {
        const unsigned long long idx = (hk[q] >> 3) + static_cast<unsigned long long>(off[q]);
        v[q] = -static_cast<double>((idx << 3) | (hk[q] & 7ull));
      }
    }
    v[4] = hb != 0 ? 1.0 : 0.0;
    PDLP_CK(cudaStreamSynchronize(s()));
    PDLP_CK(cudaMemcpyAsync(flag_.get(), v, sizeof(v), cudaMemcpyHostToDevice, s()));
    comm_->allreduce(flag_.get(), 5, true, s());
    PDLP_CK(cudaMemcpyAsync(v, flag_.get(), sizeof(v), cudaMemcpyDeviceToHost, s()));
    PDLP_CK(cudaStreamSynchronize(s()));
    for (int q = 0; q < 4; ++q) {
      hk[q] = std::isinf(v[q]) ? none : static_cast<unsigned long long>(-v[q]);
    }
    hb = v[4] > 0.5 ? 1u : 0u;
  }

  // local (n_local entries) -> this rank's block of `full`, then all-gather.
  void gather(const double* local, int64_t n_local, int64_t block, double* full) {
    if (local != full + block * comm_->rank()) {
      dev_copy(full + block * comm_->rank(), local, n_local, s());
    }
    comm_->allgather(full, static_cast<size_t>(block), s());
  }

  // A x (or A' y): on one GPU the plain product; sharded, the layout's kind
  // says whether the column-side operand is gathered first (K_g) or the
  // column-side output is reduce-scattered after (K_g^T).
  void product(const pdlpk_csr& L, int orig, const double* in, double* out) {
    if (!dist() || L.dist_kind == PDLPK_DIST_NONE) {
      PDLP_LAUNCH(pdlpk_spmv(&L, orig, in, out, parity_, s()));
      return;
    }
    const int64_t nb = xch_block();
    const int64_t nloc = xch_local();
    if (L.dist_kind == PDLPK_DIST_GATHER) {
      gather(in, nloc, nb, gbuf_.get());
      PDLP_LAUNCH(pdlpk_spmv(&L, orig, gbuf_.get(), out, 0, s()));
    } else if (peer_pbuf_ != nullptr) {
      peer_fence();
      PDLP_LAUNCH(pdlpk_spmv(&L, orig, in, peer_pbuf_, 0, s()));
      comm_->barrier(s());
      PDLP_LAUNCH(pdlpk_peer_reduce(out, &peers_, nloc, s()));
      peer_pending_ = true;
    } else {
      PDLP_LAUNCH(pdlpk_spmv(&L, orig, in, pbuf_.get(), 0, s()));
      comm_->reduce_scatter(pbuf_.get(), gbuf_.get(), static_cast<size_t>(nb), s());
      dev_copy(out, gbuf_.get(), nloc, s());
    }
  }

  // Before this rank overwrites its peer buffer: every peer has finished
  // reading it (a barrier unless a collective has intervened since).
  void peer_fence() {
    if (peer_pending_) {
      comm_->barrier(s());
      peer_pending_ = false;
    }
  }

  // Peers' last reads of this rank's buffer are done before it is freed.
  void peer_finish() {
    if (peer_pbuf_ != nullptr) peer_fence();
  }

  // Combines the reductions logged since the last read across ranks (one
  // all-gather of the slot array, rank-ordered sums / maxima).
  void combine_logged() {
    const int count = red_log_.count;
    if (count == 0) return;
    red_log_.count = 0;
    if (count > 48) throw CudaError("internal: reduction log overflow");
    uint64_t marked = 0, maxbits = 0;
    for (int i = 0; i < count; ++i) {
      const int64_t off = red_log_.out[i] - slots_.get();
      const int k = red_log_.k[i];
      if (off < 0 || off + k > kSlots) throw CudaError("internal: reduction outside the slots");
      for (int j = 0; j < k; ++j) {
        const uint64_t bit = 1ull << (off + j);
        marked |= bit;
        if ((red_log_.maxmask[i] >> j) & 1u) {
          maxbits |= bit;
        } else {
          maxbits &= ~bit;
        }
      }
    }
    double* all = slots_all_.get();
    dev_copy(all + static_cast<int64_t>(kSlots) * comm_->rank(), slots_.get(), kSlots, s());
    comm_->allgather(all, kSlots, s());
    PDLP_LAUNCH(pdlpk_combine_slots(all, comm_->world(), kSlots, marked, maxbits, slots_.get(), s()));
  }

  // One sharded attempt, all stream-ordered:
  // primal -> [AG x-bar] -> K x-bar + dual update -> K^T dy partial -> [RS]
  // -> column epilogue -> [AG 8 scalars] -> rank-ordered decision.  For the
  // dual polishing subproblem the layouts swap kinds and so do the
  // collectives (K partial + RS, K^T gathered).
  void attempt_dist(const pdlpk_problem& P, Inner& D, const pdlpk_step_args& a) {
    const int rank = comm_->rank();
    const int64_t nb = xch_block();
    const bool kg = P.K.dist_kind == PDLPK_DIST_GATHER;
    const bool ktg = P.KT.dist_kind == PDLPK_DIST_GATHER;
    // x-bar is only read inside an attempt, so one peer-mappable gathered
    // vector serves every subproblem.  Reuse needs no fence: each attempt
    // ends with the totals all-gather, which completes only after every
    // rank's row pass (the last reader) of that attempt.
    const bool push = kg && peer_gather_ != nullptr;
    double* xfull = push ? peer_gather_ : D.xbar.get();
    double* dyfull = D.dy.get();
    pdlpk_step_args b = a;
    b.xbar = kg ? xfull + nb * rank : xfull;
    if (push) {
      PDLP_LAUNCH(pdlpk_dist_primal_push(&b, &push_, s()));
    } else {
      PDLP_LAUNCH(pdlpk_dist_primal(&b, s()));
    }
    b.xbar = xfull;
    b.dy = ktg ? dyfull + nb * rank : dyfull;
    int64_t g2 = 0, g3 = 0;
    int k_acc = 0, kt_acc = 0;
    if (kg) {
      if (push) {
        comm_->barrier(s());  // every peer's x-bar block has landed
      } else {
        comm_->allgather(xfull, static_cast<size_t>(nb), s());
      }
      PDLP_LAUNCH(pdlpk_dist_row_fused(&b, s()));
      g2 = pdlpk_dist_sched_grid(&P.K);
      k_acc = 1;
    } else if (peer_pbuf_ != nullptr) {
      peer_fence();
      PDLP_LAUNCH(pdlpk_spmv(&P.K, 0, xfull, peer_pbuf_, 0, s()));
      comm_->barrier(s());
      PDLP_LAUNCH(pdlpk_dist_row_epi_peers(&b, &peers_, s()));
      peer_pending_ = true;
      g2 = pdlpk_dist_ew_grid(P.m);
    } else {
      PDLP_LAUNCH(pdlpk_spmv(&P.K, 0, xfull, D.pbuf.get(), 0, s()));
      comm_->reduce_scatter(D.pbuf.get(), D.dloc.get(), static_cast<size_t>(nb), s());
      PDLP_LAUNCH(pdlpk_dist_row_epi(&b, D.dloc.get(), s()));
      g2 = pdlpk_dist_ew_grid(P.m);
    }
    if (ktg) {
      comm_->allgather(dyfull, static_cast<size_t>(nb), s());
      b.dy = dyfull;
      PDLP_LAUNCH(pdlpk_dist_col_fused(&b, s()));
      g3 = pdlpk_dist_sched_grid(&P.KT);
      kt_acc = 1;
    } else if (peer_pbuf_ != nullptr) {
      peer_fence();
      PDLP_LAUNCH(pdlpk_spmv(&P.KT, 0, b.dy, peer_pbuf_, 0, s()));
      comm_->barrier(s());
      PDLP_LAUNCH(pdlpk_dist_col_epi_peers(&b, &peers_, s()));
      peer_pending_ = true;
      g3 = pdlpk_dist_ew_grid(P.n);
    } else {
      PDLP_LAUNCH(pdlpk_spmv(&P.KT, 0, b.dy, D.pbuf.get(), 0, s()));
      comm_->reduce_scatter(D.pbuf.get(), D.dloc.get(), static_cast<size_t>(nb), s());
      PDLP_LAUNCH(pdlpk_dist_col_epi(&b, D.dloc.get(), s()));
      g3 = pdlpk_dist_ew_grid(P.n);
    }
    double* tot = D.tot_all.get();
    PDLP_LAUNCH(pdlpk_dist_totals(&b, g2, g3, k_acc, kt_acc, tot + 8 * rank, s()));
    comm_->allgather(tot, 8, s());
    peer_pending_ = false;  // the all-gather ordered every peer's reads
    PDLP_LAUNCH(pdlpk_dist_decide(&b, tot, comm_->world(), s()));
  }

  // Whole-problem views for the gap (computed redundantly on gathered
  // vectors by every rank): the main problem, its primal polishing problem
  // (c = 0) and the swapped dual polishing problem.
  void build_full_views() {
    const int64_t nb = plan_.col_block, mb = plan_.row_block;
    const int64_t nloc = prob_.n, mloc = prob_.m;
    for (DevBuf<double>* b : {&fc_c_, &fc_lv_, &fc_uv_, &fc_zero_}) b->alloc(full_cols());
    for (DevBuf<double>* b : {&fr_lc_, &fr_uc_, &fr_zero_}) b->alloc(full_rows());
    gather(prob_.c.get(), nloc, nb, fc_c_.get());
    gather(prob_.lv.get(), nloc, nb, fc_lv_.get());
    gather(prob_.uv.get(), nloc, nb, fc_uv_.get());
    gather(prob_.lc.get(), mloc, mb, fr_lc_.get());
    gather(prob_.uc.get(), mloc, mb, fr_uc_.get());
    dev_zero(fc_zero_.get(), full_cols(), s());
    dev_zero(fr_zero_.get(), full_rows(), s());
    pdlpk_problem F{};
    F.m = m_glob_;
    F.n = n_glob_;
    F.c = F.c_o = fc_c_.get();
    F.lv = F.lv_o = fc_lv_.get();
    F.uv = F.uv_o = fc_uv_.get();
    F.lc = F.lc_o = fr_lc_.get();
    F.uc = F.uc_o = fr_uc_.get();
    full_main_ = F;
    full_primal_ = F;
    full_primal_.c = full_primal_.c_o = fc_zero_.get();
    for (DevBuf<double>* b : {&fs_lc_, &fs_uc_}) b->alloc(std::max<int64_t>(n_glob_, 1));
    for (DevBuf<double>* b : {&fs_lv_, &fs_uv_}) b->alloc(std::max<int64_t>(m_glob_, 1));
    PDLP_LAUNCH(pdlpk_dual_feas_bounds(F.c, F.lv, F.uv, n_glob_, F.lc, F.uc, m_glob_, fs_lc_.get(),
                                       fs_uc_.get(), fs_lv_.get(), fs_uv_.get(), s()));
    pdlpk_problem Q{};
    Q.m = n_glob_;
    Q.n = m_glob_;
    Q.c = Q.c_o = fr_zero_.get();
    Q.lc = Q.lc_o = fs_lc_.get();
    Q.uc = Q.uc_o = fs_uc_.get();
    Q.lv = Q.lv_o = fs_lv_.get();
    Q.uv = Q.uv_o = fs_uv_.get();
    full_dual_ = Q;
    for (auto& q : gq_) {
      for (auto& b : q) b.alloc(full_len());
    }
  }

  // Device slot layout (doubles) of one cadence batch.
  static constexpr int kSlotScrCur = 0;  // 4: primal_inf, dual_inf, pobj, penalty
  static constexpr int kSlotScrAvg = 4;  // 4
  static constexpr int kSlotDist = 8;    // dx2/dy2 of current, then of average
  static constexpr int kSlotRay = 16;    // 3 candidates x 8
  static constexpr int kSlotGap = 40;    // 2
  static constexpr int kSlotTmp = 48;    // scratch for follow-up checks
  static constexpr int kSlots = 64;

  double* slot(int i) { return slots_.get() + i; }
  // Copies slots [0, count) to the host (one sync).
  const double* read_slots(int count) {
    if (dist()) combine_logged();
    PDLP_CK(cudaMemcpyAsync(host_slots_, slots_.get(), count * sizeof(double),
                            cudaMemcpyDeviceToHost, s()));
    PDLP_CK(cudaStreamSynchronize(s()));
    return host_slots_;
  }

  // apply_rescaling (rescaling.hpp:137-143) on device, both layouts in place.
  void precondition(int ruiz_passes, bool pock_chambolle) {
    NvtxRange nvtx("pdlp:precondition");
    const auto t0 = Clock::now();
    const int64_t m = prob_.m, n = prob_.n;
    // fc spans every column of the layouts (all n under the row cut), fr
    // every row (all m under the column cut)
    const bool cc = dist() && cols_cut();
    const int64_t mr = cc ? m_glob_ : m, nc = cc ? n : n_glob_;
    DevBuf<double> fr(std::max<int64_t>(mr, 1)), fc(std::max<int64_t>(nc, 1));
    DevBuf<unsigned long long> bits(std::max<int64_t>(std::max(mr, nc), 1));
    const int64_t c0 = dist() && !cc ? plan_.col_begin : 0;
    const int64_t r0 = cc ? plan_.row_begin : 0;
    const int64_t nnz = prob_.row.view.nnz;
    (void)nnz;
    const DevBuf<int32_t>& row_of = row_of_;  // line maps built during validation
    const DevBuf<int32_t>& col_of = col_of_;
    auto pass = [&](int one_norm) {
      if (cc) {
        // column cut: the transpose of the row cut's combine -- a rank holds
        // one consecutive run (its columns) of every row: row inf-norms
        // max-combined, row 1-norms chained rank by rank, column norms local
        PDLP_LAUNCH(pdlpk_line_factors(&prob_.col.view, col_of.get(), one_norm, fc.get(), bits.get(), s()));
        if (one_norm == 0) {
          PDLP_LAUNCH(pdlpk_line_norms(&prob_.row.view, row_of.get(), 0, fr.get(), bits.get(), s()));
          comm_->allreduce(fr.get(), static_cast<size_t>(m_glob_), true, s());
        } else {
          dev_zero(fr.get(), m_glob_, s());
          for (int r = 0; r < comm_->world(); ++r) {
            if (r == comm_->rank()) PDLP_LAUNCH(pdlpk_line_onenorm_continue(&prob_.row.view, fr.get(), s()));
            comm_->allreduce(fr.get(), static_cast<size_t>(m_glob_), true, s());
          }
        }
        PDLP_LAUNCH(pdlpk_norm_to_factor(fr.get(), m_glob_, s()));
        PDLP_LAUNCH(pdlpk_apply_factors(&prob_.row.view, row_of.get(), prob_.row.value.get(), fr.get(), fc.get(), s()));
        PDLP_LAUNCH(pdlpk_apply_factors(&prob_.col.view, col_of.get(), prob_.col.value.get(), fc.get(), fr.get(), s()));
        PDLP_LAUNCH(pdlpk_apply_vec_factors(prob_.lc.get(), prob_.uc.get(), prob_.row_scale.get(),
                                            fr.get() + r0, m, prob_.c.get(), prob_.lv.get(),
                                            prob_.uv.get(), prob_.col_scale.get(), fc.get(), n, s()));
        return;
      }
      PDLP_LAUNCH(pdlpk_line_factors(&prob_.row.view, row_of.get(), one_norm, fr.get(), bits.get(), s()));
      if (dist()) {
        // A rank holds one consecutive run (its rows) of every column.
        // inf-norms: max over ranks is exact.  1-norms: continue the
        // reference's sequential sum rank by rank (rank r adds its run to the
        // carried sums, an all-reduce max publishes them since the sums only
        // grow), so the scaled problem is bit-identical to one GPU's.
        if (one_norm == 0) {
          PDLP_LAUNCH(pdlpk_line_norms(&prob_.col.view, col_of.get(), 0, fc.get(), bits.get(), s()));
          comm_->allreduce(fc.get(), static_cast<size_t>(n_glob_), true, s());
        } else {
          dev_zero(fc.get(), n_glob_, s());
          for (int r = 0; r < comm_->world(); ++r) {
            if (r == comm_->rank()) PDLP_LAUNCH(pdlpk_line_onenorm_continue(&prob_.col.view, fc.get(), s()));
            comm_->allreduce(fc.get(), static_cast<size_t>(n_glob_), true, s());
          }
        }
        PDLP_LAUNCH(pdlpk_norm_to_factor(fc.get(), n_glob_, s()));
      } else {
        PDLP_LAUNCH(pdlpk_line_factors(&prob_.col.view, col_of.get(), one_norm, fc.get(), bits.get(), s()));
      }
      PDLP_LAUNCH(pdlpk_apply_factors(&prob_.row.view, row_of.get(), prob_.row.value.get(), fr.get(), fc.get(), s()));
      PDLP_LAUNCH(pdlpk_apply_factors(&prob_.col.view, col_of.get(), prob_.col.value.get(), fc.get(), fr.get(), s()));
      PDLP_LAUNCH(pdlpk_apply_vec_factors(prob_.lc.get(), prob_.uc.get(), prob_.row_scale.get(),
                                          fr.get(), m, prob_.c.get(), prob_.lv.get(),
                                          prob_.uv.get(), prob_.col_scale.get(), fc.get() + c0, n, s()));
    };
    if (!dist() && ruiz_passes > 0) {
      // one GPU: both layouts' line inf-norms once, then each pass divides
      // and takes the next pass's norms of the result in the same sweep
      // (same maxima, same divisions as pass(0))
      DevBuf<unsigned long long> bc(std::max<int64_t>(n, 1));
      PDLP_LAUNCH(pdlpk_line_absmax(&prob_.row.view, row_of.get(), bits.get(), s()));
      PDLP_LAUNCH(pdlpk_line_absmax(&prob_.col.view, col_of.get(), bc.get(), s()));
      for (int p = 0; p < ruiz_passes; ++p) {
        const bool more = p + 1 < ruiz_passes;
        PDLP_LAUNCH(pdlpk_factors_from_bits(bits.get(), m, fr.get(), s()));
        PDLP_LAUNCH(pdlpk_factors_from_bits(bc.get(), n, fc.get(), s()));
        PDLP_LAUNCH(pdlpk_apply_factors_max(&prob_.row.view, row_of.get(), prob_.row.value.get(),
                                            fr.get(), fc.get(), more ? bits.get() : nullptr, s()));
        PDLP_LAUNCH(pdlpk_apply_factors_max(&prob_.col.view, col_of.get(), prob_.col.value.get(),
                                            fc.get(), fr.get(), more ? bc.get() : nullptr, s()));
        PDLP_LAUNCH(pdlpk_apply_vec_factors(prob_.lc.get(), prob_.uc.get(), prob_.row_scale.get(),
                                            fr.get(), m, prob_.c.get(), prob_.lv.get(),
                                            prob_.uv.get(), prob_.col_scale.get(), fc.get(), n, s()));
      }
    } else {
      for (int p = 0; p < ruiz_passes; ++p) pass(0);
    }
    if (pock_chambolle) pass(1);
    PDLP_CK(cudaStreamSynchronize(s()));
    precondition_seconds_ = std::chrono::duration<double>(Clock::now() - t0).count();
  }

  // initial_step_size (step.hpp:14-18)
  double initial_step_size() {
    const pdlpk_red r = red();
    PDLP_LAUNCH(pdlpk_abs_max(prob_.row.value.get(), prob_.row.view.nnz, &r, slot(0), s()));
    const double mx = read_slots(1)[0];
    return mx > 0.0 ? 1.0 / mx : 1.0;
  }

  // initialize_primal_weight (restarts.hpp:278-294)
  double initialize_primal_weight() {
    const pdlpk_red r = red();
    PDLP_LAUNCH(pdlpk_primal_weight_sums(prob_.c.get(), prob_.n, prob_.lc.get(), prob_.uc.get(),
                                         prob_.m, &r, slot(0), s()));
    const double* h = read_slots(2);
    const double nc = std::sqrt(h[0]);
    const double nb = std::sqrt(h[1]);
    if (nc > 1e-12 && nb > 1e-12) return nc / nb;
    return 1.0;
  }

  // Host-libm schedule factors for next_step_size (step.hpp:136-141).
  void ensure_table(int64_t len) {
    if (len <= table_len_) return;
    int64_t want = std::max<int64_t>(len, 4096);
    want = std::max(want, 2 * table_len_);
    std::vector<double> down(want), up(want);
    for (int64_t k = 0; k < want; ++k) {
      const double kk = static_cast<double>(k < 1 ? 1 : k) + 1.0;
      down[k] = 1.0 - std::pow(kk, -0.3);
      up[k] = 1.0 + std::pow(kk, -0.6);
    }
    f_down_.alloc(want);
    f_up_.alloc(want);
    PDLP_CK(cudaMemcpyAsync(f_down_.get(), down.data(), want * 8, cudaMemcpyHostToDevice, s()));
    PDLP_CK(cudaMemcpyAsync(f_up_.get(), up.data(), want * 8, cudaMemcpyHostToDevice, s()));
    PDLP_CK(cudaStreamSynchronize(s()));  // the host tables die here
    table_len_ = want;
  }

  pdlpk_step_args step_args(const pdlpk_problem& P, Inner& D) {
    pdlpk_step_args a{};
    a.P = P;
    for (int b = 0; b < 2; ++b) {
      a.x[b] = D.x[b].get();
      a.y[b] = D.y[b].get();
      a.aty[b] = D.aty[b].get();
    }
    a.xbar = D.xbar.get();
    a.dy = D.dy.get();
    a.aty_diff = D.aty_diff.get();
    a.sum_x = D.sum_x.get();
    a.sum_y = D.sum_y.get();
    a.state = D.state.get();
    a.f_down = f_down_.get();
    a.f_up = f_up_.get();
    a.table_len = table_len_;
    a.part2 = D.part2.get();
    a.part3 = D.part3.get();
    a.mode = parity_ ? PDLP_MODE_PARITY : PDLP_MODE_PERF;
    a.shards = shards_;
    a.shard_part = D.shard_part.get();
    a.line_partials = (!parity_ && !dist() && P.m <= PDLPK_LINE_PARTIALS_MAX && line_partials_on_)
                          ? 1 : 0;
    if (!parity_ && uses_sell(P)) {
      a.sell.off = sell_off_.get();
      a.sell.sidx = sell_idx_.get();
      a.sell.sval = sell_val_.get();
      a.sell.ng = sell_ng_;
      a.sell.blocks = sell_blocks_;
    }
    if (!parity_ && uses_panels(P)) {
      a.n_row_panels = panels_.np;
      a.row_panels = panels_.views.data();
      a.carry = panels_.carry.get();
    }
    return a;
  }

  void read_state(Inner& D) {
    PDLP_CK(cudaMemcpyAsync(&D.hs, D.state.get(), sizeof(pdlpk_step_state),
                            cudaMemcpyDeviceToHost, s()));
    PDLP_CK(cudaStreamSynchronize(s()));
  }
  void write_state(Inner& D) {
    PDLP_CK(cudaStreamSynchronize(s()));
    PDLP_CK(cudaMemcpyAsync(D.state.get(), &D.hs, sizeof(pdlpk_step_state), cudaMemcpyHostToDevice, s()));
    PDLP_CK(cudaStreamSynchronize(s()));
  }

  // InnerState::prepare (solver.hpp:167-192); x0 is a device vector.
  void prepare(Inner& D, const pdlpk_problem& P, const double* x0, double eta0, double omega0,
               bool fixed) {
    int64_t partials = pdlpk_step_partials(&P);
    if (uses_panels(P)) {  // the decision reads the last panel launch's partials
      pdlpk_problem Q = P;
      Q.K = panels_.views.back();
      partials = std::max(partials, pdlpk_step_partials(&Q));
    }
    if (uses_sell(P)) partials = std::max<int64_t>(partials, 2 * static_cast<int64_t>(sell_blocks_) + 64);
    if (dist()) {
      partials = std::max<int64_t>(partials, 3 * pdlpk_dist_ew_grid(std::max(P.n, P.m)) + 64);
    }
    if (D.n != P.n || D.m != P.m || static_cast<int64_t>(D.part2.size()) < partials) {
      if (dist()) {
        D.allocate(P.n, P.m, partials, shards_, xch_full(), xch_block(), comm_->world());
      } else {
        D.allocate(P.n, P.m, partials, shards_);
      }
    }
    dev_copy(D.x[0].get(), x0, P.n, s());
    dev_zero(D.y[0].get(), P.m, s());
    dev_zero(D.aty[0].get(), P.n, s());
    dev_zero(D.sum_x.get(), P.n, s());
    dev_zero(D.sum_y.get(), P.m, s());
    dev_copy(D.ref_x.get(), x0, P.n, s());
    dev_zero(D.ref_y.get(), P.m, s());
    std::memset(&D.hs, 0, sizeof(D.hs));
    D.hs.eta = eta0;
    D.hs.omega = omega0;
    D.hs.min_eta_bar = kInf;
    D.hs.max_retries = 60;
    D.hs.halt = 1;
    D.hs.fixed = fixed ? 1 : 0;
    D.omega = omega0;
    D.last_eta = eta0;
    D.mu_last = kInf;
    D.prev_candidate_mu = kInf;
    D.k_last_restart = 0;
    D.restarts = 0;
    D.next_polish_trigger = 100;
    D.polish_iterations = 0;
    D.have_sol = false;
    D.detail.clear();
    D.cert.have = false;
    write_state(D);
  }

  // Runs step attempts until k reaches target or the controller halts.
  void run_steps(const pdlpk_problem& P, Inner& D, int64_t target) {
    NvtxRange nvtx("pdlp:attempts");
    ensure_table(target + 1);
    pdlpk_step_args a = step_args(P, D);
    PDLP_LAUNCH(pdlpk_arm(D.state.get(), target, s()));
    step_begin_.record(s());
    int64_t known_k = D.hs.k;
    while (true) {
      const int64_t need = target - known_k;
      if (need <= 0) break;
      if (dist()) {
        for (int64_t t = 0; t < need; ++t) attempt_dist(P, D, a);
        read_state(D);
      } else if (profile_) {
        const int64_t attempts0 = D.hs.attempts;
        ensure_prof_events(need);
        for (int64_t t = 0; t < need; ++t) {
          PDLP_LAUNCH(pdlpk_attempt_timed(&a, prof_ev_.data() + 4 * t, s()));
        }
        read_state(D);
        const int64_t ran = std::min(need, D.hs.attempts - attempts0);
        for (int64_t t = 0; t < ran; ++t) {
          for (int q = 0; q < 3; ++q) {
            float ms = 0.0f;
            PDLP_CK(cudaEventElapsedTime(&ms, prof_ev_[4 * t + q], prof_ev_[4 * t + q + 1]));
            kernel_seconds_[q] += 1e-3 * ms;
            kernel_launches_[q] += 1;
          }
        }
      } else {
        for (int64_t t = 0; t < need; ++t) PDLP_LAUNCH(pdlpk_attempt(&a, s()));
        read_state(D);
      }
      if (D.hs.status != 0 || D.hs.k >= target) break;
      known_k = D.hs.k;
    }
    step_end_.record(s());
    step_seconds_ += elapsed_seconds(step_begin_, step_end_);
    read_state(D);
  }

  void flush_average(const pdlpk_problem& P, Inner& D) {
    pdlpk_step_args a = step_args(P, D);
    PDLP_LAUNCH(pdlpk_flush_average(&a, s()));
    D.hs.avg_pending = 0;
  }

  // --- residual screens ----------------------------------------------------
  Summary screen(const pdlpk_problem& P, int orig, const double* x, const double* y,
                 const double* ax, const double* aty, int rc_mode, double* r_out) {
    const pdlpk_red r = red();
    PDLP_LAUNCH(pdlpk_screen(&P, orig, x, y, ax, aty, rc_mode, &r, r_out, slot(0), s()));
    const double* h = read_slots(4);
    return finish_summary(h[0], h[1], h[2], -h[3]);
  }

  // recover_reduced_costs + kkt_residuals on the original data
  // (residuals.hpp:49-64, 135-158): genuine original-space products.
  Summary original_kkt(const pdlpk_problem& P, const double* x, const double* y, int rc_mode,
                       double* r_out, Inner& D) {
    product(P.K, 1, x, D.prod_m.get());
    product(P.KT, 1, y, D.prod_n.get());
    return screen(P, 1, x, y, D.prod_m.get(), D.prod_n.get(), rc_mode, r_out);
  }

  static bool screen_passes(const InnerCfg& cfg, const Summary& s) {
    return cfg.feasibility_only ? s.primal <= cfg.tol.eps_primal : check_termination(s, cfg.tol);
  }

  // screen_and_verify (solver.hpp:207-232)
  bool screen_and_verify(const pdlpk_problem& P, const InnerCfg& cfg, const double* xs,
                         const double* ys, const double* ax_s, const double* aty_s, double* rc,
                         Summary& screened, Inner& D, const char* which) {
    screened = screen(P, 0, xs, ys, ax_s, aty_s, cfg.rc_mode, rc);
    if (!screen_passes(cfg, screened)) return false;
    return verify_point(P, cfg, xs, ys, D, which);
  }

  // The verification half of screen_and_verify (solver.hpp:218-231): a
  // genuine original-space recomputation before committing to a status.
  bool verify_point(const pdlpk_problem& P, const InnerCfg& cfg, const double* xs,
                    const double* ys, Inner& D, const char* which) {
    PDLP_LAUNCH(pdlpk_scale_mul(P.col_scale, xs, D.tmp_x.get(), P.n, s()));
    PDLP_LAUNCH(pdlpk_scale_mul(P.row_scale, ys, D.tmp_y.get(), P.m, s()));
    const Summary truth = original_kkt(P, D.tmp_x.get(), D.tmp_y.get(), cfg.rc_mode, D.tmp_r.get(), D);
    const bool verified = cfg.feasibility_only ? truth.primal <= cfg.tol.eps_primal
                                               : check_termination(truth, cfg.tol);
    if (!verified) return false;
    D.sol_x.swap(D.tmp_x);
    D.sol_y.swap(D.tmp_y);
    D.sol_r.swap(D.tmp_r);
    D.sol_summary = truth;
    D.have_sol = true;
    D.detail = std::string("converged at the ") + which;
    return true;
  }

  // capture_current (solver.hpp:236-242)
  void capture_current(const pdlpk_problem& P, const InnerCfg& cfg, Inner& D) {
    const int c = D.cur();
    PDLP_LAUNCH(pdlpk_scale_mul(P.col_scale, D.x[c].get(), D.sol_x.get(), P.n, s()));
    PDLP_LAUNCH(pdlpk_scale_mul(P.row_scale, D.y[c].get(), D.sol_y.get(), P.m, s()));
    if (!parity_ && !dist() && &D == &main_ && D.fresh_products_k == D.k()) {
      // Perf mode: the cadence has just computed K x and K' y for this
      // iterate; with K = diag(1/row_scale) A diag(1/col_scale) and the
      // unscaling x = col_scale x_s, y = row_scale y_s, the original-space
      // products are A x = (K x_s) / row_scale and A' y = (K' y_s) / col_scale
      // (two elementwise passes instead of two more products).
      PDLP_LAUNCH(pdlpk_scale_div(P.row_scale, D.ax_cur.get(), D.prod_m.get(), P.m, s()));
      PDLP_LAUNCH(pdlpk_scale_div(P.col_scale, D.aty[c].get(), D.prod_n.get(), P.n, s()));
      D.sol_summary = screen(P, 1, D.sol_x.get(), D.sol_y.get(), D.prod_m.get(), D.prod_n.get(),
                             cfg.rc_mode, D.sol_r.get());
    } else {
      D.sol_summary = original_kkt(P, D.sol_x.get(), D.sol_y.get(), cfg.rc_mode, D.sol_r.get(), D);
    }
    D.have_sol = true;
  }

  // --- infeasibility rays (residuals.hpp:222-316) ---------------------------
  // Primal test on dual candidate yc; on success the ray and its completion
  // are left in ray_m / ray_n.
  bool try_primal(const pdlpk_problem& P, int orig, const double* yc, double eps_ray, Inner& D,
                  double& residual, double& objective) {
    const pdlpk_red r = red();
    PDLP_LAUNCH(pdlpk_ray_primal_prep(&P, orig, yc, D.ray_m.get(), &r, slot(0), s()));
    const double norm = read_slots(1)[0];
    if (!(norm > 0.0)) return false;
    product(P.KT, orig, D.ray_m.get(), D.prod_n.get());
    PDLP_LAUNCH(pdlpk_ray_primal_finish(&P, orig, D.ray_m.get(), D.prod_n.get(), nullptr, nullptr,
                                        D.ray_n.get(), &r, slot(0), s()));
    const double* h = read_slots(2);
    residual = h[0];
    if (residual > eps_ray * norm) return false;
    objective = -h[1];
    if (!(objective > 0.0) || !std::isfinite(objective)) return false;
    return true;
  }

  bool try_dual(const pdlpk_problem& P, int orig, const double* xc, double eps_ray, Inner& D,
                double& residual, double& objective) {
    const pdlpk_red r = red();
    PDLP_LAUNCH(pdlpk_ray_dual_prep(&P, orig, xc, &r, slot(0), s()));
    const double* h = read_slots(3);
    const double norm = h[0], box = h[1], obj = h[2];
    if (!(norm > 0.0)) return false;
    // Both conditions below must hold for a certificate; testing the cheap
    // ones first skips the product without changing the verdict.
    if (box > eps_ray * norm || !(obj < 0.0)) return false;
    product(P.K, orig, xc, D.prod_m.get());
    PDLP_LAUNCH(pdlpk_ray_dual_finish(&P, orig, D.prod_m.get(), &r, slot(0), s()));
    const double row = read_slots(1)[0];
    residual = (box < row) ? row : box;
    if (residual > eps_ray * norm) return false;
    objective = obj;
    return true;
  }

  // Ray candidates of detect_rays (solver.hpp:246-257), in the reference's order.
  struct RayCand {
    const double* x;
    const double* y;
    const double* known_aty;  // A'y already on device (same kernel), or NULL
    const char* source;
  };

  std::vector<RayCand> ray_candidates(const pdlpk_problem& P, Inner& D, bool have_avg) {
    std::vector<RayCand> cands;
    const int c = D.cur();
    if (D.k() > 0) {
      PDLP_LAUNCH(pdlpk_sub(D.x[c].get(), D.x[c ^ 1].get(), D.diff_x.get(), P.n, s()));
      PDLP_LAUNCH(pdlpk_sub(D.y[c].get(), D.y[c ^ 1].get(), D.diff_y.get(), P.m, s()));
      cands.push_back({D.diff_x.get(), D.diff_y.get(), nullptr, "difference"});
    }
    cands.push_back({D.x[c].get(), D.y[c].get(), D.aty[c].get(), "current"});
    if (have_avg) cands.push_back({D.avg_x.get(), D.avg_y.get(), D.aty_avg.get(), "average"});
    return cands;
  }

  // Enqueue the scaled-space ray tests of every candidate (no sync): slots
  // kSlotRay + 8q hold [|ray|, changed, residual, penalty, |xc|, box, c'xc].
  // When the cone projection leaves y unchanged the cached A'y is reused
  // (the product kernel is skipped on device), which is bit-identical.
  // Candidates [q0, q1) on stream st with reduction scratch r and product
  // temporary prod (the cadence runs the average's candidate on its side
  // stream).
  void enqueue_rays(const pdlpk_problem& P, Inner& D, const std::vector<RayCand>& cands,
                    size_t q0 = 0, size_t q1 = ~size_t(0), cudaStream_t st = nullptr,
                    const pdlpk_red* rs = nullptr, double* prod = nullptr) {
    const pdlpk_red r = rs != nullptr ? *rs : red();
    if (st == nullptr) st = s();
    if (prod == nullptr) prod = D.prod_n.get();
    for (size_t q = q0; q < std::min(q1, cands.size()); ++q) {
      double* sl = slot(kSlotRay + 8 * static_cast<int>(q));
      double* ray = D.ray_y[q].get();
      PDLP_LAUNCH(pdlpk_ray_primal_prep(&P, 0, cands[q].y, ray, &r, sl, st));
      if (cands[q].known_aty != nullptr && !dist()) {
        PDLP_LAUNCH(pdlpk_spmv_cond(&P.KT, 0, ray, prod, parity_, sl + 1, st));
      } else {
        product(P.KT, 0, ray, prod);  // (sharded only: always on the main stream)
      }
      // (sharded: the changed-count is still rank-local here, so the
      // product is always recomputed and the cached A'y is not used)
      PDLP_LAUNCH(pdlpk_ray_primal_finish(&P, 0, ray, prod, dist() ? nullptr : cands[q].known_aty,
                                          sl + 1, D.rhat[q].get(), &r, sl + 2, st));
      PDLP_LAUNCH(pdlpk_ray_dual_prep(&P, 0, cands[q].x, &r, sl + 4, st));
    }
  }

  // detect_rays (solver.hpp:246-280) from the batched scaled-space verdicts;
  // h = host copy of the slots.  The first certificate wins; a hit is then
  // re-verified on the original data.
  std::optional<int> detect_rays(const pdlpk_problem& P, const InnerCfg& cfg, Inner& D,
                                 const std::vector<RayCand>& cands, const double* h) {
    int kind = -1;
    size_t hit = 0;
    const double eps = cfg.eps_ray;
    for (size_t q = 0; q < cands.size() && kind < 0; ++q) {
      const double* sl = h + kSlotRay + 8 * q;
      const double norm = sl[0];
      if (norm > 0.0 && !(sl[2] > eps * norm)) {
        const double objective = -sl[3];
        if (objective > 0.0 && std::isfinite(objective)) {
          kind = PDLP_CERT_PRIMAL_INFEASIBLE;
          hit = q;
          break;
        }
      }
      const double xn = sl[4], box = sl[5], obj = sl[6];
      if (xn > 0.0 && !(box > eps * xn) && obj < 0.0) {
        const pdlpk_red r = red();
        product(P.K, 0, cands[q].x, D.prod_m.get());
        PDLP_LAUNCH(pdlpk_ray_dual_finish(&P, 0, D.prod_m.get(), &r, slot(kSlotTmp), s()));
        const double row = read_slots(kSlotTmp + 1)[kSlotTmp];
        const double residual = (box < row) ? row : box;
        if (!(residual > eps * xn)) {
          kind = PDLP_CERT_DUAL_INFEASIBLE;
          hit = q;
          dev_copy(D.ray_n.get(), cands[q].x, P.n, s());
        }
      }
    }
    if (kind < 0) return std::nullopt;
    const char* source = cands[hit].source;
    double res = 0.0, obj = 0.0;
    if (kind == PDLP_CERT_PRIMAL_INFEASIBLE) {
      dev_copy(D.ray_m.get(), D.ray_y[hit].get(), P.m, s());
      PDLP_LAUNCH(pdlpk_scale_mul(P.row_scale, D.ray_m.get(), D.tmp_y.get(), P.m, s()));
      if (try_primal(P, 1, D.tmp_y.get(), cfg.eps_ray, D, res, obj)) {
        D.cert.have = true;
        D.cert.kind = kind;
        dev_copy(D.cert.ray_y.get(), D.ray_m.get(), P.m, s());
        dev_copy(D.cert.ray_r.get(), D.ray_n.get(), P.n, s());
        D.cert.residual = res;
        D.cert.objective = obj;
        D.cert.source = source;
        D.detail = std::string("primal infeasibility certified by the ") + source + " ray";
        return kPrimalInf;
      }
    } else {
      PDLP_LAUNCH(pdlpk_scale_mul(P.col_scale, D.ray_n.get(), D.tmp_x.get(), P.n, s()));
      if (try_dual(P, 1, D.tmp_x.get(), cfg.eps_ray, D, res, obj)) {
        D.cert.have = true;
        D.cert.kind = kind;
        dev_copy(D.cert.ray_x.get(), D.tmp_x.get(), P.n, s());
        D.cert.residual = res;
        D.cert.objective = obj;
        D.cert.source = source;
        D.detail = std::string("dual infeasibility certified by the ") + source + " ray";
        return kDualInf;
      }
    }
    return std::nullopt;
  }

  // restart_progress_metric (restarts.hpp:223-231) for up to two points at
  // once: the radius sqrt(omega dx2 + dy2/omega) is evaluated on the host
  // from the device-reduced distances (same IEEE operations), then each gap
  // runs prepare -> (one sync for both event counts) -> finish -> one sync.
  struct GapQuery {
    const double *x, *y, *ax, *aty;
    double dx2, dy2;
  };
  // key0: the window-history slot of q[0] (0 current iterate, 1 window
  // average; the restart candidate's re-evaluation passes its own)
  void gaps(const InnerCfg& cfg, const pdlpk_problem& P, const GapQuery* q, int count,
            double omega, double* out, int key0 = 0) {
    NvtxRange nvtx("pdlp:gap");
    const auto gap_t0 = Clock::now();
    struct GapClock {
      double& acc;
      Clock::time_point t0;
      ~GapClock() { acc += std::chrono::duration<double>(Clock::now() - t0).count(); }
    } gap_clock{gap_seconds_, gap_t0};
    if (dist() && !gap_gathered_) {
      combine_logged();  // nothing may stay pending across the unlogged gap
      pdlpk_set_red_log(nullptr);
      for (int i = 0; i < count; ++i) out[i] = gap_dist(P, q[i], omega, i);
      pdlpk_set_red_log(&red_log_);
      if (gap_check_) {
        // the same evaluations on gathered vectors: lambda* (which the
        // crossing decides) and the gap value (a cancelling sum whose
        // rounding follows the summation order)
        double lam_d[2] = {gapd_lambda_[0], gapd_lambda_[1]}, ref[2], lam_g[2];
        gaps_gathered(cfg, P, q, count, omega, ref);
        for (int i = 0; i < count; ++i) {
          void* w = gap_work_[gap_shared_ ? 0 : i].get();
          PDLP_LAUNCH(pdlpk_gap_lambda_star(w, cfg.full->n, cfg.full->m, slot(kSlotGap + i), s()));
        }
        const double* hl = read_slots(kSlotGap + count);
        for (int i = 0; i < count; ++i) lam_g[i] = hl[kSlotGap + i];
        std::lock_guard<std::mutex> lk(gapd_stats().mu);
        auto rel = [](double a, double b) {
          return a == b ? 0.0 : std::fabs(a - b) / std::max(std::fabs(b), 1e-300);
        };
        for (int i = 0; i < count; ++i) {
          gapd_stats().max_rel = std::max(gapd_stats().max_rel, rel(out[i], ref[i]));
          gapd_stats().max_rel_lambda = std::max(gapd_stats().max_rel_lambda, rel(lam_d[i], lam_g[i]));
          ++gapd_stats().checked;
        }
      }
      return;
    }
    if (dist()) {
      gaps_gathered(cfg, P, q, count, omega, out);
      return;
    }
    gaps_local(P, q, count, omega, out, key0);
  }

  // Sharded, PDLP_GAP_GATHERED=1 (and the PDLP_GAPD_CHECK comparison): every
  // rank evaluates the same whole-problem gap on gathered vectors
  // (identical inputs -> identical mu everywhere).
  void gaps_gathered(const InnerCfg& cfg, const pdlpk_problem& P, const GapQuery* q, int count,
                     double omega, double* out) {
    {
      const int64_t nb = plan_.col_block, mb = plan_.row_block;
      const int64_t xb = cfg.swapped ? mb : nb, yb = cfg.swapped ? nb : mb;
      GapQuery g[2];
      for (int i = 0; i < count; ++i) {
        gather(q[i].x, P.n, xb, gq_[i][0].get());
        gather(q[i].aty, P.n, xb, gq_[i][1].get());
        gather(q[i].y, P.m, yb, gq_[i][2].get());
        gather(q[i].ax, P.m, yb, gq_[i][3].get());
        g[i] = {gq_[i][0].get(), gq_[i][2].get(), gq_[i][3].get(), gq_[i][1].get(), q[i].dx2, q[i].dy2};
      }
      combine_logged();  // nothing may stay pending across the unlogged gap
      pdlpk_set_red_log(nullptr);
      gaps_local(*cfg.full, g, count, omega, out);
      pdlpk_set_red_log(&red_log_);
    }
  }

  // ---- distributed normalized gap ---------------------------
  // normalized_duality_gap (restarts.hpp:107-220) over the row-sharded
  // problem without gathering a vector: each rank builds the breakpoint
  // events of its own column and row blocks; the reference's sequential
  // sweep is replaced by a bracket search over the global descending order
  // of the events.  A round picks a key s (weighted median of a strided key
  // sample of every rank's bracket), every rank reduces the masses of its
  // bracket events above / at-or-above s and counts those below, the ranks'
  // values are added in rank order, and phi(s) = C + B / lam(s)^2 (the
  // sweep's test at s) keeps the half that holds the first crossing: phi is
  // monotone in lam, so phi(s) >= r^2 means the crossing is s or above it,
  // else it is below s and the masses of [s, hi] join the base (C, B).  When
  // the bracket is small its events are all-gathered and swept by the
  // single-GPU kernels; lambda*, the candidate and the gap value follow from
  // the local blocks and one more all-gather.  Every decision depends only
  // on all-gathered values, so every rank takes the same branch and returns
  // the same gap.  Communication per round: two all-gathers of 40 and 8
  // doubles per rank.
  static double host_key_value(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double d;
    std::memcpy(&d, &b, sizeof(d));
    return d;
  }
  static uint64_t bits_of(double d) {
    uint64_t b;
    std::memcpy(&b, &d, sizeof(b));
    return b;
  }
  double* gapd_block(int64_t per_rank) {
    const int64_t need = per_rank * comm_->world();
    if (static_cast<int64_t>(gapd_buf_.size()) < need) gapd_buf_.alloc(need);
    return gapd_buf_.get();
  }
  // all-gather blocks of `count` doubles of gapd_buf_ and read them back
  const std::vector<double>& gapd_exchange(int64_t count) {
    comm_->allgather(gapd_buf_.get(), static_cast<size_t>(count), s());
    gapd_host_.resize(static_cast<size_t>(count * comm_->world()));
    PDLP_CK(cudaMemcpyAsync(gapd_host_.data(), gapd_buf_.get(), gapd_host_.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, s()));
    PDLP_CK(cudaStreamSynchronize(s()));
    return gapd_host_;
  }

  double gap_dist(const pdlpk_problem& P, const GapQuery& q, double omega, int qi) {
    const int W = comm_->world(), R = comm_->rank();
    const double radius = std::sqrt(omega * q.dx2 + q.dy2 / omega);
    gapd_lambda_[qi] = 0.0;
    if (!(radius > 0.0)) return 0.0;  // restarts.hpp:112
    const double r2 = radius * radius;
    const pdlpk_red rd = red();
    void* work = gap_work_[0].get();
    const int64_t n = P.n, m = P.m;
    constexpr int kS = 32;     // sampled keys per rank and round
    constexpr int kBlk = 40;   // doubles per rank of a sample exchange
    PDLP_LAUNCH(pdlpk_gap_prepare(&P, q.x, q.y, q.ax, q.aty, omega, &rd, work, nullptr, s()));
    double* blk = gapd_block(kBlk);
    PDLP_LAUNCH(pdlpk_gapd_stage(work, n, m, blk + 8 * R, s()));
    const std::vector<double>* h = &gapd_exchange(8);
    double B = 0.0, C = 0.0;  // masses above the bracket (incl. lam -> inf)
    std::vector<int64_t> A(W), An(W);
    int64_t At = 0;
    for (int r = 0; r < W; ++r) {
      B += (*h)[8 * r];
      C += (*h)[8 * r + 1];
      A[r] = static_cast<int64_t>((*h)[8 * r + 2]);
      At += A[r];
    }
    PDLP_LAUNCH(pdlpk_gapd_keys(work, n, m, A[R], s()));
    uint64_t* lk[2];
    int32_t* ls[2];
    pdlpk_gapd_lists(work, n, m, &lk[0], &ls[0], &lk[1], &ls[1]);
    int cur = 0;
    uint64_t lo = 0, hi = ~0ull, above_min = ~0ull;
    bool lower = false, above = false;
    int stall = 0;
    int64_t rounds = 0;
    std::vector<std::pair<uint64_t, double>> smp;
    while (At > gapd_final_ && stall < 3) {
      ++rounds;
      blk = gapd_block(kBlk);
      PDLP_LAUNCH(pdlpk_gapd_sample(lk[cur], A[R], kS, blk + kBlk * R, s()));
      h = &gapd_exchange(kBlk);
      smp.clear();
      for (int r = 0; r < W; ++r) {
        const int taken = static_cast<int>((*h)[kBlk * r + kS]);
        for (int i = 0; i < taken; ++i) {
          smp.emplace_back(bits_of((*h)[kBlk * r + i]), static_cast<double>(A[r]) / taken);
        }
      }
      std::sort(smp.begin(), smp.end(), [](const auto& a, const auto& b) {
        return a.first > b.first || (a.first == b.first && a.second < b.second);
      });
      // weighted median from the top (a quarter after a round without
      // progress: steps off a tie group at the bracket's bottom)
      const double target = static_cast<double>(At) * (stall > 0 ? 0.25 : 0.5);
      double acc = 0.0;
      uint64_t s_key = smp.back().first;
      for (const auto& e : smp) {
        acc += e.second;
        if (acc >= target) {
          s_key = e.first;
          break;
        }
      }
      blk = gapd_block(kBlk);
      PDLP_LAUNCH(pdlpk_gapd_split(work, n, m, lk[cur], ls[cur], A[R], s_key, &rd, blk + 8 * R, s()));
      h = &gapd_exchange(8);
      double cg = 0.0, bg = 0.0, ce = 0.0, be = 0.0;
      for (int r = 0; r < W; ++r) {
        cg += (*h)[8 * r];
        bg += (*h)[8 * r + 1];
        ce += (*h)[8 * r + 2];
        be += (*h)[8 * r + 3];
      }
      const double lam = host_key_value(s_key);
      const double c_sum = C + cg, b_sum = B + bg;
      uint64_t nlo = lo, nhi = hi;
      int64_t nt = 0;
      if (c_sum + b_sum / (lam * lam) >= r2) {
        nlo = s_key;  // the crossing is s or above it
        lower = true;
        for (int r = 0; r < W; ++r) An[r] = A[r] - static_cast<int64_t>((*h)[8 * r + 4]);
      } else {
        nhi = s_key - 1;  // below s: [s, hi] joins the masses above
        C += ce;
        B += be;
        above = true;
        above_min = s_key;
        for (int r = 0; r < W; ++r) An[r] = static_cast<int64_t>((*h)[8 * r + 4]);
      }
      for (int r = 0; r < W; ++r) nt += An[r];
      stall = nt == At ? stall + 1 : 0;
      if (nt != At) {
        PDLP_LAUNCH(pdlpk_gapd_compact(work, n, m, lk[cur], ls[cur], A[R], nlo, nhi, lk[cur ^ 1],
                                       ls[cur ^ 1], s()));
        cur ^= 1;
      }
      lo = nlo;
      hi = nhi;
      A.swap(An);
      At = nt;
    }
    // the bracket's events, gathered in rank order, sorted and swept
    int64_t K = 1;
    for (int r = 0; r < W; ++r) K = std::max(K, A[r]);
    blk = gapd_block(std::max<int64_t>(3 * K, kBlk));
    PDLP_LAUNCH(pdlpk_gapd_pack(work, n, m, lk[cur], ls[cur], A[R], K, blk + 3 * K * R, s()));
    comm_->allgather(blk, static_cast<size_t>(3 * K), s());
    const int64_t cap = std::max<int64_t>(At, 1);
    if (gapd_final_cap_ < cap) {
      gapd_fwork_.alloc(pdlpk_gapd_final_bytes(cap));
      gapd_final_cap_ = cap;
    }
    const double hi0 = above ? host_key_value(above_min) : std::numeric_limits<double>::infinity();
    double* lam_star = nullptr;
    PDLP_LAUNCH(pdlpk_gapd_final(gapd_fwork_.get(), gapd_final_cap_, blk, W, K, A.data(), C, B, hi0,
                                 lower ? 1 : 0, radius, &lam_star, s()));
    // (the value goes to block R after the final kernels read the blocks)
    PDLP_LAUNCH(pdlpk_gapd_value(&P, q.x, q.y, q.ax, q.aty, omega, lam_star, &rd, blk + 8 * R, s()));
    if (gap_check_) {
      PDLP_CK(cudaMemcpyAsync(&gapd_lambda_[qi], lam_star, sizeof(double), cudaMemcpyDeviceToHost, s()));
    }
    h = &gapd_exchange(8);
    double value = 0.0;
    for (int r = 0; r < W; ++r) value += (*h)[8 * r];
    {
      std::lock_guard<std::mutex> lk(gapd_stats().mu);
      ++gapd_stats().evals;
      gapd_stats().rounds += rounds;
      gapd_stats().final_events += At;
    }
    return (value > 0.0) ? value / radius : 0.0;
  }

  // Window of the next window sort for (subproblem, query): the last
  // crossing depth +- half, widened after a miss, narrowed after a hit.
  struct GapWindow {
    double depth = -1.0;  // unknown: full sort
    double half = 0.04;
  };
  GapWindow& gap_window_for(const pdlpk_problem& P, int i) {
    return gap_windows_[std::make_pair(static_cast<const void*>(P.c), i)];
  }

  void gaps_local(const pdlpk_problem& P, const GapQuery* q, int count, double omega, double* out,
                  int key0 = 0) {
    if (gap_shared_ && count > 1) {
      for (int i = 0; i < count; ++i) gaps_local(P, q + i, 1, omega, out + i, key0 + i);
      return;
    }
    const pdlpk_red r = red();
    // Two queries (current and average): the second runs on a side stream
    // with its own reduction scratch, so their chains of small, latency-bound
    // kernels overlap.  Same kernels and order per query: same values.
    const bool two = count == 2 && !gap_serial_;
    pdlpk_red r2 = r;
    if (two) {
      ensure_side();
      r2.scratch = gap_scratch2_.get();
      gap_fork_->record(s());
      PDLP_CK(cudaStreamWaitEvent(gap_side_->get(), gap_fork_->get(), 0));
    }
    auto qs = [&](int i) { return two && i == 1 ? gap_side_->get() : s(); };
    auto qr = [&](int i) { return two && i == 1 ? &r2 : &r; };
    auto join = [&] {
      if (!two) return;
      gap_join_->record(gap_side_->get());
      PDLP_CK(cudaStreamWaitEvent(s(), gap_join_->get(), 0));
    };
    static const bool gap_debug = std::getenv("PDLP_GAP_DEBUG") != nullptr;
    cudaEvent_t gev[3] = {nullptr, nullptr, nullptr};
    if (gap_debug) {
      for (auto& e : gev) cudaEventCreate(&e);
      cudaEventRecord(gev[0], s());
    }
    const auto t_prep = Clock::now();
    for (int i = 0; i < count; ++i) {
      PDLP_LAUNCH(pdlpk_gap_prepare(&P, q[i].x, q[i].y, q[i].ax, q[i].aty, omega, qr(i),
                                    gap_work_[i].get(), islots_.get() + i, qs(i)));
    }
    join();
    if (gap_debug) cudaEventRecord(gev[1], s());
    PDLP_CK(cudaMemcpyAsync(host_islots_, islots_.get(), 8 * sizeof(int), cudaMemcpyDeviceToHost, s()));
    PDLP_CK(cudaStreamSynchronize(s()));
    const auto t_fin = Clock::now();
    double qa[2] = {-1.0, -1.0}, qb[2] = {-1.0, -1.0};
    for (int i = 0; i < count; ++i) {
      const GapWindow& gw = gap_window_for(P, key0 + i);
      // Windows of the sorted breakpoints around the expected crossing: the
      // previous evaluation's depth, or, for the first evaluation of a
      // (subproblem, query), an estimate from a mass-carrying key sample
      // (qa = qb = -2).  The masses above a window are tree-summed, so the
      // gap's last bits differ from a full sort's; it stays a function of
      // its inputs (deterministic), and a window that misses the crossing
      // falls back to the full sort.  PDLP_GAP_WINDOWS=top keeps windows at
      // the top of the order (bit-identical to the full sort, rarely
      // smaller).
      if (!gap_partial_off_ && gap_any_window_) {
        // the sample estimate: the previous depth misleads after a restart
        // or an omega update (measured on C2: history windows missed 4 of
        // 8 evaluations in a 64-iteration solve, the estimate none)
        qa[i] = qb[i] = -2.0;
      } else if (!gap_partial_off_ && gw.depth >= 1.0 && gap_any_window_) {
        qa[i] = 0.9995;  // no crossing last time: only the last ~0.05 % sorted
        qb[i] = 1.0;
      } else if (!gap_partial_off_ && gw.depth >= 0.0 && gw.depth < 1.0) {
        qa[i] = gap_any_window_ ? std::max(0.0, gw.depth - gw.half) : 0.0;
        qb[i] = std::min(1.0, gw.depth + gw.half);
      }
      const double radius = std::sqrt(omega * q[i].dx2 + q[i].dy2 / omega);
      PDLP_LAUNCH(pdlpk_gap_finish(&P, q[i].x, q[i].y, q[i].ax, q[i].aty, omega, nullptr, radius,
                                   host_islots_[i], qr(i), gap_work_[i].get(),
                                   slot(kSlotGap + i), qa[i], qb[i], qs(i)));
    }
    join();
    if (gap_debug) cudaEventRecord(gev[2], s());
    const double* h = read_slots(kSlotGap + count + 2);
    float gpu_prep = 0.f, gpu_fin = 0.f;
    if (gap_debug) {
      cudaEventElapsedTime(&gpu_prep, gev[0], gev[1]);
      cudaEventElapsedTime(&gpu_fin, gev[1], gev[2]);
      for (auto& e : gev) cudaEventDestroy(e);
    }
    for (int i = 0; i < count; ++i) {
      out[i] = h[kSlotGap + i];
      const double hit = h[kSlotGap + 2 + i];
      if (gap_debug) {
        const auto t_end = Clock::now();
        std::fprintf(stderr,
                     "gap q=%d/%d c=%p E=%d window=[%.4f,%.4f] hit=%.5f prep=%.1fus "
                     "finish=%.1fus (gpu span prep %.1fus, finish %.1fus)\n",
                     i, count, static_cast<const void*>(P.c), host_islots_[i], qa[i], qb[i], hit,
                     1e6 * std::chrono::duration<double>(t_fin - t_prep).count(),
                     1e6 * std::chrono::duration<double>(t_end - t_fin).count(), 1e3 * gpu_prep,
                     1e3 * gpu_fin);
      }
      GapWindow& gw = gap_window_for(P, key0 + i);
      if (qb[i] > qa[i] && hit < 1.0 && qa[i] < 0.999) {  // did the crossing fall inside?
        const bool inside = hit >= qa[i] && hit <= qb[i];
        gw.half = inside ? std::max(0.02, 0.75 * gw.half) : std::min(0.24, 2.0 * gw.half);
      }
      gw.depth = hit;  // 1: no crossing
    }
  }

  // ---- the loop ----------------------------------------------------------
  int run_inner(const pdlpk_problem& P, const pdlpk_problem& parent_for_polish,
                const InnerCfg& cfg, Inner& D);

  bool attempt_polish(const pdlpk_problem& P, const InnerCfg& cfg, Inner& D);

  pdlpk_problem primal_feas_view(const pdlpk_problem& P) {
    pdlpk_problem Q = P;  // l_v, u_v (and their uniform flags) are P's
    Q.c = zeros_n_.get();
    Q.c_o = zeros_n_.get();
    Q.uniform = (P.uniform & ~1u) | (dist() ? 0u : 1u);  // c = +0.0 everywhere
    Q.c_u = 0.0;
    return Q;
  }

  // Which of the scaled c, l_v, u_v are bitwise uniform (one sync; after
  // preconditioning, which scales them in place).  Not on sharded solves.
  void detect_uniform() {
    prob_.uniform = 0;
    if (dist() || prob_.n == 0) return;
    DevBuf<unsigned long long> bits(6);
    const unsigned long long seed[6] = {0ull, ~0ull, 0ull, ~0ull, 0ull, ~0ull};
    PDLP_CK(cudaMemcpyAsync(bits.get(), seed, sizeof(seed), cudaMemcpyHostToDevice, s()));
    const double* v[3] = {prob_.c.get(), prob_.lv.get(), prob_.uv.get()};
    for (int q = 0; q < 3; ++q) PDLP_LAUNCH(pdlpk_uniform_bits(v[q], prob_.n, bits.get() + 2 * q, s()));
    unsigned long long h[6];
    PDLP_CK(cudaMemcpyAsync(h, bits.get(), sizeof(h), cudaMemcpyDeviceToHost, s()));
    PDLP_CK(cudaStreamSynchronize(s()));
    double* out[3] = {&prob_.c_u, &prob_.lv_u, &prob_.uv_u};
    for (int q = 0; q < 3; ++q) {
      if (h[2 * q] == h[2 * q + 1]) {
        prob_.uniform |= 1u << q;
        std::memcpy(out[q], &h[2 * q], sizeof(double));
      }
    }
  }

  pdlpk_problem dual_feas_view(const pdlpk_problem& P) {
    // build_dual_feasibility (problem.hpp:181-238) + swapped RescalingInfo
    // (solver.hpp:323-325): layouts swap roles, no matrix copy.
    if (sub_lc_.size() != static_cast<size_t>(P.n)) {
      sub_lc_.alloc(P.n);
      sub_uc_.alloc(P.n);
      sub_lv_.alloc(P.m);
      sub_uv_.alloc(P.m);
      sub_lc_o_.alloc(P.n);
      sub_uc_o_.alloc(P.n);
      sub_lv_o_.alloc(P.m);
      sub_uv_o_.alloc(P.m);
    }
    PDLP_LAUNCH(pdlpk_dual_feas_bounds(P.c, P.lv, P.uv, P.n, P.lc, P.uc, P.m, sub_lc_.get(),
                                       sub_uc_.get(), sub_lv_.get(), sub_uv_.get(), s()));
    PDLP_LAUNCH(pdlpk_dual_feas_bounds(P.c_o, P.lv_o, P.uv_o, P.n, P.lc_o, P.uc_o, P.m,
                                       sub_lc_o_.get(), sub_uc_o_.get(), sub_lv_o_.get(),
                                       sub_uv_o_.get(), s()));
    pdlpk_problem Q{};
    Q.m = P.n;
    Q.n = P.m;
    Q.K = P.KT;
    Q.KT = P.K;
    Q.c = zeros_m_.get();
    Q.c_o = zeros_m_.get();
    Q.uniform = dist() ? 0u : 1u;  // c = +0.0; the derived bounds are not checked
    Q.c_u = 0.0;
    Q.lc = sub_lc_.get();
    Q.uc = sub_uc_.get();
    Q.lv = sub_lv_.get();
    Q.uv = sub_uv_.get();
    Q.lc_o = sub_lc_o_.get();
    Q.uc_o = sub_uc_o_.get();
    Q.lv_o = sub_lv_o_.get();
    Q.uv_o = sub_uv_o_.get();
    Q.row_scale = P.col_scale;
    Q.col_scale = P.row_scale;
    return Q;
  }

  // public solve state
  pdlp_options opt_;
  bool parity_ = false;
  int shards_ = 4;
  std::unique_ptr<Stream> stream_;  // declared first: outlives every buffer
  std::unique_ptr<AllocStreamScope> alloc_scope_;
  // sharded solve
  Comm* comm_ = nullptr;
  const pdlp_shard_view* shard_in_ = nullptr;
  // column cut, during load: the shard's row layout and its by_row offsets
  const pdlp_csr_view* shard_rows_ = nullptr;
  const int64_t* shard_row_entry_offset_ = nullptr;
  // first non-finite entry (code << 3 | kind) of the column cut's row
  // layout -> its whole-problem by_row position (entries of a row keep
  // their order, rows ascend: the first local one is the first global one)
  unsigned long long col_cut_entry(unsigned long long key) const {
    if (shard_rows_ == nullptr || shard_row_entry_offset_ == nullptr || shard_rows_->start == nullptr) {
      return key;
    }
    const int64_t k = static_cast<int64_t>(key >> 3);
    const int64_t* st = shard_rows_->start;
    const int64_t r = std::upper_bound(st, st + shard_rows_->primary_dim + 1, k) - st - 1;
    const int64_t g = k + shard_row_entry_offset_[r];
    return (static_cast<unsigned long long>(g) << 3) | (key & 7ull);
  }
  pdlp_shard_plan plan_{};
  int64_t m_glob_ = 0, n_glob_ = 0;
  pdlpk_red_log red_log_{};
  DevBuf<double> gbuf_, pbuf_, slots_all_, flag_;
  // Reduce-scatter folded into the consumer (PDLP_PEER_RS=0 restores the
  // NCCL reduce-scatter): every rank writes its partial product into a
  // peer-mappable buffer; after a stream-level barrier each owner reads its
  // block from all ranks over NVLink inside the epilogue kernel.
  double* peer_pbuf_ = nullptr;
  pdlpk_peer_sum peers_{};
  // all-gather folded into the primal pass: peers store their x-bar blocks
  // straight into this rank's gathered vector
  double* peer_gather_ = nullptr;
  pdlpk_peer_sum push_{};
  bool peer_pending_ = false;  // a peer-read kernel may still be reading

  DevBuf<double> fc_c_, fc_lv_, fc_uv_, fc_zero_, fr_lc_, fr_uc_, fr_zero_;
  DevBuf<double> fs_lc_, fs_uc_, fs_lv_, fs_uv_;
  DevBuf<double> gq_[2][4];
  DevBuf<double> rows_full_;  // a sharded result's gathered vector
  pdlpk_problem full_main_{}, full_primal_{}, full_dual_{};
  DevProblem prob_;
  DevBuf<double> slots_;
  double* host_slots_ = nullptr;
  DevBuf<double> red_scratch_;
  DevBuf<char> gap_work_[2];
  bool gap_shared_ = false;  // one gap buffer, queries evaluated one at a time
  // distributed gap (sharded solves): PDLP_GAP_GATHERED=1 restores the
  // gathered evaluation, PDLP_GAPD_CHECK=1 runs both and records the
  // difference, PDLP_GAPD_FINAL = bracket size swept after the search
  bool gap_gathered_ = std::getenv("PDLP_GAP_GATHERED") != nullptr &&
                       std::getenv("PDLP_GAP_GATHERED")[0] == '1';
  bool gap_check_ = std::getenv("PDLP_GAPD_CHECK") != nullptr &&
                    std::getenv("PDLP_GAPD_CHECK")[0] == '1';
  int64_t gapd_final_ = [] {
    const char* e = std::getenv("PDLP_GAPD_FINAL");
    const long long v = e != nullptr ? std::atoll(e) : 0;
    return v > 0 ? static_cast<int64_t>(v) : int64_t(1) << 15;
  }();
  DevBuf<double> gapd_buf_;
  DevBuf<char> gapd_fwork_;
  int64_t gapd_final_cap_ = 0;
  std::vector<double> gapd_host_;
  double gapd_lambda_[2] = {0.0, 0.0};  // lambda* of the last evaluations (checks)
  bool gap_whole() const { return !dist() || gap_gathered_ || gap_check_; }
  std::map<std::pair<const void*, int>, GapWindow> gap_windows_;
  // The cadence's side stream (the window average's share, the second gap
  // query), created on first use: the engine's device is current then.
  void ensure_side() {
    if (gap_side_) return;
    gap_side_ = std::make_unique<Stream>();
    gap_fork_ = std::make_unique<Event>();
    gap_join_ = std::make_unique<Event>();
    gap_scratch2_.alloc(red_scratch_.size());
  }
  // Products on the side stream run concurrently with products of the same
  // layouts on the main stream.  A layout's multi-chunk lines combine through
  // per-layout scratch (chunk_part, chunk_cnt arrival counters, line_acc), so
  // the side stream works on a copy of the layout's view whose scratch is its
  // own (keyed by the main scratch; counters start at zero and the last CTA
  // of each line resets them).
  struct SideScratch {
    DevBuf<double> part, acc;
    DevBuf<unsigned> cnt;
  };
  std::map<const void*, SideScratch> side_scratch_;
  pdlpk_csr side_csr(const pdlpk_csr& A) {
    pdlpk_csr B = A;
    if (A.n_chunks == 0) return B;
    SideScratch& sc = side_scratch_[static_cast<const void*>(A.chunk_cnt)];
    if (sc.cnt.size() < static_cast<size_t>(A.n_chunks)) {
      sc.part.alloc(A.n_chunks);
      sc.cnt.alloc(A.n_chunks);
      PDLP_CK(cudaMemsetAsync(sc.cnt.get(), 0, A.n_chunks * sizeof(unsigned), g_alloc_stream));
      PDLP_CK(cudaStreamSynchronize(g_alloc_stream));
    }
    if (sc.acc.size() < static_cast<size_t>(A.n_multi * PDLPK_LINE_ACC)) {
      sc.acc.alloc(A.n_multi * PDLPK_LINE_ACC);
    }
    B.chunk_part = sc.part.get();
    B.chunk_cnt = sc.cnt.get();
    B.line_acc = sc.acc.get();
    return B;
  }
  pdlpk_problem side_problem(const pdlpk_problem& P) {
    pdlpk_problem Q = P;
    Q.K = side_csr(P.K);
    Q.KT = side_csr(P.KT);
    return Q;
  }
  // ---- column panels of the row pass (kernels.h n_row_panels) ----------
  // Perf mode on one GPU when the gathered x-bar is larger than L2 can keep
  // next to the pass's streams: the row layout is re-laid out as np CSR
  // matrices over consecutive column ranges of `width` columns, so each
  // launch of the row pass gathers from an x-bar range that stays in L2.
  // The panel plan's own stream (created with the engine; declared before
  // panels_ so the panel buffers, which free on it, go first).
  std::unique_ptr<Stream> panel_stream_;
  struct Panels {
    int np = 0;
    int64_t width = 0;
    std::vector<DevLayout> L;
    std::vector<pdlpk_csr> views;
    DevBuf<double> carry;
  } panels_;

  static int panel_count(int64_t n, int64_t nnz, int64_t m) {
    if (const char* e = std::getenv("PDLP_ROW_PANELS")) {
      const int v = std::atoi(e);
      return v >= 2 ? std::min(v, PDLPK_MAX_ROW_PANELS) : 0;
    }
    // x-bar above 48 MB and a matrix large enough for the gathers to
    // dominate; at most 4 panels (each launch re-reads the m-length row
    // pointers and carries)
    // each launch re-reads the row pointers and the 8-byte carries (16 B per
    // row and panel): only rows of >= 8 entries amortize that (C3's 2.5-entry
    // rows measured 331 -> 807 us with 4 panels)
    const double mb = 8.0 * static_cast<double>(n) / 1048576.0;
    if (mb <= 48.0 || nnz < (int64_t(16) << 20) || nnz < 8 * m) return 0;
    const int np = static_cast<int>(std::ceil(mb / 40.0));
    return np <= 4 ? np : 0;
  }

  // Host part (structure and schedules) from the caller's row layout; the
  // device arrays are filled from the scaled values by fill_panels().
  void plan_panels(const pdlp_csr_view& v, int64_t n, cudaStream_t ps) {
    panels_ = Panels{};
    if (parity_ || comm_ != nullptr || v.primary_dim <= 0) return;
    const int np = panel_count(n, v.nnz, v.primary_dim);
    if (np < 2) return;
    const int64_t m = v.primary_dim;
    const int64_t width = (n + np - 1) / np;
    std::vector<std::vector<int64_t>> st(static_cast<size_t>(np), std::vector<int64_t>(m + 1, 0));
    for_segments(m, 16, [&](int, int64_t lo, int64_t hi) {
      for (int64_t r = lo; r < hi; ++r) {
        const int64_t* b = v.index + v.start[r];
        const int64_t* e = v.index + v.start[r + 1];
        const int64_t* prev = b;
        for (int q = 0; q < np; ++q) {
          const int64_t* cut = q + 1 < np ? std::lower_bound(prev, e, (q + 1) * width) : e;
          st[q][r + 1] = cut - prev;  // count, prefix-summed below
          prev = cut;
        }
      }
    });
    for (int q = 0; q < np; ++q) {
      for (int64_t r = 0; r < m; ++r) st[q][r + 1] += st[q][r];
      if (st[q][m] >= (int64_t(1) << 31) - 1) return;  // 32-bit panel starts only
    }
    panels_.np = np;
    panels_.width = width;
    panels_.L.resize(static_cast<size_t>(np));
    panels_.views.resize(static_cast<size_t>(np));
    for (int q = 0; q < np; ++q) {
      DevLayout& L = panels_.L[static_cast<size_t>(q)];
      const int64_t nz = st[q][m];
      L.start32.alloc(m + 1);
      std::vector<int32_t> s32(st[q].begin(), st[q].end());
      PDLP_CK(cudaMemcpyAsync(L.start32.get(), s32.data(), (m + 1) * 4, cudaMemcpyHostToDevice, ps));
      PDLP_CK(cudaStreamSynchronize(ps));
      L.index.alloc(nz);
      L.value.alloc(nz);
      L.view.dim = m;
      L.view.nnz = nz;
      L.view.wide = 0;
      L.view.start = L.start32.get();
      L.view.index = L.index.get();
      L.view.value = L.value.get();
      L.view.value_orig = nullptr;
      // staged operands: none (first), the carry (middle), y, l_c, u_c and
      // the carry (last)
      const int32_t staged = q == 0 ? 0 : (q == np - 1 ? 4 : 1);
      const char* eb = std::getenv("PDLP_PANEL_BUDGET");
      const int32_t budget = pdlpk_stage_budget(eb != nullptr ? std::atoi(eb) : 2016);
      const char* es = std::getenv("PDLP_PANEL_SEG");
      if (es != nullptr && es[0] == '1') {
        build_seg_schedule(st[q].data(), m, L, 2048);
      } else {
        build_schedule(st[q].data(), m, L, 64, budget, staged);
      }
      panels_.views[static_cast<size_t>(q)] = L.view;
    }
    panels_.carry.alloc(m);
  }

  // The panels' host plan and schedules are built on a background thread
  // while the column layout uploads (load_parts); joined before use.
  struct Joiner {  // joins on every path, incl. a constructor that throws
    std::thread t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } panel_thread_;
  std::exception_ptr panel_err_;
  void start_panel_plan(const pdlp_csr_view& v, int64_t n) {
    if (parity_ || comm_ != nullptr || !starts_valid(v.start, v.primary_dim, v.nnz)) return;
    const int dev = opt_.device;
    if (!panel_stream_) panel_stream_ = std::make_unique<Stream>();
    const cudaStream_t ps = panel_stream_->get();
    panel_thread_.t = std::thread([this, v, n, dev, ps] {
      try {
        PDLP_CK(cudaSetDevice(dev));
        AllocStreamScope scope(ps);  // the panel buffers live on (and free on) this stream
        plan_panels(v, n, ps);
        PDLP_CK(cudaStreamSynchronize(ps));
      } catch (...) {
        panel_err_ = std::current_exception();
      }
    });
  }
  void join_panels() {
    if (panel_thread_.t.joinable()) panel_thread_.t.join();
    if (panel_err_) {
      std::exception_ptr e = panel_err_;
      panel_err_ = nullptr;
      std::rethrow_exception(e);
    }
  }

  void fill_panels() {
    if (panels_.np < 2) return;
    pdlpk_panel_ptrs pp{};
    pp.np = panels_.np;
    for (int q = 0; q < panels_.np; ++q) {
      DevLayout& L = panels_.L[static_cast<size_t>(q)];
      pp.start[q] = L.start32.get();
      pp.idx[q] = L.index.get();
      pp.val[q] = L.value.get();
    }
    PDLP_LAUNCH(pdlpk_panel_scatter(&prob_.row.view, &pp, s()));
  }

  bool uses_panels(const pdlpk_problem& P) const {
    return panels_.np >= 2 && P.K.index == prob_.row.view.index && !sell_ready_;
  }

  // ---- sliced-ELL row pass (measurement knob PDLP_ROW_SELL=1) -------------
  // Perf mode, one GPU: a SELL-32 copy of the scaled row layout (kernels.h
  // pdlpk_step_args::sell) built after preconditioning; the step's row pass
  // then runs row_pass_sell on the main problem and the primal polishing
  // subproblem (the same K).  Lab numbers and why it is off: DESIGN section 4.
  DevBuf<int64_t> sell_off_, sell_w32_;
  DevBuf<int32_t> sell_idx_;
  DevBuf<double> sell_val_;
  DevBuf<unsigned char> sell_tmp_;
  int64_t sell_ng_ = 0;
  int32_t sell_blocks_ = 0;
  bool sell_ready_ = false;
  void build_sell() {
    sell_ready_ = false;
    const char* e = std::getenv("PDLP_ROW_SELL");
    if (e == nullptr || e[0] != '1' || parity_ || comm_ != nullptr) return;
    const pdlpk_csr& K = prob_.row.view;
    if (K.dim <= 0 || K.nnz <= 0) return;
    sell_ng_ = (K.dim + 31) / 32;
    sell_off_.alloc(static_cast<size_t>(sell_ng_ + 1));
    sell_w32_.alloc(static_cast<size_t>(sell_ng_));
    size_t tb = 0;
    PDLP_LAUNCH(pdlpk_sell_plan(&K, sell_w32_.get(), sell_off_.get(), nullptr, &tb, s()));
    sell_tmp_.alloc(tb + 16);
    PDLP_LAUNCH(pdlpk_sell_plan(&K, sell_w32_.get(), sell_off_.get(), sell_tmp_.get(), &tb, s()));
    int64_t slots = 0;
    PDLP_CK(cudaMemcpyAsync(&slots, sell_off_.get() + sell_ng_, sizeof(int64_t), cudaMemcpyDeviceToHost, s()));
    PDLP_CK(cudaStreamSynchronize(s()));
    if (slots <= 0 || slots > 4 * K.nnz + 32 * sell_ng_) return;  // padding out of hand: keep the tiles
    sell_idx_.alloc(static_cast<size_t>(slots));
    sell_val_.alloc(static_cast<size_t>(slots));
    PDLP_LAUNCH(pdlpk_sell_fill(&K, sell_off_.get(), sell_idx_.get(), sell_val_.get(), s()));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, opt_.device);
    int per_sm = 4;  // PDLP_SELL_CTAS: CTAs per SM of the pass (measurement)
    if (const char* c = std::getenv("PDLP_SELL_CTAS")) per_sm = std::max(1, std::atoi(c));
    sell_blocks_ = static_cast<int32_t>(std::min<int64_t>(static_cast<int64_t>(per_sm) * sms, (sell_ng_ + 7) / 8));
    sell_ready_ = true;
    if (opt_.logging) {
      std::fprintf(stderr, "phase=setup event=row_sell slices=%lld slots=%lld padding=%.3f\n",
                   static_cast<long long>(sell_ng_), static_cast<long long>(slots),
                   static_cast<double>(slots) / static_cast<double>(K.nnz));
    }
  }
  bool uses_sell(const pdlpk_problem& P) const {
    return sell_ready_ && P.K.index == prob_.row.view.index && P.K.value == prob_.row.view.value;
  }

  // ---- multi-vector cadence products (k_multi.cu) ------------------------
  // Perf mode, one GPU, layouts of >= 16M entries: the cadence's products
  // of the current iterate, the window average and the ray candidates go
  // through one pass per layout (2 operands through K, up to 4 through K').
  // They need a segmented-span schedule on both layouts; the row layout
  // keeps its tiles for the step and gets a second, span schedule here.
  DevLayout mrow_;
  bool mrow_ready_ = false;
  DevBuf<double> multi_pack_, multi_part_, multi_prod_[2];
  void build_multi_row(const pdlp_csr_view& v) {
    mrow_ready_ = false;
    const char* e = std::getenv("PDLP_MULTI");  // 0: off; 1: also below 16M entries
    const bool force = e != nullptr && e[0] == '1';
    if (parity_ || comm_ != nullptr || (e != nullptr && e[0] == '0') ||
        (!force && prob_.row.view.nnz < (int64_t(16) << 20)) ||
        !starts_valid(v.start, v.primary_dim, v.nnz)) {
      return;
    }
    if (prob_.row.view.seg_mode) {  // the row layout's own schedule serves
      mrow_ready_ = false;
      multi_on_ = true;
      return;
    }
    build_seg_schedule(v.start, v.primary_dim, mrow_, 2048);
    const pdlpk_csr& R = prob_.row.view;
    mrow_.view.dim = R.dim;
    mrow_.view.nnz = R.nnz;
    mrow_.view.start = R.start;
    mrow_.view.wide = R.wide;
    mrow_.view.index = R.index;
    mrow_.view.value = R.value;
    mrow_.view.value_orig = R.value_orig;
    mrow_.view.dist_kind = R.dist_kind;
    mrow_ready_ = true;
    multi_on_ = true;
  }
  bool multi_on_ = false;  // multi products enabled for this problem
  // the span-scheduled view of a layout used by the multi products, or null
  const pdlpk_csr* multi_view(const pdlpk_csr& A) const {
    if (!multi_on_) return nullptr;
    if (A.seg_mode) return &A;
    if (mrow_ready_ && A.index == prob_.row.view.index) return &mrow_.view;
    return nullptr;
  }
  // out[q] = A in[q], q < k (k <= 4; padded to 2 or 4 with a scratch output)
  void multi_product(const pdlpk_csr& A, int k, double* const* in, double* const* out,
                     int64_t operand_len) {
    const pdlpk_csr* V = multi_view(A);
    const int vec = k <= 2 ? 2 : 4;
    pdlpk_multi_vecs vi{}, vo{};
    for (int q = 0; q < vec; ++q) {
      vi.v[q] = in[q < k ? q : 0];
      vo.v[q] = q < k ? out[q] : multi_prod_[1].get();
    }
    const size_t pack = static_cast<size_t>(vec) * static_cast<size_t>(std::max<int64_t>(operand_len, 1));
    if (multi_pack_.size() < pack) multi_pack_.alloc(pack);
    const size_t part = static_cast<size_t>(vec) * static_cast<size_t>(std::max<int64_t>(V->n_chunks, 1));
    if (multi_part_.size() < part) multi_part_.alloc(part);
    PDLP_LAUNCH(pdlpk_spmv_multi(V, 0, vec, &vi, operand_len, multi_pack_.get(), &vo,
                                 multi_part_.get(), s()));
  }
  DevBuf<double> side_prod_;  // the average ray's A^T product
  std::unique_ptr<Stream> gap_side_;  // second gap query's stream
  DevBuf<double> gap_scratch2_;
  std::unique_ptr<Event> gap_fork_, gap_join_;
  // PDLP_GAP_SERIAL=1: both gap queries on the main stream (measurements)
  bool gap_serial_ = [] {
    const char* e = std::getenv("PDLP_GAP_SERIAL");
    return e != nullptr && e[0] == '1';
  }();
  // PDLP_GAP_PARTIAL=0: always the full sort (measurements)
  // PDLP_LINE_PARTIALS=0: per-CTA row-pass partials (schedule-dependent)
  bool line_partials_on_ = [] {
    const char* e = std::getenv("PDLP_LINE_PARTIALS");
    return !(e != nullptr && e[0] == '0');
  }();
  bool gap_any_window_ = [] {
    const char* e = std::getenv("PDLP_GAP_WINDOWS");
    return !(e != nullptr && std::strcmp(e, "top") == 0);
  }();
  bool gap_partial_off_ = [] {
    const char* e = std::getenv("PDLP_GAP_PARTIAL");
    return e != nullptr && e[0] == '0';
  }();
  DevBuf<int> islots_;
  int* host_islots_ = nullptr;
  DevBuf<double> zeros_n_, zeros_m_;
  DevBuf<int32_t> row_of_, col_of_;  // line of each entry, both layouts
  DevBuf<double> sub_lc_, sub_uc_, sub_lv_, sub_uv_, sub_lc_o_, sub_uc_o_, sub_lv_o_, sub_uv_o_;
  DevBuf<double> f_down_, f_up_;
  int64_t table_len_ = 0;
  Event step_begin_, step_end_;
  double step_seconds_ = 0.0;
  double upload_seconds_ = 0.0;
  double precondition_seconds_ = 0.0;
  double cadence_seconds_ = 0.0;  // host time inside cadence blocks (incl. polishing)
  double polish_seconds_ = 0.0;
  double gap_seconds_ = 0.0;  // host time in normalized-gap evaluations (syncs included)
  double cad_batch_seconds_ = 0.0;    // cadence: products, screens, ray tests up to the one sync
  double cad_capture_seconds_ = 0.0;  // cadence: final original-space summary on a budget hit
  int64_t attempts_total_ = 0;
  bool profile_ = false;
  std::vector<cudaEvent_t> prof_ev_;
  double kernel_seconds_[4] = {0, 0, 0, 0};
  int64_t kernel_launches_[4] = {0, 0, 0, 0};
  int64_t timing_warmup_ = 0;
  bool timing_started_ = false;
  int64_t timed_k0_ = 0, timed_att0_ = 0;
  Event timed_begin_, timed_end_;
  Inner main_, polish_primal_, polish_dual_;
};

bool Engine::attempt_polish(const pdlpk_problem& P, const InnerCfg& cfg, Inner& D) {
  // solver.hpp:290-348
  NvtxRange nvtx("pdlp:polish");
  const auto pol_t0 = Clock::now();
  struct PolishClock {
    double& acc;
    Clock::time_point t0;
    ~PolishClock() { acc += std::chrono::duration<double>(Clock::now() - t0).count(); }
  } pol_clock{polish_seconds_, pol_t0};
  const int64_t remaining = cfg.budget - D.k() - D.polish_iterations;
  const int64_t budget = std::min(D.k() / 8, remaining);
  if (budget <= 0) return false;
  InnerCfg sub = cfg;
  sub.feasibility_only = true;
  sub.rc_mode = 0;
  sub.budget = budget;
  sub.detect_infeasibility = false;
  sub.enable_polish = false;
  sub.observer = nullptr;

  const pdlpk_problem P2 = primal_feas_view(P);
  Inner& D2 = polish_primal_;
  if (dist()) {
    sub.full = &full_primal_;
    sub.swapped = false;
  }
  prepare(D2, P2, D.avg_x.get(), D.hs.eta, D.omega, cfg.fixed_eta.has_value());
  sub.tag = "polish_primal";
  const int s2 = run_inner(P2, P2, sub, D2);
  D.polish_iterations += D2.k();
  attempts_total_ += D2.hs.attempts;
  if (s2 != kOptimal) return false;

  const pdlpk_problem P3 = dual_feas_view(P);
  Inner& D3 = polish_dual_;
  prepare(D3, P3, D.avg_y.get(), D.hs.eta, D.omega, cfg.fixed_eta.has_value());
  sub.budget = std::min(D.k() / 8, remaining - D2.k());
  if (sub.budget <= 0) return false;
  sub.tol.eps_primal = cfg.tol.eps_dual;
  sub.tag = "polish_dual";
  if (dist()) {
    sub.full = &full_dual_;
    sub.swapped = true;
  }
  const int s3 = run_inner(P3, P3, sub, D3);
  D.polish_iterations += D3.k();
  attempts_total_ += D3.hs.attempts;
  if (s3 != kOptimal) return false;

  // Stitch (x from the primal polish, y from the dual polish) and re-check.
  const Summary truth = original_kkt(P, D2.sol_x.get(), D3.sol_x.get(), 0, D.tmp_r.get(), D);
  if (!check_termination(truth, cfg.tol)) return false;
  dev_copy(D.sol_x.get(), D2.sol_x.get(), P.n, s());
  dev_copy(D.sol_y.get(), D3.sol_x.get(), P.m, s());
  D.sol_r.swap(D.tmp_r);
  D.sol_summary = truth;
  D.have_sol = true;
  D.detail = "converged at the polished point";
  return true;
}

int Engine::run_inner(const pdlpk_problem& P, const pdlpk_problem&, const InnerCfg& cfg,
                      Inner& D) {
  Summary screen_cur;
  while (true) {
    const bool budget_hit = D.k() >= cfg.budget;
    const bool at_cadence = budget_hit || (D.k() % cfg.check_interval == 0);
    if (at_cadence) {
      NvtxRange nvtx("pdlp:cadence");
      const auto cad_t0 = Clock::now();
      struct CadenceClock {  // adds the cadence's host time on every exit
        double& acc;
        Clock::time_point t0;
        ~CadenceClock() { acc += std::chrono::duration<double>(Clock::now() - t0).count(); }
      } cad_clock{cadence_seconds_, cad_t0};
      bool timed_out = cad_t0 >= cfg.deadline;
      if (dist()) timed_out = any_rank(timed_out);  // ranks must agree
      const int c = D.cur();
      flush_average(P, D);
      const bool have_avg = D.hs.avg_count > 0;
      const bool want_restart = cfg.enable_restarts && D.k() > D.k_last_restart;
      // One batch, one sync: both residual screens, every ray candidate's
      // scaled-space test, and the restart distances to the reference point.
      // Decisions below are then taken in the reference's order.  On one GPU
      // the window average's share (its products, screen, ray candidate and
      // distances) runs on the side stream with its own reduction scratch:
      // the same kernels on the same inputs, overlapped.
      const pdlpk_red rr = red();
      // multi-vector products (perf mode, both layouts span-scheduled): the
      // cadence's products in one pass per layout, all on the main stream
      const bool multi = have_avg && !dist() && !parity_ && multi_view(P.K) != nullptr &&
                         multi_view(P.KT) != nullptr;
      const bool side = have_avg && !dist() && !gap_serial_ && !multi;
      cudaStream_t sa = s();
      pdlpk_red ra = rr;
      double* prod_a = D.prod_n.get();
      pdlpk_problem Ps = P;  // the side stream's view: own chunk scratch
      if (side) {
        ensure_side();
        Ps = side_problem(P);
        sa = gap_side_->get();
        ra.scratch = gap_scratch2_.get();
        if (side_prod_.size() < static_cast<size_t>(P.n)) side_prod_.alloc(P.n);
        prod_a = side_prod_.get();
        gap_fork_->record(s());
        PDLP_CK(cudaStreamWaitEvent(sa, gap_fork_->get(), 0));
      }
      std::vector<RayCand> cands;
      if (cfg.detect_infeasibility) cands = ray_candidates(P, D, have_avg);
      std::vector<size_t> joint;  // ray candidates whose K' product joins the multi pass
      if (multi) {
        PDLP_LAUNCH(pdlpk_average_into(D.state.get(), D.sum_x.get(), D.sum_y.get(), D.avg_x.get(),
                                       D.avg_y.get(), P.n, P.m, s()));
        for (size_t q = 0; q < cands.size() && joint.size() < 2; ++q) {
          if (cands[q].known_aty != D.aty[c].get()) joint.push_back(q);  // difference, average
        }
        for (size_t q : joint) {
          PDLP_LAUNCH(pdlpk_ray_primal_prep(&P, 0, cands[q].y, D.ray_y[q].get(), &rr,
                                            slot(kSlotRay + 8 * static_cast<int>(q)), s()));
        }
        for (auto& b : multi_prod_) {
          if (b.size() < static_cast<size_t>(P.n)) b.alloc(P.n);
        }
        double* in_k[2] = {D.x[c].get(), D.avg_x.get()};
        double* out_k[2] = {D.ax_cur.get(), D.ax_avg.get()};
        multi_product(P.K, 2, in_k, out_k, P.n);
        double* in_t[4] = {D.y[c].get(), D.avg_y.get(), nullptr, nullptr};
        double* out_t[4] = {D.aty[c].get(), D.aty_avg.get(), nullptr, nullptr};
        for (size_t j = 0; j < joint.size(); ++j) {
          in_t[2 + j] = D.ray_y[joint[j]].get();
          out_t[2 + j] = j == 0 ? D.prod_n.get() : multi_prod_[0].get();
        }
        multi_product(P.KT, 2 + static_cast<int>(joint.size()), in_t, out_t, P.m);
        for (size_t j = 0; j < joint.size(); ++j) {
          const size_t q = joint[j];
          double* sl = slot(kSlotRay + 8 * static_cast<int>(q));
          PDLP_LAUNCH(pdlpk_ray_primal_finish(&P, 0, D.ray_y[q].get(), out_t[2 + j], nullptr, sl + 1,
                                              D.rhat[q].get(), &rr, sl + 2, s()));
          PDLP_LAUNCH(pdlpk_ray_dual_prep(&P, 0, cands[q].x, &rr, sl + 4, s()));
        }
        PDLP_LAUNCH(pdlpk_screen(&P, 0, D.avg_x.get(), D.avg_y.get(), D.ax_avg.get(),
                                 D.aty_avg.get(), cfg.rc_mode, &rr, D.rc_b.get(),
                                 slot(kSlotScrAvg), s()));
        if (want_restart) {
          PDLP_LAUNCH(pdlpk_diff_norm_sq(D.avg_x.get(), D.ref_x.get(), P.n, &rr, slot(kSlotDist + 2), s()));
          PDLP_LAUNCH(pdlpk_diff_norm_sq(D.avg_y.get(), D.ref_y.get(), P.m, &rr, slot(kSlotDist + 3), s()));
        }
      } else if (have_avg) {
        PDLP_LAUNCH(pdlpk_average_into(D.state.get(), D.sum_x.get(), D.sum_y.get(), D.avg_x.get(),
                                       D.avg_y.get(), P.n, P.m, sa));
        if (side) {
          PDLP_LAUNCH(pdlpk_spmv(&Ps.K, 0, D.avg_x.get(), D.ax_avg.get(), parity_, sa));
          PDLP_LAUNCH(pdlpk_spmv(&Ps.KT, 0, D.avg_y.get(), D.aty_avg.get(), parity_, sa));
          PDLP_LAUNCH(pdlpk_screen(&Ps, 0, D.avg_x.get(), D.avg_y.get(), D.ax_avg.get(),
                                   D.aty_avg.get(), cfg.rc_mode, &ra, D.rc_b.get(),
                                   slot(kSlotScrAvg), sa));
          if (cfg.detect_infeasibility) {
            enqueue_rays(Ps, D, cands, cands.size() - 1, cands.size(), sa, &ra, prod_a);
          }
          if (want_restart) {
            PDLP_LAUNCH(pdlpk_diff_norm_sq(D.avg_x.get(), D.ref_x.get(), P.n, &ra,
                                           slot(kSlotDist + 2), sa));
            PDLP_LAUNCH(pdlpk_diff_norm_sq(D.avg_y.get(), D.ref_y.get(), P.m, &ra,
                                           slot(kSlotDist + 3), sa));
          }
        }
      }
      if (!multi) {
        product(P.K, 0, D.x[c].get(), D.ax_cur.get());
        product(P.KT, 0, D.y[c].get(), D.aty[c].get());
      }
      D.fresh_products_k = D.k();
      if (have_avg && !side && !multi) {
        product(P.K, 0, D.avg_x.get(), D.ax_avg.get());
        product(P.KT, 0, D.avg_y.get(), D.aty_avg.get());
      }
      PDLP_LAUNCH(pdlpk_screen(&P, 0, D.x[c].get(), D.y[c].get(), D.ax_cur.get(), D.aty[c].get(),
                               cfg.rc_mode, &rr, D.rc_a.get(), slot(kSlotScrCur), s()));
      if (have_avg && !side && !multi) {
        PDLP_LAUNCH(pdlpk_screen(&P, 0, D.avg_x.get(), D.avg_y.get(), D.ax_avg.get(),
                                 D.aty_avg.get(), cfg.rc_mode, &rr, D.rc_b.get(),
                                 slot(kSlotScrAvg), s()));
      }
      if (cfg.detect_infeasibility) {
        if (multi) {
          for (size_t q = 0; q < cands.size(); ++q) {  // the rest (the current iterate's ray)
            if (std::find(joint.begin(), joint.end(), q) == joint.end()) enqueue_rays(P, D, cands, q, q + 1);
          }
        } else {
          enqueue_rays(P, D, cands, 0, side ? cands.size() - 1 : cands.size());
        }
      }
      if (want_restart) {
        PDLP_LAUNCH(pdlpk_diff_norm_sq(D.x[c].get(), D.ref_x.get(), P.n, &rr, slot(kSlotDist), s()));
        PDLP_LAUNCH(pdlpk_diff_norm_sq(D.y[c].get(), D.ref_y.get(), P.m, &rr, slot(kSlotDist + 1), s()));
        if (have_avg && !side && !multi) {
          PDLP_LAUNCH(pdlpk_diff_norm_sq(D.avg_x.get(), D.ref_x.get(), P.n, &rr, slot(kSlotDist + 2), s()));
          PDLP_LAUNCH(pdlpk_diff_norm_sq(D.avg_y.get(), D.ref_y.get(), P.m, &rr, slot(kSlotDist + 3), s()));
        }
      }
      if (side) {
        gap_join_->record(sa);
        PDLP_CK(cudaStreamWaitEvent(s(), gap_join_->get(), 0));
      }
      double h[kSlots];
      std::memcpy(h, read_slots(kSlots), sizeof(h));
      cad_batch_seconds_ += std::chrono::duration<double>(Clock::now() - cad_t0).count();
      screen_cur = finish_summary(h[kSlotScrCur], h[kSlotScrCur + 1], h[kSlotScrCur + 2],
                                  -h[kSlotScrCur + 3]);
      if (screen_passes(cfg, screen_cur) &&
          verify_point(P, cfg, D.x[c].get(), D.y[c].get(), D, "current iterate")) {
        return kOptimal;
      }
      Summary screen_avg;
      if (have_avg) {
        screen_avg = finish_summary(h[kSlotScrAvg], h[kSlotScrAvg + 1], h[kSlotScrAvg + 2],
                                    -h[kSlotScrAvg + 3]);
        if (screen_passes(cfg, screen_avg) &&
            verify_point(P, cfg, D.avg_x.get(), D.avg_y.get(), D, "window average")) {
          return kOptimal;
        }
      }
      if (cfg.detect_infeasibility) {
        auto st = detect_rays(P, cfg, D, cands, h);
        if (st.has_value()) {
          const std::string keep = D.detail;
          capture_current(P, cfg, D);
          D.detail = keep;
          return *st;
        }
      }
      if (cfg.enable_polish && have_avg && D.k() >= D.next_polish_trigger && !timed_out &&
          !budget_hit) {
        if (screen_avg.rel_gap <= cfg.tol.eps_rel_gap) {
          if (attempt_polish(P, cfg, D)) return kOptimal;
          while (D.next_polish_trigger <= D.k()) D.next_polish_trigger *= 2;
        }
      }
      if (want_restart) {
        // restart_progress_metric of current and average (solver.hpp:405-412)
        GapQuery q[2] = {
            {D.x[c].get(), D.y[c].get(), D.ax_cur.get(), D.aty[c].get(), h[kSlotDist],
             h[kSlotDist + 1]},
            {D.avg_x.get(), D.avg_y.get(), D.ax_avg.get(), D.aty_avg.get(), h[kSlotDist + 2],
             h[kSlotDist + 3]}};
        double mu[2] = {0.0, kInf};
        gaps(cfg, P, q, have_avg ? 2 : 1, D.omega, mu);
        const double mu_cur = mu[0];
        const double mu_avg = have_avg ? mu[1] : kInf;
        const bool use_current = mu_cur < mu_avg;
        const double cand_mu = use_current ? mu_cur : mu_avg;
        const int reason = should_restart(cand_mu, D.mu_last, D.prev_candidate_mu,
                                          D.k() - D.k_last_restart, D.k(), cfg.th);
        if (reason != kNone) {
          const GapQuery& cq = q[use_current ? 0 : 1];
          if (cfg.allow_omega_updates) {
            // diff_norm_sq(candidate, ref) is exactly the metric's distance
            D.omega = update_primal_weight(std::sqrt(cq.dx2), std::sqrt(cq.dy2), D.omega);
          }
          gaps(cfg, P, &cq, 1, D.omega, &D.mu_last, use_current ? 0 : 1);
          if (!use_current) {
            dev_copy(D.x[c].get(), D.avg_x.get(), P.n, s());
            dev_copy(D.y[c].get(), D.avg_y.get(), P.m, s());
            dev_copy(D.aty[c].get(), D.aty_avg.get(), P.n, s());
            dev_copy(D.ax_cur.get(), D.ax_avg.get(), P.m, s());  // (fresh products follow)
          }
          dev_copy(D.ref_x.get(), D.x[c].get(), P.n, s());
          dev_copy(D.ref_y.get(), D.y[c].get(), P.m, s());
          dev_zero(D.sum_x.get(), P.n, s());
          dev_zero(D.sum_y.get(), P.m, s());
          read_state(D);
          D.hs.avg_weight = 0.0;
          D.hs.avg_count = 0;
          D.hs.avg_pending = 0;
          D.hs.omega = D.omega;
          write_state(D);
          D.prev_candidate_mu = kInf;
          D.k_last_restart = D.k();
          ++D.restarts;
          if (cfg.logging) {
            std::fprintf(stderr, "phase=%s event=restart iter=%lld reason=%s omega=%.6e mu=%.6e\n",
                         cfg.tag, static_cast<long long>(D.k()), reason_name(reason), D.omega,
                         D.mu_last);
          }
        } else {
          D.prev_candidate_mu = cand_mu;
        }
      }
      if (cfg.logging) {
        std::fprintf(stderr,
                     "phase=%s iter=%lld primal_res=%.6e dual_res=%.6e rel_gap=%.6e mu=%.6e "
                     "omega=%.6e eta=%.6e restarts=%lld\n",
                     cfg.tag, static_cast<long long>(D.k()), screen_cur.primal, screen_cur.dual,
                     screen_cur.rel_gap, D.mu_last, D.omega, D.last_eta,
                     static_cast<long long>(D.restarts));
      }
      if (timed_out) {
        capture_current(P, cfg, D);
        D.detail = "time limit reached";
        return kTimeLimit;
      }
      if (budget_hit) {
        const auto tc = Clock::now();
        capture_current(P, cfg, D);
        PDLP_CK(cudaStreamSynchronize(s()));
        cad_capture_seconds_ += std::chrono::duration<double>(Clock::now() - tc).count();
        D.detail = "iteration limit reached";
        return kIterLimit;
      }
    }

    maybe_start_timer(D);
    // Accepted steps up to the next cadence point (or one, with an observer).
    int64_t target = (D.k() / cfg.check_interval + 1) * cfg.check_interval;
    target = std::min(target, cfg.budget);
    if (cfg.observer != nullptr) target = D.k() + 1;
    // A timed run whose warm-up ends inside this block stops there first, so
    // the timed region opens exactly after the warm-up (block boundaries
    // only decide when the host reads the controller: same values).
    if (!timing_started_ && &D == &main_ && timing_warmup_ > D.k() && timing_warmup_ < target) {
      target = timing_warmup_;
    }
    if (cfg.fixed_eta.has_value() && D.hs.eta != *cfg.fixed_eta) {
      D.hs.eta = *cfg.fixed_eta;
      write_state(D);
    }
    run_steps(P, D, target);
    D.last_eta = D.hs.eta_used;
    if (D.hs.status != 0) {
      if (!cfg.fixed_eta.has_value()) {
        // One recovery screen of the last good point and the window average
        // (solver.hpp:494-516).
        const int c = D.cur();
        product(P.K, 0, D.x[c].get(), D.ax_cur.get());
        Summary tmp;
        if (screen_and_verify(P, cfg, D.x[c].get(), D.y[c].get(), D.ax_cur.get(), D.aty[c].get(),
                              D.rc_a.get(), tmp, D, "current iterate after a numerical error")) {
          return kOptimal;
        }
        if (D.hs.avg_count > 0) {
          flush_average(P, D);
          PDLP_LAUNCH(pdlpk_average_into(D.state.get(), D.sum_x.get(), D.sum_y.get(),
                                         D.avg_x.get(), D.avg_y.get(), P.n, P.m, s()));
          product(P.K, 0, D.avg_x.get(), D.ax_avg.get());
          product(P.KT, 0, D.avg_y.get(), D.aty_avg.get());
          if (screen_and_verify(P, cfg, D.avg_x.get(), D.avg_y.get(), D.ax_avg.get(),
                                D.aty_avg.get(), D.rc_b.get(), tmp, D,
                                "window average after a numerical error")) {
            return kOptimal;
          }
        }
        capture_current(P, cfg, D);
        D.detail = "adaptive step failed to find a usable step size";
        return kNumErr;
      }
      capture_current(P, cfg, D);
      D.detail = "fixed-size step produced non-finite values";
      return kNumErr;
    }
    if (cfg.observer != nullptr) {
      const int c = D.cur();
      std::vector<double> hx(P.n), hy(P.m);
      if (P.n > 0) PDLP_CK(cudaMemcpyAsync(hx.data(), D.x[c].get(), P.n * 8, cudaMemcpyDeviceToHost, s()));
      if (P.m > 0) PDLP_CK(cudaMemcpyAsync(hy.data(), D.y[c].get(), P.m * 8, cudaMemcpyDeviceToHost, s()));
      PDLP_CK(cudaStreamSynchronize(s()));
      pdlp_iteration_record rec{};
      rec.iteration = D.k();
      rec.x = hx.data();
      rec.x_len = P.n;
      rec.y = hy.data();
      rec.y_len = P.m;
      rec.eta = D.hs.eta_used;
      rec.omega = D.omega;
      cfg.observer(cfg.observer_user, &rec);
    }
  }
}

void copy_to_host(double* dst, const double* src, int64_t n, cudaStream_t s) {
  if (dst != nullptr && n > 0) stage_d2h(dst, src, static_cast<size_t>(n) * 8, s);
}

// solve (solver.hpp:535-608)
// Inner state of an (n, m) loop: 24 n-vectors and 17 m-vectors (Inner::allocate).
int64_t inner_bytes(int64_t n, int64_t m) { return 8 * (24 * n + 17 * m) + 64 * 41; }

// comm != nullptr: this process/thread is one rank of a row-sharded solve.
void solve(const pdlp_problem_view* problem, const pdlp_options* opts, pdlp_result* res,
           Comm* comm = nullptr, const pdlp_shard_view* shard = nullptr) {
  const auto t0 = Clock::now();
  // sharded: one log (rank 0); every rank computes the same trajectory
  pdlp_options local = *opts;
  if (comm != nullptr && comm->rank() != 0) local.logging = 0;
  const pdlp_options* o = &local;
  g_alloc_seconds = 0.0;
  Engine E(problem, *o, comm, shard);  // uploads and validates on device
  if (o->enable_scaling) E.precondition(o->ruiz_passes, o->pock_chambolle != 0);
  if (std::getenv("PDLP_NO_UNIFORM") == nullptr) E.detect_uniform();
  if (!E.dist()) {
    E.join_panels();
    E.fill_panels();
    E.build_sell();
  }
  if (E.dist() && E.gap_whole()) E.build_full_views();
  // Polishing is only considered at a cadence point k >= 100 below the
  // iteration budget (solver.hpp:395-401; the first trigger is 100).
  const int64_t ci = o->check_interval > 0 ? o->check_interval : 64;
  const int64_t first_polish_k = (100 + ci - 1) / ci * ci;
  if (o->enable_polish && first_polish_k < o->iteration_limit) {
    // The polishing subproblems' states are allocated mid-loop, the first
    // time polishing triggers.  Growing the pool then costs 10-300 ms of
    // driver time; reserve it now (freed blocks stay in the retaining pool
    // and are sub-allocated later).  (A solve whose budget ends before the
    // first possible trigger skips it: the 4.7 GB reserve of C2 costs
    // 40-55 ms even on a warm pool.)
    // (Straight to the pool: through DevBuf the block would park in the
    // block cache instead of growing the pool.)
    const int64_t nl = E.problem().n, ml = E.problem().m;
    void* reserve = nullptr;
    const size_t rb = static_cast<size_t>(inner_bytes(nl, ml) + inner_bytes(ml, nl));
    const auto tr = std::chrono::steady_clock::now();
    if (cudaMallocAsync(&reserve, rb, E.s()) == cudaSuccess) {
      cudaFreeAsync(reserve, E.s());
    } else {
      cudaGetLastError();
    }
    g_alloc_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - tr).count();
  }
  const pdlpk_problem P = E.problem().view();

  InnerCfg cfg;
  cfg.tol.eps_primal = o->eps_primal;
  cfg.tol.eps_dual = o->eps_dual;
  cfg.tol.eps_rel_gap = o->eps_rel_gap;
  cfg.feasibility_only = false;
  cfg.rc_mode = o->enable_polish ? 0 : 1;
  cfg.budget = o->iteration_limit;
  if (std::isfinite(o->time_limit_seconds)) {
    cfg.deadline = t0 + std::chrono::duration_cast<Clock::duration>(
                            std::chrono::duration<double>(o->time_limit_seconds));
  }
  cfg.enable_restarts = o->enable_restarts != 0;
  cfg.detect_infeasibility = o->detect_infeasibility != 0;
  cfg.enable_polish = o->enable_polish != 0;
  cfg.eps_ray = o->eps_ray;
  cfg.check_interval = o->check_interval > 0 ? o->check_interval : 64;
  cfg.th.sufficient = o->restart_sufficient;
  cfg.th.necessary = o->restart_necessary;
  cfg.th.artificial = o->restart_artificial;
  if (o->has_fixed_step_size) cfg.fixed_eta = o->fixed_step_size;
  cfg.allow_omega_updates = o->has_fixed_primal_weight == 0;
  cfg.observer = o->observer;
  cfg.observer_user = o->observer_user;
  cfg.logging = o->logging != 0;
  cfg.tag = "main";
  if (E.dist()) cfg.full = &E.full_main_;

  const double eta0 = o->has_fixed_step_size ? o->fixed_step_size : E.initial_step_size();
  const double omega0 =
      o->has_fixed_primal_weight ? o->fixed_primal_weight : E.initialize_primal_weight();
  Inner& D = E.main_;
  {
    DevBuf<double> x0(P.n);
    PDLP_LAUNCH(pdlpk_initial_point(P.lv, P.uv, x0.get(), P.n, E.s()));
    E.prepare(D, P, x0.get(), eta0, omega0, cfg.fixed_eta.has_value());
  }
  E.ensure_table(std::min<int64_t>(o->iteration_limit, 1 << 20) + 2);

  E.profile_ = o->profile_kernels != 0;
  E.timing_warmup_ = std::max<int64_t>(0, o->timing_warmup_iterations);
  const auto loop_t0 = Clock::now();
  const double prep_seconds = std::chrono::duration<double>(loop_t0 - t0).count() -
                              E.upload_seconds_ - E.precondition_seconds_;
  const int status = E.run_inner(P, P, cfg, D);
  E.timed_end_.record(E.s());
  PDLP_CK(cudaStreamSynchronize(E.s()));
  const double loop_seconds = std::chrono::duration<double>(Clock::now() - loop_t0).count();
  if (E.timing_started_) {
    res->timed_seconds = elapsed_seconds(E.timed_begin_, E.timed_end_);
    res->timed_iterations = D.k() - E.timed_k0_;
    res->timed_attempts = D.hs.attempts - E.timed_att0_;
  }
  for (int q = 0; q < 4; ++q) {
    res->kernel_seconds[q] = E.kernel_seconds_[q];
    res->kernel_launches[q] = E.kernel_launches_[q];
  }

  res->status = status;
  // Sharded: every rank gathers the whole vectors (collectively, so every
  // rank makes the same calls) and returns the whole result.
  auto out_vec = [&](double* host, const double* dev, bool col_side) {
    if (!E.dist()) {
      copy_to_host(host, dev, col_side ? P.n : P.m, E.s());
      return;
    }
    const int64_t need = col_side ? E.full_cols() : E.full_rows();
    if (E.rows_full_.size() < static_cast<size_t>(need)) E.rows_full_.alloc(need);
    double* full = E.rows_full_.get();
    E.gather(dev, col_side ? P.n : P.m, col_side ? E.plan_.col_block : E.plan_.row_block, full);
    copy_to_host(host, full, col_side ? E.n_glob_ : E.m_glob_, E.s());
    PDLP_CK(cudaStreamSynchronize(E.s()));
  };
  const auto results_t0 = Clock::now();
  out_vec(res->x, D.sol_x.get(), true);
  out_vec(res->y, D.sol_y.get(), false);
  out_vec(res->reduced_costs, D.sol_r.get(), true);
  res->summary.primal_residual_inf = D.sol_summary.primal;
  res->summary.dual_residual_inf = D.sol_summary.dual;
  res->summary.primal_objective = D.sol_summary.pobj;
  res->summary.dual_objective = D.sol_summary.dobj;
  res->summary.abs_gap = D.sol_summary.abs_gap;
  res->summary.rel_gap = D.sol_summary.rel_gap;
  res->has_certificate = D.cert.have ? 1 : 0;
  if (D.cert.have) {
    res->cert_kind = D.cert.kind;
    if (D.cert.kind == PDLP_CERT_PRIMAL_INFEASIBLE) {
      out_vec(res->cert_ray_y, D.cert.ray_y.get(), false);
      out_vec(res->cert_ray_r, D.cert.ray_r.get(), true);
    } else {
      out_vec(res->cert_ray_x, D.cert.ray_x.get(), true);
    }
    res->cert_residual_inf = D.cert.residual;
    res->cert_objective = D.cert.objective;
    std::snprintf(res->cert_source, sizeof(res->cert_source), "%s", D.cert.source.c_str());
  }
  PDLP_CK(cudaStreamSynchronize(E.s()));
  res->iterations = D.k();
  res->polish_iterations = D.polish_iterations;
  res->restarts = D.restarts;
  res->step_retries = D.hs.retries;
  res->final_step_size = D.hs.eta;
  res->final_primal_weight = D.omega;
  res->min_step_size_limit = D.hs.min_eta_bar;
  res->attempts = D.hs.attempts + E.attempts_total_;
  res->upload_seconds = E.upload_seconds_;
  res->precondition_seconds = E.precondition_seconds_;
  res->loop_seconds = loop_seconds;
  res->step_seconds = E.step_seconds_;
  E.peer_finish();
  res->solve_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
  std::snprintf(res->termination_detail, sizeof(res->termination_detail), "%s", D.detail.c_str());
  if (o->logging) {
    std::fprintf(stderr,
                 "phase=main event=done status=%s iters=%lld polish_iters=%lld detail=\"%s\"\n",
                 status_name(status), static_cast<long long>(res->iterations),
                 static_cast<long long>(res->polish_iterations), res->termination_detail);
  }
  if (o->logging || std::getenv("PDLP_TIMING") != nullptr) {
    int64_t wt = 0, wd = 0;
    pdlpk_gap_window_stats(&wt, &wd);
    std::fprintf(stderr,
                 "phase=main event=timing solve=%.4f upload=%.4f precondition=%.4f loop=%.4f "
                 "steps=%.4f cadence=%.4f cad_batch=%.4f cad_capture=%.4f gap=%.4f "
                 "gap_windows=%lld/%lld polish=%.4f alloc=%.4f prep=%.4f results=%.4f\n",
                 res->solve_seconds, res->upload_seconds, res->precondition_seconds,
                 res->loop_seconds, res->step_seconds, E.cadence_seconds_, E.cad_batch_seconds_,
                 E.cad_capture_seconds_, E.gap_seconds_,
                 static_cast<long long>(wd), static_cast<long long>(wt), E.polish_seconds_,
                 g_alloc_seconds, prep_seconds,
                 std::chrono::duration<double>(Clock::now() - results_t0).count());
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PDLP_OK;
  } catch (const std::invalid_argument& e) {  // InvalidProblem, shard extraction
    g_last_error = e.what();
    return PDLP_ERR_INVALID_PROBLEM;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return PDLP_ERR_CUDA;
  } catch (const std::bad_alloc& e) {
    g_last_error = e.what();
    return PDLP_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PDLP_ERR_INTERNAL;
  }
}

}  // namespace pdlp_host

// =========================================================== public C-ABI ===
using namespace pdlp_host;

extern "C" {

void pdlp_default_options(pdlp_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->eps_primal = 1e-8;
  o->eps_dual = 1e-8;
  o->eps_rel_gap = 1e-2;
  o->iteration_limit = 200000;
  o->time_limit_seconds = kInf;
  o->threads = 1;
  o->shards_per_thread = 4;
  o->enable_scaling = 1;
  o->ruiz_passes = 10;
  o->pock_chambolle = 1;
  o->enable_polish = 1;
  o->enable_restarts = 1;
  o->detect_infeasibility = 1;
  o->eps_ray = 1e-12;
  o->check_interval = 64;
  o->restart_sufficient = 0.1;
  o->restart_necessary = 0.9;
  o->restart_artificial = 0.5;
  o->mode = PDLP_MODE_PERF;
  o->device = 0;
  o->reserved0 = 0;
}

int pdlp_solve(const pdlp_problem_view* problem, const pdlp_options* options,
               pdlp_result* result) {
  if (problem == nullptr || options == nullptr || result == nullptr) {
    g_last_error = "null argument";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] { solve(problem, options, result); });
}

const char* pdlp_last_error(void) { return g_last_error.c_str(); }

int pdlp_shard_plan_for(int64_t rows, int64_t cols, int32_t rank, int32_t world,
                        pdlp_shard_plan* out) {
  if (out == nullptr || world < 1 || rank < 0 || rank >= world || rows < 0 || cols < 0) {
    g_last_error = "invalid shard request";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  *out = shard_plan(rows, cols, rank, world, auto_cut(rows, cols));
  return PDLP_OK;
}

int pdlp_shard_extract_cut(const pdlp_problem_view* problem, int32_t rank, int32_t world,
                           int32_t cut, pdlp_shard_view* out, void** owner) {
  if (problem == nullptr || out == nullptr || owner == nullptr || world < 1 || rank < 0 ||
      rank >= world || (cut != PDLP_CUT_ROWS && cut != PDLP_CUT_COLS)) {
    g_last_error = "invalid shard request";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    auto d = std::make_unique<ShardData>();
    extract_shard(*problem, rank, world, cut, *d);
    *out = d->view;
    *owner = d.release();
  });
}

int pdlp_shard_extract(const pdlp_problem_view* problem, int32_t rank, int32_t world,
                       pdlp_shard_view* out, void** owner) {
  if (problem == nullptr) {
    g_last_error = "invalid shard request";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  return pdlp_shard_extract_cut(problem, rank, world, auto_cut(problem->rows, problem->cols), out,
                                owner);
}

void pdlp_shard_free(void* owner) { delete static_cast<ShardData*>(owner); }

int pdlp_nccl_unique_id(unsigned char out[128]) {
  const char* why = "";
  if (out == nullptr) {
    g_last_error = "null argument";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  if (!nccl_unique_id(out, &why)) {
    g_last_error = why;
    return PDLP_ERR_CUDA;
  }
  return PDLP_OK;
}

// A caller-built shard must be the one pdlp_shard_plan_for assigns to this
// rank (equal blocks: the collectives exchange equal counts).
static int check_shard_view(const pdlp_shard_view* v, int32_t rank, int32_t world,
                            pdlp_shard_view* fixed) {
  if (v == nullptr) {
    g_last_error = "null shard";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  if (world < 1 || rank < 0 || rank >= world || v->plan.rows < 0 || v->plan.cols < 0 ||
      (v->plan.cut != PDLP_CUT_ROWS && v->plan.cut != PDLP_CUT_COLS)) {
    g_last_error = "invalid shard request";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  // the shard's own cut (a caller may build either); the ranges must be
  // the equal blocks of pdlp_shard_plan_for
  const pdlp_shard_plan want = shard_plan(v->plan.rows, v->plan.cols, rank, world, v->plan.cut);
  if (want.row_begin != v->plan.row_begin || want.row_end != v->plan.row_end ||
      want.col_begin != v->plan.col_begin || want.col_end != v->plan.col_end) {
    g_last_error = "shard ranges differ from pdlp_shard_plan_for(rows, cols, rank, world)";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  const bool cols_cut = want.cut == PDLP_CUT_COLS;
  const int64_t rows_dim = cols_cut ? v->plan.rows : want.row_end - want.row_begin;
  const int64_t cols_dim = cols_cut ? want.col_end - want.col_begin : v->plan.cols;
  if (v->rows.primary_dim != rows_dim || v->cols.primary_dim != cols_dim ||
      v->rows.nnz != v->cols.nnz) {
    g_last_error = "invalid problem: row/column layouts disagree (index -1)";
    return PDLP_ERR_INVALID_PROBLEM;
  }
  *fixed = *v;
  fixed->plan = want;
  return PDLP_OK;
}

static int check_sharded_args(const pdlp_problem_view* problem, const pdlp_options* o,
                              int32_t rank, int32_t world, const pdlp_result* result) {
  if (problem == nullptr || o == nullptr || result == nullptr || world < 1 || rank < 0 ||
      rank >= world) {
    g_last_error = "invalid sharded-solve arguments";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  if (o->mode != PDLP_MODE_PERF) {
    g_last_error = "the sharded solve runs in perf mode only (parity needs one GPU)";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  if (o->observer != nullptr) {
    g_last_error = "the sharded solve does not support an observer";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  return PDLP_OK;
}

int pdlp_solve_sharded(const pdlp_problem_view* problem, const pdlp_options* options,
                       int32_t rank, int32_t world, const unsigned char nccl_id[128],
                       pdlp_result* result) {
  int rc = check_sharded_args(problem, options, rank, world, result);
  if (rc != PDLP_OK) return rc;
  if (nccl_id == nullptr) {
    g_last_error = "null nccl id";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    std::unique_ptr<Comm> comm = make_nccl_comm(nccl_id, rank, world, options->device);
    solve(problem, options, result, comm.get());
  });
}

int pdlp_solve_sharded_emulated(const pdlp_problem_view* problem, const pdlp_options* options,
                                int32_t world, pdlp_result* result) {
  int rc = check_sharded_args(problem, options, 0, world, result);
  if (rc != PDLP_OK) return rc;
  const size_t n = static_cast<size_t>(std::max<int64_t>(problem->cols, 0));
  const size_t m = static_cast<size_t>(std::max<int64_t>(problem->rows, 0));
  // ranks > 0 fill private copies of the (identical) result
  std::vector<pdlp_result> res(static_cast<size_t>(world));
  struct Bufs {
    std::vector<double> x, y, r, rx, ry, rr;
  };
  std::vector<Bufs> store(static_cast<size_t>(world));
  for (int r = 0; r < world; ++r) {
    if (r == 0) {
      res[0] = *result;
      continue;
    }
    Bufs& b = store[r];
    for (auto* v : {&b.x, &b.r, &b.rx, &b.rr}) v->assign(n + 1, 0.0);
    for (auto* v : {&b.y, &b.ry}) v->assign(m + 1, 0.0);
    res[r] = pdlp_result{};
    res[r].x = b.x.data();
    res[r].y = b.y.data();
    res[r].reduced_costs = b.r.data();
    res[r].cert_ray_x = b.rx.data();
    res[r].cert_ray_y = b.ry.data();
    res[r].cert_ray_r = b.rr.data();
  }
  std::shared_ptr<ThreadHub> hub = make_thread_hub(world);
  std::vector<int> codes(static_cast<size_t>(world), PDLP_OK);
  std::vector<std::string> errs(static_cast<size_t>(world));
  std::vector<std::thread> th;
  for (int r = 0; r < world; ++r) {
    th.emplace_back([&, r] {
      codes[r] = guarded([&] {
        std::unique_ptr<Comm> comm = make_thread_comm(hub, r);
        solve(problem, options, &res[r], comm.get());
      });
      if (codes[r] != PDLP_OK) {
        errs[r] = g_last_error;
        abort_thread_hub(*hub);
      }
    });
  }
  for (auto& t : th) t.join();
  // report the first rank's own failure (not the "another rank failed" echo)
  int pick = -1;
  for (int r = 0; r < world; ++r) {
    if (codes[r] != PDLP_OK && errs[r].find("another rank of the group failed") == std::string::npos) {
      pick = r;
      break;
    }
  }
  if (pick < 0) {
    for (int r = 0; r < world && pick < 0; ++r) {
      if (codes[r] != PDLP_OK) pick = r;
    }
  }
  if (pick >= 0) {
    g_last_error = errs[pick];
    return codes[pick];
  }
  const pdlp_result user = *result;
  *result = res[0];
  // keep the caller's buffer pointers (res[0] was filled through them)
  result->x = user.x;
  result->y = user.y;
  result->reduced_costs = user.reduced_costs;
  result->cert_ray_x = user.cert_ray_x;
  result->cert_ray_y = user.cert_ray_y;
  result->cert_ray_r = user.cert_ray_r;
  return PDLP_OK;
}

int pdlp_host_register(void* ptr, size_t bytes) {
  if (ptr == nullptr || bytes == 0) return PDLP_OK;
  return guarded([&] { PDLP_CK(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable)); });
}

int pdlp_host_unregister(void* ptr) {
  if (ptr == nullptr) return PDLP_OK;
  return guarded([&] { PDLP_CK(cudaHostUnregister(ptr)); });
}

int pdlp_host_alloc(size_t bytes, void** out) {
  if (out == nullptr) {
    g_last_error = "null argument";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  if (bytes == 0) return PDLP_OK;
  return guarded([&] { PDLP_CK(cudaHostAlloc(out, bytes, cudaHostAllocPortable)); });
}

int pdlp_host_free(void* ptr) {
  if (ptr == nullptr) return PDLP_OK;
  return guarded([&] { PDLP_CK(cudaFreeHost(ptr)); });
}

int pdlp_trim_device_memory(int device) {
  return guarded([&] {
    cudaMemPool_t pool;
    PDLP_CK(cudaSetDevice(device));
    PDLP_CK(cudaDeviceSynchronize());
    BlockCache::get().trim(device);
    PDLP_CK(cudaDeviceGetDefaultMemPool(&pool, device));
    PDLP_CK(cudaMemPoolTrimTo(pool, 0));
  });
}

void pdlp_gap_dist_stats(int64_t* out, double* max_rel, int32_t reset) {
  /* max_rel[0]: the gap values, max_rel[1]: lambda* */
  auto& g = pdlp_host::gapd_stats();
  std::lock_guard<std::mutex> lk(g.mu);
  if (out != nullptr) {
    out[0] = g.evals;
    out[1] = g.rounds;
    out[2] = g.final_events;
    out[3] = g.checked;
  }
  if (max_rel != nullptr) {
    max_rel[0] = g.max_rel;
    max_rel[1] = g.max_rel_lambda;
  }
  if (reset) {
    g.evals = g.rounds = g.final_events = g.checked = 0;
    g.max_rel = g.max_rel_lambda = 0.0;
  }
}

int pdlp_abi_version(void) { return PDLP_ABI_VERSION; }

int pdlp_device_count(void) {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    g_last_error = cudaGetErrorString(e);
    return PDLP_ERR_CUDA;
  }
  return n;
}

}  // extern "C"

// ------------------------------------------------- component entry points ---
namespace pdlp_host {

struct Component {
  pdlp_options o;
  std::unique_ptr<Engine> E;
  Component(const pdlp_problem_view* p, int mode, int shards) {
    pdlp_default_options(&o);
    o.mode = mode;
    o.threads = 1;
    o.shards_per_thread = shards > 0 ? shards : 4;
    E = std::make_unique<Engine>(p, o);
  }
};

DevBuf<double> to_dev(const double* h, int64_t n, cudaStream_t s) { return upload_vec(h, n, s); }

void from_dev(double* h, const DevBuf<double>& d, int64_t n, cudaStream_t s) {
  if (h != nullptr && n > 0) {
    PDLP_CK(cudaMemcpyAsync(h, d.get(), n * 8, cudaMemcpyDeviceToHost, s));
    PDLP_CK(cudaStreamSynchronize(s));
  }
}

}  // namespace pdlp_host

extern "C" {

int pdlp_pdhg_step(const pdlp_problem_view* problem, const double* x, const double* y,
                   double omega, double eta, int32_t mode, int32_t shards, double* x_out,
                   double* y_out, int32_t* finite) {
  return guarded([&] {
    Component C(problem, mode, shards);
    Engine& E = *C.E;
    const pdlpk_problem P = E.problem().view();
    Inner& D = E.main_;
    DevBuf<double> x0 = to_dev(x, P.n, E.s());
    E.prepare(D, P, x0.get(), eta, omega, true);
    if (P.m > 0) PDLP_CK(cudaMemcpyAsync(D.y[0].get(), y, P.m * 8, cudaMemcpyHostToDevice, E.s()));
    PDLP_LAUNCH(pdlpk_spmv(&P.KT, 0, D.y[0].get(), D.aty[0].get(), E.parity(), E.s()));
    E.run_steps(P, D, 1);
    // On a non-finite trial the controller keeps the old iterate; the trial
    // itself sits in the other buffer.
    const int c = D.hs.status == 0 ? D.cur() : (D.cur() ^ 1);
    std::vector<double> hx(P.n), hy(P.m);
    from_dev(hx.data(), D.x[c], P.n, E.s());
    from_dev(hy.data(), D.y[c], P.m, E.s());
    // pdhg_step (step.hpp:100-115) reports nullopt on any non-finite entry.
    bool all_finite = true;
    for (double v : hx) all_finite = all_finite && std::isfinite(v);
    for (double v : hy) all_finite = all_finite && std::isfinite(v);
    *finite = all_finite ? 1 : 0;
    if (x_out != nullptr && P.n > 0) std::memcpy(x_out, hx.data(), P.n * 8);
    if (y_out != nullptr && P.m > 0) std::memcpy(y_out, hy.data(), P.m * 8);
  });
}

int pdlp_adaptive_step(const pdlp_problem_view* problem, double* x, double* y, double* aty,
                       double* io_state, int32_t mode, int32_t shards, double* prev_x,
                       double* prev_y, double* stats, int32_t* outcome) {
  return guarded([&] {
    Component C(problem, mode, shards);
    Engine& E = *C.E;
    const pdlpk_problem P = E.problem().view();
    Inner& D = E.main_;
    DevBuf<double> x0 = to_dev(x, P.n, E.s());
    E.prepare(D, P, x0.get(), io_state[0], io_state[3], false);
    if (P.m > 0) PDLP_CK(cudaMemcpyAsync(D.y[0].get(), y, P.m * 8, cudaMemcpyHostToDevice, E.s()));
    if (P.n > 0) PDLP_CK(cudaMemcpyAsync(D.aty[0].get(), aty, P.n * 8, cudaMemcpyHostToDevice, E.s()));
    D.hs.k = static_cast<int64_t>(io_state[1]);
    D.hs.max_retries = static_cast<int32_t>(io_state[2]);
    E.write_state(D);
    E.run_steps(P, D, D.hs.k + 1);
    *outcome = D.hs.status == 0 ? 0 : 1;
    const int c = D.cur();
    from_dev(x, D.x[c], P.n, E.s());
    from_dev(y, D.y[c], P.m, E.s());
    from_dev(aty, D.aty[c], P.n, E.s());
    from_dev(prev_x, D.x[c ^ 1], P.n, E.s());
    from_dev(prev_y, D.y[c ^ 1], P.m, E.s());
    io_state[0] = D.hs.eta;
    io_state[1] = static_cast<double>(D.hs.k);
    stats[0] = static_cast<double>(D.hs.accepted);
    stats[1] = static_cast<double>(D.hs.retries);
    stats[2] = D.hs.min_eta_bar;
    stats[3] = D.hs.eta_used;
  });
}

int pdlp_spmv(const pdlp_problem_view* problem, const double* x, double* out, int32_t mode) {
  return guarded([&] {
    Component C(problem, mode, 4);
    Engine& E = *C.E;
    const pdlpk_problem P = E.problem().view();
    DevBuf<double> dx = to_dev(x, P.n, E.s()), dout(P.m);
    PDLP_LAUNCH(pdlpk_spmv(&P.K, 0, dx.get(), dout.get(), E.parity(), E.s()));
    from_dev(out, dout, P.m, E.s());
  });
}

int pdlp_spmv_transpose(const pdlp_problem_view* problem, const double* y, double* out,
                        int32_t mode) {
  return guarded([&] {
    Component C(problem, mode, 4);
    Engine& E = *C.E;
    const pdlpk_problem P = E.problem().view();
    DevBuf<double> dy = to_dev(y, P.m, E.s()), dout(P.n);
    PDLP_LAUNCH(pdlpk_spmv(&P.KT, 0, dy.get(), dout.get(), E.parity(), E.s()));
    from_dev(out, dout, P.n, E.s());
  });
}

int pdlp_apply_rescaling(const pdlp_problem_view* problem, int32_t ruiz_passes,
                         int32_t pock_chambolle, double* row_values, double* col_values,
                         double* objective, double* con_lower, double* con_upper,
                         double* var_lower, double* var_upper, double* row_scale,
                         double* col_scale) {
  return guarded([&] {
    Component C(problem, PDLP_MODE_PARITY, 4);
    Engine& E = *C.E;
    E.precondition(ruiz_passes, pock_chambolle != 0);
    const DevProblem& Q = E.problem();
    from_dev(row_values, Q.row.value, Q.row.view.nnz, E.s());
    from_dev(col_values, Q.col.value, Q.col.view.nnz, E.s());
    from_dev(objective, Q.c, Q.n, E.s());
    from_dev(con_lower, Q.lc, Q.m, E.s());
    from_dev(con_upper, Q.uc, Q.m, E.s());
    from_dev(var_lower, Q.lv, Q.n, E.s());
    from_dev(var_upper, Q.uv, Q.n, E.s());
    from_dev(row_scale, Q.row_scale, Q.m, E.s());
    from_dev(col_scale, Q.col_scale, Q.n, E.s());
  });
}

int pdlp_normalized_duality_gap(const pdlp_problem_view* problem, const double* x,
                                const double* y, const double* ax, const double* aty,
                                double omega, double r, int32_t mode, double* gap) {
  return guarded([&] {
    Component C(problem, mode, 4);
    Engine& E = *C.E;
    const pdlpk_problem P = E.problem().view();
    DevBuf<double> dx = to_dev(x, P.n, E.s()), dy = to_dev(y, P.m, E.s());
    DevBuf<double> dax = to_dev(ax, P.m, E.s()), daty = to_dev(aty, P.n, E.s());
    const pdlpk_red red = E.red();
    PDLP_LAUNCH(pdlpk_gap_prepare(&P, dx.get(), dy.get(), dax.get(), daty.get(), omega, &red,
                                  E.gap_work_[0].get(), E.islots_.get(), E.s()));
    int events = 0;
    PDLP_CK(cudaMemcpyAsync(&events, E.islots_.get(), sizeof(int), cudaMemcpyDeviceToHost, E.s()));
    PDLP_CK(cudaStreamSynchronize(E.s()));
    // PDLP_GAP_WINDOW="qa:qb" forces a window sort (tests of the perf path)
    double qa = -1.0, qb = -1.0;
    if (const char* wv = std::getenv("PDLP_GAP_WINDOW")) std::sscanf(wv, "%lf:%lf", &qa, &qb);
    PDLP_LAUNCH(pdlpk_gap_finish(&P, dx.get(), dy.get(), dax.get(), daty.get(), omega, nullptr, r,
                                 events, &red, E.gap_work_[0].get(), E.slot(0), qa, qb, E.s()));
    *gap = E.read_slots(1)[0];
  });
}

int pdlp_kkt_residuals(const pdlp_problem_view* problem, const double* x, const double* y,
                       int32_t rc_mode, int32_t mode, double* r_out,
                       pdlp_residual_summary* summary) {
  return guarded([&] {
    Component C(problem, mode, 4);
    Engine& E = *C.E;
    const pdlpk_problem P = E.problem().view();
    Inner& D = E.main_;
    D.allocate(P.n, P.m, pdlpk_step_partials(&P), 4);
    DevBuf<double> dx = to_dev(x, P.n, E.s()), dy = to_dev(y, P.m, E.s());
    // rc_mode 2: r_out carries the reduced costs to use (kkt_residuals with r,
    // residuals.hpp:135-158), else it receives the recovered ones
    DevBuf<double> dr = rc_mode == 2 ? to_dev(r_out, P.n, E.s()) : DevBuf<double>(P.n);
    const Summary s = E.original_kkt(P, dx.get(), dy.get(), rc_mode, dr.get(), D);
    if (rc_mode != 2) from_dev(r_out, dr, P.n, E.s());
    summary->primal_residual_inf = s.primal;
    summary->dual_residual_inf = s.dual;
    summary->primal_objective = s.pobj;
    summary->dual_objective = s.dobj;
    summary->abs_gap = s.abs_gap;
    summary->rel_gap = s.rel_gap;
  });
}

int pdlp_check_certificate(const pdlp_problem_view* problem, int32_t kind, const double* ray,
                           double eps_ray, int32_t* verified, double* residual,
                           double* objective) {
  if (problem == nullptr || ray == nullptr || verified == nullptr || (kind != 0 && kind != 1)) {
    g_last_error = "invalid certificate check";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    Component C(problem, PDLP_MODE_PERF, 4);
    Engine& E = *C.E;
    const pdlpk_problem P = E.problem().view();
    Inner& D = E.main_;
    D.allocate(P.n, P.m, pdlpk_step_partials(&P), 4);
    double res = kInf, obj = 0.0;
    bool ok;
    if (kind == PDLP_CERT_PRIMAL_INFEASIBLE) {
      DevBuf<double> dy = to_dev(ray, P.m, E.s());
      ok = E.try_primal(P, 1, dy.get(), eps_ray, D, res, obj);
    } else {
      DevBuf<double> dx = to_dev(ray, P.n, E.s());
      ok = E.try_dual(P, 1, dx.get(), eps_ray, D, res, obj);
    }
    *verified = ok ? 1 : 0;
    if (residual != nullptr) *residual = res;
    if (objective != nullptr) *objective = obj;
  });
}

int pdlp_feasibility_run(const pdlp_problem_view* a, const double* b, const double* x0,
                         double eta, int64_t restart_length, int32_t rounds, int32_t mode,
                         int32_t device, double* restart_points, double* residuals,
                         int32_t* recorded, int32_t* finite) {
  if (a == nullptr || b == nullptr || x0 == nullptr || residuals == nullptr ||
      recorded == nullptr || finite == nullptr || restart_length < 1 || rounds < 0 ||
      (mode != PDLP_MODE_PERF && mode != PDLP_MODE_PARITY)) {
    g_last_error = "invalid feasibility run";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    const int64_t m = a->rows, n = a->cols;
    // The harness reads only A and b: an LP view around them (c = 0,
    // A x = b, x >= 0) lets the engine upload, validate and schedule A.
    std::vector<double> zero(static_cast<size_t>(std::max<int64_t>(n, 1)), 0.0);
    std::vector<double> inf(static_cast<size_t>(std::max<int64_t>(n, 1)), kInf);
    pdlp_problem_view v = *a;
    v.objective = zero.data();
    v.var_lower = zero.data();
    v.var_upper = inf.data();
    v.con_lower = b;
    v.con_upper = b;
    pdlp_options o;
    pdlp_default_options(&o);
    o.mode = mode;
    o.device = device;
    o.threads = 1;
    o.shards_per_thread = 1;  // one shard: the residual sums run in row order
    Engine E(&v, o);
    const DevProblem& Q = E.problem();
    const cudaStream_t s = E.s();
    const int parity = mode == PDLP_MODE_PARITY ? 1 : 0;
    DevBuf<double> x = to_dev(x0, n, s), xs = to_dev(x0, n, s), db = to_dev(b, m, s);
    DevBuf<double> xsum(n), y(m), aty(n), scr(n), axm(m), ax(m);
    DevBuf<int32_t> flag(1);
    dev_zero(xsum.get(), n, s);
    const int32_t one = 1;
    PDLP_CK(cudaMemcpyAsync(flag.get(), &one, sizeof(one), cudaMemcpyHostToDevice, s));
    const pdlpk_red red = E.red();
    // feasibility_residual (feasibility_method.hpp:26-34): ||A x - b||_2
    auto residual = [&](const double* pt) {
      PDLP_LAUNCH(pdlpk_spmv(&Q.row.view, 0, pt, ax.get(), parity, s));
      PDLP_LAUNCH(pdlpk_diff_norm_sq(ax.get(), db.get(), m, &red, E.slot(0), s));
      return std::sqrt(E.read_slots(1)[0]);
    };
    // One feasibility_step (:42-57): aty = A^T y; primal half; A scratch;
    // dual half.  Rounds replay captured graphs of up to 64 steps.
    auto enqueue_steps = [&](int64_t steps) {
      for (int64_t t = 0; t < steps; ++t) {
        PDLP_LAUNCH(pdlpk_spmv(&Q.col.view, 0, y.get(), aty.get(), parity, s));
        PDLP_LAUNCH(pdlpk_feas_primal(x.get(), aty.get(), scr.get(), xsum.get(), eta, n, s));
        PDLP_LAUNCH(pdlpk_spmv(&Q.row.view, 0, scr.get(), axm.get(), parity, s));
        PDLP_LAUNCH(pdlpk_feas_dual(y.get(), db.get(), axm.get(), eta, m, s));
      }
    };
    struct Graph {
      cudaGraphExec_t exec = nullptr;
      ~Graph() {
        if (exec != nullptr) cudaGraphExecDestroy(exec);
      }
    };
    auto capture = [&](int64_t steps, Graph& g) {
      if (steps == 0) return;
      cudaGraph_t graph = nullptr;
      PDLP_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      enqueue_steps(steps);
      PDLP_CK(cudaStreamEndCapture(s, &graph));
      const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
      cudaGraphDestroy(graph);
      PDLP_CK(e);
    };
    const int64_t chunk = std::min<int64_t>(restart_length, 64);
    const int64_t reps = restart_length / chunk, rest = restart_length % chunk;
    Graph body, tail;
    capture(chunk, body);
    capture(rest, tail);

    auto record = [&](int32_t k) {
      if (restart_points != nullptr && n > 0) {
        PDLP_CK(cudaMemcpyAsync(restart_points + static_cast<int64_t>(k) * n, xs.get(), n * 8,
                                cudaMemcpyDeviceToHost, s));
      }
      residuals[k] = residual(xs.get());
    };
    record(0);
    int32_t rec = 1, ok = 1;
    for (int32_t r = 0; r < rounds; ++r) {
      dev_zero(y.get(), m, s);  // y reset (:67)
      for (int64_t q = 0; q < reps; ++q) PDLP_CK(cudaGraphLaunch(body.exec, s));
      if (rest > 0) PDLP_CK(cudaGraphLaunch(tail.exec, s));
      PDLP_LAUNCH(pdlpk_feas_average(xs.get(), x.get(), xsum.get(),
                                     static_cast<double>(restart_length), n, flag.get(), s));
      PDLP_CK(cudaMemcpyAsync(&ok, flag.get(), sizeof(ok), cudaMemcpyDeviceToHost, s));
      PDLP_CK(cudaStreamSynchronize(s));
      if (!ok) break;
      record(rec);
      ++rec;
    }
    PDLP_CK(cudaStreamSynchronize(s));
    *recorded = rec;
    *finite = ok;
  });
}

int pdlp_step_size_rules(double movement, double curvature, double eta_bar, double eta,
                         int64_t k, double* limit_out, double* next_out) {
  // Scalar rules (step.hpp:126-141), evaluated with the host table values the
  // device decision kernel reads.
  const double denom = 2.0 * std::abs(curvature);
  *limit_out = (denom > 0.0) ? movement / denom : kInf;
  const double kk = static_cast<double>(k < 1 ? 1 : k) + 1.0;
  const double down = (1.0 - std::pow(kk, -0.3)) * eta_bar;
  const double up = (1.0 + std::pow(kk, -0.6)) * eta;
  *next_out = (up < down) ? up : down;
  return PDLP_OK;
}

}  // extern "C"

// ------------------------------------------------ shard-local ingest ---
// Every rank passes only its shard: nothing of the whole
// problem is materialized on any host; x, y and the reduced costs are still
// gathered to every rank's result (n- and m-length buffers).
int pdlp_solve_sharded_local(const pdlp_shard_view* shard, const pdlp_options* options,
                             int32_t rank, int32_t world, const unsigned char nccl_id[128],
                             pdlp_result* result) {
  pdlp_problem_view dummy{};
  int rc = check_sharded_args(&dummy, options, rank, world, result);
  if (rc != PDLP_OK) return rc;
  pdlp_shard_view v{};
  rc = check_shard_view(shard, rank, world, &v);
  if (rc != PDLP_OK) return rc;
  if (nccl_id == nullptr) {
    g_last_error = "null nccl id";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    std::unique_ptr<Comm> comm = make_nccl_comm(nccl_id, rank, world, options->device);
    solve(nullptr, options, result, comm.get(), &v);
  });
}

int pdlp_solve_sharded_local_emulated(const pdlp_shard_view* const* shards,
                                      const pdlp_options* options, int32_t world,
                                      pdlp_result* result) {
  pdlp_problem_view dummy{};
  int rc = check_sharded_args(&dummy, options, 0, world, result);
  if (rc != PDLP_OK) return rc;
  if (shards == nullptr) {
    g_last_error = "null shards";
    return PDLP_ERR_INVALID_ARGUMENT;
  }
  std::vector<pdlp_shard_view> v(static_cast<size_t>(world));
  for (int r = 0; r < world; ++r) {
    rc = check_shard_view(shards[r], r, world, &v[static_cast<size_t>(r)]);
    if (rc != PDLP_OK) return rc;
  }
  const size_t n = static_cast<size_t>(std::max<int64_t>(v[0].plan.cols, 0));
  const size_t m = static_cast<size_t>(std::max<int64_t>(v[0].plan.rows, 0));
  std::vector<pdlp_result> res(static_cast<size_t>(world));
  struct Bufs {
    std::vector<double> x, y, r, rx, ry, rr;
  };
  std::vector<Bufs> store(static_cast<size_t>(world));
  for (int r = 0; r < world; ++r) {
    if (r == 0) {
      res[0] = *result;
      continue;
    }
    Bufs& b = store[r];
    for (auto* q : {&b.x, &b.r, &b.rx, &b.rr}) q->assign(n + 1, 0.0);
    for (auto* q : {&b.y, &b.ry}) q->assign(m + 1, 0.0);
    res[r] = pdlp_result{};
    res[r].x = b.x.data();
    res[r].y = b.y.data();
    res[r].reduced_costs = b.r.data();
    res[r].cert_ray_x = b.rx.data();
    res[r].cert_ray_y = b.ry.data();
    res[r].cert_ray_r = b.rr.data();
  }
  std::shared_ptr<ThreadHub> hub = make_thread_hub(world);
  std::vector<int> codes(static_cast<size_t>(world), PDLP_OK);
  std::vector<std::string> errs(static_cast<size_t>(world));
  std::vector<std::thread> th;
  for (int r = 0; r < world; ++r) {
    th.emplace_back([&, r] {
      codes[r] = guarded([&] {
        std::unique_ptr<Comm> comm = make_thread_comm(hub, r);
        solve(nullptr, options, &res[r], comm.get(), &v[static_cast<size_t>(r)]);
      });
      if (codes[r] != PDLP_OK) {
        errs[r] = g_last_error;
        abort_thread_hub(*hub);
      }
    });
  }
  for (auto& t : th) t.join();
  for (int r = 0; r < world; ++r) {
    if (codes[r] != PDLP_OK && errs[r].find("another rank of the group failed") == std::string::npos) {
      g_last_error = errs[r];
      return codes[r];
    }
  }
  for (int r = 0; r < world; ++r) {
    if (codes[r] != PDLP_OK) {
      g_last_error = errs[r];
      return codes[r];
    }
  }
  const pdlp_result user = *result;
  *result = res[0];
  result->x = user.x;
  result->y = user.y;
  result->reduced_costs = user.reduced_costs;
  result->cert_ray_x = user.cert_ray_x;
  result->cert_ray_y = user.cert_ray_y;
  result->cert_ray_r = user.cert_ray_r;
  return PDLP_OK;
}
