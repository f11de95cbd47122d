// Row-sharded partition, host side (see shard.hpp).
#include "shard.hpp"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>

namespace pdlp_host {
namespace {

int64_t even_block(int64_t total, int world) {
  if (total <= 0) return 0;
  const int64_t b = (total + world - 1) / world;
  return (b + 1) / 2 * 2;
}

[[noreturn]] void broken(const char* what) {
  throw std::invalid_argument(std::string("invalid problem: ") + what + " (index -1)");
}

void check_pointers(const pdlp_csr_view& v, int64_t dim) {
  if (v.primary_dim != dim || v.nnz < 0) broken("row/column layouts disagree");
  if (v.start == nullptr) {
    if (v.nnz != 0) broken("row/column layouts disagree");
    return;
  }
  if (v.start[0] != 0 || v.start[dim] != v.nnz) broken("row/column layouts disagree");
  for (int64_t i = 0; i < dim; ++i) {
    if (v.start[i + 1] < v.start[i]) broken("row/column layouts disagree");
  }
}

template <class F>
void parallel_lines(int64_t dim, F f) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t T = std::max<int64_t>(1, std::min<int64_t>({static_cast<int64_t>(hw), 16, dim / 65536 + 1}));
  if (T == 1) {
    f(int64_t(0), dim);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (dim + T - 1) / T;
  for (int64_t t = 0; t < T; ++t) {
    const int64_t lo = std::min(dim, t * per), hi = std::min(dim, lo + per);
    th.emplace_back([=, &f] { f(lo, hi); });
  }
  for (auto& t : th) t.join();
}

}  // namespace

static const bool g_auto_cols = true;

int auto_cut(int64_t m, int64_t n) {
  if (const char* e = std::getenv("PDLP_SHARD_CUT")) {
    if (std::strcmp(e, "rows") == 0) return PDLP_CUT_ROWS;
    if (std::strcmp(e, "cols") == 0) return PDLP_CUT_COLS;
    if (std::strcmp(e, "auto") == 0) return m < n ? PDLP_CUT_COLS : PDLP_CUT_ROWS;
  }
  return g_auto_cols && m < n ? PDLP_CUT_COLS : PDLP_CUT_ROWS;
}

pdlp_shard_plan shard_plan(int64_t m, int64_t n, int rank, int world, int cut) {
  pdlp_shard_plan p{};
  p.cut = cut == PDLP_CUT_COLS ? PDLP_CUT_COLS : PDLP_CUT_ROWS;
  p.rank = rank;
  p.world = world;
  p.rows = m;
  p.cols = n;
  p.row_block = even_block(m, world);
  p.col_block = even_block(n, world);
  p.row_begin = std::min(m, p.row_block * rank);
  p.row_end = std::min(m, p.row_block * (rank + 1));
  p.col_begin = std::min(n, p.col_block * rank);
  p.col_end = std::min(n, p.col_block * (rank + 1));
  return p;
}

static void extract_cols(const pdlp_problem_view& p, const pdlp_shard_plan& plan,
                         const int64_t* rstart, const int64_t* cs, ShardData& out);

void extract_shard(const pdlp_problem_view& p, int rank, int world, int cut, ShardData& out) {
  const int64_t m = p.rows, n = p.cols;
  if (m < 0 || n < 0 || p.by_row.nnz != p.by_col.nnz) broken("row/column layouts disagree");
  check_pointers(p.by_row, m);
  check_pointers(p.by_col, n);
  // an empty matrix may come without line pointers
  std::vector<int64_t> zr, zc;
  const int64_t* rstart = p.by_row.start;
  const int64_t* cs = p.by_col.start;
  if (rstart == nullptr) {
    zr.assign(static_cast<size_t>(m + 1), 0);
    rstart = zr.data();
  }
  if (cs == nullptr) {
    zc.assign(static_cast<size_t>(n + 1), 0);
    cs = zc.data();
  }
  const pdlp_shard_plan plan = shard_plan(m, n, rank, world, cut);
  if (plan.cut == PDLP_CUT_COLS) {
    extract_cols(p, plan, rstart, cs, out);
    return;
  }
  const int64_t r0 = plan.row_begin, r1 = plan.row_end;
  const int64_t c0 = plan.col_begin, c1 = plan.col_end;
  pdlp_shard_view& v = out.view;
  v = pdlp_shard_view{};
  v.plan = plan;

  // K_g: a window of the caller's row layout, pointers rebased.
  const int64_t e0 = rstart[r0], e1 = rstart[r1];
  out.row_start.resize(static_cast<size_t>(r1 - r0 + 1));
  for (int64_t i = r0; i <= r1; ++i) out.row_start[static_cast<size_t>(i - r0)] = rstart[i] - e0;
  v.rows.primary_dim = r1 - r0;
  v.rows.nnz = e1 - e0;
  v.rows.start = out.row_start.data();
  v.rows.index = p.by_row.index ? p.by_row.index + e0 : nullptr;
  v.rows.value = p.by_row.value ? p.by_row.value + e0 : nullptr;
  v.entry_offset = e0;

  // K_g^T: each column's entries with a row in [r0, r1) are one contiguous
  // run (rows ascend within a column): binary-search it, then copy.
  const int64_t* ci = p.by_col.index;
  const double* cv = p.by_col.value;
  out.col_start.assign(static_cast<size_t>(n + 1), 0);
  std::atomic<bool> bad{false};
  parallel_lines(n, [&](int64_t lo, int64_t hi) {
    for (int64_t j = lo; j < hi; ++j) {
      const int64_t a = cs[j], b = cs[j + 1];
      for (int64_t k = a; k < b; ++k) {
        if (ci[k] < 0 || ci[k] >= m || (k > a && ci[k] <= ci[k - 1])) {
          bad = true;
          return;
        }
      }
      const int64_t* first = std::lower_bound(ci + a, ci + b, r0);
      const int64_t* last = std::lower_bound(first, ci + b, r1);
      out.col_start[static_cast<size_t>(j + 1)] = last - first;
    }
  });
  if (bad) broken("row/column layouts disagree");
  for (int64_t j = 0; j < n; ++j) out.col_start[static_cast<size_t>(j + 1)] += out.col_start[static_cast<size_t>(j)];
  const int64_t nnz_t = out.col_start[static_cast<size_t>(n)];
  out.col_index.resize(static_cast<size_t>(nnz_t));
  out.col_value.resize(static_cast<size_t>(nnz_t));
  parallel_lines(n, [&](int64_t lo, int64_t hi) {
    for (int64_t j = lo; j < hi; ++j) {
      const int64_t a = cs[j], b = cs[j + 1];
      const int64_t k0 = std::lower_bound(ci + a, ci + b, r0) - ci;
      int64_t o = out.col_start[static_cast<size_t>(j)];
      const int64_t o1 = out.col_start[static_cast<size_t>(j + 1)];
      for (int64_t k = k0; o < o1; ++k, ++o) {
        out.col_index[static_cast<size_t>(o)] = ci[k] - r0;
        out.col_value[static_cast<size_t>(o)] = cv[k];
      }
    }
  });
  v.cols.primary_dim = n;
  v.cols.nnz = nnz_t;
  v.cols.start = out.col_start.data();
  v.cols.index = out.col_index.data();
  v.cols.value = out.col_value.data();

  v.objective = p.objective ? p.objective + c0 : nullptr;
  v.var_lower = p.var_lower ? p.var_lower + c0 : nullptr;
  v.var_upper = p.var_upper ? p.var_upper + c0 : nullptr;
  v.con_lower = p.con_lower ? p.con_lower + r0 : nullptr;
  v.con_upper = p.con_upper ? p.con_upper + r0 : nullptr;
  (void)c1;
}

// PDLP_CUT_COLS: K_g^T is a window of the caller's column layout (lines
// [c0, c1), global row indices); K_g keeps every row and, of each row, the
// one contiguous run of entries with a column in [c0, c1) (columns ascend
// within a row), column indices made local.
static void extract_cols(const pdlp_problem_view& p, const pdlp_shard_plan& plan,
                         const int64_t* rstart, const int64_t* cs, ShardData& out) {
  const int64_t m = p.rows;
  const int64_t r0 = plan.row_begin, c0 = plan.col_begin, c1 = plan.col_end;
  pdlp_shard_view& v = out.view;
  v = pdlp_shard_view{};
  v.plan = plan;

  const int64_t e0 = cs[c0], e1 = cs[c1];
  out.col_start.resize(static_cast<size_t>(c1 - c0 + 1));
  for (int64_t j = c0; j <= c1; ++j) out.col_start[static_cast<size_t>(j - c0)] = cs[j] - e0;
  v.cols.primary_dim = c1 - c0;
  v.cols.nnz = e1 - e0;
  v.cols.start = out.col_start.data();
  v.cols.index = p.by_col.index ? p.by_col.index + e0 : nullptr;
  v.cols.value = p.by_col.value ? p.by_col.value + e0 : nullptr;
  v.entry_offset = 0;

  const int64_t* ri = p.by_row.index;
  const double* rv = p.by_row.value;
  out.row_start.assign(static_cast<size_t>(m + 1), 0);
  out.row_entry_offset.assign(static_cast<size_t>(m), 0);
  std::atomic<bool> bad{false};
  parallel_lines(m, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t a = rstart[i], b = rstart[i + 1];
      for (int64_t k = a; k < b; ++k) {
        if (ri[k] < 0 || ri[k] >= p.cols || (k > a && ri[k] <= ri[k - 1])) {
          bad = true;
          return;
        }
      }
      const int64_t* first = std::lower_bound(ri + a, ri + b, c0);
      const int64_t* last = std::lower_bound(first, ri + b, c1);
      out.row_start[static_cast<size_t>(i + 1)] = last - first;
      out.row_entry_offset[static_cast<size_t>(i)] = first - ri;  // by_row position (rebased below)
    }
  });
  if (bad) broken("row/column layouts disagree");
  for (int64_t i = 0; i < m; ++i) out.row_start[static_cast<size_t>(i + 1)] += out.row_start[static_cast<size_t>(i)];
  for (int64_t i = 0; i < m; ++i) out.row_entry_offset[static_cast<size_t>(i)] -= out.row_start[static_cast<size_t>(i)];
  const int64_t nnz_r = out.row_start[static_cast<size_t>(m)];
  out.row_index.resize(static_cast<size_t>(nnz_r));
  out.row_value.resize(static_cast<size_t>(nnz_r));
  parallel_lines(m, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      int64_t o = out.row_start[static_cast<size_t>(i)];
      const int64_t o1 = out.row_start[static_cast<size_t>(i + 1)];
      for (int64_t k = o + out.row_entry_offset[static_cast<size_t>(i)]; o < o1; ++k, ++o) {
        out.row_index[static_cast<size_t>(o)] = ri[k] - c0;
        out.row_value[static_cast<size_t>(o)] = rv[k];
      }
    }
  });
  v.rows.primary_dim = m;
  v.rows.nnz = nnz_r;
  v.rows.start = out.row_start.data();
  v.rows.index = out.row_index.data();
  v.rows.value = out.row_value.data();
  v.row_entry_offset = out.row_entry_offset.data();

  v.objective = p.objective ? p.objective + c0 : nullptr;
  v.var_lower = p.var_lower ? p.var_lower + c0 : nullptr;
  v.var_upper = p.var_upper ? p.var_upper + c0 : nullptr;
  v.con_lower = p.con_lower ? p.con_lower + r0 : nullptr;
  v.con_upper = p.con_upper ? p.con_upper + r0 : nullptr;
}

}  // namespace pdlp_host
