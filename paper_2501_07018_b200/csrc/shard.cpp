// Row-sharded partition, host side (see shard.hpp).
#include "shard.hpp"

#include <algorithm>
#include <atomic>
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

pdlp_shard_plan shard_plan(int64_t m, int64_t n, int rank, int world) {
  pdlp_shard_plan p{};
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

void extract_shard(const pdlp_problem_view& p, int rank, int world, ShardData& out) {
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
  const pdlp_shard_plan plan = shard_plan(m, n, rank, world);
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

}  // namespace pdlp_host
