// Seeded synthetic LP instances for the BASELINE.json configs (libpdlp_gen.so).
//
// Host-only data plumbing: builds the test/benchmark inputs, never part of the
// timed solve path.  Recipes restate BASELINE.json configs[0..4] as concrete
// seeded samplers; the splitmix64 engine and the raw
// 53-bit-to-double mapping follow the reference generator's style
// (proj/include/pdhglp/generator.hpp:75-94) so every instance is identical on
// every platform for a given seed.  The layout builder reproduces the
// reference's from_triplets semantics (sparse.hpp:48-115) so the emitted
// row/column layouts pass the reference's validate()/layouts_consistent().

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <vector>

#include <thread>

#include "pdlp_gen.h"

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct SplitMix {
  uint64_t s;
  explicit SplitMix(uint64_t seed) : s(seed * 0x2545f4914f6cdd1dull + 0x9e3779b97f4a7c15ull) {}
  uint64_t next() {
    s += 0x9e3779b97f4a7c15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  // Strictly inside (0, 1): safe for log().
  double u01_open() { return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * u01(); }
  double normal() {
    const double u1 = u01_open();
    const double u2 = u01();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  int64_t below(int64_t n) { return static_cast<int64_t>(next() % static_cast<uint64_t>(n)); }
};

struct Layout {
  std::vector<int64_t> start, index;
  std::vector<double> value;
};

}  // namespace

struct pdlp_instance {
  int64_t rows = 0, cols = 0;
  Layout by_row, by_col;
  std::vector<double> objective, con_lower, con_upper, var_lower, var_upper;
  std::vector<double> feasible_point;
};

namespace {

// from_triplets semantics for one orientation: counting sort by primary
// index (stable in input order), stable sort of each line by secondary index,
// duplicates summed left to right in input order.
void build_layout(int64_t primary_dim, int64_t count, const int64_t* prim, const int64_t* sec,
                  const double* val, Layout& out) {
  std::vector<int64_t> start(static_cast<size_t>(primary_dim) + 1, 0);
  for (int64_t k = 0; k < count; ++k) ++start[static_cast<size_t>(prim[k]) + 1];
  for (int64_t p = 0; p < primary_dim; ++p) start[p + 1] += start[p];
  std::vector<int64_t> order(static_cast<size_t>(count));
  {
    std::vector<int64_t> cursor(start.begin(), start.end() - 1);
    for (int64_t k = 0; k < count; ++k) order[cursor[prim[k]]++] = k;
  }
  out.start.assign(static_cast<size_t>(primary_dim) + 1, 0);
  out.index.clear();
  out.value.clear();
  out.index.reserve(static_cast<size_t>(count));
  out.value.reserve(static_cast<size_t>(count));
  for (int64_t p = 0; p < primary_dim; ++p) {
    int64_t* lo = order.data() + start[p];
    int64_t* hi = order.data() + start[p + 1];
    bool sorted = true;
    for (int64_t* q = lo; q + 1 < hi; ++q) {
      if (sec[q[1]] < sec[q[0]]) {
        sorted = false;
        break;
      }
    }
    if (!sorted) std::stable_sort(lo, hi, [&](int64_t a, int64_t b) { return sec[a] < sec[b]; });
    for (int64_t* q = lo; q < hi;) {
      double sum = val[*q];
      int64_t* e = q + 1;
      while (e < hi && sec[*e] == sec[*q]) {
        sum += val[*e];
        ++e;
      }
      out.index.push_back(sec[*q]);
      out.value.push_back(sum);
      q = e;
    }
    out.start[p + 1] = static_cast<int64_t>(out.index.size());
  }
}

struct Triplets {
  std::vector<int64_t> r, c;
  std::vector<double> v;
  void push(int64_t rr, int64_t cc, double vv) {
    r.push_back(rr);
    c.push_back(cc);
    v.push_back(vv);
  }
};

void build_both(pdlp_instance* inst, const Triplets& t) {
  const int64_t count = static_cast<int64_t>(t.v.size());
  build_layout(inst->rows, count, t.r.data(), t.c.data(), t.v.data(), inst->by_row);
  build_layout(inst->cols, count, t.c.data(), t.r.data(), t.v.data(), inst->by_col);
}

// Row-layout product in storage order (same order the reference's
// row_product uses, generator.hpp:108-120).
std::vector<double> row_product(const pdlp_instance* inst, const std::vector<double>& x) {
  std::vector<double> out(static_cast<size_t>(inst->rows), 0.0);
  for (int64_t r = 0; r < inst->rows; ++r) {
    double acc = 0.0;
    for (int64_t k = inst->by_row.start[r]; k < inst->by_row.start[r + 1]; ++k) {
      acc += inst->by_row.value[k] * x[inst->by_row.index[k]];
    }
    out[r] = acc;
  }
  return out;
}

std::vector<double> col_product(const pdlp_instance* inst, const std::vector<double>& y) {
  std::vector<double> out(static_cast<size_t>(inst->cols), 0.0);
  for (int64_t c = 0; c < inst->cols; ++c) {
    double acc = 0.0;
    for (int64_t k = inst->by_col.start[c]; k < inst->by_col.start[c + 1]; ++k) {
      acc += inst->by_col.value[k] * y[inst->by_col.index[k]];
    }
    out[c] = acc;
  }
  return out;
}

int64_t sample_count(SplitMix& rng, const pdlp_gen_params& p) {
  if (p.count_kind == 0) return p.count_fixed;
  // Continuous Pareto inverse CDF, floored: P(K >= k) ~ (kmin/k)^(alpha-1).
  for (;;) {
    const double u = rng.u01_open();
    const double k = std::floor(static_cast<double>(p.kmin) * std::pow(u, -1.0 / (p.alpha - 1.0)));
    if (k <= static_cast<double>(p.kmax)) return static_cast<int64_t>(k);
  }
}

double sample_value(SplitMix& rng, const pdlp_gen_params& p) {
  double mag;
  if (p.value_kind == 0) {
    mag = rng.uniform(p.value_lo, p.value_hi);
  } else {
    const double a = std::log(p.value_lo), b = std::log(p.value_hi);
    mag = std::exp(a + (b - a) * rng.u01());
  }
  return (rng.next() & 1u) ? mag : -mag;
}

}  // namespace

extern "C" {

void pdlp_gen_c0_params(pdlp_gen_params* p, uint64_t seed) {
  std::memset(p, 0, sizeof(*p));
  p->rows = 1000;
  p->cols = 2000;
  p->count_kind = 0;
  p->count_fixed = 10;
  p->value_kind = 0;
  p->value_lo = 0.1;
  p->value_hi = 10.0;
  p->eq_frac = 0.5;
  p->eq_rows_first = 1;
  p->bound_kind = 0;
  p->box_hi = 10.0;
  p->slack_hi = 1.0;
  p->seed = seed;
}

void pdlp_gen_c2_params(pdlp_gen_params* p, uint64_t seed) {
  std::memset(p, 0, sizeof(*p));
  p->rows = 5000000;
  p->cols = 10000000;
  p->count_kind = 1;
  p->alpha = 2.0;
  p->kmin = 2;
  p->kmax = 10000;
  p->value_kind = 1;
  p->value_lo = 1e-3;
  p->value_hi = 1e3;
  p->eq_frac = 0.7;
  p->eq_rows_first = 0;
  p->bound_kind = 1;
  p->box_hi = 10.0;
  p->slack_hi = 1.0;
  p->seed = seed;
}

void pdlp_gen_c4_params(pdlp_gen_params* p, uint64_t seed) {
  pdlp_gen_c2_params(p, seed);
  p->rows = 150000000;
  p->cols = 300000000;
  p->alpha = 2.2;
  p->value_lo = 1e-2;
  p->value_hi = 1e2;
  p->eq_frac = 0.5;
  p->bound_kind = 0;
}

pdlp_instance* pdlp_gen_random_lp(const pdlp_gen_params* params) {
  const pdlp_gen_params& p = *params;
  if (p.rows < 1 || p.cols < 1) return nullptr;
  SplitMix rng(p.seed);
  auto* inst = new pdlp_instance;
  inst->rows = p.rows;
  inst->cols = p.cols;
  const int64_t m = p.rows, n = p.cols;

  // Matrix, generated column by column (triplets in column-major order).
  Triplets t;
  for (int64_t c = 0; c < n; ++c) {
    const int64_t k = sample_count(rng, p);
    for (int64_t e = 0; e < k; ++e) t.push(rng.below(m), c, sample_value(rng, p));
  }
  build_both(inst, t);
  t = Triplets{};

  // Variable bounds and a feasible point x*, reduced-cost cone per type.
  inst->var_lower.resize(n);
  inst->var_upper.resize(n);
  std::vector<double> xs(n), rs(n);
  for (int64_t i = 0; i < n; ++i) {
    int kind = 0;  // 0 = [0, hi] (C0 box) or [0, inf); 1 = [l, u]; 2 = free
    if (p.bound_kind == 1) {
      const double u = rng.u01();
      kind = u < 0.6 ? 0 : (u < 0.9 ? 1 : 2);
    }
    if (kind == 0) {
      inst->var_lower[i] = 0.0;
      inst->var_upper[i] = p.bound_kind == 0 ? p.box_hi : kInf;
      xs[i] = rng.uniform(0.0, p.box_hi);
      rs[i] = std::fabs(rng.normal());
    } else if (kind == 1) {
      const double l = rng.uniform(-p.box_hi, 0.0);
      const double u = l + rng.uniform(1.0, 2.0 * p.box_hi);
      inst->var_lower[i] = l;
      inst->var_upper[i] = u;
      xs[i] = rng.uniform(l, u);
      rs[i] = rng.normal();
    } else {
      inst->var_lower[i] = -kInf;
      inst->var_upper[i] = kInf;
      xs[i] = p.box_hi * 0.5 * rng.normal();
      rs[i] = 0.0;
    }
  }

  // Rows: b = A x*, equality or <= with slack; dual point y* in its cone.
  const std::vector<double> ax = row_product(inst, xs);
  inst->con_lower.resize(m);
  inst->con_upper.resize(m);
  std::vector<double> ys(m);
  const int64_t n_eq_first = static_cast<int64_t>(std::llround(p.eq_frac * static_cast<double>(m)));
  for (int64_t j = 0; j < m; ++j) {
    const bool eq = p.eq_rows_first ? (j < n_eq_first) : (rng.u01() < p.eq_frac);
    if (eq) {
      inst->con_lower[j] = ax[j];
      inst->con_upper[j] = ax[j];
      ys[j] = rng.normal();
    } else {
      inst->con_lower[j] = -kInf;
      inst->con_upper[j] = ax[j] + rng.uniform(0.0, p.slack_hi);
      ys[j] = -std::fabs(rng.normal());
    }
  }
  // c = A'y* + r*: (y*, r*) is dual feasible, so the LP is bounded.
  const std::vector<double> aty = col_product(inst, ys);
  inst->objective.resize(n);
  for (int64_t i = 0; i < n; ++i) inst->objective[i] = aty[i] + rs[i];
  inst->feasible_point = std::move(xs);
  return inst;
}

// Rows [r0, r1) of the random-LP family as a standalone LP (SURVEY 8(f) 1:
// a C4 row shard is 18.75M x 300M with 375M entries; the whole instance, 3B
// entries, is never built).  Every column and every row has its own
// counter-based stream, so the draws parallelize over host threads and a
// window's entries do not depend on the window: the matrix of window [r0, r1)
// is exactly the rows r0..r1-1 of window [0, m).  Bounds, x*, y*, r* follow
// the sequential recipe per index; b = A_w x* and c = A_w' y*_w + r* are
// formed over the window, so the window LP is feasible and bounded on its
// own.  (Draws differ from pdlp_gen_random_lp's single sequential stream.)
static pdlp_instance* random_lp_window(const pdlp_gen_params* params, int64_t r0, int64_t r1,
                                       int64_t* entries_before);

pdlp_instance* pdlp_gen_random_lp_window(const pdlp_gen_params* params, int64_t r0, int64_t r1) {
  return random_lp_window(params, r0, r1, nullptr);
}

// entries_before (optional): entries of the whole instance in rows < r0, i.e.
// the by_row position of the window's first entry.
static pdlp_instance* random_lp_window(const pdlp_gen_params* params, int64_t r0, int64_t r1,
                                       int64_t* entries_before) {
  const pdlp_gen_params& p = *params;
  if (p.rows < 1 || p.cols < 1 || r0 < 0 || r1 > p.rows || r0 >= r1) return nullptr;
  const int64_t m = p.rows, n = p.cols, mw = r1 - r0;
  auto stream = [&](uint64_t kind, int64_t i) {
    SplitMix h(p.seed ^ (kind * 0xd1b54a32d192ed03ull));
    h.s += static_cast<uint64_t>(i) * 0x9e3779b97f4a7c15ull;
    return SplitMix(h.next());
  };
  const int T = static_cast<int>(std::max<unsigned>(1u, std::min(32u, std::thread::hardware_concurrency())));
  auto parallel = [&](int64_t count, auto&& body) {
    std::vector<std::thread> th;
    const int64_t per = (count + T - 1) / T;
    for (int t = 0; t < T; ++t) {
      const int64_t lo = std::min(count, per * t), hi = std::min(count, lo + per);
      th.emplace_back([&, t, lo, hi] { body(t, lo, hi); });
    }
    for (auto& x : th) x.join();
  };
  // Matrix: column streams, entries of the window kept (column-major order).
  std::vector<Triplets> part(static_cast<size_t>(T));
  std::vector<int64_t> before(static_cast<size_t>(T), 0);
  parallel(n, [&](int t, int64_t lo, int64_t hi) {
    Triplets& tr = part[static_cast<size_t>(t)];
    int64_t b = 0;
    std::vector<int64_t> above;  // this column's rows < r0 (duplicates merge)
    for (int64_t c = lo; c < hi; ++c) {
      SplitMix rng = stream(1, c);
      const int64_t k = sample_count(rng, p);
      above.clear();
      for (int64_t e = 0; e < k; ++e) {
        const int64_t row = rng.below(m);
        const double v = sample_value(rng, p);
        if (row >= r0 && row < r1) tr.push(row - r0, c, v);
        if (entries_before != nullptr && row < r0) above.push_back(row);
      }
      if (!above.empty()) {
        std::sort(above.begin(), above.end());
        b += std::unique(above.begin(), above.end()) - above.begin();
      }
    }
    before[static_cast<size_t>(t)] = b;
  });
  if (entries_before != nullptr) {
    *entries_before = 0;
    for (int64_t b : before) *entries_before += b;
  }
  Triplets all;
  size_t total = 0;
  for (const auto& tr : part) total += tr.v.size();
  all.r.reserve(total);
  all.c.reserve(total);
  all.v.reserve(total);
  for (auto& tr : part) {
    all.r.insert(all.r.end(), tr.r.begin(), tr.r.end());
    all.c.insert(all.c.end(), tr.c.begin(), tr.c.end());
    all.v.insert(all.v.end(), tr.v.begin(), tr.v.end());
    tr = Triplets{};
  }
  auto* inst = new pdlp_instance;
  inst->rows = mw;
  inst->cols = n;
  build_both(inst, all);
  all = Triplets{};

  inst->var_lower.resize(n);
  inst->var_upper.resize(n);
  std::vector<double> xs(n), rs(n);
  parallel(n, [&](int, int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      SplitMix rng = stream(2, i);
      int kind = 0;
      if (p.bound_kind == 1) {
        const double u = rng.u01();
        kind = u < 0.6 ? 0 : (u < 0.9 ? 1 : 2);
      }
      if (kind == 0) {
        inst->var_lower[i] = 0.0;
        inst->var_upper[i] = p.bound_kind == 0 ? p.box_hi : kInf;
        xs[i] = rng.uniform(0.0, p.box_hi);
        rs[i] = std::fabs(rng.normal());
      } else if (kind == 1) {
        const double l = rng.uniform(-p.box_hi, 0.0);
        const double u = l + rng.uniform(1.0, 2.0 * p.box_hi);
        inst->var_lower[i] = l;
        inst->var_upper[i] = u;
        xs[i] = rng.uniform(l, u);
        rs[i] = rng.normal();
      } else {
        inst->var_lower[i] = -kInf;
        inst->var_upper[i] = kInf;
        xs[i] = p.box_hi * 0.5 * rng.normal();
        rs[i] = 0.0;
      }
    }
  });
  const std::vector<double> ax = row_product(inst, xs);
  inst->con_lower.resize(mw);
  inst->con_upper.resize(mw);
  std::vector<double> ys(mw);
  const int64_t n_eq_first = static_cast<int64_t>(std::llround(p.eq_frac * static_cast<double>(m)));
  parallel(mw, [&](int, int64_t lo, int64_t hi) {
    for (int64_t j = lo; j < hi; ++j) {
      const int64_t g = r0 + j;
      SplitMix rng = stream(3, g);
      const bool eq = p.eq_rows_first ? (g < n_eq_first) : (rng.u01() < p.eq_frac);
      if (eq) {
        inst->con_lower[j] = ax[j];
        inst->con_upper[j] = ax[j];
        ys[j] = rng.normal();
      } else {
        inst->con_lower[j] = -kInf;
        inst->con_upper[j] = ax[j] + rng.uniform(0.0, p.slack_hi);
        ys[j] = -std::fabs(rng.normal());
      }
    }
  });
  const std::vector<double> aty = col_product(inst, ys);
  inst->objective.resize(n);
  for (int64_t i = 0; i < n; ++i) inst->objective[i] = aty[i] + rs[i];
  inst->feasible_point = std::move(xs);
  return inst;
}

// One rank's shard of the counter-based instance (the window generator over
// all m rows): rows [r0, r1) in both layouts exactly as the window generator
// draws them, and for the column block [c0, c1) the bounds and the GLOBAL
// objective c = A'y* + r* (every entry of the block's columns, all rows).
// Work O(entries of the whole instance) for the matrix pass (each column's
// stream is drawn to find its window rows) plus O(entries of the block) for
// the objective; memory O(shard).
struct pdlp_gen_shard {
  pdlp_instance* win = nullptr;
  int64_t rows = 0, cols = 0, r0 = 0, r1 = 0, c0 = 0, c1 = 0, entry_offset = 0;
  std::vector<double> objective, var_lower, var_upper;
  // column cut: the block's layouts and the window rows' bounds
  int32_t cut = 0;
  std::vector<int64_t> rstart, rindex, cstart, cindex;
  std::vector<double> rvalue, cvalue, con_lower, con_upper;
  ~pdlp_gen_shard() { delete win; }
};

static pdlp_gen_shard* build_shard(const pdlp_gen_params* params, int64_t r0, int64_t r1,
                                   int64_t c0, int64_t c1, int32_t cut);

pdlp_gen_shard* pdlp_gen_random_lp_shard(const pdlp_gen_params* params, int64_t r0, int64_t r1,
                                         int64_t c0, int64_t c1) {
  return build_shard(params, r0, r1, c0, c1, 0);
}

static pdlp_gen_shard* build_shard(const pdlp_gen_params* params, int64_t r0, int64_t r1,
                                   int64_t c0, int64_t c1, int32_t cut) {
  const pdlp_gen_params& p = *params;
  if (c0 < 0 || c1 > p.cols || c0 > c1) return nullptr;
  auto* sh = new pdlp_gen_shard;
  sh->cut = cut;
  int64_t before = 0;
  sh->win = random_lp_window(params, r0, r1, &before);
  if (sh->win == nullptr) {
    delete sh;
    return nullptr;
  }
  sh->rows = p.rows;
  sh->cols = p.cols;
  sh->r0 = r0;
  sh->r1 = r1;
  sh->c0 = c0;
  sh->c1 = c1;
  sh->entry_offset = before;
  const int64_t m = p.rows, nb = c1 - c0;
  sh->var_lower.assign(sh->win->var_lower.begin() + c0, sh->win->var_lower.begin() + c1);
  sh->var_upper.assign(sh->win->var_upper.begin() + c0, sh->win->var_upper.begin() + c1);
  sh->objective.assign(static_cast<size_t>(nb), 0.0);
  auto stream = [&](uint64_t kind, int64_t i) {
    SplitMix h(p.seed ^ (kind * 0xd1b54a32d192ed03ull));
    h.s += static_cast<uint64_t>(i) * 0x9e3779b97f4a7c15ull;
    return SplitMix(h.next());
  };
  const int64_t n_eq_first = static_cast<int64_t>(std::llround(p.eq_frac * static_cast<double>(m)));
  // y*_g from row g's stream, as the window generator draws it
  auto ystar = [&](int64_t g) {
    SplitMix rng = stream(3, g);
    const bool eq = p.eq_rows_first ? (g < n_eq_first) : (rng.u01() < p.eq_frac);
    if (eq) return rng.normal();
    (void)rng.uniform(0.0, p.slack_hi);
    return -std::fabs(rng.normal());
  };
  // r*_i from column i's bound stream
  auto rstar = [&](int64_t i) {
    SplitMix rng = stream(2, i);
    int kind = 0;
    if (p.bound_kind == 1) {
      const double u = rng.u01();
      kind = u < 0.6 ? 0 : (u < 0.9 ? 1 : 2);
    }
    if (kind == 0) {
      (void)rng.uniform(0.0, p.box_hi);
      return std::fabs(rng.normal());
    }
    if (kind == 1) {
      const double l = rng.uniform(-p.box_hi, 0.0);
      const double u = l + rng.uniform(1.0, 2.0 * p.box_hi);
      (void)rng.uniform(l, u);
      return rng.normal();
    }
    (void)rng.normal();
    return 0.0;
  };
  const int T = static_cast<int>(std::max<unsigned>(1u, std::min(32u, std::thread::hardware_concurrency())));
  std::vector<std::thread> th;
  const int64_t per = (nb + T - 1) / T;
  // column cut: the block's columns as stored (per thread, joined below)
  std::vector<std::vector<int64_t>> t_len(static_cast<size_t>(T)), t_row(static_cast<size_t>(T));
  std::vector<std::vector<double>> t_val(static_cast<size_t>(T));
  const bool keep = sh->cut == 1;
  for (int t = 0; t < T; ++t) {
    const int64_t lo = std::min(nb, per * t), hi = std::min(nb, lo + per);
    th.emplace_back([&, t, lo, hi] {
      std::vector<std::pair<int64_t, double>> col;
      for (int64_t q = lo; q < hi; ++q) {
        const int64_t c = c0 + q;
        SplitMix rng = stream(1, c);
        const int64_t k = sample_count(rng, p);
        col.clear();
        for (int64_t e = 0; e < k; ++e) {
          const int64_t row = rng.below(m);
          col.emplace_back(row, sample_value(rng, p));
        }
        // the column as build_layout stores it: rows ascending, duplicates
        // summed in draw order; then the product in storage order
        std::stable_sort(col.begin(), col.end(),
                         [](const auto& a, const auto& b) { return a.first < b.first; });
        double acc = 0.0;
        int64_t len = 0;
        for (size_t e = 0; e < col.size();) {
          double v = col[e].second;
          size_t f = e + 1;
          while (f < col.size() && col[f].first == col[e].first) v += col[f++].second;
          acc += v * ystar(col[e].first);
          if (keep) {
            t_row[static_cast<size_t>(t)].push_back(col[e].first);
            t_val[static_cast<size_t>(t)].push_back(v);
            ++len;
          }
          e = f;
        }
        if (keep) t_len[static_cast<size_t>(t)].push_back(len);
        sh->objective[static_cast<size_t>(q)] = acc + rstar(c);
      }
    });
  }
  for (auto& x : th) x.join();
  if (keep) {
    // K_g^T: the block's columns in order; K_g: its transpose over all rows
    // (a counting sort keeps columns ascending within each row)
    sh->cstart.assign(1, 0);
    for (int t = 0; t < T; ++t) {
      for (int64_t len : t_len[static_cast<size_t>(t)]) sh->cstart.push_back(sh->cstart.back() + len);
      sh->cindex.insert(sh->cindex.end(), t_row[static_cast<size_t>(t)].begin(), t_row[static_cast<size_t>(t)].end());
      sh->cvalue.insert(sh->cvalue.end(), t_val[static_cast<size_t>(t)].begin(), t_val[static_cast<size_t>(t)].end());
      t_row[static_cast<size_t>(t)] = {};
      t_val[static_cast<size_t>(t)] = {};
    }
    const int64_t nnz = static_cast<int64_t>(sh->cindex.size());
    sh->rstart.assign(static_cast<size_t>(m + 1), 0);
    for (int64_t r : sh->cindex) ++sh->rstart[static_cast<size_t>(r + 1)];
    for (int64_t r = 0; r < m; ++r) sh->rstart[static_cast<size_t>(r + 1)] += sh->rstart[static_cast<size_t>(r)];
    sh->rindex.resize(static_cast<size_t>(nnz));
    sh->rvalue.resize(static_cast<size_t>(nnz));
    std::vector<int64_t> fill(sh->rstart.begin(), sh->rstart.end() - 1);
    for (int64_t q = 0; q < nb; ++q) {
      for (int64_t k = sh->cstart[static_cast<size_t>(q)]; k < sh->cstart[static_cast<size_t>(q + 1)]; ++k) {
        const int64_t o = fill[static_cast<size_t>(sh->cindex[static_cast<size_t>(k)])]++;
        sh->rindex[static_cast<size_t>(o)] = q;
        sh->rvalue[static_cast<size_t>(o)] = sh->cvalue[static_cast<size_t>(k)];
      }
    }
    // only the window rows' bounds are kept from the window
    sh->con_lower = sh->win->con_lower;
    sh->con_upper = sh->win->con_upper;
    delete sh->win;
    sh->win = nullptr;
  }
  return sh;
}

pdlp_gen_shard* pdlp_gen_random_lp_colshard(const pdlp_gen_params* params, int64_t r0, int64_t r1,
                                            int64_t c0, int64_t c1) {
  return build_shard(params, r0, r1, c0, c1, 1);
}

void pdlp_gen_shard_view(const pdlp_gen_shard* sh, pdlp_shard_view* out) {
  std::memset(out, 0, sizeof(*out));
  out->plan.rows = sh->rows;
  out->plan.cols = sh->cols;
  out->plan.row_begin = sh->r0;
  out->plan.row_end = sh->r1;
  out->plan.col_begin = sh->c0;
  out->plan.col_end = sh->c1;
  out->plan.cut = sh->cut;
  if (sh->cut == 1) {
    out->rows = {sh->rows, static_cast<int64_t>(sh->rvalue.size()), sh->rstart.data(),
                 sh->rindex.data(), sh->rvalue.data()};
    out->cols = {sh->c1 - sh->c0, static_cast<int64_t>(sh->cvalue.size()), sh->cstart.data(),
                 sh->cindex.data(), sh->cvalue.data()};
    out->objective = sh->objective.data();
    out->var_lower = sh->var_lower.data();
    out->var_upper = sh->var_upper.data();
    out->con_lower = sh->con_lower.data();
    out->con_upper = sh->con_upper.data();
    out->entry_offset = 0;
    out->row_entry_offset = nullptr;
    return;
  }
  const pdlp_instance* w = sh->win;
  out->rows = {w->rows, static_cast<int64_t>(w->by_row.value.size()), w->by_row.start.data(),
               w->by_row.index.data(), w->by_row.value.data()};
  out->cols = {w->cols, static_cast<int64_t>(w->by_col.value.size()), w->by_col.start.data(),
               w->by_col.index.data(), w->by_col.value.data()};
  out->objective = sh->objective.data();
  out->var_lower = sh->var_lower.data();
  out->var_upper = sh->var_upper.data();
  out->con_lower = w->con_lower.data();
  out->con_upper = w->con_upper.data();
  out->entry_offset = sh->entry_offset;
}

void pdlp_gen_shard_free(pdlp_gen_shard* sh) { delete sh; }

pdlp_instance* pdlp_gen_transport(int64_t sources, int64_t sinks, uint64_t seed) {
  if (sources < 1 || sinks < 1) return nullptr;
  SplitMix rng(seed);
  auto* inst = new pdlp_instance;
  const int64_t m = sources + sinks, n = sources * sinks;
  inst->rows = m;
  inst->cols = n;
  std::vector<double> supply(sources), demand(sinks);
  double total_s = 0.0, total_d = 0.0;
  for (auto& s : supply) {
    s = static_cast<double>(50 + rng.below(101));
    total_s += s;
  }
  for (auto& d : demand) {
    d = static_cast<double>(50 + rng.below(101));
    total_d += d;
  }
  const double scale = 0.95 * total_s / total_d;
  for (auto& d : demand) d *= scale;

  // Row layout: supply row s holds columns s*sinks .. s*sinks+sinks-1;
  // demand row d holds columns d, sinks+d, 2 sinks+d, ...
  Layout& R = inst->by_row;
  R.start.resize(m + 1);
  R.index.resize(2 * n);
  R.value.assign(2 * n, 1.0);
  R.start[0] = 0;
  for (int64_t s = 0; s < sources; ++s) {
    R.start[s + 1] = R.start[s] + sinks;
    for (int64_t d = 0; d < sinks; ++d) R.index[R.start[s] + d] = s * sinks + d;
  }
  for (int64_t d = 0; d < sinks; ++d) {
    const int64_t row = sources + d;
    R.start[row + 1] = R.start[row] + sources;
    for (int64_t s = 0; s < sources; ++s) R.index[R.start[row] + s] = s * sinks + d;
  }
  // Column layout: column (s, d) holds rows s and sources + d (sorted).
  Layout& C = inst->by_col;
  C.start.resize(n + 1);
  C.index.resize(2 * n);
  C.value.assign(2 * n, 1.0);
  for (int64_t v = 0; v <= n; ++v) C.start[v] = 2 * v;
  for (int64_t s = 0; s < sources; ++s) {
    for (int64_t d = 0; d < sinks; ++d) {
      const int64_t v = s * sinks + d;
      C.index[2 * v] = s;
      C.index[2 * v + 1] = sources + d;
    }
  }
  inst->objective.resize(n);
  for (auto& c : inst->objective) c = rng.uniform(1.0, 100.0);
  inst->var_lower.assign(n, 0.0);
  inst->var_upper.assign(n, kInf);
  inst->con_lower.resize(m);
  inst->con_upper.resize(m);
  for (int64_t s = 0; s < sources; ++s) {
    inst->con_lower[s] = -kInf;
    inst->con_upper[s] = supply[s];
  }
  for (int64_t d = 0; d < sinks; ++d) {
    inst->con_lower[sources + d] = demand[d];
    inst->con_upper[sources + d] = kInf;
  }
  // Proportional split x_sd = s_s d_d / S: row sums 0.95 s_s <= s_s, column
  // sums d_d, so the instance is feasible (total demand = 0.95 total supply).
  inst->feasible_point.resize(n);
  for (int64_t s = 0; s < sources; ++s) {
    for (int64_t d = 0; d < sinks; ++d) {
      inst->feasible_point[s * sinks + d] = supply[s] * demand[d] / total_s;
    }
  }
  return inst;
}

pdlp_instance* pdlp_gen_unit_commitment(int64_t periods, int64_t generators, uint64_t seed) {
  if (periods < 2 || generators < 1) return nullptr;
  SplitMix rng(seed);
  const int64_t T = periods, G = generators;
  auto* inst = new pdlp_instance;
  const int64_t n = 2 * T * G;
  const int64_t m = T + (T - 1) * G + T * G;
  inst->rows = m;
  inst->cols = n;
  std::vector<double> cap(G), ramp(G), cost(G);
  double total_cap = 0.0;
  for (int64_t g = 0; g < G; ++g) {
    cap[g] = rng.uniform(50.0, 500.0);
    ramp[g] = rng.uniform(0.2, 0.6) * cap[g];
    cost[g] = rng.uniform(10.0, 200.0);
    total_cap += cap[g];
  }
  std::vector<double> demand(T);
  for (int64_t t = 0; t < T; ++t) {
    const double season = 1.0 + 0.3 * std::sin(6.283185307179586 * static_cast<double>(t) / 24.0);
    demand[t] = 0.5 * total_cap * season * (1.0 + 0.05 * rng.normal());
  }
  auto pvar = [&](int64_t t, int64_t g) { return t * G + g; };
  auto uvar = [&](int64_t t, int64_t g) { return T * G + t * G + g; };
  Triplets tr;
  tr.r.reserve(5 * T * G);
  tr.c.reserve(5 * T * G);
  tr.v.reserve(5 * T * G);
  inst->con_lower.resize(m);
  inst->con_upper.resize(m);
  for (int64_t t = 0; t < T; ++t) {  // demand balance
    for (int64_t g = 0; g < G; ++g) tr.push(t, pvar(t, g), 1.0);
    inst->con_lower[t] = demand[t];
    inst->con_upper[t] = demand[t];
  }
  for (int64_t t = 1; t < T; ++t) {  // ramps
    for (int64_t g = 0; g < G; ++g) {
      const int64_t row = T + (t - 1) * G + g;
      tr.push(row, pvar(t - 1, g), -1.0);
      tr.push(row, pvar(t, g), 1.0);
      inst->con_lower[row] = -ramp[g];
      inst->con_upper[row] = ramp[g];
    }
  }
  for (int64_t t = 0; t < T; ++t) {  // capacity
    for (int64_t g = 0; g < G; ++g) {
      const int64_t row = T + (T - 1) * G + t * G + g;
      tr.push(row, pvar(t, g), 1.0);
      tr.push(row, uvar(t, g), -cap[g]);
      inst->con_lower[row] = -kInf;
      inst->con_upper[row] = 0.0;
    }
  }
  build_both(inst, tr);
  inst->objective.resize(n);
  inst->var_lower.assign(n, 0.0);
  inst->var_upper.resize(n);
  for (int64_t t = 0; t < T; ++t) {
    for (int64_t g = 0; g < G; ++g) {
      inst->objective[pvar(t, g)] = cost[g];
      inst->objective[uvar(t, g)] = 0.1 * cost[g] * cap[g] / 100.0;
      inst->var_upper[pvar(t, g)] = kInf;
      inst->var_upper[uvar(t, g)] = 1.0;
    }
  }
  inst->feasible_point.resize(n);
  for (int64_t t = 0; t < T; ++t) {
    for (int64_t g = 0; g < G; ++g) {
      const double pg = demand[t] * cap[g] / total_cap;
      inst->feasible_point[pvar(t, g)] = pg;
      inst->feasible_point[uvar(t, g)] = pg / cap[g];
    }
  }
  return inst;
}

pdlp_instance* pdlp_instance_from_triplets(int64_t rows, int64_t cols, int64_t count,
                                           const int64_t* r, const int64_t* c,
                                           const double* v, const double* objective,
                                           const double* con_lower, const double* con_upper,
                                           const double* var_lower, const double* var_upper) {
  if (rows < 0 || cols < 0 || count < 0) return nullptr;
  for (int64_t k = 0; k < count; ++k) {
    if (r[k] < 0 || r[k] >= rows || c[k] < 0 || c[k] >= cols) return nullptr;
  }
  auto* inst = new pdlp_instance;
  inst->rows = rows;
  inst->cols = cols;
  build_layout(rows, count, r, c, v, inst->by_row);
  build_layout(cols, count, c, r, v, inst->by_col);
  inst->objective.assign(objective, objective + cols);
  inst->con_lower.assign(con_lower, con_lower + rows);
  inst->con_upper.assign(con_upper, con_upper + rows);
  inst->var_lower.assign(var_lower, var_lower + cols);
  inst->var_upper.assign(var_upper, var_upper + cols);
  return inst;
}

void pdlp_instance_view(const pdlp_instance* inst, pdlp_problem_view* view) {
  view->rows = inst->rows;
  view->cols = inst->cols;
  view->by_row = {inst->rows, static_cast<int64_t>(inst->by_row.value.size()),
                  inst->by_row.start.data(), inst->by_row.index.data(),
                  inst->by_row.value.data()};
  view->by_col = {inst->cols, static_cast<int64_t>(inst->by_col.value.size()),
                  inst->by_col.start.data(), inst->by_col.index.data(),
                  inst->by_col.value.data()};
  view->objective = inst->objective.data();
  view->con_lower = inst->con_lower.data();
  view->con_upper = inst->con_upper.data();
  view->var_lower = inst->var_lower.data();
  view->var_upper = inst->var_upper.data();
}

const double* pdlp_instance_feasible_point(const pdlp_instance* inst) {
  return inst->feasible_point.empty() ? nullptr : inst->feasible_point.data();
}

void pdlp_instance_free(pdlp_instance* inst) { delete inst; }

}  // extern "C"
