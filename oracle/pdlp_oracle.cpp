// oracle/pdlp_oracle.cpp — TEST INFRASTRUCTURE ONLY (never linked into the
// product).  An independent CPU restatement of the reference PDHG path, used
// as the parity checker when the reference library itself is not built.  It
// is pinned bit-for-bit against oracle/_ref (the reference compiled in place)
// and against the reference's known-answer tests (tests/test_oracle.py).
//
// Arithmetic order follows the reference for threads=1 and S shards:
//   line products sequential in storage order   kernels.hpp:30-59
//   sharded sums, ascending shard combine       kernels.hpp:69-97, shard.hpp:24-40
//   plain sequential loops elsewhere            residuals.hpp, restarts.hpp
// Build: oracle/Makefile (g++ -O2 -ffp-contract=off, no -march).
// Exposes the same ref_* C-ABI as ref_capi.cpp.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "pdlp_b200.h"

namespace orc {

using Vec = std::vector<double>;
constexpr double INF = std::numeric_limits<double>::infinity();
thread_local std::string last_error;

// ------------------------------------------------------------ data model ---
struct Lines {  // one compressed orientation
  std::vector<int64_t> ptr, idx;
  Vec val;
  int64_t dim() const { return static_cast<int64_t>(ptr.size()) - 1; }
};

struct Lp {
  int64_t m = 0, n = 0;
  Lines rows, cols;  // by_row, by_col
  Vec c, lc, uc, lv, uv;
};

Lp from_view(const pdlp_problem_view* v) {
  Lp p;
  p.m = v->rows;
  p.n = v->cols;
  auto lines = [](const pdlp_csr_view& s) {
    Lines L;
    L.ptr.assign(s.start, s.start + s.primary_dim + 1);
    L.idx.assign(s.index, s.index + s.nnz);
    L.val.assign(s.value, s.value + s.nnz);
    return L;
  };
  p.rows = lines(v->by_row);
  p.cols = lines(v->by_col);
  p.c.assign(v->objective, v->objective + p.n);
  p.lc.assign(v->con_lower, v->con_lower + p.m);
  p.uc.assign(v->con_upper, v->con_upper + p.m);
  p.lv.assign(v->var_lower, v->var_lower + p.n);
  p.uv.assign(v->var_upper, v->var_upper + p.n);
  return p;
}

// ---------------------------------------------------------------- scalars ---
inline double zmul(double a, double b) { return (a == 0.0 || b == 0.0) ? 0.0 : a * b; }
inline double box(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }
inline double dist(double v, double lo, double hi) {
  return v < lo ? lo - v : (v > hi ? v - hi : 0.0);
}
inline double keepmax(double a, double v) { return (a < v) ? v : a; }

enum { CONE_ZERO, CONE_NONPOS, CONE_NONNEG, CONE_FREE };
inline int mult_cone(double lo, double hi) {  // sign cone of a bound pair
  const bool a = lo > -INF, b = hi < INF;
  return (a && b) ? CONE_FREE : a ? CONE_NONNEG : b ? CONE_NONPOS : CONE_ZERO;
}
inline int rec_cone(double lo, double hi) {  // recession cone
  const bool a = lo > -INF, b = hi < INF;
  return (a && b) ? CONE_ZERO : a ? CONE_NONNEG : b ? CONE_NONPOS : CONE_FREE;
}
inline double proj(double v, int k) {
  if (k == CONE_ZERO) return 0.0;
  if (k == CONE_NONPOS) return v < 0.0 ? v : 0.0;
  if (k == CONE_NONNEG) return v > 0.0 ? v : 0.0;
  return v;
}

// ------------------------------------------------------------ products ---
void line_products(const Lines& L, const Vec& v, Vec& out) {
  out.assign(static_cast<size_t>(L.dim()), 0.0);
  for (int64_t r = 0; r < L.dim(); ++r) {
    double s = 0.0;
    for (int64_t k = L.ptr[r]; k < L.ptr[r + 1]; ++k) s += L.val[k] * v[L.idx[k]];
    out[r] = s;
  }
}

// S contiguous shards, earlier ones larger by one; partial sums combined in
// ascending order.
struct Plan {
  int64_t dim, S;
  int64_t lo(int64_t s) const { return s * (dim / S) + std::min(s, dim % S); }
  int64_t hi(int64_t s) const { return lo(s + 1); }
};

template <class F>
double shard_sum(const Plan& pl, F&& term) {
  double total = 0.0;
  for (int64_t s = 0; s < pl.S; ++s) {
    double part = 0.0;
    for (int64_t i = pl.lo(s); i < pl.hi(s); ++i) part += term(i);
    total += part;
  }
  return total;
}

template <class F>
double shard_max(const Plan& pl, F&& term) {
  double total = 0.0;
  for (int64_t s = 0; s < pl.S; ++s) {
    double part = 0.0;
    for (int64_t i = pl.lo(s); i < pl.hi(s); ++i) part = keepmax(part, term(i));
    total = keepmax(total, part);
  }
  return total;
}

double sqdist(const Plan& pl, const Vec& a, const Vec& b) {
  return shard_sum(pl, [&](int64_t i) {
    const double d = a[i] - b[i];
    return d * d;
  });
}

// --------------------------------------------------------- rescaling ---
struct Scales {
  Vec row, col;
};

// Divide every entry by f_row * f_col and fold the factors into the problem.
void divide_by(Lp& p, Scales& sc, const Vec& fr, const Vec& fc) {
  for (int64_t r = 0; r < p.m; ++r)
    for (int64_t k = p.rows.ptr[r]; k < p.rows.ptr[r + 1]; ++k)
      p.rows.val[k] /= fr[r] * fc[p.rows.idx[k]];
  for (int64_t c = 0; c < p.n; ++c)
    for (int64_t k = p.cols.ptr[c]; k < p.cols.ptr[c + 1]; ++k)
      p.cols.val[k] /= fc[c] * fr[p.cols.idx[k]];
  for (int64_t j = 0; j < p.m; ++j) {
    p.lc[j] /= fr[j];
    p.uc[j] /= fr[j];
    sc.row[j] /= fr[j];
  }
  for (int64_t i = 0; i < p.n; ++i) {
    p.c[i] /= fc[i];
    p.lv[i] *= fc[i];
    p.uv[i] *= fc[i];
    sc.col[i] /= fc[i];
  }
}

Vec line_factor(const Lines& L, bool one_norm) {
  Vec f(static_cast<size_t>(L.dim()));
  for (int64_t r = 0; r < L.dim(); ++r) {
    double a = 0.0;
    for (int64_t k = L.ptr[r]; k < L.ptr[r + 1]; ++k) {
      a = one_norm ? a + std::fabs(L.val[k]) : std::max(a, std::fabs(L.val[k]));
    }
    f[r] = a > 0.0 ? std::sqrt(a) : 1.0;
  }
  return f;
}

Scales precondition(Lp& p, int ruiz, bool pc) {
  Scales sc{Vec(p.m, 1.0), Vec(p.n, 1.0)};
  for (int it = 0; it < ruiz + (pc ? 1 : 0); ++it) {
    const bool one = it >= ruiz;
    const Vec fr = line_factor(p.rows, one), fc = line_factor(p.cols, one);
    divide_by(p, sc, fr, fc);
  }
  return sc;
}

// ------------------------------------------------------------- summaries ---
struct Summary {
  double pres = INF, dres = INF, pobj = 0.0, dobj = 0.0, agap = INF, rgap = INF;
};

Summary summarize(double pres, double dres, double pobj, double dobj) {
  Summary s{pres, dres, pobj, dobj, INF, INF};
  if (!std::isfinite(dobj)) return s;
  s.agap = std::fabs(pobj - dobj);
  s.rgap = s.agap == 0.0 ? 0.0 : s.agap / std::max(std::fabs(pobj), std::fabs(dobj));
  return s;
}

struct Tols {
  double p = 1e-8, d = 1e-8, g = 1e-2;
};
bool meets(const Summary& s, const Tols& t) { return s.pres <= t.p && s.dres <= t.d && s.rgap <= t.g; }

// reduced cost of coordinate i; mode 0 natural (cone projection), 1 robust
double rcost(const Lp& p, int64_t i, double xi, double atyi, int mode) {
  const double v = p.c[i] - atyi;
  if (mode == 0) return proj(v, mult_cone(p.lv[i], p.uv[i]));
  if (v > 0.0 && xi - p.lv[i] <= std::fabs(xi)) return v;
  if (v < 0.0 && p.uv[i] - xi <= std::fabs(xi)) return v;
  return 0.0;
}

// -p(-y; l_c, u_c) - p(-r; l_v, u_v) accumulated rows first, then columns.
double dual_obj(const Lp& p, const Vec& y, const Vec& r) {
  double pen = 0.0;
  auto add = [&](double w, double lo, double hi) {
    const double v = -w;
    if (v > 0.0) pen += zmul(hi, v);
    else if (v < 0.0) pen += zmul(lo, v);
  };
  for (int64_t j = 0; j < p.m; ++j) add(y[j], p.lc[j], p.uc[j]);
  for (int64_t i = 0; i < p.n; ++i) add(r[i], p.lv[i], p.uv[i]);
  return -pen;
}

// Residual summary from products; scales == nullptr means original space.
Summary residuals(const Lp& p, const Scales* sc, const Vec& x, const Vec& y, const Vec& r,
                  const Vec& ax, const Vec& aty) {
  double pres = 0.0;
  for (int64_t j = 0; j < p.m; ++j) {
    const double d = dist(ax[j], p.lc[j], p.uc[j]);
    pres = std::max(pres, sc ? d / sc->row[j] : d);
  }
  for (int64_t i = 0; i < p.n; ++i) {
    const double d = dist(x[i], p.lv[i], p.uv[i]);
    pres = std::max(pres, sc ? d * sc->col[i] : d);
  }
  double dres = 0.0, pobj = 0.0;
  for (int64_t i = 0; i < p.n; ++i) {
    const double d = std::fabs(p.c[i] - aty[i] - r[i]);
    dres = std::max(dres, sc ? d / sc->col[i] : d);
    pobj += p.c[i] * x[i];
  }
  return summarize(pres, dres, pobj, dual_obj(p, y, r));
}

Vec rcosts(const Lp& p, const Vec& x, const Vec& aty, int mode) {
  Vec r(static_cast<size_t>(p.n));
  for (int64_t i = 0; i < p.n; ++i) r[i] = rcost(p, i, x[i], aty[i], mode);
  return r;
}

// Original-space KKT from scratch (products recomputed).
Summary kkt(const Lp& p, const Vec& x, const Vec& y, int mode, Vec& r) {
  Vec ax, aty;
  line_products(p.rows, x, ax);
  line_products(p.cols, y, aty);
  r = rcosts(p, x, aty, mode);
  return residuals(p, nullptr, x, y, r, ax, aty);
}

// --------------------------------------------------------- gap / restarts ---
struct Break {
  double lam, dc, di;
};

double ball_gap(const Lp& p, const Vec& x, const Vec& y, const Vec& ax, const Vec& aty, double w,
                double r) {
  if (!(r > 0.0)) return 0.0;
  const double r2 = r * r;
  std::vector<Break> ev;
  double cm = 0.0, bm = 0.0;
  for (int64_t i = 0; i < p.n; ++i) {
    const double g = aty[i] - p.c[i];
    if (g == 0.0) continue;
    const double off = (g > 0.0 ? p.uv[i] : p.lv[i]) - x[i];
    if (off == 0.0) continue;
    bm += g * g / w;
    if (std::isfinite(off)) ev.push_back({g / (w * off), w * off * off, -g * g / w});
  }
  for (int64_t j = 0; j < p.m; ++j) {
    const double yj = y[j], lo = ax[j] - p.uc[j], hi = ax[j] - p.lc[j];
    const double mass = yj * yj / w;
    if (yj > 0.0) {
      if (hi <= 0.0) {
        if (hi < 0.0) bm += w * hi * hi;
        continue;
      }
      if (std::isfinite(hi)) {
        bm += w * hi * hi;
        ev.push_back({w * hi / yj, mass, -w * hi * hi});
      } else {
        cm += mass;
      }
      if (lo > 0.0) ev.push_back({w * lo / yj, -mass, w * lo * lo});
    } else if (yj < 0.0) {
      if (lo >= 0.0) {
        if (lo > 0.0) bm += w * lo * lo;
        continue;
      }
      if (std::isfinite(lo)) {
        bm += w * lo * lo;
        ev.push_back({w * lo / yj, mass, -w * lo * lo});
      } else {
        cm += mass;
      }
      if (hi < 0.0) ev.push_back({w * hi / yj, -mass, w * hi * hi});
    } else {
      if (lo > 0.0) bm += w * lo * lo;
      else if (hi < 0.0) bm += w * hi * hi;
    }
  }
  std::sort(ev.begin(), ev.end(), [](const Break& a, const Break& b) { return a.lam > b.lam; });
  double csum = cm, bsum = bm, top = INF, lam_star = -1.0;
  size_t k = 0;
  while (k < ev.size()) {
    const double lam = ev[k].lam;
    if (csum + bsum / (lam * lam) >= r2) {
      lam_star = (bsum > 0.0 && r2 > csum) ? std::sqrt(bsum / (r2 - csum)) : lam;
      lam_star = box(lam_star, lam, top);
      break;
    }
    for (; k < ev.size() && ev[k].lam == lam; ++k) {
      csum += ev[k].dc;
      bsum += ev[k].di;
    }
    top = lam;
  }
  if (lam_star < 0.0) {
    if (bsum > 0.0 && r2 > csum) lam_star = std::min(std::sqrt(bsum / (r2 - csum)), top);
    else if (bsum > 0.0) lam_star = top;
    else lam_star = std::isfinite(top) ? top / 2.0 : 1.0;
  }
  if (!std::isfinite(lam_star)) lam_star = 1e300;
  if (lam_star <= 0.0) lam_star = 1e-300;
  // candidate and value
  double val = 0.0;
  for (int64_t i = 0; i < p.n; ++i) {
    const double xh = box(x[i] + (aty[i] - p.c[i]) / (lam_star * w), p.lv[i], p.uv[i]);
    val += p.c[i] * (x[i] - xh) + aty[i] * xh;
  }
  const double nu = lam_star / w;
  for (int64_t j = 0; j < p.m; ++j) {
    const double lo = ax[j] - p.uc[j], hi = ax[j] - p.lc[j], t = nu * y[j];
    double v = t >= hi ? y[j] - hi / nu : (t <= lo ? y[j] - lo / nu : 0.0);
    v = proj(v, mult_cone(p.lc[j], p.uc[j]));
    val -= v * ax[j];
    if (v > 0.0) val -= zmul(-p.lc[j], v);
    else if (v < 0.0) val -= zmul(-p.uc[j], v);
    if (y[j] > 0.0) val += zmul(-p.lc[j], y[j]);
    else if (y[j] < 0.0) val += zmul(-p.uc[j], y[j]);
  }
  return val > 0.0 ? val / r : 0.0;
}

double weight0(const Lp& p) {
  double c2 = 0.0, b2 = 0.0;
  for (double v : p.c) c2 += v * v;
  for (int64_t j = 0; j < p.m; ++j) {
    double a = 0.0;
    if (std::isfinite(p.lc[j])) a = std::max(a, std::fabs(p.lc[j]));
    if (std::isfinite(p.uc[j])) a = std::max(a, std::fabs(p.uc[j]));
    b2 += a * a;
  }
  const double nc = std::sqrt(c2), nb = std::sqrt(b2);
  return (nc > 1e-12 && nb > 1e-12) ? nc / nb : 1.0;
}

double reweight(double dx, double dy, double w) {
  if (!(dx > 1e-12) || !(dy > 1e-12)) return w;
  return std::exp(0.5 * std::log(dy / dx) + (1.0 - 0.5) * std::log(w));
}

double eta0(const Lp& p) {
  double mx = 0.0;
  for (double v : p.rows.val) mx = std::max(mx, std::fabs(v));
  return mx > 0.0 ? 1.0 / mx : 1.0;
}

// ------------------------------------------------------------- the step ---
struct Trial {
  Vec x, y, aty, ext, dy, daty;
};

void trial_step(const Lp& p, const Vec& x, const Vec& y, const Vec& aty, double tau,
                double sigma, Trial& t) {
  t.x.resize(p.n);
  for (int64_t i = 0; i < p.n; ++i) t.x[i] = box(x[i] - tau * (p.c[i] - aty[i]), p.lv[i], p.uv[i]);
  t.ext.assign(p.m, 0.0);
  for (int64_t r = 0; r < p.m; ++r) {
    double s = 0.0;
    for (int64_t k = p.rows.ptr[r]; k < p.rows.ptr[r + 1]; ++k) {
      const int64_t c = p.rows.idx[k];
      s += p.rows.val[k] * (2.0 * t.x[c] - x[c]);
    }
    t.ext[r] = s;
  }
  t.y.resize(p.m);
  t.dy.resize(p.m);
  for (int64_t j = 0; j < p.m; ++j) {
    const double yh = y[j] - sigma * t.ext[j];
    t.y[j] = yh - sigma * box(yh / sigma, -p.uc[j], -p.lc[j]);
    t.dy[j] = t.y[j] - y[j];
  }
  line_products(p.cols, t.dy, t.daty);
  t.aty.resize(p.n);
  for (int64_t i = 0; i < p.n; ++i) t.aty[i] = aty[i] + t.daty[i];
}

struct Iter {
  Vec x, y, aty;
};

struct Ctrl {
  double eta_hat = 1.0;
  int64_t k = 0;
  int max_retries = 60;
  int64_t accepted = 0, retries = 0;
  double min_bar = INF;
};

double next_eta(double bar, double eta, int64_t k) {
  const double kk = static_cast<double>(k < 1 ? 1 : k) + 1.0;
  return std::min((1.0 - std::pow(kk, -0.3)) * bar, (1.0 + std::pow(kk, -0.6)) * eta);
}

double limit(double movement, double curv) {
  const double d = 2.0 * std::fabs(curv);
  return d > 0.0 ? movement / d : INF;
}

// One accepted step; false on numerical failure (state untouched).
bool adaptive(const Lp& p, const Plan& xp, const Plan& yp, Iter& z, double w, Ctrl& ct,
              Trial& t, double& used) {
  double eta = ct.eta_hat;
  for (int a = 0; a <= ct.max_retries; ++a) {
    if (!(eta > 0.0) || !std::isfinite(eta)) return false;
    trial_step(p, z.x, z.y, z.aty, eta / w, eta * w, t);
    const double dx2 = sqdist(xp, t.x, z.x);
    const double dy2 = sqdist(yp, t.y, z.y);
    const double mv = w * dx2 + dy2 / w;
    const double cv = shard_sum(xp, [&](int64_t i) { return t.daty[i] * (t.x[i] - z.x[i]); });
    if (!std::isfinite(mv) || !std::isfinite(cv)) return false;
    const double bar = limit(mv, cv);
    if (std::isfinite(bar)) ct.min_bar = std::min(ct.min_bar, bar);
    const double nxt = next_eta(bar, eta, ct.k);
    if (eta <= bar) {
      std::swap(z.x, t.x);
      std::swap(z.y, t.y);
      std::swap(z.aty, t.aty);
      ct.eta_hat = nxt;
      ct.k += 1;
      ct.accepted += 1;
      used = eta;
      return true;
    }
    ct.retries += 1;
    eta = nxt;
  }
  return false;
}

// ------------------------------------------------------------ the driver ---
struct Cert {
  int kind = 0;
  Vec rx, ry, rr;
  double res = INF, obj = 0.0;
  std::string src;
};

std::optional<Cert> primal_ray(const Lp& p, const Vec& yc, double eps, const char* src) {
  Vec ray(static_cast<size_t>(p.m));
  double nrm = 0.0;
  for (int64_t j = 0; j < p.m; ++j) {
    ray[j] = proj(yc[j], mult_cone(p.lc[j], p.uc[j]));
    nrm = std::max(nrm, std::fabs(ray[j]));
  }
  if (!(nrm > 0.0)) return std::nullopt;
  Vec aty;
  line_products(p.cols, ray, aty);
  Vec rh(static_cast<size_t>(p.n));
  double res = 0.0;
  for (int64_t i = 0; i < p.n; ++i) {
    rh[i] = proj(-aty[i], mult_cone(p.lv[i], p.uv[i]));
    res = std::max(res, std::fabs(aty[i] + rh[i]));
  }
  if (res > eps * nrm) return std::nullopt;
  const double obj = dual_obj(p, ray, rh);
  if (!(obj > 0.0) || !std::isfinite(obj)) return std::nullopt;
  return Cert{PDLP_CERT_PRIMAL_INFEASIBLE, {}, ray, rh, res, obj, src};
}

std::optional<Cert> dual_ray(const Lp& p, const Vec& xc, double eps, const char* src) {
  double nrm = 0.0;
  for (double v : xc) nrm = std::max(nrm, std::fabs(v));
  if (!(nrm > 0.0)) return std::nullopt;
  double res = 0.0, obj = 0.0;
  for (int64_t i = 0; i < p.n; ++i) res = std::max(res, std::fabs(xc[i] - proj(xc[i], rec_cone(p.lv[i], p.uv[i]))));
  for (int64_t i = 0; i < p.n; ++i) obj += p.c[i] * xc[i];
  Vec ax;
  line_products(p.rows, xc, ax);
  for (int64_t j = 0; j < p.m; ++j) res = std::max(res, std::fabs(ax[j] - proj(ax[j], rec_cone(p.lc[j], p.uc[j]))));
  if (res > eps * nrm || !(obj < 0.0)) return std::nullopt;
  return Cert{PDLP_CERT_DUAL_INFEASIBLE, xc, {}, {}, res, obj, src};
}

struct Cfg {
  Tols tol;
  bool feas_only = false;
  int rc_mode = 0;
  int64_t budget = 0;
  std::chrono::steady_clock::time_point deadline = std::chrono::steady_clock::time_point::max();
  bool restarts = true, rays = true, polish = false;
  double eps_ray = 1e-12;
  int64_t every = 64;
  double th_suff = 0.1, th_nec = 0.9, th_art = 0.5;
  std::optional<double> fixed_eta;
  bool reweight = true;
  int S = 4;
  const pdlp_options* obs = nullptr;
  bool log = false;
  const char* tag = "main";
};

struct State {
  Iter z;
  Trial t;
  Ctrl ct;
  Vec sx, sy;
  double sw = 0.0;
  int64_t cnt = 0;
  double w = 1.0, last_eta = 0.0, mu_last = INF, mu_prev = INF;
  Vec refx, refy;
  int64_t k = 0, k_restart = 0, restarts = 0, trigger = 100, polished = 0;
  Vec solx, soly, solr;
  Summary sol;
  std::optional<Cert> cert;
  std::string detail;

  void init(const Lp& p, const Vec& x0, double e0, double w0) {
    z.x = x0;
    z.y.assign(p.m, 0.0);
    z.aty.assign(p.n, 0.0);
    t = Trial{};
    t.x.assign(p.n, 0.0);
    t.y.assign(p.m, 0.0);
    ct = Ctrl{};
    ct.eta_hat = e0;
    sx.assign(p.n, 0.0);
    sy.assign(p.m, 0.0);
    sw = 0.0;
    cnt = 0;
    w = w0;
    last_eta = e0;
    refx = z.x;
    refy = z.y;
  }
  void averaged(Vec& ax_, Vec& ay_) const {
    const double inv = 1.0 / sw;
    ax_.resize(sx.size());
    ay_.resize(sy.size());
    for (size_t i = 0; i < sx.size(); ++i) ax_[i] = inv * sx[i];
    for (size_t j = 0; j < sy.size(); ++j) ay_[j] = inv * sy[j];
  }
};

class Engine {
 public:
  Engine(const Lp& orig, const Lp& scaled, const Scales& sc) : O(orig), Sp(scaled), sc(sc) {}

  int run(const Cfg& cfg, State& st);

 private:
  const Lp& O;
  const Lp& Sp;
  const Scales& sc;

  bool screen(const Cfg& cfg, const Vec& xs, const Vec& ys, const Vec& axs, const Vec& atys,
              Summary& out, State& st, const char* which) {
    const Vec rs = rcosts(Sp, xs, atys, cfg.rc_mode);
    out = residuals(Sp, &sc, xs, ys, rs, axs, atys);
    const bool pass = cfg.feas_only ? out.pres <= cfg.tol.p : meets(out, cfg.tol);
    if (!pass) return false;
    Vec x(xs.size()), y(ys.size()), r;
    for (size_t i = 0; i < xs.size(); ++i) x[i] = sc.col[i] * xs[i];
    for (size_t j = 0; j < ys.size(); ++j) y[j] = sc.row[j] * ys[j];
    const Summary truth = kkt(O, x, y, cfg.rc_mode, r);
    if (!(cfg.feas_only ? truth.pres <= cfg.tol.p : meets(truth, cfg.tol))) return false;
    st.solx = x;
    st.soly = y;
    st.solr = r;
    st.sol = truth;
    st.detail = std::string("converged at the ") + which;
    return true;
  }

  void capture(const Cfg& cfg, State& st) {
    st.solx.resize(st.z.x.size());
    st.soly.resize(st.z.y.size());
    for (size_t i = 0; i < st.z.x.size(); ++i) st.solx[i] = sc.col[i] * st.z.x[i];
    for (size_t j = 0; j < st.z.y.size(); ++j) st.soly[j] = sc.row[j] * st.z.y[j];
    st.sol = kkt(O, st.solx, st.soly, cfg.rc_mode, st.solr);
  }

  std::optional<int> rays(const Cfg& cfg, State& st, bool have_avg, const Vec& avx,
                          const Vec& avy) {
    struct C {
      const Vec* x;
      const Vec* y;
      const char* s;
    };
    std::vector<C> cs;
    Vec dx, dy;
    if (st.k > 0) {
      dx.resize(st.z.x.size());
      dy.resize(st.z.y.size());
      for (size_t i = 0; i < dx.size(); ++i) dx[i] = st.z.x[i] - st.t.x[i];
      for (size_t j = 0; j < dy.size(); ++j) dy[j] = st.z.y[j] - st.t.y[j];
      cs.push_back({&dx, &dy, "difference"});
    }
    cs.push_back({&st.z.x, &st.z.y, "current"});
    if (have_avg) cs.push_back({&avx, &avy, "average"});
    std::optional<Cert> hit;
    for (const C& c : cs) {
      hit = primal_ray(Sp, *c.y, cfg.eps_ray, c.s);
      if (hit) break;
      hit = dual_ray(Sp, *c.x, cfg.eps_ray, c.s);
      if (hit) break;
    }
    if (!hit) return std::nullopt;
    if (hit->kind == PDLP_CERT_PRIMAL_INFEASIBLE) {
      Vec ray(hit->ry.size());
      for (size_t j = 0; j < ray.size(); ++j) ray[j] = sc.row[j] * hit->ry[j];
      auto v = primal_ray(O, ray, cfg.eps_ray, hit->src.c_str());
      if (v) {
        st.cert = v;
        st.detail = "primal infeasibility certified by the " + hit->src + " ray";
        return PDLP_STATUS_PRIMAL_INFEASIBLE;
      }
    } else {
      Vec ray(hit->rx.size());
      for (size_t i = 0; i < ray.size(); ++i) ray[i] = sc.col[i] * hit->rx[i];
      auto v = dual_ray(O, ray, cfg.eps_ray, hit->src.c_str());
      if (v) {
        st.cert = v;
        st.detail = "dual infeasibility certified by the " + hit->src + " ray";
        return PDLP_STATUS_DUAL_INFEASIBLE;
      }
    }
    return std::nullopt;
  }

  double metric(const Cfg& cfg, const Vec& x, const Vec& y, const Vec& ax, const Vec& aty,
                const State& st, double w) {
    const double dx2 = sqdist(Plan{Sp.n, cfg.S}, x, st.refx);
    const double dy2 = sqdist(Plan{Sp.m, cfg.S}, y, st.refy);
    return ball_gap(Sp, x, y, ax, aty, w, std::sqrt(w * dx2 + dy2 / w));
  }

  bool polish(const Cfg& cfg, State& st, const Vec& avx, const Vec& avy);
};

Lp primal_feas(const Lp& p) {
  Lp q = p;
  q.c.assign(p.n, 0.0);
  return q;
}

Lp dual_feas(const Lp& p) {
  Lp q;
  q.m = p.n;
  q.n = p.m;
  q.rows = p.cols;
  q.cols = p.rows;
  q.c.assign(p.m, 0.0);
  q.lc.resize(p.n);
  q.uc.resize(p.n);
  for (int64_t i = 0; i < p.n; ++i) {
    switch (mult_cone(p.lv[i], p.uv[i])) {
      case CONE_ZERO: q.lc[i] = p.c[i]; q.uc[i] = p.c[i]; break;
      case CONE_NONNEG: q.lc[i] = -INF; q.uc[i] = p.c[i]; break;
      case CONE_NONPOS: q.lc[i] = p.c[i]; q.uc[i] = INF; break;
      default: q.lc[i] = -INF; q.uc[i] = INF; break;
    }
  }
  q.lv.resize(p.m);
  q.uv.resize(p.m);
  for (int64_t j = 0; j < p.m; ++j) {
    switch (mult_cone(p.lc[j], p.uc[j])) {
      case CONE_ZERO: q.lv[j] = 0.0; q.uv[j] = 0.0; break;
      case CONE_NONNEG: q.lv[j] = 0.0; q.uv[j] = INF; break;
      case CONE_NONPOS: q.lv[j] = -INF; q.uv[j] = 0.0; break;
      default: q.lv[j] = -INF; q.uv[j] = INF; break;
    }
  }
  return q;
}

bool Engine::polish(const Cfg& cfg, State& st, const Vec& avx, const Vec& avy) {
  const int64_t left = cfg.budget - st.k - st.polished;
  Cfg sub = cfg;
  sub.feas_only = true;
  sub.rc_mode = 0;
  sub.budget = std::min(st.k / 8, left);
  sub.rays = false;
  sub.polish = false;
  sub.obs = nullptr;
  if (sub.budget <= 0) return false;
  const Lp ps = primal_feas(Sp), po = primal_feas(O);
  State s2;
  s2.init(ps, avx, st.ct.eta_hat, st.w);
  sub.tag = "polish_primal";
  Engine e2(po, ps, sc);
  const int r2 = e2.run(sub, s2);
  st.polished += s2.k;
  if (r2 != PDLP_STATUS_OPTIMAL) return false;
  const Lp ds = dual_feas(Sp), dd = dual_feas(O);
  const Scales sw{sc.col, sc.row};
  State s3;
  s3.init(ds, avy, st.ct.eta_hat, st.w);
  sub.budget = std::min(st.k / 8, left - s2.k);
  if (sub.budget <= 0) return false;
  sub.tol.p = cfg.tol.d;
  sub.tag = "polish_dual";
  Engine e3(dd, ds, sw);
  const int r3 = e3.run(sub, s3);
  st.polished += s3.k;
  if (r3 != PDLP_STATUS_OPTIMAL) return false;
  Vec r;
  const Summary truth = kkt(O, s2.solx, s3.solx, 0, r);
  if (!meets(truth, cfg.tol)) return false;
  st.solx = s2.solx;
  st.soly = s3.solx;
  st.solr = r;
  st.sol = truth;
  st.detail = "converged at the polished point";
  return true;
}

int Engine::run(const Cfg& cfg, State& st) {
  const Plan xp{Sp.n, cfg.S}, yp{Sp.m, cfg.S};
  Vec ax, avx, avy, axa, atya;
  Summary cur;
  while (true) {
    const bool out_of_budget = st.k >= cfg.budget;
    if (out_of_budget || st.k % cfg.every == 0) {
      const bool late = std::chrono::steady_clock::now() >= cfg.deadline;
      line_products(Sp.rows, st.z.x, ax);
      line_products(Sp.cols, st.z.y, st.z.aty);
      const bool have_avg = st.cnt > 0;
      if (have_avg) {
        st.averaged(avx, avy);
        line_products(Sp.rows, avx, axa);
        line_products(Sp.cols, avy, atya);
      }
      if (screen(cfg, st.z.x, st.z.y, ax, st.z.aty, cur, st, "current iterate")) return PDLP_STATUS_OPTIMAL;
      Summary avg;
      if (have_avg && screen(cfg, avx, avy, axa, atya, avg, st, "window average")) return PDLP_STATUS_OPTIMAL;
      if (cfg.rays) {
        if (auto s = rays(cfg, st, have_avg, avx, avy)) {
          capture(cfg, st);
          return *s;
        }
      }
      if (cfg.polish && have_avg && st.k >= st.trigger && !late && !out_of_budget &&
          avg.rgap <= cfg.tol.g) {
        if (polish(cfg, st, avx, avy)) return PDLP_STATUS_OPTIMAL;
        while (st.trigger <= st.k) st.trigger *= 2;
      }
      if (cfg.restarts && st.k > st.k_restart) {
        const double mc = metric(cfg, st.z.x, st.z.y, ax, st.z.aty, st, st.w);
        const double ma = have_avg ? metric(cfg, avx, avy, axa, atya, st, st.w) : INF;
        const bool use_cur = mc < ma;
        const double mu = use_cur ? mc : ma;
        int why = 0;
        if (std::isfinite(st.mu_last)) {
          if (mu <= cfg.th_suff * st.mu_last) why = 1;
          else if (mu <= cfg.th_nec * st.mu_last && mu > st.mu_prev) why = 2;
        }
        if (why == 0 && static_cast<double>(st.k - st.k_restart) >= cfg.th_art * static_cast<double>(st.k)) why = 3;
        if (why != 0) {
          const Vec& cx = use_cur ? st.z.x : avx;
          const Vec& cy = use_cur ? st.z.y : avy;
          const Vec& cax = use_cur ? ax : axa;
          const Vec& caty = use_cur ? st.z.aty : atya;
          if (cfg.reweight) {
            st.w = reweight(std::sqrt(sqdist(xp, cx, st.refx)), std::sqrt(sqdist(yp, cy, st.refy)), st.w);
          }
          st.mu_last = metric(cfg, cx, cy, cax, caty, st, st.w);
          if (!use_cur) {
            st.z.x = avx;
            st.z.y = avy;
            st.z.aty = atya;
          }
          st.refx = st.z.x;
          st.refy = st.z.y;
          st.sx.assign(Sp.n, 0.0);
          st.sy.assign(Sp.m, 0.0);
          st.sw = 0.0;
          st.cnt = 0;
          st.mu_prev = INF;
          st.k_restart = st.k;
          ++st.restarts;
          if (cfg.log) {
            static const char* names[] = {"none", "sufficient", "stalled", "artificial"};
            std::fprintf(stderr, "phase=%s event=restart iter=%lld reason=%s omega=%.6e mu=%.6e\n",
                         cfg.tag, static_cast<long long>(st.k), names[why], st.w, st.mu_last);
          }
        } else {
          st.mu_prev = mu;
        }
      }
      if (cfg.log) {
        std::fprintf(stderr,
                     "phase=%s iter=%lld primal_res=%.6e dual_res=%.6e rel_gap=%.6e mu=%.6e "
                     "omega=%.6e eta=%.6e restarts=%lld\n",
                     cfg.tag, static_cast<long long>(st.k), cur.pres, cur.dres, cur.rgap,
                     st.mu_last, st.w, st.last_eta, static_cast<long long>(st.restarts));
      }
      if (late) {
        capture(cfg, st);
        st.detail = "time limit reached";
        return PDLP_STATUS_TIME_LIMIT;
      }
      if (out_of_budget) {
        capture(cfg, st);
        st.detail = "iteration limit reached";
        return PDLP_STATUS_ITERATION_LIMIT;
      }
    }
    double used = 0.0;
    if (cfg.fixed_eta) {
      const double e = *cfg.fixed_eta;
      trial_step(Sp, st.z.x, st.z.y, st.z.aty, e / st.w, e * st.w, st.t);
      const double ix = shard_max(xp, [&](int64_t i) { return std::fabs(st.t.x[i]); });
      const double iy = shard_max(yp, [&](int64_t j) { return std::fabs(st.t.y[j]); });
      if (!std::isfinite(ix) || !std::isfinite(iy)) {
        capture(cfg, st);
        st.detail = "fixed-size step produced non-finite values";
        return PDLP_STATUS_NUMERICAL_ERROR;
      }
      std::swap(st.z.x, st.t.x);
      std::swap(st.z.y, st.t.y);
      std::swap(st.z.aty, st.t.aty);
      ++st.ct.accepted;
      used = e;
    } else if (!adaptive(Sp, xp, yp, st.z, st.w, st.ct, st.t, used)) {
      line_products(Sp.rows, st.z.x, ax);
      Summary tmp;
      if (screen(cfg, st.z.x, st.z.y, ax, st.z.aty, tmp, st, "current iterate after a numerical error"))
        return PDLP_STATUS_OPTIMAL;
      if (st.cnt > 0) {
        st.averaged(avx, avy);
        line_products(Sp.rows, avx, axa);
        line_products(Sp.cols, avy, atya);
        if (screen(cfg, avx, avy, axa, atya, tmp, st, "window average after a numerical error"))
          return PDLP_STATUS_OPTIMAL;
      }
      capture(cfg, st);
      st.detail = "adaptive step failed to find a usable step size";
      return PDLP_STATUS_NUMERICAL_ERROR;
    }
    ++st.k;
    st.last_eta = used;
    for (int64_t i = 0; i < Sp.n; ++i) st.sx[i] += used * st.z.x[i];
    for (int64_t j = 0; j < Sp.m; ++j) st.sy[j] += used * st.z.y[j];
    st.sw += used;
    st.cnt += 1;
    if (cfg.obs != nullptr && cfg.obs->observer != nullptr) {
      pdlp_iteration_record rec{st.k, st.z.x.data(), Sp.n, st.z.y.data(), Sp.m, used, st.w};
      cfg.obs->observer(cfg.obs->observer_user, &rec);
    }
  }
}

void validate(const Lp& p) {
  auto bad = [](const std::string& m, int64_t i) {
    throw std::invalid_argument("invalid problem: " + m + " (index " + std::to_string(i) + ")");
  };
  for (int64_t i = 0; i < p.n; ++i) if (!std::isfinite(p.c[i])) bad("objective entry not finite", i);
  for (int64_t i = 0; i < p.n; ++i) {
    if (std::isnan(p.lv[i]) || std::isnan(p.uv[i])) bad("variable bound is NaN", i);
    if (p.lv[i] == INF) bad("variable lower bound is +inf", i);
    if (p.uv[i] == -INF) bad("variable upper bound is -inf", i);
    if (p.lv[i] > p.uv[i]) bad("variable bounds crossed", i);
  }
  for (int64_t j = 0; j < p.m; ++j) {
    if (std::isnan(p.lc[j]) || std::isnan(p.uc[j])) bad("constraint bound is NaN", j);
    if (p.lc[j] == INF) bad("constraint lower bound is +inf", j);
    if (p.uc[j] == -INF) bad("constraint upper bound is -inf", j);
    if (p.lc[j] > p.uc[j]) bad("constraint bounds crossed", j);
  }
  for (size_t k = 0; k < p.rows.val.size(); ++k)
    if (!std::isfinite(p.rows.val[k])) bad("matrix entry not finite", static_cast<int64_t>(k));
  // layouts: rebuild the row form from the column form and compare
  std::vector<std::vector<std::pair<int64_t, double>>> byrow(p.m);
  for (int64_t c = 0; c < p.n; ++c)
    for (int64_t k = p.cols.ptr[c]; k < p.cols.ptr[c + 1]; ++k) byrow[p.cols.idx[k]].push_back({c, p.cols.val[k]});
  bool ok = p.rows.val.size() == p.cols.val.size();
  for (int64_t r = 0; ok && r < p.m; ++r) {
    auto& l = byrow[r];
    std::stable_sort(l.begin(), l.end(), [](auto& a, auto& b) { return a.first < b.first; });
    std::vector<std::pair<int64_t, double>> merged;
    for (auto& e : l) {
      if (!merged.empty() && merged.back().first == e.first) merged.back().second += e.second;
      else merged.push_back(e);
    }
    if (static_cast<int64_t>(merged.size()) != p.rows.ptr[r + 1] - p.rows.ptr[r]) ok = false;
    for (size_t q = 0; ok && q < merged.size(); ++q) {
      const int64_t k = p.rows.ptr[r] + static_cast<int64_t>(q);
      if (merged[q].first != p.rows.idx[k] || merged[q].second != p.rows.val[k]) ok = false;
    }
  }
  if (!ok) bad("row/column layouts disagree", -1);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PDLP_OK;
  } catch (const std::invalid_argument& e) {
    last_error = e.what();
    return PDLP_ERR_INVALID_PROBLEM;
  } catch (const std::exception& e) {
    last_error = e.what();
    return PDLP_ERR_INTERNAL;
  }
}

void put(const Vec& v, double* dst) {
  if (dst != nullptr && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
}

}  // namespace orc

using namespace orc;

extern "C" {

const char* ref_last_error(void) { return orc::last_error.c_str(); }

void ref_default_options(pdlp_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->eps_primal = 1e-8;
  o->eps_dual = 1e-8;
  o->eps_rel_gap = 1e-2;
  o->iteration_limit = 200000;
  o->time_limit_seconds = INF;
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
}

int ref_solve(const pdlp_problem_view* pv, const pdlp_options* o, pdlp_result* res) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const Lp orig = from_view(pv);
    validate(orig);
    Lp scaled = orig;
    const Scales sc = o->enable_scaling ? precondition(scaled, o->ruiz_passes, o->pock_chambolle != 0)
                                        : Scales{Vec(orig.m, 1.0), Vec(orig.n, 1.0)};
    Cfg cfg;
    cfg.tol = {o->eps_primal, o->eps_dual, o->eps_rel_gap};
    cfg.rc_mode = o->enable_polish ? 0 : 1;
    cfg.budget = o->iteration_limit;
    if (std::isfinite(o->time_limit_seconds)) {
      cfg.deadline = t0 + std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                              std::chrono::duration<double>(o->time_limit_seconds));
    }
    cfg.restarts = o->enable_restarts != 0;
    cfg.rays = o->detect_infeasibility != 0;
    cfg.polish = o->enable_polish != 0;
    cfg.eps_ray = o->eps_ray;
    cfg.every = o->check_interval;
    cfg.th_suff = o->restart_sufficient;
    cfg.th_nec = o->restart_necessary;
    cfg.th_art = o->restart_artificial;
    if (o->has_fixed_step_size) cfg.fixed_eta = o->fixed_step_size;
    cfg.reweight = o->has_fixed_primal_weight == 0;
    cfg.S = std::max(1, o->threads) * std::max(1, o->shards_per_thread);
    cfg.obs = o;
    cfg.log = o->logging != 0;
    State st;
    Vec x0(static_cast<size_t>(scaled.n));
    for (int64_t i = 0; i < scaled.n; ++i) x0[i] = box(0.0, scaled.lv[i], scaled.uv[i]);
    st.init(scaled, x0, o->has_fixed_step_size ? o->fixed_step_size : eta0(scaled),
            o->has_fixed_primal_weight ? o->fixed_primal_weight : weight0(scaled));
    Engine eng(orig, scaled, sc);
    const int status = eng.run(cfg, st);
    res->status = status;
    put(st.solx, res->x);
    put(st.soly, res->y);
    put(st.solr, res->reduced_costs);
    res->summary = {st.sol.pres, st.sol.dres, st.sol.pobj, st.sol.dobj, st.sol.agap, st.sol.rgap};
    res->has_certificate = st.cert ? 1 : 0;
    if (st.cert) {
      res->cert_kind = st.cert->kind;
      put(st.cert->rx, res->cert_ray_x);
      put(st.cert->ry, res->cert_ray_y);
      put(st.cert->rr, res->cert_ray_r);
      res->cert_residual_inf = st.cert->res;
      res->cert_objective = st.cert->obj;
      std::snprintf(res->cert_source, sizeof(res->cert_source), "%s", st.cert->src.c_str());
    }
    res->iterations = st.k;
    res->polish_iterations = st.polished;
    res->restarts = st.restarts;
    res->step_retries = st.ct.retries;
    res->final_step_size = st.ct.eta_hat;
    res->final_primal_weight = st.w;
    res->min_step_size_limit = st.ct.min_bar;
    res->solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::snprintf(res->termination_detail, sizeof(res->termination_detail), "%s", st.detail.c_str());
  });
}

int ref_pdhg_step(const pdlp_problem_view* pv, const double* x, const double* y, double omega,
                  double eta, double* x_out, double* y_out, int32_t* finite) {
  return guarded([&] {
    const Lp p = from_view(pv);
    const Vec xv(x, x + p.n), yv(y, y + p.m);
    Vec aty;
    line_products(p.cols, yv, aty);
    Trial t;
    trial_step(p, xv, yv, aty, eta / omega, eta * omega, t);
    bool ok = true;
    for (double v : t.x) ok = ok && std::isfinite(v);
    for (double v : t.y) ok = ok && std::isfinite(v);
    *finite = ok ? 1 : 0;
    if (ok) {
      put(t.x, x_out);
      put(t.y, y_out);
    }
  });
}

int ref_adaptive_step(const pdlp_problem_view* pv, double* x, double* y, double* aty,
                      double* io, int32_t threads, int32_t spt, double* prev_x, double* prev_y,
                      double* stats, int32_t* outcome) {
  return guarded([&] {
    const Lp p = from_view(pv);
    const int64_t S = static_cast<int64_t>(std::max(1, threads)) * std::max(1, spt);
    Iter z{Vec(x, x + p.n), Vec(y, y + p.m), Vec(aty, aty + p.n)};
    Trial t;
    t.x.assign(p.n, 0.0);
    t.y.assign(p.m, 0.0);
    Ctrl ct;
    ct.eta_hat = io[0];
    ct.k = static_cast<int64_t>(io[1]);
    ct.max_retries = static_cast<int>(io[2]);
    double used = 0.0;
    const bool ok = adaptive(p, Plan{p.n, S}, Plan{p.m, S}, z, io[3], ct, t, used);
    *outcome = ok ? 0 : 1;
    put(z.x, x);
    put(z.y, y);
    put(z.aty, aty);
    put(t.x, prev_x);
    put(t.y, prev_y);
    io[0] = ct.eta_hat;
    io[1] = static_cast<double>(ct.k);
    stats[0] = static_cast<double>(ct.accepted);
    stats[1] = static_cast<double>(ct.retries);
    stats[2] = ct.min_bar;
    stats[3] = used;
  });
}

int ref_spmv(const pdlp_problem_view* pv, const double* x, double* out, int32_t, int32_t) {
  return guarded([&] {
    const Lp p = from_view(pv);
    Vec o;
    line_products(p.rows, Vec(x, x + p.n), o);
    put(o, out);
  });
}

int ref_spmv_transpose(const pdlp_problem_view* pv, const double* y, double* out, int32_t,
                       int32_t) {
  return guarded([&] {
    const Lp p = from_view(pv);
    Vec o;
    line_products(p.cols, Vec(y, y + p.m), o);
    put(o, out);
  });
}

int ref_apply_rescaling(const pdlp_problem_view* pv, int32_t ruiz, int32_t pc, double* rv,
                        double* cv, double* obj, double* lc, double* uc, double* lv, double* uv,
                        double* rs, double* cs) {
  return guarded([&] {
    Lp p = from_view(pv);
    const Scales sc = precondition(p, ruiz, pc != 0);
    put(p.rows.val, rv);
    put(p.cols.val, cv);
    put(p.c, obj);
    put(p.lc, lc);
    put(p.uc, uc);
    put(p.lv, lv);
    put(p.uv, uv);
    put(sc.row, rs);
    put(sc.col, cs);
  });
}

int ref_normalized_duality_gap(const pdlp_problem_view* pv, const double* x, const double* y,
                               const double* ax, const double* aty, double omega, double r,
                               double* gap) {
  return guarded([&] {
    const Lp p = from_view(pv);
    *gap = ball_gap(p, Vec(x, x + p.n), Vec(y, y + p.m), Vec(ax, ax + p.m), Vec(aty, aty + p.n),
                    omega, r);
  });
}

int ref_kkt_residuals(const pdlp_problem_view* pv, const double* x, const double* y,
                      int32_t rc_mode, double* r_out, pdlp_residual_summary* s) {
  return guarded([&] {
    const Lp p = from_view(pv);
    Vec r;
    const Summary k = kkt(p, Vec(x, x + p.n), Vec(y, y + p.m), rc_mode, r);
    put(r, r_out);
    *s = {k.pres, k.dres, k.pobj, k.dobj, k.agap, k.rgap};
  });
}

int ref_step_size_rules(double movement, double curvature, double eta_bar, double eta, int64_t k,
                        double* lim, double* nxt) {
  *lim = limit(movement, curvature);
  *nxt = next_eta(eta_bar, eta, k);
  return PDLP_OK;
}

double ref_initialize_primal_weight(const pdlp_problem_view* pv) { return weight0(from_view(pv)); }

double ref_initial_step_size(const pdlp_problem_view* pv) { return eta0(from_view(pv)); }

// Appendix-B fixed-restart feasibility harness, restated from the
// reference's test harness (proj/tests/feasibility_method.hpp:40-85):
// residual ||A x - b||_2 in row order (:26-34); one step = A^T y by columns,
// x' = max(0, x - eta A^T y), mid = 2x' - x, y -= eta (b - A mid) (:42-57);
// a round averages its restart_length primal iterates (:62-81).
int ref_feasibility_run(const pdlp_problem_view* pv, const double* b, const double* x0,
                        double eta, int64_t restart_length, int32_t rounds, double* points,
                        double* residuals, int32_t* recorded, int32_t* finite) {
  return guarded([&] {
    const Lp p = from_view(pv);
    const size_t m = static_cast<size_t>(p.m), n = static_cast<size_t>(p.n);
    const Vec rhs(b, b + m);
    Vec start(x0, x0 + n), x, y, sum, aty, mid, ax;
    auto residual = [&](const Vec& pt) {
      line_products(p.rows, pt, ax);
      double acc = 0.0;
      for (size_t j = 0; j < m; ++j) acc += (ax[j] - rhs[j]) * (ax[j] - rhs[j]);
      return std::sqrt(acc);
    };
    auto keep = [&](int32_t k) {
      if (points != nullptr) std::copy(start.begin(), start.end(), points + k * static_cast<int64_t>(n));
      residuals[k] = residual(start);
    };
    keep(0);
    int32_t count = 1, ok = 1;
    for (int32_t r = 0; r < rounds && ok; ++r) {
      x = start;
      y.assign(m, 0.0);
      sum.assign(n, 0.0);
      mid.assign(n, 0.0);
      for (int64_t t = 0; t < restart_length; ++t) {
        line_products(p.cols, y, aty);
        for (size_t i = 0; i < n; ++i) {
          const double cand = x[i] - eta * aty[i];
          const double nx = 0.0 < cand ? cand : 0.0;
          mid[i] = 2.0 * nx - x[i];
          x[i] = nx;
        }
        line_products(p.rows, mid, ax);
        for (size_t j = 0; j < m; ++j) y[j] = y[j] - eta * (rhs[j] - ax[j]);
        for (size_t i = 0; i < n; ++i) sum[i] += x[i];
      }
      for (size_t i = 0; i < n; ++i) start[i] = sum[i] / static_cast<double>(restart_length);
      for (double v : start) ok &= std::isfinite(v) ? 1 : 0;
      if (ok) keep(count++);
    }
    *recorded = count;
    *finite = ok;
  });
}

int ref_validate(const pdlp_problem_view* pv, char* msg, int32_t len) {
  try {
    validate(from_view(pv));
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(msg, static_cast<size_t>(len), "%s", e.what());
    return 1;
  }
}

}  // extern "C"
