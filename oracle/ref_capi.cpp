// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (never linked into the
// product).  A thin C-ABI over the UNMODIFIED reference library compiled from
// /root/reference/proj/include (header-only C++20), so that Python tests and
// bench.py's cpu_baseline / --impl reference arm can call the reference
// implementation of the PDHG path through the same plain-pointer structs the
// product exposes (include/pdlp_b200.h).  Built by oracle/Makefile into
// oracle/_ref/libpdhglp_ref.so with  g++ -std=c++20 -O2 -ffp-contract=off
// (no -march: FMA contraction breaks the reference, SURVEY.md §0 finding 6).
//
// Only marshalling lives here; every number comes from the reference code.

#include <pdhglp/generator.hpp>
#include <pdhglp/mps.hpp>
#include <pdhglp/rescaling.hpp>
#include <pdhglp/residuals.hpp>
#include <pdhglp/restarts.hpp>
#include <pdhglp/solver.hpp>
#include <pdhglp/step.hpp>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "feasibility_method.hpp"  // proj/tests: the Appendix-B harness
#include "pdlp_b200.h"

using namespace pdhglp;

namespace {

thread_local std::string g_err;

CompressedLayout to_layout(const pdlp_csr_view& v) {
  CompressedLayout out;
  out.start.assign(v.start, v.start + v.primary_dim + 1);
  out.index.assign(v.index, v.index + v.nnz);
  out.value.assign(v.value, v.value + v.nnz);
  return out;
}

LpProblem to_problem(const pdlp_problem_view* pv) {
  LpProblem p;
  p.a.rows = pv->rows;
  p.a.cols = pv->cols;
  p.a.by_row = to_layout(pv->by_row);
  p.a.by_col = to_layout(pv->by_col);
  p.objective.assign(pv->objective, pv->objective + pv->cols);
  p.con_lower.assign(pv->con_lower, pv->con_lower + pv->rows);
  p.con_upper.assign(pv->con_upper, pv->con_upper + pv->rows);
  p.var_lower.assign(pv->var_lower, pv->var_lower + pv->cols);
  p.var_upper.assign(pv->var_upper, pv->var_upper + pv->cols);
  return p;
}

void copy_out(const Vector& v, double* dst) {
  if (dst != nullptr && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
}

SolverOptions to_options(const pdlp_options* o) {
  SolverOptions s;
  s.tolerances.eps_primal = o->eps_primal;
  s.tolerances.eps_dual = o->eps_dual;
  s.tolerances.eps_rel_gap = o->eps_rel_gap;
  s.iteration_limit = o->iteration_limit;
  s.time_limit_seconds = o->time_limit_seconds;
  s.threads = o->threads;
  s.shards_per_thread = o->shards_per_thread;
  s.enable_scaling = o->enable_scaling != 0;
  s.ruiz_passes = o->ruiz_passes;
  s.pock_chambolle = o->pock_chambolle != 0;
  s.enable_polish = o->enable_polish != 0;
  s.enable_restarts = o->enable_restarts != 0;
  s.detect_infeasibility = o->detect_infeasibility != 0;
  s.eps_ray = o->eps_ray;
  s.check_interval = o->check_interval;
  s.restart_thresholds.sufficient = o->restart_sufficient;
  s.restart_thresholds.necessary = o->restart_necessary;
  s.restart_thresholds.artificial = o->restart_artificial;
  if (o->has_fixed_step_size) s.fixed_step_size = o->fixed_step_size;
  if (o->has_fixed_primal_weight) s.fixed_primal_weight = o->fixed_primal_weight;
  s.logging = o->logging != 0;
  if (o->observer != nullptr) {
    pdlp_observer_fn fn = o->observer;
    void* user = o->observer_user;
    s.observer = [fn, user](const IterationRecord& rec) {
      pdlp_iteration_record r;
      r.iteration = rec.iteration;
      r.x = rec.x->data();
      r.x_len = static_cast<int64_t>(rec.x->size());
      r.y = rec.y->data();
      r.y_len = static_cast<int64_t>(rec.y->size());
      r.eta = rec.eta;
      r.omega = rec.omega;
      fn(user, &r);
    };
  }
  return s;
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PDLP_ERR_INVALID_PROBLEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PDLP_ERR_INTERNAL;
  }
}

struct RefInstance {
  GeneratedInstance inst;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_default_options(pdlp_options* o) {
  const SolverOptions s{};
  std::memset(o, 0, sizeof(*o));
  o->eps_primal = s.tolerances.eps_primal;
  o->eps_dual = s.tolerances.eps_dual;
  o->eps_rel_gap = s.tolerances.eps_rel_gap;
  o->iteration_limit = s.iteration_limit;
  o->time_limit_seconds = s.time_limit_seconds;
  o->threads = s.threads;
  o->shards_per_thread = s.shards_per_thread;
  o->enable_scaling = s.enable_scaling;
  o->ruiz_passes = s.ruiz_passes;
  o->pock_chambolle = s.pock_chambolle;
  o->enable_polish = s.enable_polish;
  o->enable_restarts = s.enable_restarts;
  o->detect_infeasibility = s.detect_infeasibility;
  o->eps_ray = s.eps_ray;
  o->check_interval = s.check_interval;
  o->restart_sufficient = s.restart_thresholds.sufficient;
  o->restart_necessary = s.restart_thresholds.necessary;
  o->restart_artificial = s.restart_thresholds.artificial;
  o->logging = s.logging;
}

int ref_solve(const pdlp_problem_view* pv, const pdlp_options* o, pdlp_result* res) {
  return guarded([&] {
    const LpProblem p = to_problem(pv);
    const SolverOptions s = to_options(o);
    SolveResult r = solve(p, s);
    res->status = static_cast<int32_t>(r.status);
    copy_out(r.x, res->x);
    copy_out(r.y, res->y);
    copy_out(r.reduced_costs, res->reduced_costs);
    res->summary.primal_residual_inf = r.summary.primal_residual_inf;
    res->summary.dual_residual_inf = r.summary.dual_residual_inf;
    res->summary.primal_objective = r.summary.primal_objective;
    res->summary.dual_objective = r.summary.dual_objective;
    res->summary.abs_gap = r.summary.abs_gap;
    res->summary.rel_gap = r.summary.rel_gap;
    res->has_certificate = r.certificate.has_value() ? 1 : 0;
    if (r.certificate) {
      res->cert_kind = static_cast<int32_t>(r.certificate->kind);
      copy_out(r.certificate->ray_x, res->cert_ray_x);
      copy_out(r.certificate->ray_y, res->cert_ray_y);
      copy_out(r.certificate->ray_r, res->cert_ray_r);
      res->cert_residual_inf = r.certificate->residual_inf;
      res->cert_objective = r.certificate->objective;
      std::strncpy(res->cert_source, r.certificate->source, sizeof(res->cert_source) - 1);
    }
    res->iterations = r.iterations;
    res->polish_iterations = r.polish_iterations;
    res->restarts = r.restarts;
    res->step_retries = r.step_retries;
    res->final_step_size = r.final_step_size;
    res->final_primal_weight = r.final_primal_weight;
    res->min_step_size_limit = r.min_step_size_limit;
    res->solve_seconds = r.solve_seconds;
    std::strncpy(res->termination_detail, r.termination_detail.c_str(),
                 sizeof(res->termination_detail) - 1);
    return PDLP_OK;
  });
}

int ref_pdhg_step(const pdlp_problem_view* pv, const double* x, const double* y, double omega,
                  double eta, double* x_out, double* y_out, int32_t* finite) {
  return guarded([&] {
    const LpProblem p = to_problem(pv);
    PrimalDualIterate z{Vector(x, x + pv->cols), Vector(y, y + pv->rows)};
    auto next = pdhg_step(p, z, omega, eta);
    *finite = next.has_value() ? 1 : 0;
    if (next) {
      copy_out(next->x, x_out);
      copy_out(next->y, y_out);
    }
    return PDLP_OK;
  });
}

// io_state = {eta_hat, k, max_retries, omega}; stats = {accepted, retries,
// min_eta_bar, eta_used}.
int ref_adaptive_step(const pdlp_problem_view* pv, double* x, double* y, double* aty,
                      double* io_state, int32_t threads, int32_t spt, double* prev_x,
                      double* prev_y, double* stats, int32_t* outcome) {
  return guarded([&] {
    const LpProblem p = to_problem(pv);
    Executor ex(p.cols(), p.rows(), threads, spt);
    PdhgIterate z{Vector(x, x + pv->cols), Vector(y, y + pv->rows),
                  Vector(aty, aty + pv->cols)};
    PdhgWorkspace ws;
    ws.resize(p.cols(), p.rows());
    StepSizeControl ctrl;
    ctrl.eta_hat = io_state[0];
    ctrl.k = static_cast<Index>(io_state[1]);
    ctrl.max_retries = static_cast<int>(io_state[2]);
    const double omega = io_state[3];
    StepStats st;
    Scalar eta_used = 0.0;
    const StepOutcome out = adaptive_step(p, ex, z, omega, ctrl, ws, st, eta_used);
    *outcome = out == StepOutcome::Accepted ? 0 : 1;
    copy_out(z.x, x);
    copy_out(z.y, y);
    copy_out(z.aty, aty);
    copy_out(ws.x_trial, prev_x);
    copy_out(ws.y_trial, prev_y);
    io_state[0] = ctrl.eta_hat;
    io_state[1] = static_cast<double>(ctrl.k);
    stats[0] = static_cast<double>(st.accepted_steps);
    stats[1] = static_cast<double>(st.retries);
    stats[2] = st.min_eta_bar;
    stats[3] = eta_used;
    return PDLP_OK;
  });
}

int ref_spmv(const pdlp_problem_view* pv, const double* x, double* out, int32_t threads,
             int32_t spt) {
  return guarded([&] {
    const LpProblem p = to_problem(pv);
    Executor ex(p.cols(), p.rows(), threads, spt);
    Vector xv(x, x + pv->cols), o(static_cast<size_t>(pv->rows));
    kernels::spmv(ex.pool, ex.y_plan, p.a, xv, o);
    copy_out(o, out);
    return PDLP_OK;
  });
}

int ref_spmv_transpose(const pdlp_problem_view* pv, const double* y, double* out,
                       int32_t threads, int32_t spt) {
  return guarded([&] {
    const LpProblem p = to_problem(pv);
    Executor ex(p.cols(), p.rows(), threads, spt);
    Vector yv(y, y + pv->rows), o(static_cast<size_t>(pv->cols));
    kernels::spmv_transpose(ex.pool, ex.x_plan, p.a, yv, o);
    copy_out(o, out);
    return PDLP_OK;
  });
}

int ref_apply_rescaling(const pdlp_problem_view* pv, int32_t ruiz, int32_t pc,
                        double* row_values, double* col_values, double* objective,
                        double* con_lower, double* con_upper, double* var_lower,
                        double* var_upper, double* row_scale, double* col_scale) {
  return guarded([&] {
    const LpProblem p = to_problem(pv);
    ScaledProblem sp = apply_rescaling(p, ruiz, pc != 0);
    copy_out(sp.problem.a.by_row.value, row_values);
    copy_out(sp.problem.a.by_col.value, col_values);
    copy_out(sp.problem.objective, objective);
    copy_out(sp.problem.con_lower, con_lower);
    copy_out(sp.problem.con_upper, con_upper);
    copy_out(sp.problem.var_lower, var_lower);
    copy_out(sp.problem.var_upper, var_upper);
    copy_out(sp.info.row_scale, row_scale);
    copy_out(sp.info.col_scale, col_scale);
    return PDLP_OK;
  });
}

int ref_normalized_duality_gap(const pdlp_problem_view* pv, const double* x, const double* y,
                               const double* ax, const double* aty, double omega, double r,
                               double* gap) {
  return guarded([&] {
    const LpProblem p = to_problem(pv);
    GapWorkspace ws;
    *gap = normalized_duality_gap(p, Vector(x, x + pv->cols), Vector(y, y + pv->rows),
                                  Vector(ax, ax + pv->rows), Vector(aty, aty + pv->cols), omega,
                                  r, ws);
    return PDLP_OK;
  });
}

int ref_kkt_residuals(const pdlp_problem_view* pv, const double* x, const double* y,
                      int32_t rc_mode, double* r_out, pdlp_residual_summary* s) {
  return guarded([&] {
    const LpProblem p = to_problem(pv);
    const Vector xv(x, x + pv->cols), yv(y, y + pv->rows);
    const Vector r = recover_reduced_costs(
        p, xv, yv, rc_mode == 0 ? ReducedCostMode::Natural : ReducedCostMode::BoundRobust);
    const ResidualSummary rs = kkt_residuals(p, xv, yv, r);
    copy_out(r, r_out);
    s->primal_residual_inf = rs.primal_residual_inf;
    s->dual_residual_inf = rs.dual_residual_inf;
    s->primal_objective = rs.primal_objective;
    s->dual_objective = rs.dual_objective;
    s->abs_gap = rs.abs_gap;
    s->rel_gap = rs.rel_gap;
    return PDLP_OK;
  });
}

int ref_step_size_rules(double movement, double curvature, double eta_bar, double eta,
                        int64_t k, double* limit_out, double* next_out) {
  *limit_out = step_size_limit(movement, curvature);
  *next_out = next_step_size(eta_bar, eta, k);
  return PDLP_OK;
}

// ---- MPS: the reference's parse_mps / write_mps (mps.hpp:87-535) -------
struct RefMps {
  MpsModel model;
};

int ref_mps_parse(const char* text, size_t len, void** out) {
  try {
    *out = new RefMps{parse_mps(std::string_view(text ? text : "", len))};
    return PDLP_OK;
  } catch (const MpsParseError& e) {
    g_err = e.what();
    return PDLP_ERR_INVALID_PROBLEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PDLP_ERR_INTERNAL;
  }
}

void ref_mps_view(const void* h, pdlp_problem_view* v) {
  const LpProblem& p = static_cast<const RefMps*>(h)->model.problem;
  v->rows = p.a.rows;
  v->cols = p.a.cols;
  v->by_row = {p.a.rows, static_cast<int64_t>(p.a.by_row.value.size()), p.a.by_row.start.data(),
               p.a.by_row.index.data(), p.a.by_row.value.data()};
  v->by_col = {p.a.cols, static_cast<int64_t>(p.a.by_col.value.size()), p.a.by_col.start.data(),
               p.a.by_col.index.data(), p.a.by_col.value.data()};
  v->objective = p.objective.data();
  v->con_lower = p.con_lower.data();
  v->con_upper = p.con_upper.data();
  v->var_lower = p.var_lower.data();
  v->var_upper = p.var_upper.data();
}

int32_t ref_mps_maximize(const void* h) { return static_cast<const RefMps*>(h)->model.maximize ? 1 : 0; }
const char* ref_mps_name(const void* h) { return static_cast<const RefMps*>(h)->model.name.c_str(); }
const char* ref_mps_objective_name(const void* h) {
  return static_cast<const RefMps*>(h)->model.objective_name.c_str();
}
const char* ref_mps_row_name(const void* h, int64_t j) {
  return static_cast<const RefMps*>(h)->model.row_names[static_cast<size_t>(j)].c_str();
}
const char* ref_mps_col_name(const void* h, int64_t i) {
  return static_cast<const RefMps*>(h)->model.col_names[static_cast<size_t>(i)].c_str();
}
void ref_mps_free(void* h) { delete static_cast<RefMps*>(h); }

int ref_mps_write(const pdlp_problem_view* pv, const char* name, int32_t maximize, char** text,
                  size_t* len) {
  return guarded([&] {
    const std::string s = write_mps(to_problem(pv), name ? name : "", maximize != 0);
    char* buf = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(buf, s.c_str(), s.size() + 1);
    *text = buf;
    *len = s.size();
    return PDLP_OK;
  });
}

void ref_mps_free_text(char* t) { std::free(t); }

double ref_initialize_primal_weight(const pdlp_problem_view* pv) {
  return initialize_primal_weight(to_problem(pv));
}

double ref_initial_step_size(const pdlp_problem_view* pv) {
  return initial_step_size(to_problem(pv));
}

// ---- Appendix-B harness (tests/feasibility_method.hpp:60-85), as is -------

int ref_feasibility_run(const pdlp_problem_view* pv, const double* b, const double* x0,
                        double eta, int64_t restart_length, int32_t rounds, double* points,
                        double* residuals, int32_t* recorded, int32_t* finite) {
  return guarded([&]() -> int {
    const LpProblem p = to_problem(pv);
    const Vector rhs(b, b + pv->rows), start(x0, x0 + pv->cols);
    const testharness::FeasibilityRun run =
        testharness::fixed_restart_feasibility(p.a, rhs, start, eta, restart_length, rounds);
    for (size_t k = 0; k < run.restart_points.size(); ++k) {
      if (points != nullptr) copy_out(run.restart_points[k], points + k * pv->cols);
      residuals[k] = run.residuals[k];
    }
    *recorded = static_cast<int32_t>(run.restart_points.size());
    *finite = run.finite ? 1 : 0;
    return PDLP_OK;
  });
}

// Strictly positive point of a feasibility-system instance (A x = b), for
// the criterion-10 starts; NaN-filled when the instance kind has none.
void ref_instance_feasible_point(void* h, double* out) {
  const auto& inst = static_cast<RefInstance*>(h)->inst;
  const size_t n = static_cast<size_t>(inst.problem.cols());
  for (size_t i = 0; i < n; ++i) {
    out[i] = i < inst.feasible_point.size() ? inst.feasible_point[i] : std::nan("");
  }
}

// ---- instances from the reference generator (generator.hpp:347-374) ------

void* ref_generate(int32_t kind, int64_t rows, int64_t cols, double density, uint64_t seed) {
  try {
    GeneratorSpec spec;
    spec.kind = static_cast<InstanceKind>(kind);
    spec.rows = rows;
    spec.cols = cols;
    spec.density = density;
    spec.seed = seed;
    auto* h = new RefInstance{generate_instance(spec)};
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Builds an instance from triplets with the reference's from_triplets
// (sparse.hpp:107-115); bounds/objective copied from the given arrays.
void* ref_from_triplets(int64_t rows, int64_t cols, int64_t count, const int64_t* r,
                        const int64_t* c, const double* v, const double* objective,
                        const double* con_lower, const double* con_upper,
                        const double* var_lower, const double* var_upper) {
  try {
    std::vector<Triplet> t(static_cast<size_t>(count));
    for (int64_t k = 0; k < count; ++k) t[static_cast<size_t>(k)] = {r[k], c[k], v[k]};
    auto* h = new RefInstance{};
    LpProblem& p = h->inst.problem;
    p.a = SparseMatrix::from_triplets(rows, cols, t);
    p.objective.assign(objective, objective + cols);
    p.con_lower.assign(con_lower, con_lower + rows);
    p.con_upper.assign(con_upper, con_upper + rows);
    p.var_lower.assign(var_lower, var_lower + cols);
    p.var_upper.assign(var_upper, var_upper + cols);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_instance_view(void* h, pdlp_problem_view* pv) {
  const LpProblem& p = static_cast<RefInstance*>(h)->inst.problem;
  pv->rows = p.rows();
  pv->cols = p.cols();
  pv->by_row = {p.a.by_row.primary_dim(), p.a.by_row.nonzeros(), p.a.by_row.start.data(),
                p.a.by_row.index.data(), p.a.by_row.value.data()};
  pv->by_col = {p.a.by_col.primary_dim(), p.a.by_col.nonzeros(), p.a.by_col.start.data(),
                p.a.by_col.index.data(), p.a.by_col.value.data()};
  pv->objective = p.objective.data();
  pv->con_lower = p.con_lower.data();
  pv->con_upper = p.con_upper.data();
  pv->var_lower = p.var_lower.data();
  pv->var_upper = p.var_upper.data();
}

// Optimal objective of a random-feasible instance (NaN when unknown).
double ref_instance_optimal_objective(void* h) {
  const auto& inst = static_cast<RefInstance*>(h)->inst;
  return inst.optimal_objective.has_value() ? *inst.optimal_objective : std::nan("");
}

void ref_instance_free(void* h) { delete static_cast<RefInstance*>(h); }

int ref_validate(const pdlp_problem_view* pv, char* msg, int32_t msg_len) {
  const LpProblem p = to_problem(pv);
  auto issue = validate(p);
  if (!issue) return 0;
  std::snprintf(msg, static_cast<size_t>(msg_len), "%s (index %lld)", issue->message.c_str(),
                static_cast<long long>(issue->index));
  return 1;
}

// Timing harness of the bench's reference arm (bench.py --impl reference):
// the unmodified solve() with tolerances unreachable, an iteration limit of
// warmup + steps, and an observer that only takes a steady_clock stamp
// (solver.hpp:521-529 calls it after every accepted main-loop step; no copy
// of x or y).  The window runs from the stamp of iteration `warmup` to the
// return of solve(): `steps` iterations plus the budget-hit cadence at the
// end (solver.hpp:358-360), the same span the GPU arm's timed region covers.
// out[0] = window seconds, out[1] = iterations in the window, out[2] =
// seconds from the call to the window start (problem build, validation,
// rescaling, warm-up iterations), out[3] = total seconds, out[4] = restarts,
// out[5] = step retries.  stamps (optional, n_stamps doubles): seconds since
// the call of each accepted iteration k at stamps[k].
int ref_time_window(const pdlp_problem_view* pv, int32_t threads, int32_t shards_per_thread,
                    int64_t warmup, int64_t steps, double* out, double* stamps,
                    int64_t n_stamps) {
  return guarded([&] {
    using Clock = std::chrono::steady_clock;
    const auto t0 = Clock::now();
    const int64_t w = warmup < 1 ? 1 : warmup;
    const LpProblem p = to_problem(pv);
    SolverOptions s{};
    s.tolerances.eps_primal = 0.0;
    s.tolerances.eps_dual = 0.0;
    s.tolerances.eps_rel_gap = 0.0;
    s.iteration_limit = w + steps;
    s.threads = threads;
    s.shards_per_thread = shards_per_thread;
    Clock::time_point tw = t0;
    Index kw = -1;
    s.observer = [&](const IterationRecord& rec) {
      const auto now = Clock::now();
      if (stamps != nullptr && rec.iteration >= 0 && rec.iteration < n_stamps) {
        stamps[rec.iteration] = std::chrono::duration<double>(now - t0).count();
      }
      if (kw < 0 && rec.iteration >= w) {
        kw = rec.iteration;
        tw = now;
      }
    };
    const SolveResult r = solve(p, s);
    const auto t1 = Clock::now();
    if (kw < 0) {
      g_err = "ref_time_window: the solve stopped before the window opened (" +
              std::string(solve_status_name(r.status)) + ")";
      return PDLP_ERR_INTERNAL;
    }
    out[0] = std::chrono::duration<double>(t1 - tw).count();
    out[1] = static_cast<double>(r.iterations - kw);
    out[2] = std::chrono::duration<double>(tw - t0).count();
    out[3] = std::chrono::duration<double>(t1 - t0).count();
    out[4] = static_cast<double>(r.restarts);
    out[5] = static_cast<double>(r.step_retries);
    return PDLP_OK;
  });
}

}  // extern "C"
