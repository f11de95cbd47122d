// Drop-in replacement for the reference's proj/include/pdhglp/solver.hpp.
//
// Put include/pdhglp_b200 ahead of the reference's include directory and link
// libpdlp_b200.so: every caller of pdhglp::solve (tools/main.cpp:99, the
// reference's tests and acceptance criteria) then runs the B200 solver, with
// no source change.  The reference's other headers keep providing LpProblem,
// SparseMatrix, TerminationTolerances, ResidualSummary, InfeasibilityCertificate
// and RestartThresholds; this header re-declares only what solver.hpp owned,
// field for field (solver.hpp:35-108), and implements solve() by marshalling
// onto the C-ABI of include/pdlp_b200.h.
//
// Define PDHGLP_B200_STANDALONE to build without the reference headers
// (pdhglp_b200/types.hpp then provides the same structs).
//
// B200 additions are extra SolverOptions fields with defaults, so existing code
// compiles unchanged: b200_mode (PDLP_MODE_PERF / PDLP_MODE_PARITY; -1 reads
// the PDLP_MODE environment variable, default perf) and b200_device.
#pragma once

#include <cstdlib>
#include <cstring>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef PDHGLP_B200_STANDALONE
#include "pdhglp_b200/types.hpp"
#else
#include "pdhglp/problem.hpp"
#include "pdhglp/residuals.hpp"
#include "pdhglp/restarts.hpp"
#endif

#include "pdlp_b200.h"

namespace pdhglp {

enum class SolveStatus {
  Optimal,
  PrimalInfeasible,
  DualInfeasible,
  IterationLimit,
  TimeLimit,
  NumericalError,
};

inline const char* solve_status_name(SolveStatus s) {
  switch (s) {
    case SolveStatus::Optimal: return "optimal";
    case SolveStatus::PrimalInfeasible: return "primal_infeasible";
    case SolveStatus::DualInfeasible: return "dual_infeasible";
    case SolveStatus::IterationLimit: return "iteration_limit";
    case SolveStatus::TimeLimit: return "time_limit";
    case SolveStatus::NumericalError: return "numerical_error";
  }
  return "numerical_error";
}

struct IterationRecord {
  Index iteration = 0;
  const Vector* x = nullptr;
  const Vector* y = nullptr;
  Scalar eta = 0.0;
  Scalar omega = 1.0;
};

using IterationObserver = std::function<void(const IterationRecord&)>;

struct SolverOptions {
  TerminationTolerances tolerances{};
  Index iteration_limit = 200000;
  Scalar time_limit_seconds = kInf;
  int threads = 1;
  int shards_per_thread = 4;
  bool enable_scaling = true;
  int ruiz_passes = 10;
  bool pock_chambolle = true;
  bool enable_polish = true;
  bool enable_restarts = true;
  bool detect_infeasibility = true;
  Scalar eps_ray = 1e-12;
  Index check_interval = 64;
  RestartThresholds restart_thresholds{};
  std::optional<Scalar> fixed_step_size;
  std::optional<Scalar> fixed_primal_weight;
  bool logging = false;
  IterationObserver observer;
  // B200 extensions (additive)
  int b200_mode = -1;
  int b200_device = 0;
};

struct SolveResult {
  SolveStatus status = SolveStatus::NumericalError;
  Vector x;
  Vector y;
  Vector reduced_costs;
  ResidualSummary summary;
  std::optional<InfeasibilityCertificate> certificate;
  Index iterations = 0;
  Index polish_iterations = 0;
  Index restarts = 0;
  Index step_retries = 0;
  Scalar final_step_size = 0.0;
  Scalar final_primal_weight = 1.0;
  Scalar min_step_size_limit = kInf;
  Scalar solve_seconds = 0.0;
  std::string termination_detail;
};

namespace b200_detail {

inline pdlp_csr_view layout_view(const CompressedLayout& L) {
  pdlp_csr_view v;
  v.primary_dim = static_cast<int64_t>(L.start.size()) - 1;
  v.nnz = static_cast<int64_t>(L.value.size());
  v.start = L.start.data();
  v.index = L.index.data();
  v.value = L.value.data();
  return v;
}

struct ObserverBridge {
  const IterationObserver* fn;
  Vector x, y;
  static void call(void* user, const pdlp_iteration_record* rec) {
    auto* self = static_cast<ObserverBridge*>(user);
    self->x.assign(rec->x, rec->x + rec->x_len);
    self->y.assign(rec->y, rec->y + rec->y_len);
    IterationRecord r;
    r.iteration = rec->iteration;
    r.x = &self->x;
    r.y = &self->y;
    r.eta = rec->eta;
    r.omega = rec->omega;
    (*self->fn)(r);
  }
};

// Certificate sources are string literals in the reference (solver.hpp:254-257).
inline const char* static_source(const char* s) {
  if (std::strcmp(s, "difference") == 0) return "difference";
  if (std::strcmp(s, "current") == 0) return "current";
  if (std::strcmp(s, "average") == 0) return "average";
  return "";
}

inline int mode_from_env() {
  const char* m = std::getenv("PDLP_MODE");
  return (m != nullptr && std::strcmp(m, "parity") == 0) ? PDLP_MODE_PARITY : PDLP_MODE_PERF;
}

}  // namespace b200_detail

// pdhglp::solve (solver.hpp:535-608) on the GPU.  Same contract: throws
// std::invalid_argument for a malformed problem, every algorithmic outcome is
// a SolveStatus.  Device failures (no usable GPU) throw std::runtime_error —
// there is no CPU fallback.
inline SolveResult solve(const LpProblem& problem, const SolverOptions& options = {}) {
  const auto n = static_cast<size_t>(problem.cols());
  const auto m = static_cast<size_t>(problem.rows());
  auto bad_len = [](const char* what) {
    throw std::invalid_argument(std::string("invalid problem: ") + what + " (index -1)");
  };
  if (problem.objective.size() != n) bad_len("objective length != cols");
  if (problem.con_lower.size() != m) bad_len("con_lower length != rows");
  if (problem.con_upper.size() != m) bad_len("con_upper length != rows");
  if (problem.var_lower.size() != n) bad_len("var_lower length != cols");
  if (problem.var_upper.size() != n) bad_len("var_upper length != cols");

  pdlp_problem_view view;
  view.rows = problem.rows();
  view.cols = problem.cols();
  view.by_row = b200_detail::layout_view(problem.a.by_row);
  view.by_col = b200_detail::layout_view(problem.a.by_col);
  view.objective = problem.objective.data();
  view.con_lower = problem.con_lower.data();
  view.con_upper = problem.con_upper.data();
  view.var_lower = problem.var_lower.data();
  view.var_upper = problem.var_upper.data();

  pdlp_options o;
  pdlp_default_options(&o);
  o.eps_primal = options.tolerances.eps_primal;
  o.eps_dual = options.tolerances.eps_dual;
  o.eps_rel_gap = options.tolerances.eps_rel_gap;
  o.iteration_limit = options.iteration_limit;
  o.time_limit_seconds = options.time_limit_seconds;
  o.threads = options.threads;
  o.shards_per_thread = options.shards_per_thread;
  o.enable_scaling = options.enable_scaling;
  o.ruiz_passes = options.ruiz_passes;
  o.pock_chambolle = options.pock_chambolle;
  o.enable_polish = options.enable_polish;
  o.enable_restarts = options.enable_restarts;
  o.detect_infeasibility = options.detect_infeasibility;
  o.eps_ray = options.eps_ray;
  o.check_interval = options.check_interval;
  o.restart_sufficient = options.restart_thresholds.sufficient;
  o.restart_necessary = options.restart_thresholds.necessary;
  o.restart_artificial = options.restart_thresholds.artificial;
  o.has_fixed_step_size = options.fixed_step_size.has_value();
  o.fixed_step_size = options.fixed_step_size.value_or(0.0);
  o.has_fixed_primal_weight = options.fixed_primal_weight.has_value();
  o.fixed_primal_weight = options.fixed_primal_weight.value_or(0.0);
  o.logging = options.logging;
  o.mode = options.b200_mode >= 0 ? options.b200_mode : b200_detail::mode_from_env();
  o.device = options.b200_device;
  b200_detail::ObserverBridge bridge{&options.observer, {}, {}};
  if (options.observer) {
    o.observer = &b200_detail::ObserverBridge::call;
    o.observer_user = &bridge;
  }

  SolveResult out;
  out.x.assign(n, 0.0);
  out.y.assign(m, 0.0);
  out.reduced_costs.assign(n, 0.0);
  Vector rx(n), ry(m), rr(n);
  pdlp_result r;
  std::memset(&r, 0, sizeof(r));
  r.x = out.x.data();
  r.y = out.y.data();
  r.reduced_costs = out.reduced_costs.data();
  r.cert_ray_x = rx.data();
  r.cert_ray_y = ry.data();
  r.cert_ray_r = rr.data();
  const int rc = pdlp_solve(&view, &o, &r);
  if (rc == PDLP_ERR_INVALID_PROBLEM) throw std::invalid_argument(pdlp_last_error());
  if (rc != PDLP_OK) throw std::runtime_error(std::string("pdlp_solve: ") + pdlp_last_error());

  out.status = static_cast<SolveStatus>(r.status);
  out.summary.primal_residual_inf = r.summary.primal_residual_inf;
  out.summary.dual_residual_inf = r.summary.dual_residual_inf;
  out.summary.primal_objective = r.summary.primal_objective;
  out.summary.dual_objective = r.summary.dual_objective;
  out.summary.abs_gap = r.summary.abs_gap;
  out.summary.rel_gap = r.summary.rel_gap;
  if (r.has_certificate) {
    InfeasibilityCertificate cert;
    cert.kind = r.cert_kind == PDLP_CERT_PRIMAL_INFEASIBLE ? CertificateKind::PrimalInfeasible
                                                           : CertificateKind::DualInfeasible;
    if (cert.kind == CertificateKind::PrimalInfeasible) {
      cert.ray_y = std::move(ry);
      cert.ray_r = std::move(rr);
    } else {
      cert.ray_x = std::move(rx);
    }
    cert.residual_inf = r.cert_residual_inf;
    cert.objective = r.cert_objective;
    cert.source = b200_detail::static_source(r.cert_source);
    out.certificate = std::move(cert);
  }
  out.iterations = r.iterations;
  out.polish_iterations = r.polish_iterations;
  out.restarts = r.restarts;
  out.step_retries = r.step_retries;
  out.final_step_size = r.final_step_size;
  out.final_primal_weight = r.final_primal_weight;
  out.min_step_size_limit = r.min_step_size_limit;
  out.solve_seconds = r.solve_seconds;
  out.termination_detail = r.termination_detail;
  return out;
}

}  // namespace pdhglp
