// Uses the drop-in header exactly like reference code would
// (test_solver.cpp:54-84): #include <pdhglp/solver.hpp>, call pdhglp::solve.
// Build standalone: g++ -std=c++20 -DPDHGLP_B200_STANDALONE -Iinclude/pdhglp_b200 -Iinclude
//                   examples/dropin_tiny.cpp -Lpaper_2501_07018_b200 -lpdlp_b200
#include <pdhglp/solver.hpp>

#include <cmath>
#include <cstdio>

int main() {
  using namespace pdhglp;
  LpProblem p;  // min -x1 - 2 x2, x1 + x2 <= 1, x >= 0
  p.a = SparseMatrix::from_triplets(1, 2, {{0, 0, 1.0}, {0, 1, 1.0}});
  p.objective = {-1.0, -2.0};
  p.con_lower = {-kInf};
  p.con_upper = {1.0};
  p.var_lower = {0.0, 0.0};
  p.var_upper = {kInf, kInf};
  SolverOptions opt;
  opt.tolerances.eps_rel_gap = 1e-9;
  const SolveResult r = solve(p, opt);
  std::printf("status=%s x=(%.9f, %.9f) y=%.9f obj=%.9f iters=%lld detail=\"%s\"\n",
              solve_status_name(r.status), r.x[0], r.x[1], r.y[0], r.summary.primal_objective,
              static_cast<long long>(r.iterations), r.termination_detail.c_str());
  const bool ok = r.status == SolveStatus::Optimal && std::abs(r.x[1] - 1.0) < 1e-6 &&
                  std::abs(r.summary.primal_objective + 2.0) < 1e-7;
  return ok ? 0 : 1;
}
