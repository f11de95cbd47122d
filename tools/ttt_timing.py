"""C1 time-to-tolerance solve with the phase report (PDLP_TIMING)."""
import os
os.environ["PDLP_TIMING"] = "1"
import paper_2501_07018_b200 as P  # noqa: E402

p = P.generate("c1", 0)
tol = P.relative_tolerances(p)
for _ in range(2):
    r = P.solve(p, P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=100000))
    print(P.solve_status_name(r.status), r.iterations, r.polish_iterations, r.restarts, flush=True)
