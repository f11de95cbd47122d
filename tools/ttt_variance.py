"""Repeat the C1 time-to-tolerance solve and split its time (variance hunt)."""
import time
import paper_2501_07018_b200 as P

p = P.generate("c1", 0)
tol = P.relative_tolerances(p)
for i in range(5):
    o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=100000)
    t0 = time.perf_counter()
    r = P.solve(p, o)
    w = time.perf_counter() - t0
    print(f"{i}: wall {w:.3f} solve {r.solve_seconds:.3f} loop {r.loop_seconds:.3f} "
          f"steps {r.step_seconds:.3f} upload {r.upload_seconds:.3f} it {r.iterations}+{r.polish_iterations} "
          f"attempts {r.attempts}", flush=True)
