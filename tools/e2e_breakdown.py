"""Break the e2e pdlp_solve() wall time of the bench workload into phases."""
import time
import paper_2501_07018_b200 as P

p = P.generate("c1", 0)
K = 2048
o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), iteration_limit=K,
                    mode="perf")
for i in range(4):
    t0 = time.perf_counter()
    r = P.solve(p, o)
    w = time.perf_counter() - t0
    print(f"call {i}: wall {w:.3f}s upload {r.upload_seconds:.3f} precond {r.precondition_seconds:.3f} "
          f"loop {r.loop_seconds:.3f} rest {w - r.upload_seconds - r.precondition_seconds - r.loop_seconds:.3f} "
          f"solve_seconds {r.solve_seconds:.3f} iters {r.iterations}")
