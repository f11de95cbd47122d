"""C1 (transport 2000x2000) to BASELINE's 1e-4 relative KKT over seeds 0-4:
the GPU (perf mode) next to the compiled reference (16 host
threads x 4 shards) on the same instances.  One JSON line per seed."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2501_07018_b200 as P  # noqa: E402

ref = oracle.get()
T = os.cpu_count() or 1
for seed in range(5):
    p = P.generate("c1", seed)
    tol = P.relative_tolerances(p)
    row = {"seed": seed}
    for name, fn, mode in (("gpu_perf", P.solve, "perf"), ("reference", ref.solve, None)):
        o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=200000,
                            time_limit_seconds=600.0, threads=T, shards_per_thread=4)
        if mode:
            o.mode = mode
        t0 = time.perf_counter()
        r = fn(p, o)
        row[name] = {"status": P.solve_status_name(r.status), "iterations": r.iterations,
                     "polish_iterations": r.polish_iterations, "restarts": r.restarts,
                     "seconds": time.perf_counter() - t0,
                     "objective": r.summary.primal_objective}
    print(json.dumps(row), flush=True)
