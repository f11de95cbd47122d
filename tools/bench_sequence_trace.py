"""The bench's solve sequence on C1 with phase timings (logging), to find
where occasional host-side time goes."""
import sys
import paper_2501_07018_b200 as P

p = P.generate("c1", 0)
tol = P.relative_tolerances(p)


def opts(k, w, **kw):
    o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), iteration_limit=w + k,
                        timing_warmup_iterations=w, mode="perf", logging=True)
    for a, b in kw.items():
        setattr(o, a, b)
    return o


for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    print("rep", rep, file=sys.stderr, flush=True)
    P.solve(p, opts(64, 0))
    P.solve(p, opts(2048, 64))
    P.solve(p, opts(2048, 0))
    P.solve(p, opts(2048, 64, profile_kernels=True))
    P.solve(p, P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=100000,
                               logging=True))
