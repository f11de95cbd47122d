import paper_2501_07018_b200 as P
from paper_2501_07018_b200 import sharded as S
for p in (P.generate("c0", 3), P.generate("c1", 3, sources=45, sinks=55)):
    tol = P.relative_tolerances(p, 1e-4)
    o = P.SolverOptions(mode="perf", tolerances=P.TerminationTolerances(*tol))
    r = S.solve_sharded_emulated(p, o, 2)
    print(p.rows(), p.cols(), r.status, r.iterations, "polish", r.polish_iterations)
