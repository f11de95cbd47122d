import numpy as np
import paper_2501_07018_b200 as P
from paper_2501_07018_b200 import sharded as S


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


p = P.generate("c2", 2, rows=800, cols=1600, kmax=600)
print("m n nnz", p.rows(), p.cols(), p.a.nonzeros(), "max row", np.diff(p.a.by_row.start).max(),
      "max col", np.diff(p.a.by_col.start).max())
for kw in ({}, {"enable_restarts": False, "detect_infeasibility": False}, {"enable_scaling": False}):
    for it in (1, 2, 3, 10, 63, 64, 65, 100):
        o = P.SolverOptions(mode="perf", iteration_limit=it,
                            tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), **kw)
        a = P.solve(p, o)
        row = [kw, it]
        for w in (2, 3, 4):
            b = S.solve_sharded_emulated(p, o, w)
            row.append((w, f"{rel(b.x, a.x):.1e}", f"{rel(b.y, a.y):.1e}", b.restarts - a.restarts))
        print(*row, flush=True)
