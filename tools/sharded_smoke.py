"""Sharded solve (threads-emulated ranks and 1-rank NCCL) vs the single-GPU solve."""
import sys
import time

import numpy as np

import paper_2501_07018_b200 as P
from paper_2501_07018_b200 import sharded as S


def opts(**kw):
    o = P.SolverOptions(mode="perf")
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


cases = [("c0", P.generate("c0", 0)), ("transport", P.generate("c1", 0, sources=60, sinks=60))]
for name, p in cases:
    tol = P.relative_tolerances(p, 1e-4) if hasattr(P, "relative_tolerances") else None
    for it in (100,):
        o = opts(iteration_limit=it, tolerances=P.TerminationTolerances(0.0, 0.0, 0.0))
        a = P.solve(p, o)
        for w in (1, 2, 3):
            t = time.time()
            b = S.solve_sharded_emulated(p, o, w)
            print(name, "iters", it, "world", w, "x rel", rel(b.x, a.x), "y rel", rel(b.y, a.y),
                  b.iterations, a.iterations, f"{time.time()-t:.2f}s", flush=True)
    o = opts(tolerances=P.TerminationTolerances(*tol))
    a = P.solve(p, o)
    for w in (1, 2, 4):
        b = S.solve_sharded_emulated(p, o, w)
        print(name, "full", "world", w, a.status.name, b.status.name, a.iterations, b.iterations,
              a.summary.primal_objective, b.summary.primal_objective, b.termination_detail, flush=True)
    nid = S.nccl_unique_id()
    b = S.solve_sharded(p, o, 0, 1, nid)
    print(name, "nccl world 1", b.status.name, b.iterations, b.summary.primal_objective, flush=True)
