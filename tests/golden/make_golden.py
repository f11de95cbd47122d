"""Generate tests/golden/golden.{npz,json} from the COMPILED REFERENCE
(oracle/_ref/libpdhglp_ref.so, built from /root/reference by oracle/Makefile).

Run in the build container (the reference sources are not on the GPU box):
    python tests/golden/make_golden.py
The fixtures pin the oracle restatement and the GPU parity mode without the
reference library: full-solve outcomes and solution vectors on seeded
BASELINE-family instances, plus an observer trace of the first 100 C0
iterates (checksummed; iterations 1, 10, 50, 100 stored in full).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2501_07018_b200 as P  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

SOLVES = {
    "c0_seed0": dict(config="c0", seed=0, size={}, rel=True, iteration_limit=200000),
    "c1_small": dict(config="c1", seed=3, size=dict(sources=30, sinks=40), rel=True,
                     iteration_limit=200000),
    "c2_small": dict(config="c2", seed=1, size=dict(rows=500, cols=1000), rel=True,
                     iteration_limit=640),
    "c3_small": dict(config="c3", seed=2, size=dict(periods=24, generators=8), rel=True,
                     iteration_limit=1280),
}


def main():
    R = oracle.reference()
    arrays, meta = {}, {"generator": "oracle/_ref (reference compiled in place)", "solves": {}}
    for name, spec in SOLVES.items():
        p = P.generate(spec["config"], spec["seed"], **spec["size"])
        tol = P.relative_tolerances(p) if spec["rel"] else (1e-8, 1e-8, 1e-2)
        o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol),
                            iteration_limit=spec["iteration_limit"])
        r = R.solve(p, o)
        arrays[name + "_x"] = r.x
        arrays[name + "_y"] = r.y
        meta["solves"][name] = dict(config=spec["config"], seed=spec["seed"], size=spec["size"],
                                    tol=list(tol), iteration_limit=spec["iteration_limit"],
                                    status=int(r.status), iterations=int(r.iterations),
                                    polish_iterations=int(r.polish_iterations),
                                    restarts=int(r.restarts),
                                    objective=r.summary.primal_objective)
        print(name, P.solve_status_name(r.status), r.iterations, r.polish_iterations, r.restarts)
    # first-100 trace on C0 seed 0
    p = P.generate("c0", 0)
    o = P.SolverOptions(tolerances=P.TerminationTolerances(*P.relative_tolerances(p)),
                        iteration_limit=100)
    xs, ys = [], []
    o.observer = lambda rec: (xs.append(rec.x), ys.append(rec.y))
    R.solve(p, o)
    xs, ys = np.array(xs), np.array(ys)
    for k in (1, 10, 50, 100):
        arrays[f"trace_x_{k}"] = xs[k - 1]
        arrays[f"trace_y_{k}"] = ys[k - 1]
    meta["trace"] = dict(config="c0", seed=0, iterations=100,
                         x_bits_xor=int(np.bitwise_xor.reduce(xs.view(np.uint64).ravel())),
                         y_bits_xor=int(np.bitwise_xor.reduce(ys.view(np.uint64).ravel())))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    json.dump(meta, open(os.path.join(HERE, "golden.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
