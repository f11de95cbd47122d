"""A few C2 iterations (ncu target for the full-size power-law config)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_07018_b200 as P  # noqa: E402

p = P.generate("c2", 0, row_window=(0, 5_000_000))  # the benchmarked instance (bench.py)
o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), iteration_limit=12)
P.solve(p, o)
