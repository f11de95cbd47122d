"""Cadence share of a fixed-work solve per config (PDLP_TIMING line)."""
import os
import sys

os.environ["PDLP_TIMING"] = "1"
import paper_2501_07018_b200 as P  # noqa: E402

for cfg in sys.argv[1:] or ["c1"]:
    p = P.generate(cfg, 0)
    o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), iteration_limit=512)
    P.solve(p, o)
    print(cfg, "---", file=sys.stderr, flush=True)
    P.solve(p, o)
