"""One C1 solve of 320 iterations (5 cadences) for an ncu launch list of the
cadence kernels (tools/gap_report.py summarizes it)."""
import paper_2501_07018_b200 as P

p = P.generate("c1", 0)
o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), iteration_limit=320)
P.solve(p, o)
