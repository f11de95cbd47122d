"""Small solves covering every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per run): staged tiles, warp
lines, CTA chunks, segmented spans (forced), column panels (forced), the
cadence (screens, rays, gap), polishing, and parity mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_07018_b200 as P  # noqa: E402


def run(tag, p, **kw):
    tol = P.relative_tolerances(p)
    o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=300, **kw)
    r = P.solve(p, o)
    print(f"{tag}: {P.solve_status_name(r.status)} it={r.iterations} polish={r.polish_iterations}",
          flush=True)


c0 = P.generate("c0", 0, rows=200, cols=400)
c1 = P.generate("c1", 0, sources=30, sinks=40)
c2 = P.generate("c2", 1, rows=3000, cols=6000, kmax=3000)
run("c0 perf", c0)
run("c0 parity", c0, mode="parity")
run("c1 perf", c1)
run("c2 perf (tiles / warp lines / CTA chunks)", c2)
os.environ["PDLP_SEG"] = "1"
run("c2 perf (segmented spans)", c2)
os.environ["PDLP_ROW_PANELS"] = "2"
run("c2 perf (segmented spans + column panels)", c2)
del os.environ["PDLP_SEG"]
run("c2 perf (tiles + column panels)", c2)
