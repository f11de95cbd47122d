"""C2 cadence breakdown (PDLP_TIMING line): W=5 warm-up + K=20 timed, as the
driver's bench window."""
import os
import sys

os.environ["PDLP_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_07018_b200 as P  # noqa: E402
from paper_2501_07018_b200.problem import load_problem, save_problem  # noqa: E402

inst = "/dev/shm/pdlp_c2_0"
if not os.path.exists(os.path.join(inst, "shape.json")):
    save_problem(P.generate("c2", 0), inst)
p = load_problem(inst)
P.solve(p, bench._options(P, 16, 0))
for k in (20, 64):
    r = P.solve(p, bench._options(P, k, 5))
    print(f"K={k}: {r.timed_iterations / r.timed_seconds:.1f} it/s, timed {r.timed_seconds * 1e3:.2f} ms", flush=True)
