"""C1 end-to-end breakdown (PDLP_TIMING): pdlp_solve of 20 iterations from
page-locked host buffers, as bench.py's c1 e2e key."""
import os
import sys
import time

os.environ["PDLP_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_07018_b200 as P  # noqa: E402

p = P.generate("c1", 0)
pp = P.pinned_copy(p)
out = {"x": P.pinned_empty(p.cols()), "y": P.pinned_empty(p.rows()),
       "reduced_costs": P.pinned_empty(p.cols())}
P.solve(pp, bench._options(P, 20, 0), out=out)
for _ in range(3):
    t0 = time.perf_counter()
    r = P.solve(pp, bench._options(P, 20, 0), out=out)
    w = time.perf_counter() - t0
    print(f"C1 e2e K=20: wall {1e3 * w:.2f} ms -> {20 / w:.1f} it/s", flush=True)
