"""C2 end-to-end breakdown (PDLP_TIMING): pdlp_solve from host buffers for
K = 20 iterations, as the bench's e2e."""
import os
import sys
import time

os.environ["PDLP_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_07018_b200 as P  # noqa: E402

p = bench.generate("c2")
P.solve(p, bench._options(P, 16, 0))
for _ in range(2):
    t0 = time.perf_counter()
    r = P.solve(p, bench._options(P, 20, 0))
    print(f"e2e K=20: wall {time.perf_counter() - t0:.3f}s -> {20 / (time.perf_counter() - t0):.1f} it/s",
          flush=True)
