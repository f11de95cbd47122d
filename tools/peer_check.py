import numpy as np
import paper_2501_07018_b200 as P
from paper_2501_07018_b200 import sharded as S
for world in (2, 3):
    p = P.generate("c1", 5, sources=23, sinks=31)
    o = P.SolverOptions(mode="perf", iteration_limit=400, logging=(world == 2))
    b = S.solve_sharded_emulated(p, o, world)
    print(world, b.status, b.iterations)
