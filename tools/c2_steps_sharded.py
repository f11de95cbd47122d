"""A few C2 iterations through the sharded engine at world 1 (column cut,
shard-local ingest, 1-rank NCCL communicator): the ncu target for the
per-rank attempt of `bench.py --gpus N`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_07018_b200 as P  # noqa: E402
from paper_2501_07018_b200 import sharded as S  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

name, seed, kw = bench.WORKLOADS["c2"]["gen"]
kw = {k: v for k, v in kw.items() if k != "row_window"}
shard = S.generate_shard(name, seed, 0, 1, cut="auto", **kw)
o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), iteration_limit=12)
S.solve_sharded_local(shard, o, 0, 1, S.nccl_unique_id())
