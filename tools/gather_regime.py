"""Row/column pass cost per entry vs the size of the gathered vector
(C2 family): does an L2-resident x-bar change the regime?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_07018_b200 as P  # noqa: E402

for rows, cols in ((5_000_000, 2_500_000), (5_000_000, 5_000_000), (5_000_000, 10_000_000),
                   (1_250_000, 10_000_000)):
    p = P.generate("c2", 0, rows=rows, cols=cols)
    m, n, nnz = p.rows(), p.cols(), p.a.nonzeros()
    prof = P.solve(p, bench._options(P, 32, 4, profile_kernels=True))
    out = {"m": m, "n": n, "nnz": nnz, "xbar_MB": n * 8 / 2**20, "dy_MB": m * 8 / 2**20}
    for q, nm in enumerate(["primal_pass", "row_pass", "col_pass"]):
        t = prof.kernel_seconds[q] / max(prof.kernel_launches[q], 1)
        out[nm + "_us"] = round(t * 1e6, 1)
        if nm != "primal_pass":
            out[nm + "_ps_per_nnz"] = round(t / nnz * 1e12, 1)
    print(json.dumps(out), flush=True)
