"""The bench's reference arm (oracle/ref_arm.py) runs the compiled reference
alone: loaded by path, it imports no module of the product package and maps
no library of this repo other than oracle/_ref/libpdhglp_ref.so (VERDICT r1:
round 1's arm imported the package and mapped its libraries)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "libpdhglp_ref.so")

CHILD = r"""
import importlib.util, json, os, sys
spec = importlib.util.spec_from_file_location("ra", os.path.join(sys.argv[1], "oracle", "ref_arm.py"))
ra = importlib.util.module_from_spec(spec); spec.loader.exec_module(ra)
d = ra.load_arrays(sys.argv[2])
w = ra.time_window(d, 2, 2, 3)
maps = open("/proc/self/maps").read()
repo_libs = sorted({l.split()[-1] for l in maps.splitlines()
                    if l.split()[-1].startswith(sys.argv[1]) and l.split()[-1].endswith(".so")})
print(json.dumps({"w": w, "libs": repo_libs,
                  "pkg": [m for m in sys.modules if m.startswith("paper_2501_07018_b200")]}))
"""


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")
def test_reference_arm_maps_only_the_reference(tmp_path):
    import json

    import paper_2501_07018_b200 as P
    from paper_2501_07018_b200.problem import save_problem
    p = P.generate("c0", 1, rows=120, cols=240)
    save_problem(p, str(tmp_path / "inst"))
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(tmp_path / "inst")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["pkg"] == []
    assert out["libs"] == [REF]
    w = out["w"]
    assert w["iterations"] == 3 and w["window_seconds"] > 0.0 and w["value"] > 0.0


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")
def test_bench_reference_window_matches_a_direct_solve():
    """ref_time_window runs the unmodified reference solve: over the same
    iterations it reaches the same state as oracle.solve (same restarts)."""
    import importlib.util

    import numpy as np
    import oracle
    import paper_2501_07018_b200 as P
    spec = importlib.util.spec_from_file_location("ra", os.path.join(ROOT, "oracle", "ref_arm.py"))
    ra = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ra)
    p = P.generate("c0", 2, rows=150, cols=300)
    d = {"rows": p.rows(), "cols": p.cols(), "row_start": p.a.by_row.start, "row_index": p.a.by_row.index,
         "row_value": p.a.by_row.value, "col_start": p.a.by_col.start, "col_index": p.a.by_col.index,
         "col_value": p.a.by_col.value, "objective": p.objective, "con_lower": p.con_lower,
         "con_upper": p.con_upper, "var_lower": p.var_lower, "var_upper": p.var_upper}
    w = ra.time_window(d, 1, 3, 100)
    o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), iteration_limit=103,
                        threads=1, shards_per_thread=4)
    r = oracle.get().solve(p, o)
    assert w["iterations"] == 100 and r.iterations == 103
    assert w["restarts"] == r.restarts and w["step_retries"] == r.step_retries
    assert np.isfinite(w["value"])
