"""The SpMV schedule (tiles, warp lines, CTA chunks) built by host threads
equals the sequential greedy build: perf-mode iterates depend on the tiling
through the per-CTA partial sums of the step reductions, so solves with one
and with many schedule threads must agree bit for bit."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2501_07018_b200 as P


def _mixed_lp(seed: int, rows: int, cols: int):
    """Columns of mixed lengths: mostly 1-3 entries (tiled), some ~100
    (warp lines) and a few ~3000 (CTA chunks) -- every segment kind, with
    enough lines (>= 2^19) for the threaded build to split them."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 4, cols)
    lens[rng.choice(cols, 300, replace=False)] = 100
    lens[rng.choice(cols, 5, replace=False)] = 3000
    c = np.repeat(np.arange(cols), lens)
    r = rng.integers(0, rows, c.size)
    v = rng.uniform(-1, 1, c.size)
    key = r.astype(np.int64) * cols + c
    _, first = np.unique(key, return_index=True)
    r, c, v = r[first], c[first], v[first]
    trip = list(zip(r.tolist(), c.tolist(), v.tolist()))
    xs = rng.uniform(0, 1, cols)
    A = np.zeros(rows)
    np.add.at(A, r, v * xs[c])
    return P.problem(rows, cols, trip, rng.normal(size=cols), A - 1.0, A + 1.0,
                     np.zeros(cols), np.full(cols, 5.0))


@pytest.mark.gpu
def test_threaded_schedule_equals_sequential(gpu, monkeypatch):
    cases = [P.generate("c1", 0, sources=1100, sinks=1000), _mixed_lp(3, 20000, 700000)]
    for p in cases:
        o = P.SolverOptions(mode="perf", iteration_limit=300,
                            tolerances=P.TerminationTolerances(0.0, 0.0, 0.0))
        monkeypatch.setenv("PDLP_SCHED_THREADS", "1")
        a = P.solve(p, o)
        monkeypatch.setenv("PDLP_SCHED_THREADS", "7")
        b = P.solve(p, o)
        assert a.iterations == b.iterations == 300
        np.testing.assert_array_equal(a.x.view(np.int64), b.x.view(np.int64))
        np.testing.assert_array_equal(a.y.view(np.int64), b.y.view(np.int64))


@pytest.mark.gpu
def test_uniform_vectors_are_bit_identical(gpu, monkeypatch):
    """Bitwise-uniform scaled c / l_v / u_v (x >= 0 problems; the polishing
    subproblems' zero objective) are read as scalars by the primal pass: the
    same values, so the same bits as streaming them."""
    cases = [P.generate("c1", 6, sources=300, sinks=400),      # l_v = 0, u_v = inf everywhere
             P.generate("c0", 7, rows=300, cols=600)]           # mixed bounds: no flags but c' = 0 in polish
    for p in cases:
        tol = P.relative_tolerances(p, 1e-4)
        o = P.SolverOptions(mode="perf", tolerances=P.TerminationTolerances(*tol))
        monkeypatch.setenv("PDLP_NO_UNIFORM", "1")
        a = P.solve(p, o)
        monkeypatch.delenv("PDLP_NO_UNIFORM")
        b = P.solve(p, o)
        assert (a.status, a.iterations, a.polish_iterations) == (b.status, b.iterations, b.polish_iterations)
        np.testing.assert_array_equal(a.x.view(np.int64), b.x.view(np.int64))
        np.testing.assert_array_equal(a.y.view(np.int64), b.y.view(np.int64))


def _solve_in_subprocess(env_extra, cfg, kw):
    """A solve in a fresh process (PDLP_NO_PDL is read once per process)."""
    import json
    import os
    import subprocess
    import sys
    code = (
        "import json, numpy as np, paper_2501_07018_b200 as P\n"
        f"p = P.generate({cfg!r}, 8, **{kw!r})\n"
        "tol = P.relative_tolerances(p, 1e-4)\n"
        "r = P.solve(p, P.SolverOptions(mode='perf', tolerances=P.TerminationTolerances(*tol)))\n"
        "print(json.dumps({'it': r.iterations, 'pol': r.polish_iterations,"
        " 'x': r.x.view(np.int64).tolist()[:2000], 'hx': int(np.bitwise_xor.reduce(r.x.view(np.int64))),"
        " 'hy': int(np.bitwise_xor.reduce(r.y.view(np.int64)))}))\n")
    env = dict(os.environ, **env_extra)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


@pytest.mark.gpu
def test_programmatic_dependent_launch_is_bit_identical(gpu):
    """The step chain and the cadence's kernels launched with programmatic
    dependent launch (each waits on griddepcontrol.wait) give the same bits as
    plain launches: whole solves to 1e-4, polishing included."""
    for cfg, kw in (("c1", {"sources": 300, "sinks": 400}), ("c0", {"rows": 400, "cols": 800})):
        a = _solve_in_subprocess({"PDLP_NO_PDL": "1"}, cfg, kw)
        b = _solve_in_subprocess({}, cfg, kw)
        assert a == b


@pytest.mark.gpu
def test_interleaved_warp_lines_are_bit_identical(gpu, monkeypatch):
    """With per-line row-pass partials the step's reductions do not depend on
    the SpMV schedule: interleaving the row layout's warp lines changes no
    bit of the iterates."""
    for p in (P.generate("c1", 9, sources=300, sinks=400), P.generate("c0", 9, rows=500, cols=900)):
        tol = P.relative_tolerances(p, 1e-4)
        o = P.SolverOptions(mode="perf", tolerances=P.TerminationTolerances(*tol))
        monkeypatch.setenv("PDLP_NO_INTERLEAVE", "1")
        a = P.solve(p, o)
        monkeypatch.delenv("PDLP_NO_INTERLEAVE")
        b = P.solve(p, o)
        assert (a.iterations, a.polish_iterations) == (b.iterations, b.polish_iterations)
        np.testing.assert_array_equal(a.x.view(np.int64), b.x.view(np.int64))
        np.testing.assert_array_equal(a.y.view(np.int64), b.y.view(np.int64))


@pytest.mark.gpu
def test_interleaved_warp_lines_polishing_bit_identical(gpu, monkeypatch):
    """The dual polishing subproblem runs its column pass over the (interleaved)
    row layout; that pass takes the split form (product, then an elementwise
    epilogue whose partials follow the line index), so polishing is
    bit-identical with and without interleaving too."""
    p = P.generate("c1", 9, sources=300, sinks=400)
    tp, td, _ = P.relative_tolerances(p, 1e-7)
    o = P.SolverOptions(mode="perf", tolerances=P.TerminationTolerances(tp, td, 0.5),
                        iteration_limit=20000)
    monkeypatch.setenv("PDLP_NO_INTERLEAVE", "1")
    a = P.solve(p, o)
    monkeypatch.delenv("PDLP_NO_INTERLEAVE")
    b = P.solve(p, o)
    assert a.polish_iterations > 0
    assert (a.status, a.iterations, a.polish_iterations) == (b.status, b.iterations, b.polish_iterations)
    np.testing.assert_array_equal(a.x.view(np.int64), b.x.view(np.int64))
    np.testing.assert_array_equal(a.y.view(np.int64), b.y.view(np.int64))
