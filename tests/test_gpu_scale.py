"""Parity on the benchmarked workloads at full size (BASELINE
north_star: iterates within 1e-9 relative over the first iterations, the same
restart/termination decisions, final objective and residuals meeting the same
tolerances).

The oracle is the compiled reference (oracle/_ref) run here on the box's host
cores.  Iterates are compared through per-iterate strided samples plus the full
vectors at the last compared iterate (a full trace of C2 would be GBs).
Drift is measured as max_k ||g_k - r_k||_inf / max(||g_k||, ||r_k||) (helpers.
max_rel); the perf-mode bar is max(1e-9, 2x the reference's own spread when
only its shard plan changes), measured in the same test.
"""
import os

import numpy as np
import pytest

import paper_2501_07018_b200 as P
from tests.helpers import max_rel, same_bits

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = os.cpu_count() or 1


def _opts(n_iter, mode="perf", spt=4, tol=(0.0, 0.0, 0.0)):
    o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=n_iter,
                        threads=THREADS, shards_per_thread=spt)
    o.mode = mode
    return o


_REF_TRACES = {}  # reference traces shared by the parity and the perf test of one instance


def _ref_trace(ref, p, n_iter, stride_x, stride_y, spt=4):
    """The compiled reference's sampled trace (threads = nproc, spt shards per
    thread), computed once per (instance, window, shard plan): a C2 reference
    run costs ~1 minute of host time."""
    key = (id(p), n_iter, stride_x, stride_y, spt)
    if key not in _REF_TRACES:  # the entry keeps p alive, so its id cannot be reused
        _REF_TRACES[key] = (p, _sampled_trace(ref.solve, p, _opts(n_iter, spt=spt), n_iter, stride_x, stride_y))
    return _REF_TRACES[key][1]


def _sampled_trace(solver_fn, p, o, n_iter, stride_x, stride_y):
    """Strided samples of x and y after each of the first n_iter accepted
    steps, and the full vectors after the last one."""
    xs, ys, last = [], [], {}

    def obs(rec):
        if rec.iteration <= n_iter:
            xs.append(rec.x[::stride_x].copy())
            ys.append(rec.y[::stride_y].copy())
            if rec.iteration == n_iter:
                last["x"], last["y"] = rec.x.copy(), rec.y.copy()

    o.observer = obs
    o.iteration_limit = n_iter
    solver_fn(p, o)
    return np.array(xs), np.array(ys), last


def _perf_drift_case(ref, p, n_iter, stride_x, stride_y, spts=(4, 1, 16)):
    """(drift of the GPU perf trace vs the reference, the reference's own
    spread across shard plans)."""
    rx, ry, rl = _ref_trace(ref, p, n_iter, stride_x, stride_y, spt=spts[0])
    spread = 0.0
    for spt in spts[1:]:
        sx, sy, sl = _ref_trace(ref, p, n_iter, stride_x, stride_y, spt=spt)
        spread = max(spread, max_rel(sx, rx), max_rel(sy, ry), max_rel(sl["x"], rl["x"]),
                     max_rel(sl["y"], rl["y"]))
    gx, gy, gl = _sampled_trace(P.solve, p, _opts(n_iter), n_iter, stride_x, stride_y)
    assert gx.shape == rx.shape and gy.shape == ry.shape
    drift = max(max_rel(gx, rx), max_rel(gy, ry), max_rel(gl["x"], rl["x"]), max_rel(gl["y"], rl["y"]))
    return drift, spread


# --------------------------------------------------------------- C1 full ---
@pytest.fixture(scope="module")
def c1():
    return P.generate("c1", 0)


def test_c1_full_first_100_iterates_parity(gpu, ref, c1):
    """Parity mode on the full 2000x2000 transport LP: the first 100 iterates
    are the reference's bit for bit (same shard plan)."""
    rx, ry, rl = _ref_trace(ref, c1, 100, 997, 1)
    gx, gy, gl = _sampled_trace(P.solve, c1, _opts(100, mode="parity"), 100, 997, 1)
    assert same_bits(gx, rx) and same_bits(gy, ry)
    assert same_bits(gl["x"], rl["x"]) and same_bits(gl["y"], rl["y"])


def test_c1_full_first_100_iterates_perf(gpu, ref, c1):
    drift, spread = _perf_drift_case(ref, c1, 100, 997, 1)
    print(f"C1 full, first 100 iterates: perf drift {drift:.3e}, reference spread {spread:.3e}")
    assert drift <= max(1e-9, 2.0 * spread), (drift, spread)


def test_c1_full_solve_to_1e4(gpu, ref, c1):
    """The 1e-4 solve of the benchmarked C1 instance: perf mode reaches the
    reference's status with residuals and objective inside the same
    tolerances, in an iteration count within the spread the reference shows
    across its own shard plans (x1.5 margin)."""
    tol = P.relative_tolerances(c1)
    r4 = ref.solve(c1, _opts(200000, spt=4, tol=tol))
    # a second shard plan of the reference (~45 s of host time) only on request:
    # its spread is recorded over 5 seeds in profiles/r2_c1_seeds_vs_reference.jsonl
    r1 = ref.solve(c1, _opts(200000, spt=1, tol=tol)) if os.environ.get("PDLP_LONG_TESTS") == "1" else r4
    g = P.solve(c1, _opts(200000, tol=tol))
    assert g.status == r4.status == r1.status == P.SolveStatus.OPTIMAL
    s = g.summary
    assert s.primal_residual_inf <= tol[0] and s.dual_residual_inf <= tol[1] and s.rel_gap <= tol[2]
    ref_obj = r4.summary.primal_objective
    assert abs(s.primal_objective - ref_obj) <= 1e-4 * (1.0 + abs(ref_obj))
    lo = min(r4.iterations, r1.iterations)
    hi = max(r4.iterations, r1.iterations)
    print(f"C1 1e-4: gpu perf {g.iterations} it ({g.restarts} restarts), reference "
          f"{r4.iterations} (S=4x{THREADS})" + (f" / {r1.iterations} (S=1x{THREADS})" if r1 is not r4 else ""))
    assert lo / 1.5 <= g.iterations <= hi * 1.5


@pytest.mark.skipif(os.environ.get("PDLP_LONG_TESTS") != "1",
                    reason="~5 min: parity-mode C1 solve to 1e-4 (set PDLP_LONG_TESTS=1)")
def test_c1_full_solve_to_1e4_parity(gpu, ref, c1):
    """Parity mode reproduces the reference's whole 1e-4 run on the full C1
    instance: iterations, restarts, polishing and the solution bits."""
    tol = P.relative_tolerances(c1)
    r4 = ref.solve(c1, _opts(200000, spt=4, tol=tol))
    g = P.solve(c1, _opts(200000, mode="parity", spt=4, tol=tol))
    assert g.status == r4.status == P.SolveStatus.OPTIMAL
    assert (g.iterations, g.restarts, g.polish_iterations) == (r4.iterations, r4.restarts, r4.polish_iterations)
    assert same_bits(g.x, r4.x) and same_bits(g.y, r4.y)


# --------------------------------------------------------------- C2 full ---
@pytest.fixture(scope="module")
def c2():
    # the benchmarked instance (bench.py WORKLOADS["c2"]: counter-based streams)
    return P.generate("c2", 0, row_window=(0, 5_000_000))


def test_c2_full_first_iterates_parity(gpu, ref, c2):
    """The headline workload (5M x 10M, ~165M nonzeros): parity mode's first
    12 iterates equal the reference's bit for bit."""
    n = 12
    rx, ry, rl = _ref_trace(ref, c2, n, 4999, 2503)
    gx, gy, gl = _sampled_trace(P.solve, c2, _opts(n, mode="parity"), n, 4999, 2503)
    assert same_bits(gx, rx) and same_bits(gy, ry)
    assert same_bits(gl["x"], rl["x"]) and same_bits(gl["y"], rl["y"])


def test_c2_full_first_iterates_perf(gpu, ref, c2):
    """Perf mode on the headline workload -- the column panels of the row
    pass and the segmented spans of the column pass -- tracks the reference
    within max(1e-9, 2x its own shard-plan spread) over the first 12
    iterates."""
    drift, spread = _perf_drift_case(ref, c2, 12, 4999, 2503, spts=(4, 1))
    print(f"C2 full, first 12 iterates: perf drift {drift:.3e}, reference spread {spread:.3e}")
    assert drift <= max(1e-9, 2.0 * spread), (drift, spread)


# ------------------------------------------------------ C2 / C3 mid-size ---
def test_c2_full_perf_mode_is_deterministic(gpu, c2):
    """on layouts of >= 16M entries the schedule is a
    function of the line lengths (no timed autotuning), the step reductions
    combine in a fixed order and the gap's window placement is a function of
    its inputs -- two perf solves of the headline instance across a 64-step
    cadence (screens, ray tests, gap evaluations, a restart decision) give
    the same bits."""
    o = _opts(70)
    a, b = P.solve(c2, o), P.solve(c2, o)
    assert (a.iterations, a.restarts, a.step_retries) == (b.iterations, b.restarts, b.step_retries)
    assert a.final_step_size == b.final_step_size and a.final_primal_weight == b.final_primal_weight
    assert same_bits(a.x, b.x) and same_bits(a.y, b.y)


@pytest.mark.parametrize("force", [None, "seg", "panels"])
def test_c2_mid_first_100_iterates_perf(gpu, ref, monkeypatch, force):
    """C2 recipe at 200k x 400k: first 100 iterates, with the default
    schedule, with segmented spans forced on both layouts, and with column
    panels forced on the row pass."""
    p = P.generate("c2", 0, rows=200_000, cols=400_000)
    if force == "seg":
        monkeypatch.setenv("PDLP_SEG", "1")
    elif force == "panels":
        monkeypatch.setenv("PDLP_ROW_PANELS", "2")
    drift, spread = _perf_drift_case(ref, p, 100, 97, 53)
    print(f"C2 200k x 400k ({force}): perf drift {drift:.3e}, reference spread {spread:.3e}")
    assert drift <= max(1e-9, 2.0 * spread), (drift, spread)


def test_c3_mid_first_100_iterates_perf(gpu, ref):
    """C3 unit-commitment recipe at 168 periods x 100 generators."""
    p = P.generate("c3", 0, periods=168, generators=100)
    drift, spread = _perf_drift_case(ref, p, 100, 7, 11)
    print(f"C3 168x100: perf drift {drift:.3e}, reference spread {spread:.3e}")
    assert drift <= max(1e-9, 2.0 * spread), (drift, spread)


def test_c3_mid_first_100_iterates_parity(gpu, ref):
    p = P.generate("c3", 0, periods=168, generators=100)
    rx, ry, rl = _sampled_trace(ref.solve, p, _opts(100), 100, 7, 11)
    gx, gy, gl = _sampled_trace(P.solve, p, _opts(100, mode="parity"), 100, 7, 11)
    assert same_bits(gx, rx) and same_bits(gy, ry)
    assert same_bits(gl["x"], rl["x"]) and same_bits(gl["y"], rl["y"])


# ------------------------------------------------------ sharded, at scale ---
@pytest.mark.parametrize("cut", ["rows", "cols"])
def test_c2_full_sharded_world2_tracks_single_gpu(gpu, c2, monkeypatch, cut):
    """The sharded solve on the headline instance (both cuts, 2 emulated
    ranks on one GPU: shards extracted on the host, segmented spans, long
    multi-chunk columns, peer-read epilogues, the distributed gap) tracks the
    single-GPU solve within 1e-9 relative over the first 12 iterates.  (With
    tolerances unreachable and 12 < 64 no restart or gap decision is taken,
    so the comparison isolates the per-rank kernels and the exchanges.)"""
    from paper_2501_07018_b200 import sharded as S
    monkeypatch.setenv("PDLP_SHARD_CUT", cut)
    o = P.SolverOptions(mode="perf", iteration_limit=12,
                        tolerances=P.TerminationTolerances(0.0, 0.0, 0.0))
    a = P.solve(c2, o)
    b = S.solve_sharded_emulated(c2, o, 2)
    assert a.iterations == b.iterations == 12
    rel = lambda u, v: float(np.max(np.abs(u - v)) / max(1e-300, np.max(np.abs(v))))  # noqa: E731
    assert rel(b.x, a.x) <= 1e-9 and rel(b.y, a.y) <= 1e-9, (rel(b.x, a.x), rel(b.y, a.y))
