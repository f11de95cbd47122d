"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar: PARITY mode is bit-exact with the reference for the same shard plan;
PERF mode stays within the reference's own cross-shard-plan spread
(1e-9 relative over the first 100 iterations); written
tolerances below.
"""
import math

import numpy as np
import pytest

import paper_2501_07018_b200 as P
from tests.helpers import (INF, box_interior_point, clamp_free_row, contradictory_rows, dense,
                           equality_lp, max_rel, one_var_equality, overflow_lp, random_box_lp,
                           rejection_lp, same_bits, slack_row_box_lp, tiny_lp, unbounded_lp)

pytestmark = pytest.mark.gpu

MODES = ["parity", "perf"]


# ------------------------------------------------------------ single step ---
@pytest.mark.parametrize("mode", MODES)
def test_step_known_answers(gpu, mode):
    # test_step.cpp:116-130
    x, y = P.pdhg_step(one_var_equality(), [0.0], [0.0], 1.0, 0.5, mode=mode)
    assert x[0] == 0.0 and y[0] == 0.5
    # test_step.cpp:132-148: one-sided clamp, free row multiplier exactly 0
    x, y = P.pdhg_step(clamp_free_row(), [3.0], [0.0, 5.0], 1.0, 1.0, mode=mode)
    assert x[0] == 3.0 and y[0] == -1.0 and y[1] == 0.0


@pytest.mark.parametrize("mode", MODES)
def test_step_matches_reference(gpu, ref, mode):
    # test_step.cpp:150-171 (40 random box LPs, one step)
    rng = np.random.default_rng(20240801)
    for _ in range(40):
        p = random_box_lp(rng, 1 + rng.integers(8), 1 + rng.integers(8))
        x = box_interior_point(rng, p)
        y = rng.uniform(-1.5, 1.5, p.rows())
        omega = math.exp(rng.uniform(-1.5, 1.5))
        eta = math.exp(rng.uniform(-2.0, 0.0))
        g = P.pdhg_step(p, x, y, omega, eta, mode=mode)
        r = ref.pdhg_step(p, x, y, omega, eta)
        assert (g is None) == (r is None)
        if mode == "parity":
            assert same_bits(g[0], r[0]) and same_bits(g[1], r[1])
        else:
            np.testing.assert_allclose(g[0], r[0], rtol=0, atol=1e-12)
            np.testing.assert_allclose(g[1], r[1], rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode", MODES)
def test_rejection_then_accept(gpu, mode):
    # test_step.cpp:274-304
    out = P.adaptive_step(rejection_lp(), [0.0], [1.0], [1.0], eta_hat=4.0, mode=mode)
    assert out["accepted"]
    assert out["retries"] == 1 and out["accepted_steps"] == 1 and out["k"] == 1
    assert out["min_eta_bar"] == 1.25
    assert out["eta_used"] == pytest.approx((1.0 - 2.0 ** -0.3) * 1.25, rel=1e-15)
    ref_step = P.pdhg_step(rejection_lp(), [0.0], [1.0], 1.0, out["eta_used"], mode=mode)
    assert out["x"][0] == ref_step[0][0] and out["y"][0] == ref_step[1][0]
    assert out["prev_x"][0] == 0.0 and out["prev_y"][0] == 1.0


@pytest.mark.parametrize("mode", MODES)
def test_retry_exhaustion_and_overflow(gpu, mode):
    # test_step.cpp:306-345
    out = P.adaptive_step(rejection_lp(), [0.0], [1.0], [1.0], eta_hat=4.0, max_retries=0, mode=mode)
    assert not out["accepted"] and out["retries"] == 1 and out["accepted_steps"] == 0
    assert out["x"][0] == 0.0 and out["y"][0] == 1.0 and out["aty"][0] == 1.0
    out = P.adaptive_step(overflow_lp(), [0.0], [0.0], [0.0], eta_hat=1e8, mode=mode)
    assert not out["accepted"]


def test_adaptive_step_matches_reference(gpu, ref):
    rng = np.random.default_rng(555123)
    for _ in range(25):
        p = random_box_lp(rng, 1 + rng.integers(6), 1 + rng.integers(6))
        x = box_interior_point(rng, p)
        y = rng.uniform(-1, 1, p.rows())
        aty = ref.spmv_transpose(p, y)
        eta0 = ref.initial_step_size(p)
        g = P.adaptive_step(p, x, y, aty, eta_hat=eta0, mode="parity")
        r = ref.adaptive_step(p, x, y, aty, eta_hat=eta0)
        assert g["accepted"] == r["accepted"]
        for key in ("x", "y", "aty", "prev_x", "prev_y"):
            assert same_bits(g[key], r[key]), key
        for key in ("eta_hat", "retries", "min_eta_bar", "eta_used"):
            assert same_bits(g[key], r[key]), key


# ------------------------------------------------------------- components ---
@pytest.mark.parametrize("mode", MODES)
def test_spmv_matches_reference(gpu, ref, mode):
    rng = np.random.default_rng(3)
    for _ in range(10):
        p = random_box_lp(rng, 1 + rng.integers(40), 1 + rng.integers(40))
        x = rng.uniform(-1, 1, p.cols())
        y = rng.uniform(-1, 1, p.rows())
        gx, gy = P.spmv(p, x, mode=mode), P.spmv_transpose(p, y, mode=mode)
        rx, ry = ref.spmv(p, x), ref.spmv_transpose(p, y)
        if mode == "parity":
            assert same_bits(gx, rx) and same_bits(gy, ry)
        else:
            np.testing.assert_allclose(gx, rx, rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(gy, ry, rtol=1e-12, atol=1e-12)


def test_spmv_skewed_schedule(gpu, ref):
    # C2-style power-law columns exercise the warp and CTA segments.
    p = P.generate("c2", 3, rows=5000, cols=6000, kmax=5000)
    assert np.diff(p.a.by_col.start).max() > 2048  # > PDLPK_CHUNK: multi-chunk lines
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, p.cols())
    y = rng.uniform(-1, 1, p.rows())
    np.testing.assert_allclose(P.spmv(p, x, mode="perf"), ref.spmv(p, x), rtol=1e-11, atol=1e-9)
    np.testing.assert_allclose(P.spmv_transpose(p, y, mode="perf"), ref.spmv_transpose(p, y),
                               rtol=1e-11, atol=1e-9)


def test_rescaling_matches_reference(gpu, ref):
    for p in (P.generate("c0", 0, rows=200, cols=400), P.generate("c2", 1, rows=500, cols=1000),
              P.generate("c1", 0, sources=20, sinks=30), tiny_lp()):
        g = P.apply_rescaling(p)
        r = ref.apply_rescaling(p)
        for k in r:
            assert same_bits(g[k], r[k]), k


@pytest.mark.parametrize("mode", MODES)
def test_gap_matches_reference(gpu, ref, mode):
    rng = np.random.default_rng(42100)
    for _ in range(20):
        p = random_box_lp(rng, 1 + rng.integers(6), 1 + rng.integers(6))
        x = box_interior_point(rng, p)
        y = rng.uniform(-1, 1, p.rows())
        ax, aty = ref.spmv(p, x), ref.spmv_transpose(p, y)
        omega = math.exp(rng.uniform(-1, 1))
        for r in (0.0, -1.0, 0.25, 1.0, 4.0):
            g = P.normalized_duality_gap(p, x, y, ax, aty, omega, r, mode=mode)
            e = ref.normalized_duality_gap(p, x, y, ax, aty, omega, r)
            if mode == "parity":
                assert same_bits(g, e)
            else:
                assert g == pytest.approx(e, rel=1e-11, abs=1e-14)


def test_gap_closed_form(gpu):
    # test_restarts.cpp:149-172
    p = P.problem(0, 1, [], [1.5], [], [], [-1.0], [INF])
    for omega in (1.0, 2.0):
        for r in (0.25, 1.0, 4.0):
            travel = min(r / math.sqrt(omega), 1.2)
            g = P.normalized_duality_gap(p, [0.2], [], [], [0.0], omega, r)
            assert g == pytest.approx(1.5 * travel / r, rel=1e-12)


@pytest.mark.parametrize("mode", MODES)
def test_kkt_matches_reference(gpu, ref, mode):
    rng = np.random.default_rng(991100)
    for _ in range(15):
        p = random_box_lp(rng, 2 + rng.integers(6), 2 + rng.integers(6))
        x = rng.uniform(-1, 1, p.cols())
        y = rng.uniform(-1, 1, p.rows())
        for rc in (0, 1):
            gr, gs = P.kkt_residuals(p, x, y, rc, mode=mode)
            rr, rs = ref.kkt_residuals(p, x, y, rc)
            if mode == "parity":
                assert same_bits(gr, rr)
                assert same_bits([gs.primal_residual_inf, gs.dual_residual_inf, gs.primal_objective,
                                  gs.dual_objective],
                                 [rs.primal_residual_inf, rs.dual_residual_inf, rs.primal_objective,
                                  rs.dual_objective])
            else:
                np.testing.assert_allclose(gr, rr, rtol=1e-12, atol=1e-12)
                assert gs.primal_objective == pytest.approx(rs.primal_objective, rel=1e-12, abs=1e-12)


# ------------------------------------------------------------ full solves ---
def _opts(**kw):
    tol = kw.pop("tol", None)
    o = P.SolverOptions(**kw)
    if tol is not None:
        o.tolerances = P.TerminationTolerances(*tol)
    return o


@pytest.mark.parametrize("mode", MODES)
def test_tiny_lp_solves(gpu, mode):
    # test_solver.cpp:54-84
    out = P.solve(tiny_lp(), _opts(tol=(1e-8, 1e-8, 1e-9), mode=mode))
    assert out.status == P.SolveStatus.OPTIMAL
    assert out.x == pytest.approx([0.0, 1.0], abs=1e-6)
    assert out.y == pytest.approx([-2.0], abs=1e-6)
    assert out.reduced_costs == pytest.approx([1.0, 0.0], abs=1e-6)
    assert out.summary.primal_objective == pytest.approx(-2.0, abs=1e-7)
    assert out.iterations > 0 and out.termination_detail


def _assert_same_solve(g, r):
    assert g.status == r.status
    assert g.iterations == r.iterations
    assert g.polish_iterations == r.polish_iterations
    assert g.restarts == r.restarts
    assert g.step_retries == r.step_retries
    assert g.termination_detail == r.termination_detail
    assert same_bits(g.final_step_size, r.final_step_size)
    assert same_bits(g.final_primal_weight, r.final_primal_weight)
    assert same_bits(g.x, r.x) and same_bits(g.y, r.y) and same_bits(g.reduced_costs, r.reduced_costs)


def test_parity_solve_c0_bit_exact(gpu, ref):
    p = P.generate("c0", 0)
    tol = P.relative_tolerances(p)
    for spt in (4, 16):
        o = _opts(tol=tol, shards_per_thread=spt, mode="parity")
        _assert_same_solve(P.solve(p, o), ref.solve(p, o))


@pytest.mark.parametrize("seed", [1, 2])
def test_parity_solve_reference_kinds(gpu, ref, seed):
    for p in (equality_lp(np.random.default_rng(seed), 12, 16),
              P.generate("c1", seed, sources=8, sinks=9),
              slack_row_box_lp(np.random.default_rng(seed), 6, 10)):
        o = _opts(tol=(1e-8, 1e-8, 1e-9), mode="parity")
        _assert_same_solve(P.solve(p, o), ref.solve(p, o))


def _trace(solver_fn, p, o, n_iter=100):
    xs, ys = [], []

    def obs(rec):
        if rec.iteration <= n_iter:
            xs.append(rec.x)
            ys.append(rec.y)

    o.observer = obs
    o.iteration_limit = n_iter
    solver_fn(p, o)
    return np.array(xs), np.array(ys)


@pytest.mark.parametrize("seed", [0, 1, 3])
def test_first_100_iterates_parity(gpu, ref, seed):
    """BASELINE: per-iteration iterates within 1e-9 relative over the first
    100 iterations — bit-exact in parity mode, for two shard plans."""
    p = P.generate("c0", seed)
    tol = P.relative_tolerances(p)
    for spt in (4, 32):
        gx, gy = _trace(P.solve, p, _opts(tol=tol, shards_per_thread=spt, mode="parity"))
        rx, ry = _trace(ref.solve, p, _opts(tol=tol, shards_per_thread=spt))
        assert gx.shape == rx.shape == (100, p.cols())
        assert same_bits(gx, rx) and same_bits(gy, ry)


@pytest.mark.parametrize("seed", [0, 1, 3])
def test_first_100_iterates_perf(gpu, ref, seed):
    """Perf mode reorders sums (tree reductions, split long lines), which the
    reference itself does when only its shard plan changes.  Bar: drift vs the
    oracle <= max(1e-9, 2x the oracle's own spread across shard plans
    S in {1, 8, 32, 64}) — measured here, not assumed."""
    p = P.generate("c0", seed)
    tol = P.relative_tolerances(p)
    rx, ry = _trace(ref.solve, p, _opts(tol=tol))
    spread = 0.0
    for spt in (1, 8, 32, 64):
        sx, sy = _trace(ref.solve, p, _opts(tol=tol, shards_per_thread=spt))
        spread = max(spread, max_rel(sx, rx), max_rel(sy, ry))
    gx, gy = _trace(P.solve, p, _opts(tol=tol, mode="perf"))
    drift = max(max_rel(gx, rx), max_rel(gy, ry))
    assert drift <= max(1e-9, 2.0 * spread), (drift, spread)


def test_perf_solve_c0_decisions(gpu, ref):
    """Perf mode: termination within the oracle's own shard-plan spread; the
    final point meets the same tolerances."""
    p = P.generate("c0", 0)
    tol = P.relative_tolerances(p)
    g = P.solve(p, _opts(tol=tol, mode="perf"))
    r = ref.solve(p, _opts(tol=tol))
    assert g.status == r.status == P.SolveStatus.OPTIMAL
    assert g.summary.primal_residual_inf <= tol[0]
    assert g.summary.dual_residual_inf <= tol[1]
    assert g.summary.rel_gap <= tol[2]
    assert abs(g.summary.primal_objective - r.summary.primal_objective) <= 1e-3 * abs(r.summary.primal_objective)
    total_g = g.iterations + g.polish_iterations
    total_r = r.iterations + r.polish_iterations
    assert 0.5 * total_r <= total_g <= 2.0 * total_r


@pytest.mark.parametrize("mode", MODES)
def test_infeasibility_certificates(gpu, ref, mode):
    # test_solver.cpp:119-162
    out = P.solve(contradictory_rows(), _opts(mode=mode))
    assert out.status == P.SolveStatus.PRIMAL_INFEASIBLE
    assert out.certificate.kind == P.CertificateKind.PRIMAL_INFEASIBLE
    assert out.certificate.objective > 0.0
    out = P.solve(unbounded_lp(), _opts(mode=mode))
    assert out.status == P.SolveStatus.DUAL_INFEASIBLE
    assert out.certificate.objective < 0.0
    if mode == "parity":
        for p in (contradictory_rows(), unbounded_lp()):
            _assert_same_solve(P.solve(p, _opts(mode="parity")), ref.solve(p, _opts()))


@pytest.mark.parametrize("mode", MODES)
def test_fixed_step_and_limits(gpu, mode):
    # test_solver.cpp:188-204, 227-247, 286-303
    out = P.solve(tiny_lp(), _opts(tol=(1e-8, 1e-8, 1e-9), fixed_step_size=0.4,
                                   fixed_primal_weight=1.0, enable_restarts=False,
                                   enable_polish=False, mode=mode))
    assert out.status == P.SolveStatus.OPTIMAL
    assert out.final_step_size == 0.4 and out.final_primal_weight == 1.0
    assert out.restarts == 0 and out.step_retries == 0 and out.min_step_size_limit == INF
    out = P.solve(tiny_lp(), _opts(tol=(1e-8, 1e-8, 1e-12), iteration_limit=5, mode=mode))
    assert out.status == P.SolveStatus.ITERATION_LIMIT and out.iterations == 5
    out = P.solve(tiny_lp(), _opts(time_limit_seconds=0.0, mode=mode))
    assert out.status == P.SolveStatus.TIME_LIMIT and out.iterations == 0
    p = rejection_lp()
    p.con_lower[:] = 1.0
    p.con_upper[:] = 1.0
    out = P.solve(p, _opts(fixed_step_size=10.0, enable_scaling=False, enable_restarts=False,
                           detect_infeasibility=False, enable_polish=False, mode=mode))
    assert out.status == P.SolveStatus.NUMERICAL_ERROR and out.termination_detail


def test_polishing_runs(gpu, ref):
    # test_solver.cpp:269-284
    p = equality_lp(np.random.default_rng(11), 20, 30)
    o = _opts(tol=(1e-11, 1e-6, 0.5), mode="parity")
    g = P.solve(p, o)
    assert g.status == P.SolveStatus.OPTIMAL and g.polish_iterations > 0
    _assert_same_solve(g, ref.solve(p, o))


def test_observer_sees_every_step(gpu):
    seen = []
    o = _opts(tol=(1e-8, 1e-8, 1e-9))
    o.observer = lambda rec: seen.append(rec.iteration)
    out = P.solve(tiny_lp(), o)
    assert out.status == P.SolveStatus.OPTIMAL
    assert seen == list(range(1, out.iterations + 1))


def test_invalid_problem_rejected(gpu):
    q = tiny_lp()
    q.var_lower[0] = 2.0
    q.var_upper[0] = 1.0
    with pytest.raises(ValueError, match="variable bounds crossed"):
        P.solve(q)


def _tamper(kind):
    p = P.generate("c0", 0, rows=40, cols=60)
    nan = float("nan")
    if kind == "objective":
        p.objective[7] = nan
    elif kind == "var_nan":
        p.var_upper[3] = nan
    elif kind == "var_lo_inf":
        p.var_lower[5] = INF
    elif kind == "var_crossed":
        p.var_lower[9], p.var_upper[9] = 3.0, 1.0
    elif kind == "con_hi_neginf":
        p.con_upper[4] = -INF
    elif kind == "con_crossed":
        p.con_lower[11], p.con_upper[11] = 5.0, 4.0
    elif kind == "matrix_inf":
        p.a.by_row.value[13] = INF
    elif kind == "layout_value":
        p.a.by_col.value[2] += 1.0
    elif kind == "layout_index":
        p.a.by_row.index[0] = p.cols() + 3
    elif kind == "layout_order":
        L = p.a.by_row
        r = next(r for r in range(p.rows()) if L.start[r + 1] - L.start[r] >= 2)
        k = L.start[r]
        L.index[k], L.index[k + 1] = L.index[k + 1], L.index[k]
        L.value[k], L.value[k + 1] = L.value[k + 1], L.value[k]
    elif kind == "index_wraps":  # 2^32 + 5 would truncate to a valid 5
        p.a.by_row.index[3] = (1 << 32) + 5
    elif kind == "index_huge":
        p.a.by_col.index[1] = (1 << 40)
    elif kind == "index_negative":
        p.a.by_row.index[2] = -7
    elif kind == "start_wraps":
        p.a.by_col.start[5] = (1 << 32) + int(p.a.by_col.start[5])
    elif kind == "index_wraps_staged":  # > 1 MB of indices: the pinned-ring path
        p = P.generate("c0", 1, rows=7000, cols=14000)
        assert p.a.nonzeros() * 8 > (1 << 20)
        p.a.by_row.index[p.a.nonzeros() - 2] = (1 << 32) + 1
    elif kind == "first_of_many":
        p.var_lower[20], p.var_upper[20] = 3.0, 1.0
        p.var_upper[8] = nan
        p.con_lower[2] = INF
    return p


@pytest.mark.parametrize("kind", ["objective", "var_nan", "var_lo_inf", "var_crossed",
                                  "con_hi_neginf", "con_crossed", "matrix_inf", "layout_value",
                                  "layout_index", "layout_order", "first_of_many"])
def test_validation_messages_match_reference(gpu, ref, kind):
    """validate (problem.hpp:119-154) runs on device; same first failure and
    message as the reference's std::invalid_argument."""
    p = _tamper(kind)
    with pytest.raises(ValueError) as ours:
        P.solve(p)
    with pytest.raises(ValueError) as theirs:
        ref.solve(p)
    assert str(ours.value) == str(theirs.value)


@pytest.mark.parametrize("kind", ["value", "row_swap", "dup_row", "none"])
def test_layout_consistency_rebuild_on_large_layouts(gpu, kind):
    """Layouts of >= 2^20 entries are checked by rebuilding the row form from
    the column form (stable radix sort by row) and comparing position by
    position: a changed value, two rows exchanged inside a column, or a
    column listing one row twice are rejected with the reference's message;
    consistent layouts solve."""
    p = P.generate("c2", 1, rows=100000, cols=200000)
    assert p.a.nonzeros() >= 1 << 20
    C = p.a.by_col
    j = next(j for j in range(p.cols()) if C.start[j + 1] - C.start[j] >= 3)
    k = C.start[j]
    if kind == "value":
        C.value[k + 1] *= 1.0 + 2.0 ** -40
    elif kind == "row_swap":  # two entries of the column trade rows
        C.index[k], C.index[k + 1] = C.index[k + 1], C.index[k]
    elif kind == "dup_row":
        C.index[k + 1] = C.index[k]
    o = P.SolverOptions(mode="perf", iteration_limit=2)
    if kind == "none":
        assert P.solve(p, o).iterations == 2
        return
    with pytest.raises(ValueError, match="row/column layouts disagree"):
        P.solve(p, o)


@pytest.mark.parametrize("kind", ["index_wraps", "index_huge", "index_negative", "start_wraps",
                                  "index_wraps_staged"])
def test_out_of_range_layout_values_are_rejected(gpu, ref, kind):
    """Indices and line starts far outside the problem (beyond int32, where a
    plain narrowing would wrap them into range; negative) are rejected with
    the reference's layout error.  The compiled reference itself indexes with
    such values before validating and crashes, so the expected message is
    the one it gives for an index just past the last column."""
    with pytest.raises(ValueError) as theirs:
        ref.solve(_tamper("layout_index"))
    want = str(theirs.value)
    with pytest.raises(ValueError) as ours:
        P.solve(_tamper(kind))
    assert str(ours.value) == want


def test_perf_mode_deterministic_on_skewed_instance(gpu, ref):
    """Power-law columns put long lines on the chunked warp path (multi-chunk
    lines combine partials in chunk order and write their epilogue terms to
    fixed slots): two perf runs must be bitwise identical, and the iterates
    must track the reference."""
    p = P.generate("c2", 5, rows=5000, cols=6000, kmax=5000)
    assert np.diff(p.a.by_col.start).max() > 2048  # > PDLPK_CHUNK: multi-chunk lines
    o = _opts(iteration_limit=200, tol=(0.0, 0.0, 0.0), mode="perf")
    a, b = P.solve(p, o), P.solve(p, o)
    assert same_bits(a.x, b.x) and same_bits(a.y, b.y)
    assert a.iterations == b.iterations == 200 and a.restarts == b.restarts
    gx, gy = _trace(P.solve, p, _opts(tol=(0.0, 0.0, 0.0), mode="perf"), n_iter=30)
    rx, ry = _trace(ref.solve, p, _opts(tol=(0.0, 0.0, 0.0)), n_iter=30)
    assert max_rel(gx, rx) <= 1e-9 and max_rel(gy, ry) <= 1e-9


# ------------------------------------------- segmented spans / row panels ---
def _skewed_cases():
    rng = np.random.default_rng(77)
    cases = [P.generate("c2", 3, rows=5000, cols=6000, kmax=5000),
             P.generate("c1", 0, sources=40, sinks=50)]
    for _ in range(6):  # small random LPs: empty rows/columns, ragged lines
        cases.append(random_box_lp(rng, 1 + rng.integers(60), 1 + rng.integers(60)))
    return cases


def test_spmv_segmented_spans(gpu, ref, monkeypatch):
    # The segmented-span schedule (spmv.cuh seg_spans: lane-contiguous
    # entries, segmented scan across lanes, chunked long lines, empty lines)
    # forced on every layout; the products must match the reference's.
    monkeypatch.setenv("PDLP_SEG", "1")
    rng = np.random.default_rng(5)
    for p in _skewed_cases():
        x = rng.uniform(-1, 1, p.cols())
        y = rng.uniform(-1, 1, p.rows())
        np.testing.assert_allclose(P.spmv(p, x, mode="perf"), ref.spmv(p, x), rtol=1e-11, atol=1e-9)
        np.testing.assert_allclose(P.spmv_transpose(p, y, mode="perf"), ref.spmv_transpose(p, y),
                                   rtol=1e-11, atol=1e-9)


def test_solve_segmented_spans_tracks_tiles(gpu, ref, monkeypatch):
    # A perf-mode solve with the segmented spans on both layouts reaches the
    # same outcome as with the tile schedule and as the reference.
    p = P.generate("c2", 1, rows=500, cols=1000)
    tol = P.relative_tolerances(p)
    o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=100000)
    monkeypatch.setenv("PDLP_SEG", "0")
    a = P.solve(p, o)
    monkeypatch.setenv("PDLP_SEG", "1")
    b = P.solve(p, o)
    r = ref.solve(p, o)
    assert a.status == b.status == r.status
    for res in (a, b):
        s = res.summary
        assert s.primal_residual_inf <= tol[0] and s.dual_residual_inf <= tol[1]
        assert abs(s.primal_objective - r.summary.primal_objective) <= 1e-3 * (1 + abs(r.summary.primal_objective))


def test_row_panels_bit_identical(gpu, monkeypatch):
    # Column panels chain each row's running sum from panel to panel in
    # storage order, and the step's row-pass reductions are per line
    # (m <= PDLPK_LINE_PARTIALS_MAX): iterates with and without panels are
    # bit-identical.
    p = P.generate("c2", 2, rows=20000, cols=40000, kmax=400)
    assert np.diff(p.a.by_row.start).max() <= 64  # every row in the storage-order tile path
    o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), iteration_limit=300)
    monkeypatch.setenv("PDLP_ROW_PANELS", "0")
    a = P.solve(p, o)
    for np_ in ("2", "3"):
        monkeypatch.setenv("PDLP_ROW_PANELS", np_)
        b = P.solve(p, o)
        assert a.iterations == b.iterations and a.restarts == b.restarts
        assert same_bits(a.x, b.x) and same_bits(a.y, b.y), np_


def test_row_sell_bit_identical(gpu, monkeypatch):
    # The sliced-ELL row pass (PDLP_ROW_SELL=1: lane per row, coalesced
    # slice-column-major streams) adds each row's products in storage order,
    # like the tile path's short lines, and the step's row-pass reductions are
    # per line here (m <= PDLPK_LINE_PARTIALS_MAX): bit-identical iterates,
    # across cadences, restarts and polishing attempts.
    p = P.generate("c2", 2, rows=20000, cols=40000, kmax=400)
    assert np.diff(p.a.by_row.start).max() <= 64  # every row in the storage-order tile path
    tol = P.relative_tolerances(p)
    o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=600)
    monkeypatch.setenv("PDLP_ROW_PANELS", "0")
    a = P.solve(p, o)
    monkeypatch.setenv("PDLP_ROW_SELL", "1")
    b = P.solve(p, o)
    assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
    assert same_bits(a.x, b.x) and same_bits(a.y, b.y)
    assert a.iterations == 600 or a.status == P.SolveStatus.OPTIMAL


def test_multi_vector_cadence_products_bit_identical(gpu, monkeypatch):
    # The cadence's products through one multi-vector pass per layout
    # (k_multi.cu: current + average through K; current + average + the
    # difference and average rays through K') equal the single-vector
    # products on the same span schedules bit for bit, so whole solves are
    # identical with and without them.
    p = P.generate("c2", 3, rows=4000, cols=8000, kmax=3000)
    tol = P.relative_tolerances(p)
    o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=700)
    monkeypatch.setenv("PDLP_SEG", "1")
    monkeypatch.setenv("PDLP_MULTI", "0")
    a = P.solve(p, o)
    monkeypatch.setenv("PDLP_MULTI", "1")
    b = P.solve(p, o)
    assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
    assert same_bits(a.x, b.x) and same_bits(a.y, b.y)
    assert a.restarts > 0  # the cadence (incl. restarts to the average) ran


@pytest.mark.parametrize("mode", ["perf", "parity"])
def test_side_stream_cadence_on_multi_chunk_lines(gpu, monkeypatch, mode):
    # The cadence's window-average share runs on a side stream with its own
    # chunk scratch (chunk partials, arrival counters, line accumulators)
    # while the main stream runs the same kernels on the same layouts.  On
    # a layout with lines cut into several CTA chunks (> 2,048 entries) the
    # overlapped cadence must give the bits of the serial one
    # (PDLP_GAP_SERIAL=1), restart decisions included.
    p = P.generate("c2", 5, rows=5000, cols=6000, kmax=5000)
    assert np.diff(p.a.by_col.start).max() > 2048
    tol = P.relative_tolerances(p)
    o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=1500)
    o.mode = mode
    monkeypatch.setenv("PDLP_SEG", "0")    # tile schedule with chunked lines
    monkeypatch.setenv("PDLP_MULTI", "0")  # single-vector cadence products: the side stream is used
    monkeypatch.setenv("PDLP_GAP_SERIAL", "1")
    a = P.solve(p, o)
    monkeypatch.setenv("PDLP_GAP_SERIAL", "0")
    for _ in range(3):
        b = P.solve(p, o)
        assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
        assert same_bits(a.x, b.x) and same_bits(a.y, b.y)
    assert a.restarts > 0


@pytest.mark.parametrize("knobs", [{"PDLP_ROW_PANELS": "2"}, {"PDLP_ROW_PANELS": "3", "PDLP_SEG": "1"},
                                   {"PDLP_SEG": "1", "PDLP_MULTI": "1"}, {"PDLP_ROW_SELL": "1"}])
def test_forced_schedules_on_ragged_problems(gpu, ref, monkeypatch, knobs):
    # Column panels, segmented spans and multi-vector cadence products forced
    # onto small ragged LPs (empty rows and columns, lines shorter and longer
    # than the tiles): the solves reach the reference's outcome.
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(91)
    cases = [random_box_lp(rng, 30 + rng.integers(40), 30 + rng.integers(60)) for _ in range(4)]
    cases.append(P.generate("c2", 4, rows=1500, cols=3000, kmax=2500))
    for p in cases:
        tol = (1e-7, 1e-7, 1e-8)
        o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=20000)
        g, r = P.solve(p, o), ref.solve(p, o)
        assert g.status == r.status
        if r.status == P.SolveStatus.OPTIMAL:
            assert abs(g.summary.primal_objective - r.summary.primal_objective) <= 1e-5 * (
                1.0 + abs(r.summary.primal_objective))


def test_pinned_problem_and_outputs_solve_identically(gpu):
    """A problem held in page-locked memory (pinned_copy) uploads by DMA with
    its 64-bit indices narrowed on the device, and page-locked result buffers
    are filled by DMA: the solve is the pageable one bit for bit."""
    p = P.generate("c2", 3, rows=60000, cols=120000)  # layouts above the 1 MB direct-copy size
    o = P.SolverOptions(mode="perf", iteration_limit=40,
                        tolerances=P.TerminationTolerances(0.0, 0.0, 0.0))
    a = P.solve(p, o)
    pp = P.pinned_copy(p)
    out = {"x": P.pinned_empty(p.cols()), "y": P.pinned_empty(p.rows()),
           "reduced_costs": P.pinned_empty(p.cols())}
    b = P.solve(pp, o, out=out)
    assert b.x is out["x"]
    assert a.iterations == b.iterations == 40
    assert same_bits(a.x, b.x) and same_bits(a.y, b.y)
    assert same_bits(a.reduced_costs, b.reduced_costs)
