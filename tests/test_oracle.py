"""CPU: the oracle restatement (oracle/pdlp_oracle.cpp) pinned against the
compiled reference (oracle/_ref) and the reference's own known-answer tests
(proj/tests/*.cpp, cited per case), plus the committed golden fixtures."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import paper_2501_07018_b200 as P
from tests.helpers import (INF, box_interior_point, clamp_free_row, contradictory_rows,
                           equality_lp, one_var_equality, random_box_lp, rejection_lp, same_bits,
                           slack_row_box_lp, tiny_lp, unbounded_lp)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def port():
    if not oracle.have_port():
        oracle.build(with_reference=False)
    return oracle.port()


def test_known_answers(port):
    # test_step.cpp:116-148
    x, y = port.pdhg_step(one_var_equality(), [0.0], [0.0], 1.0, 0.5)
    assert x[0] == 0.0 and y[0] == 0.5
    x, y = port.pdhg_step(clamp_free_row(), [3.0], [0.0, 5.0], 1.0, 1.0)
    assert (x[0], y[0], y[1]) == (3.0, -1.0, 0.0)
    # test_step.cpp:173-196
    assert port.step_size_rules(2.0, 0.5, 1, 1, 0)[0] == 2.0
    assert port.step_size_rules(1.0, -3.0, 1, 1, 0)[0] == 1.0 / 6.0
    assert port.step_size_rules(0, 0, 1.0, 1.0, 9)[1] == pytest.approx(0.4988127663727278, rel=1e-15)
    # test_step.cpp:274-304
    out = port.adaptive_step(rejection_lp(), [0.0], [1.0], [1.0], eta_hat=4.0)
    assert out["retries"] == 1 and out["min_eta_bar"] == 1.25
    assert out["eta_used"] == pytest.approx((1 - 2 ** -0.3) * 1.25, rel=1e-15)
    # test_restarts.cpp:310-335 (omega init)
    p = P.problem(1, 2, [(0, 0, 1.0), (0, 1, 1.0)], [3.0, 4.0], [-INF], [2.0], [-INF, -INF], [INF, INF])
    assert port.initialize_primal_weight(p) == pytest.approx(2.5, rel=1e-15)
    # test_rescaling.cpp:35-57
    d = P.problem(2, 2, [(0, 0, 4.0), (1, 1, 9.0)], [1, 1], [-1, -1], [1, 1], [0, 0], [2, 2])
    s = port.apply_rescaling(d, 1, False)
    assert s["row_values"].tolist() == [1.0, 1.0] and s["row_scale"].tolist() == [0.5, 1 / 3]
    pc = P.problem(2, 2, [(0, 0, 1.0), (0, 1, 1.0), (1, 1, 2.0)], [1, 1], [-1, -1], [1, 1], [0, 0], [2, 2])
    s = port.apply_rescaling(pc, 0, True)
    assert s["row_values"] == pytest.approx([1 / math.sqrt(2), 1 / math.sqrt(6), 2 / math.sqrt(6)], rel=1e-15)
    # test_residuals.cpp:49-69
    r, s = port.kkt_residuals(tiny_lp(), [0.0, 1.0], [-2.0])
    assert r.tolist() == [1.0, 0.0] and s.primal_residual_inf == 0.0 and s.rel_gap == 0.0
    _, s = port.kkt_residuals(tiny_lp(), [0.0, 1.0], [1.0])
    assert s.dual_objective == -INF and s.rel_gap == INF
    # test_solver.cpp:54-84
    out = port.solve(tiny_lp(), P.SolverOptions(tolerances=P.TerminationTolerances(1e-8, 1e-8, 1e-9)))
    assert out.status == 0 and out.x == pytest.approx([0, 1], abs=1e-6)
    assert port.solve(contradictory_rows()).status == P.SolveStatus.PRIMAL_INFEASIBLE
    assert port.solve(unbounded_lp()).status == P.SolveStatus.DUAL_INFEASIBLE


def _same(a, b):
    assert a.status == b.status and a.iterations == b.iterations
    assert a.polish_iterations == b.polish_iterations and a.restarts == b.restarts
    assert a.termination_detail == b.termination_detail
    assert same_bits(a.x, b.x) and same_bits(a.y, b.y) and same_bits(a.reduced_costs, b.reduced_costs)


@pytest.mark.skipif(not oracle.have_reference(), reason="reference library not built")
def test_port_matches_reference_bitwise(port):
    R = oracle.reference()
    rng = np.random.default_rng(5)
    for _ in range(10):
        p = random_box_lp(rng, 1 + rng.integers(8), 1 + rng.integers(8))
        x = box_interior_point(rng, p)
        y = rng.uniform(-1, 1, p.rows())
        a, b = port.pdhg_step(p, x, y, 1.3, 0.4), R.pdhg_step(p, x, y, 1.3, 0.4)
        assert (a is None) == (b is None)
        if a is not None:
            assert same_bits(a[0], b[0]) and same_bits(a[1], b[1])
        aty = R.spmv_transpose(p, y)
        for kk in ("x", "y", "aty", "prev_x", "eta_hat", "min_eta_bar"):
            assert same_bits(port.adaptive_step(p, x, y, aty, 0.9, k=3)[kk],
                             R.adaptive_step(p, x, y, aty, 0.9, k=3)[kk])
        ax = R.spmv(p, x)
        for r in (0.3, 2.0):
            assert same_bits(port.normalized_duality_gap(p, x, y, ax, aty, 0.7, r),
                             R.normalized_duality_gap(p, x, y, ax, aty, 0.7, r))
    for p in (P.generate("c0", 0, rows=300, cols=600), P.generate("c2", 2, rows=400, cols=800)):
        a, b = port.apply_rescaling(p), R.apply_rescaling(p)
        assert all(same_bits(a[k], b[k]) for k in a)
    c0 = P.generate("c0", 0)
    cases = [(c0, P.relative_tolerances(c0))] + [
        (p, (1e-8, 1e-8, 1e-9)) for p in (
            tiny_lp(), contradictory_rows(), unbounded_lp(),
            equality_lp(np.random.default_rng(11), 20, 30), P.generate("c1", 1, sources=8, sinks=9),
            slack_row_box_lp(np.random.default_rng(7), 6, 9))]
    for p, tol in cases:
        for spt in (4, 16):
            o = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), shards_per_thread=spt)
            _same(port.solve(p, o), R.solve(p, o))
    p = equality_lp(np.random.default_rng(11), 20, 30)
    o = P.SolverOptions(tolerances=P.TerminationTolerances(1e-11, 1e-6, 0.5))
    _same(port.solve(p, o), R.solve(p, o))


def test_port_matches_golden(port):
    """Fixtures made by tests/golden/make_golden.py from the compiled reference."""
    path = os.path.join(GOLDEN, "golden.npz")
    if not os.path.exists(path):
        pytest.skip("golden fixtures not generated")
    g = np.load(path)
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))
    for name, info in meta["solves"].items():
        p = P.generate(info["config"], info["seed"], **info["size"])
        o = P.SolverOptions(tolerances=P.TerminationTolerances(*info["tol"]),
                            iteration_limit=info["iteration_limit"])
        out = port.solve(p, o)
        assert out.iterations == info["iterations"] and out.restarts == info["restarts"]
        assert int(out.status) == info["status"]
        assert same_bits(out.x, g[name + "_x"]) and same_bits(out.y, g[name + "_y"])
