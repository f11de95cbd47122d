"""Row-window instances (a row shard of a large instance as a
standalone LP, without building the whole instance)."""
import numpy as np
import pytest

import paper_2501_07018_b200 as P
from tests.helpers import dense


def test_window_rows_are_rows_of_the_full_window():
    full = P.generate("c0", 4, row_window=(0, 1000))
    part = P.generate("c0", 4, row_window=(250, 640))
    assert part.rows() == 390 and part.cols() == full.cols()
    np.testing.assert_array_equal(dense(part), dense(full)[250:640])
    # per-column / per-row streams: bounds and equality pattern agree too
    np.testing.assert_array_equal(part.var_lower, full.var_lower)
    np.testing.assert_array_equal(np.isinf(part.con_lower), np.isinf(full.con_lower[250:640]))


def test_window_lp_is_feasible_and_bounded(ref):
    p, xs = P.generate_with_point("c2", 1, rows=600, cols=1200, kmax=400, row_window=(100, 400))
    a = dense(p)
    ax = a @ xs
    assert np.all(ax >= p.con_lower - 1e-9) and np.all(ax <= p.con_upper + 1e-9)
    assert np.all(xs >= p.var_lower) and np.all(xs <= p.var_upper)
    # bounded: the C0 family (box variables) solves to optimality by the oracle
    q = P.generate("c0", 2, row_window=(200, 700))
    tol = P.relative_tolerances(q)
    r = ref.solve(q, P.SolverOptions(tolerances=P.TerminationTolerances(*tol)))
    assert r.status == P.SolveStatus.OPTIMAL


@pytest.mark.parametrize("window", [(0, 0), (-1, 5), (10, 5), (0, 10**9)])
def test_window_rejects_bad_ranges(window):
    with pytest.raises(Exception):
        P.generate("c0", 0, row_window=window)
