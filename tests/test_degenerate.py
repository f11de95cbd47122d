"""Degenerate shapes (no rows, empty rows / columns, single entries) solve
like the reference on the GPU, in both modes."""
import numpy as np
import pytest

import paper_2501_07018_b200 as P
from paper_2501_07018_b200.problem import problem

INF = np.inf
CASES = {
    # min x1 - x2 with bounds only (no constraints)
    "no-rows": lambda: problem(0, 2, [], [1.0, -1.0], [], [], [0.0, -3.0], [2.0, 4.0]),
    # an all-zero row and a column that appears in no row
    "empty-row-and-col": lambda: problem(2, 3, [(1, 0, 1.0), (1, 2, 2.0)], [1.0, 0.5, -1.0],
                                         [-INF, 1.0], [5.0, 6.0], [0.0, 0.0, 0.0], [10.0, 1.0, 10.0]),
    # a single variable and a single equality
    "one-by-one": lambda: problem(1, 1, [(0, 0, 2.0)], [3.0], [4.0], [4.0], [-INF], [INF]),
    # free variables only
    "free-vars": lambda: problem(2, 2, [(0, 0, 1.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, -1.0)],
                                 [1.0, 2.0], [1.0, -1.0], [1.0, -1.0], [-INF, -INF], [INF, INF]),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("mode", ["parity", "perf"])
def test_degenerate_shapes_match_reference(gpu, ref, name, mode):
    p = CASES[name]()
    o = P.SolverOptions(tolerances=P.TerminationTolerances(1e-8, 1e-8, 1e-6), mode=mode,
                        iteration_limit=20000)
    g = P.solve(p, o)
    r = ref.solve(p, o)
    assert g.status == r.status, (g.termination_detail, r.termination_detail)
    if r.status == P.SolveStatus.OPTIMAL:
        np.testing.assert_allclose(g.x, r.x, rtol=1e-6, atol=1e-6)
        assert g.summary.primal_objective == pytest.approx(r.summary.primal_objective, rel=1e-6, abs=1e-6)
    if mode == "parity":
        assert g.iterations == r.iterations
