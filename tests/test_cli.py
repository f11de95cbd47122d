"""JSON result documents (solution_io.hpp) and the command line front end
(tools/main.cpp: solve / check / generate, its report lines and exit codes)."""
from __future__ import annotations

import json
import math

import numpy as np
import pytest

import paper_2501_07018_b200 as P
from paper_2501_07018_b200 import cli
from paper_2501_07018_b200 import solution_io as S
from paper_2501_07018_b200.mps import write_mps
from tests.helpers import contradictory_rows, tiny_lp


def _fake_result(**kw):
    base = dict(status=P.SolveStatus.OPTIMAL, x=np.array([1.0, math.inf]), y=np.array([-0.5]),
                reduced_costs=np.array([0.0, math.nan]),
                summary=P.ResidualSummary(1e-9, 2e-9, 3.5, 3.25, 0.25, 0.07),
                certificate=None, iterations=64, polish_iterations=8, restarts=2, step_retries=1,
                final_step_size=0.5, final_primal_weight=math.inf, min_step_size_limit=0.1,
                solve_seconds=0.01, termination_detail="converged at the current iterate")
    base.update(kw)
    return P.SolveResult(**base)


def test_document_round_trip_with_non_finite_values():
    doc = S.make_document(_fake_result(), maximize=True, include_solution=True)
    assert list(doc) == ["schema_version", "status", "termination_detail", "sense", "objective",
                         "residuals", "statistics", "solution"]
    assert doc["objective"]["primal"] == -3.5 and doc["sense"] == "max"
    text = S.solution_to_json(doc)
    raw = json.loads(text)
    assert raw["solution"]["x"][1] == "inf" and raw["solution"]["reduced_costs"][1] == "nan"
    assert raw["statistics"]["final_primal_weight"] == "inf"
    back = S.solution_from_json(text)
    assert back["maximize"] and back["status"] == "optimal"
    assert back["x"][0] == 1.0 and math.isinf(back["x"][1]) and math.isnan(back["reduced_costs"][1])
    assert back["iterations"] == 64 and back["objective_primal"] == -3.5


@pytest.mark.parametrize("text,msg", [
    ("[1, 2]", "top level is not an object"),
    ('{"schema_version": 2, "status": "optimal"}', "unsupported schema_version"),
    ('{"schema_version": 1}', "missing status"),
    ('{"schema_version": 1, "status": "optimal", "solution": {"x": 5, "y": [], "reduced_costs": []}}',
     "solution.x is not an array"),
    ('{"schema_version": 1, "status": "optimal", "objective": {"primal": "big", "dual": 0}}',
     "bad number in objective.primal"),
    ("{not json", "solution file: "),
])
def test_document_errors(text, msg):
    with pytest.raises(ValueError, match=msg):
        S.solution_from_json(text)


def test_generate_writes_a_parsable_model(tmp_path):
    out = tmp_path / "g.mps"
    assert cli.main(["generate", "--kind", "c0", "--rows", "30", "--cols", "50", "--seed", "2",
                     "--out", str(out)]) == 0
    m = P.read_mps(str(out))
    ref = P.generate("c0", 2, rows=30, cols=50)
    np.testing.assert_array_equal(m.problem.objective, ref.objective)
    assert m.name == "c0-30x50-s2"


def test_input_errors_exit_5(tmp_path, capsys):
    bad = tmp_path / "bad.mps"
    bad.write_text("ROWS\n N obj\n Q r\n")
    assert cli.main(["solve", str(bad), "--quiet"]) == 5
    assert "line 3: unknown row type 'Q'" in capsys.readouterr().err
    assert cli.main(["check", str(bad), str(tmp_path / "none.json")]) == 5


@pytest.mark.gpu
def test_solve_then_check(gpu, tmp_path, capsys):
    model = tmp_path / "m.mps"
    model.write_text(write_mps(P.generate("c0", 5, rows=80, cols=160), "m"))
    out = tmp_path / "m.json"
    assert cli.main(["solve", str(model), "--out", str(out), "--quiet", "--eps-primal", "1e-6",
                     "--eps-dual", "1e-6", "--rel-gap", "1e-6"]) == 0
    doc = json.loads(out.read_text())
    assert doc["status"] == "optimal" and len(doc["solution"]["x"]) == 160
    capsys.readouterr()
    assert cli.main(["check", str(model), str(out), "--eps-primal", "1e-6", "--eps-dual", "1e-6",
                     "--rel-gap", "1e-6"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert len(lines) == 4 and all(": ok" in ln for ln in lines)
    # a tampered objective fails the consistency check
    doc["objective"]["primal"] = doc["objective"]["primal"] * 1.5 + 1.0
    out.write_text(json.dumps(doc))
    assert cli.main(["check", str(model), str(out)]) == 1
    assert "reported objective matches: FAIL" in capsys.readouterr().out


@pytest.mark.gpu
def test_infeasible_model_certificate_round_trip(gpu, tmp_path, capsys):
    model = tmp_path / "inf.mps"
    model.write_text(write_mps(contradictory_rows(), "inf"))
    out = tmp_path / "inf.json"
    assert cli.main(["solve", str(model), "--out", str(out), "--quiet", "--no-solution"]) == 2
    doc = json.loads(out.read_text())
    assert doc["status"] == "primal_infeasible" and doc["certificate"]["kind"] == "primal_infeasible"
    capsys.readouterr()
    assert cli.main(["check", str(model), str(out)]) == 0
    assert "primal infeasibility certificate verifies: ok" in capsys.readouterr().out


@pytest.mark.gpu
def test_given_reduced_cost_residuals_match_oracle(gpu, ref):
    p = P.generate("c0", 6, rows=50, cols=90)
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 10, p.cols())
    y = rng.normal(size=p.rows())
    r, want = ref.kkt_residuals(p, x, y)
    got = P.solver.kkt_residuals_given(p, x, y, r)
    for f in ("primal_residual_inf", "dual_residual_inf", "primal_objective", "dual_objective"):
        assert getattr(got, f) == pytest.approx(getattr(want, f), rel=1e-12, abs=1e-12), f


@pytest.mark.gpu
def test_check_certificate_rejects_a_wrong_ray(gpu):
    p = contradictory_rows()
    res = P.solve(p, P.SolverOptions())
    assert res.certificate is not None
    ok, _, _ = P.solver.check_certificate(p, 0, res.certificate.ray_y)
    assert ok
    bad, _, _ = P.solver.check_certificate(p, 0, -res.certificate.ray_y)
    assert not bad
