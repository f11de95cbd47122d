"""MPS reader / writer against the reference's own parse_mps /
write_mps (proj/include/pdhglp/mps.hpp, compiled in oracle/_ref): the same
model, the same error messages, byte-identical output; round trips of the
seeded instances; a GPU solve from an MPS model."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2501_07018_b200 as P
from paper_2501_07018_b200 import mps as M
from tests.helpers import random_box_lp

# Handcrafted models (own content) exercising every section and rule.
MODELS = {
    "all-row-kinds": """NAME kinds
ROWS
 N cost
 L cap
 G need
 E bal
 N spare
COLUMNS
 x cost 1.5 cap 2
 x need 1 bal -1
 y cost -2 cap 1
 y spare 4
 z bal 3
RHS
 rhs cap 10 need 2
 rhs bal 1.5
 rhs spare 99
ENDATA
""",
    "ranges-and-bounds": """NAME rb
ROWS
 N obj
 L r1
 G r2
 E r3
 E r4
COLUMNS
 a obj 1 r1 1
 a r2 1 r3 2
 b obj -1 r1 3
 b r4 1
 c obj 2 r2 -1
 d obj 0 r3 1
 e obj 1 r4 2
RHS
 B r1 8 r2 1
 B r3 4 r4 -2
RANGES
 R r1 2.5 r2 -3
 R r3 1.5
 R r4 -0.5
BOUNDS
 UP BND a -2
 LO BND b -1
 UP BND b 5
 FX BND c 3.25
 FR BND d
 MI BND e
 PL BND e
ENDATA
""",
    "set-names-omitted": """NAME nos
ROWS
 N obj
 L r1
 G r2
COLUMNS
 x obj 1 r1 1
 x r2 1
 y obj 1 r1 1
RHS
 r1 4 r2 1
RANGES
 r2 2
BOUNDS
 UP x 3
 FR y
ENDATA
""",
    "max-inline": """NAME m
OBJSENSE MAX
ROWS
 N obj
 L r
COLUMNS
 x obj 3 r 1
 y obj 2 r 1
RHS
 rhs r 4
ENDATA
""",
    "max-next-line": """NAME m2
OBJSENSE
    MAXIMIZE
ROWS
 N obj
 L r
COLUMNS
 x obj 3 r 1
RHS
 rhs r 4
ENDATA
""",
    "duplicates-and-comments": """* a comment
NAME dup

ROWS
 N obj
 L r1
COLUMNS
* another comment
 x obj 1 r1 1
 x r1 2
 x obj 0.5
 y r1 1 obj 1
RHS
 rhs r1 5
ENDATA
""",
    "bounds-three-token-forms": """NAME b3
ROWS
 N obj
 L r
COLUMNS
 x obj 1 r 1
 y obj 1 r 1
 z obj 1 r 1
RHS
 rhs r 1
BOUNDS
 FR BND x
 MI y 0
 PL BND z
 LO BND z -4
ENDATA
""",
    "negative-up-after-lo": """NAME nu
ROWS
 N obj
 L r
COLUMNS
 x obj 1 r 1
 y obj 1 r 1
RHS
 rhs r 1
BOUNDS
 LO BND x -5
 UP BND x -1
 UP BND y -3
ENDATA
""",
    "crlf-and-tabs": "NAME\tcr\r\nROWS\r\n N\tobj\r\n G\tg1\r\nCOLUMNS\r\n\tx\tobj\t2\tg1\t1\r\nRHS\r\n\trhs\tg1\t3\r\nENDATA\r\n",
    "markers-intend-only": """NAME mk
ROWS
 N obj
 L r
COLUMNS
 MARK1 'MARKER' 'INTEND'
 x obj 1 r 1
RHS
 rhs r 2
ENDATA
""",
}

BROKEN = [
    "ROWS\n N obj\nCOLUMNS\n x obj 1\nfoo\n",
    " x obj 1\n",
    "NAME a\n x\n",
    "NAME a\nCOLUMNS\n",
    "ROWS\n N obj\n Q r\n",
    "ROWS\n N obj\n L r\n L r\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x obj 1 q 2\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x obj abc\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x obj 1 r\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n M 'MARKER' 'INTORG'\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n M 'MARKER' 'WHAT'\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nRHS\n rhs r\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nRANGES\n R obj 1\n",
    "ROWS\n N obj\n N f\n L r\nCOLUMNS\n x r 1\nRANGES\n R f 1\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nBOUNDS\n BV BND x\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nBOUNDS\n XX BND x 1\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nBOUNDS\n UP BND w 1\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nBOUNDS\n UP BND x\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nBOUNDS\n UP\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nSOS\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nWEIRD\n",
    "OBJSENSE\n",
    "OBJSENSE SIDEWAYS\n",
    "NAME x\n",
    "ROWS\n L r\nCOLUMNS\n x r 1\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r 1\nBOUNDS\n LO BND x 5\n UP BND x 1\nENDATA\n",
    "ROWS\n N obj\n L r\nCOLUMNS\n x r nan\nENDATA\n",
]


def _same(a: M.MpsModel, b: M.MpsModel):
    pa, pb = a.problem, b.problem
    for f in ("objective", "con_lower", "con_upper", "var_lower", "var_upper"):
        np.testing.assert_array_equal(getattr(pa, f), getattr(pb, f), err_msg=f)
    for side in ("by_row", "by_col"):
        la, lb = getattr(pa.a, side), getattr(pb.a, side)
        np.testing.assert_array_equal(la.start, lb.start)
        np.testing.assert_array_equal(la.index, lb.index)
        np.testing.assert_array_equal(la.value.view(np.int64), lb.value.view(np.int64))
    assert (a.maximize, a.name, a.objective_name) == (b.maximize, b.name, b.objective_name)
    assert a.row_names == b.row_names and a.col_names == b.col_names


@pytest.fixture(scope="module")
def refmps():
    import oracle
    try:
        return oracle.reference()
    except FileNotFoundError:
        pytest.skip("compiled reference (oracle/_ref) not built")


@pytest.mark.parametrize("name", sorted(MODELS))
def test_parse_matches_reference(refmps, name):
    _same(M.parse_mps(MODELS[name]), refmps.parse_mps(MODELS[name]))


@pytest.mark.parametrize("text", BROKEN)
def test_errors_match_reference(refmps, text):
    with pytest.raises(ValueError) as ours:
        M.parse_mps(text)
    with pytest.raises(ValueError) as theirs:
        refmps.parse_mps(text)
    assert str(ours.value) == str(theirs.value)


def _instances():
    rng = np.random.default_rng(11)
    yield P.generate("c0", 1, rows=60, cols=90)
    yield P.generate("c1", 2, sources=7, sinks=9)
    yield P.generate("c2", 3, rows=40, cols=80, kmax=30)
    yield P.generate("c3", 4, periods=6, generators=5)
    yield random_box_lp(rng, 25, 35)


@pytest.mark.parametrize("maximize", [False, True])
def test_writer_is_byte_identical(refmps, maximize):
    for p in _instances():
        assert M.write_mps(p, "inst", maximize) == refmps.write_mps(p, "inst", maximize)


@pytest.mark.parametrize("maximize", [False, True])
def test_round_trip_reproduces_the_problem(maximize, tmp_path):
    for k, p in enumerate(_instances()):
        path = tmp_path / f"p{k}.mps"
        M.write_mps_file(str(path), p, f"p{k}", maximize)
        back = M.read_mps(str(path))
        assert back.maximize == maximize
        for f in ("objective", "con_lower", "con_upper", "var_lower", "var_upper"):
            np.testing.assert_array_equal(getattr(back.problem, f), getattr(p, f))
        np.testing.assert_array_equal(back.problem.a.by_row.value, p.a.by_row.value)
        np.testing.assert_array_equal(back.problem.a.by_col.index, p.a.by_col.index)


def test_missing_file_is_reported():
    with pytest.raises(ValueError, match="cannot open"):
        M.read_mps("/nonexistent/model.mps")


@pytest.mark.gpu
def test_gpu_solve_from_mps_matches_oracle(gpu, refmps):
    model = M.parse_mps(MODELS["ranges-and-bounds"])
    o = P.SolverOptions(tolerances=P.TerminationTolerances(1e-8, 1e-8, 1e-6), mode="parity")
    g = P.solve(model.problem, o)
    r = refmps.solve(model.problem, o)
    assert g.status == r.status
    assert g.iterations == r.iterations
    np.testing.assert_array_equal(g.x.view(np.int64), r.x.view(np.int64))
