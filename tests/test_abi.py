"""CPU-only checks of the C-ABI boundary: the libraries load and export every
symbol include/*.h declares; the host logic that needs no device behaves.
No compute calls reach the GPU here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2501_07018_b200 as P
from paper_2501_07018_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header: str) -> list[str]:
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pdlp_[a-z0-9_]+)\s*\(", text)))


def _exported(path: str) -> set[str]:
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_solver_library_exports_header():
    names = _declared("pdlp_b200.h")
    assert "pdlp_solve" in names and len(names) >= 10
    exported = _exported(N.LIB_PATH)
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = N.lib()
    for n in names:
        assert getattr(lib, n) is not None
    assert lib.pdlp_abi_version() == 1


def test_generator_library_exports_header():
    names = _declared("pdlp_gen.h")
    exported = _exported(N.GEN_LIB_PATH)
    assert not [n for n in names if n not in exported]


def test_sm100a_code_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_default_options_match_reference():
    o = N.Options()
    N.lib().pdlp_default_options(C.byref(o))
    d = P.SolverOptions()
    assert (o.eps_primal, o.eps_dual, o.eps_rel_gap) == (1e-8, 1e-8, 1e-2)
    assert o.iteration_limit == d.iteration_limit == 200000
    assert o.threads == 1 and o.shards_per_thread == 4 and o.check_interval == 64
    assert o.ruiz_passes == 10 and o.pock_chambolle == 1 and o.eps_ray == 1e-12
    assert (o.restart_sufficient, o.restart_necessary, o.restart_artificial) == (0.1, 0.9, 0.5)


def test_host_step_rules_known_answers():
    # test_step.cpp:173-196 (host scalar rules; no device needed)
    lim, _ = P.step_size_rules(2.0, 0.5, 1.0, 1.0, 0)
    assert lim == 2.0
    assert P.step_size_rules(1.0, 0.0, 1.0, 1.0, 0)[0] == float("inf")
    assert P.step_size_rules(1.0, -3.0, 1.0, 1.0, 0)[0] == 1.0 / 6.0
    _, nxt = P.step_size_rules(0, 0, 1.0, 1.0, 9)
    assert nxt == pytest.approx(0.4988127663727278, rel=1e-15)
    _, grown = P.step_size_rules(0, 0, 100.0, 1.0, 9)
    assert grown == pytest.approx(1.0 + 10.0 ** -0.6, rel=1e-15)


def test_from_triplets_semantics():
    # duplicates summed in input order, lines sorted (sparse.hpp:48-103)
    a = P.SparseMatrix.from_triplets(2, 3, [(1, 2, 1.0), (0, 1, 2.0), (1, 0, 3.0), (1, 2, 0.5)])
    assert a.by_row.start.tolist() == [0, 1, 3]
    assert a.by_row.index.tolist() == [1, 0, 2]
    assert a.by_row.value.tolist() == [2.0, 3.0, 1.5]
    assert a.by_col.start.tolist() == [0, 1, 2, 3]
    assert a.by_col.index.tolist() == [1, 0, 1]


@pytest.mark.parametrize("cfg,kw", [("c0", {}), ("c1", dict(sources=40, sinks=50)),
                                    ("c2", dict(rows=2000, cols=4000)),
                                    ("c3", dict(periods=24, generators=10))])
def test_generators_are_valid_and_deterministic(cfg, kw):
    p1, feas = P.generate_with_point(cfg, 7, **kw)
    p2 = P.generate(cfg, 7, **kw)
    assert np.array_equal(p1.a.by_row.value, p2.a.by_row.value)
    assert np.array_equal(p1.objective, p2.objective)
    # both layouts describe the same matrix
    A = np.zeros((p1.rows(), p1.cols()))
    L = p1.a.by_row
    rows = np.repeat(np.arange(p1.rows()), np.diff(L.start))
    A[rows, L.index] = L.value
    Lc = p1.a.by_col
    cols = np.repeat(np.arange(p1.cols()), np.diff(Lc.start))
    assert np.array_equal(A[Lc.index, cols], Lc.value)
    # the construction point is feasible
    if feas is not None:
        ax = A @ feas
        scale = 1.0 + np.abs(ax).max()
        assert np.all(ax >= p1.con_lower - 1e-9 * scale)
        assert np.all(ax <= p1.con_upper + 1e-9 * scale)
        assert np.all(feas >= p1.var_lower) and np.all(feas <= p1.var_upper)


def test_c1_shape():
    p = P.generate("c1", 0, sources=20, sinks=30)
    assert p.rows() == 50 and p.cols() == 600 and p.a.nonzeros() == 1200
    assert np.all(p.a.by_row.value == 1.0)
