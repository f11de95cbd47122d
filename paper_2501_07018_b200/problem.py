"""LP data model mirroring the reference structs.

    CompressedLayout  <- pdhglp::CompressedLayout (proj/include/pdhglp/sparse.hpp:21-28)
    SparseMatrix      <- pdhglp::SparseMatrix     (sparse.hpp:33-42, from_triplets :107-115)
    LpProblem         <- pdhglp::LpProblem        (problem.hpp:15-25)

Arrays are numpy (int64 indices, float64 values, as in the reference); the
solver copies them to HBM once per solve.  Instances from the seeded
generators (libpdlp_gen.so) are zero-copy views into generator-owned memory.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

INF = float("inf")


@dataclass
class CompressedLayout:
    start: np.ndarray
    index: np.ndarray
    value: np.ndarray

    def primary_dim(self) -> int:
        return int(self.start.shape[0]) - 1

    def nonzeros(self) -> int:
        return int(self.value.shape[0])


@dataclass
class SparseMatrix:
    rows: int
    cols: int
    by_row: CompressedLayout
    by_col: CompressedLayout

    def nonzeros(self) -> int:
        return self.by_row.nonzeros()

    @staticmethod
    def from_triplets(rows: int, cols: int, triplets) -> "SparseMatrix":
        """reference SparseMatrix::from_triplets (sparse.hpp:107-115): lines
        sorted by secondary index, duplicates summed in input order."""
        if len(triplets) == 0:
            r = np.zeros(0, np.int64)
            c = np.zeros(0, np.int64)
            v = np.zeros(0, np.float64)
        else:
            r = np.ascontiguousarray([t[0] for t in triplets], dtype=np.int64)
            c = np.ascontiguousarray([t[1] for t in triplets], dtype=np.int64)
            v = np.ascontiguousarray([t[2] for t in triplets], dtype=np.float64)
        return SparseMatrix.from_arrays(rows, cols, r, c, v)

    @staticmethod
    def from_arrays(rows: int, cols: int, r, c, v) -> "SparseMatrix":
        r = np.ascontiguousarray(r, dtype=np.int64)
        c = np.ascontiguousarray(c, dtype=np.int64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        zc = np.zeros(cols, np.float64)
        zr = np.zeros(rows, np.float64)
        h = N.gen().pdlp_instance_from_triplets(
            rows, cols, r.shape[0], _p64(r), _p64(c), _pd(v), _pd(zc), _pd(zr), _pd(zr),
            _pd(zc), _pd(zc))
        if not h:
            raise ValueError("triplet index out of range")
        try:
            view = N.ProblemView()
            N.gen().pdlp_instance_view(h, C.byref(view))
            return SparseMatrix(rows, cols, _copy_layout(view.by_row), _copy_layout(view.by_col))
        finally:
            N.gen().pdlp_instance_free(h)


@dataclass
class LpProblem:
    a: SparseMatrix
    objective: np.ndarray
    con_lower: np.ndarray
    con_upper: np.ndarray
    var_lower: np.ndarray
    var_upper: np.ndarray
    _owner: object = field(default=None, repr=False, compare=False)

    def rows(self) -> int:
        return self.a.rows

    def cols(self) -> int:
        return self.a.cols

    def view(self) -> N.ProblemView:
        """A pdlp_problem_view over this problem's arrays (borrowed)."""
        for name in ("objective", "con_lower", "con_upper", "var_lower", "var_upper"):
            arr = getattr(self, name)
            if not (isinstance(arr, np.ndarray) and arr.dtype == np.float64 and arr.flags.c_contiguous):
                setattr(self, name, np.ascontiguousarray(arr, dtype=np.float64))
        if self.objective.shape[0] != self.cols():
            raise ValueError("invalid problem: objective length != cols (index -1)")
        if self.con_lower.shape[0] != self.rows():
            raise ValueError("invalid problem: con_lower length != rows (index -1)")
        if self.con_upper.shape[0] != self.rows():
            raise ValueError("invalid problem: con_upper length != rows (index -1)")
        if self.var_lower.shape[0] != self.cols():
            raise ValueError("invalid problem: var_lower length != cols (index -1)")
        if self.var_upper.shape[0] != self.cols():
            raise ValueError("invalid problem: var_upper length != cols (index -1)")
        v = N.ProblemView()
        v.rows = self.rows()
        v.cols = self.cols()
        v.by_row = _layout_view(self.a.by_row)
        v.by_col = _layout_view(self.a.by_col)
        v.objective = _pd(self.objective)
        v.con_lower = _pd(self.con_lower)
        v.con_upper = _pd(self.con_upper)
        v.var_lower = _pd(self.var_lower)
        v.var_upper = _pd(self.var_upper)
        return v

    def copy(self) -> "LpProblem":
        lay = lambda L: CompressedLayout(L.start.copy(), L.index.copy(), L.value.copy())
        return LpProblem(SparseMatrix(self.a.rows, self.a.cols, lay(self.a.by_row), lay(self.a.by_col)),
                         self.objective.copy(), self.con_lower.copy(), self.con_upper.copy(),
                         self.var_lower.copy(), self.var_upper.copy())


def problem(rows, cols, triplets, objective, con_lower, con_upper, var_lower, var_upper) -> LpProblem:
    f = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    return LpProblem(SparseMatrix.from_triplets(rows, cols, triplets), f(objective), f(con_lower),
                     f(con_upper), f(var_lower), f(var_upper))


# ------------------------------------------------------------------ helpers ---
def _pd(a: np.ndarray):
    return a.ctypes.data_as(N.c_double_p)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(N.c_int64_p)


def _layout_view(L: CompressedLayout) -> N.CsrView:
    for name, dt in (("start", np.int64), ("index", np.int64), ("value", np.float64)):
        arr = getattr(L, name)
        if not (arr.dtype == dt and arr.flags.c_contiguous):
            setattr(L, name, np.ascontiguousarray(arr, dtype=dt))
    v = N.CsrView()
    v.primary_dim = L.primary_dim()
    v.nnz = L.nonzeros()
    v.start = _p64(L.start)
    v.index = _p64(L.index)
    v.value = _pd(L.value)
    return v


def _as_array(ptr, n: int, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).view(dtype)


def _copy_layout(v: N.CsrView) -> CompressedLayout:
    return CompressedLayout(_as_array(v.start, v.primary_dim + 1, np.int64).copy(),
                            _as_array(v.index, v.nnz, np.int64).copy(),
                            _as_array(v.value, v.nnz, np.float64).copy())


class _Instance:
    """Owns a generator instance; frees it when the last view goes away."""

    def __init__(self, handle):
        if not handle:
            raise ValueError("instance generation failed")
        self.handle = handle

    def __del__(self):
        if getattr(self, "handle", None):
            N.gen().pdlp_instance_free(self.handle)
            self.handle = None


def _wrap(handle) -> tuple[LpProblem, np.ndarray | None]:
    inst = _Instance(handle)
    v = N.ProblemView()
    N.gen().pdlp_instance_view(inst.handle, C.byref(v))
    lay = lambda L: CompressedLayout(_as_array(L.start, L.primary_dim + 1, np.int64),
                                     _as_array(L.index, L.nnz, np.int64),
                                     _as_array(L.value, L.nnz, np.float64))
    m, n = v.rows, v.cols
    p = LpProblem(SparseMatrix(m, n, lay(v.by_row), lay(v.by_col)),
                  _as_array(v.objective, n, np.float64), _as_array(v.con_lower, m, np.float64),
                  _as_array(v.con_upper, m, np.float64), _as_array(v.var_lower, n, np.float64),
                  _as_array(v.var_upper, n, np.float64), _owner=inst)
    fp = N.gen().pdlp_instance_feasible_point(inst.handle)
    feas = _as_array(fp, n, np.float64) if fp else None
    return p, feas


def generate(config: str, seed: int = 0, **overrides) -> LpProblem:
    """Seeded instance for a BASELINE.json config ('c0'..'c4'); size
    overrides (rows/cols, sources/sinks, periods/generators) give scaled-down
    members of the same family for parity tests."""
    return generate_with_point(config, seed, **overrides)[0]


def generate_with_point(config: str, seed: int = 0, **overrides):
    g = N.gen()
    cfg = config.lower()
    if cfg in ("c0", "c2", "c4"):
        prm = N.GenParams()
        getattr(g, f"pdlp_gen_{cfg}_params")(C.byref(prm), seed)
        window = overrides.pop("row_window", None)
        for k, val in overrides.items():
            setattr(prm, k, val)
        if window is not None:
            # rows [r0, r1) as a standalone LP (counter-based streams, threaded)
            r0, r1 = window
            return _wrap(g.pdlp_gen_random_lp_window(C.byref(prm), int(r0), int(r1)))
        return _wrap(g.pdlp_gen_random_lp(C.byref(prm)))
    if cfg in ("c1", "transport"):
        return _wrap(g.pdlp_gen_transport(overrides.get("sources", 2000),
                                          overrides.get("sinks", 2000), seed))
    if cfg == "c3":
        return _wrap(g.pdlp_gen_unit_commitment(overrides.get("periods", 8760),
                                                overrides.get("generators", 1000), seed))
    raise ValueError(f"unknown config {config!r}")


def relative_tolerances(p: LpProblem, eps: float = 1e-4) -> tuple[float, float, float]:
    """BASELINE '1e-4 relative KKT' mapped onto the reference's absolute
    tolerances: eps_primal = eps (1 + max finite |l_c, u_c|),
    eps_dual = eps (1 + |c|_inf), eps_rel_gap = eps."""
    b = np.concatenate([p.con_lower, p.con_upper])
    b = b[np.isfinite(b)]
    bmax = float(np.max(np.abs(b))) if b.size else 0.0
    cmax = float(np.max(np.abs(p.objective))) if p.objective.size else 0.0
    return eps * (1.0 + bmax), eps * (1.0 + cmax), eps


# On-disk form of an LpProblem: one .npy per array plus the shape, so a large
# seeded instance is generated once and memory-mapped by later processes (the
# bench's reference arm reads it without importing this package).
_ARRAYS = ("row_start", "row_index", "row_value", "col_start", "col_index", "col_value",
           "objective", "con_lower", "con_upper", "var_lower", "var_upper")


def save_problem(p: LpProblem, path: str) -> None:
    import json
    import os
    os.makedirs(path, exist_ok=True)
    arrs = (p.a.by_row.start, p.a.by_row.index, p.a.by_row.value, p.a.by_col.start,
            p.a.by_col.index, p.a.by_col.value, p.objective, p.con_lower, p.con_upper,
            p.var_lower, p.var_upper)
    for name, a in zip(_ARRAYS, arrs):
        np.save(os.path.join(path, name + ".npy"), np.ascontiguousarray(a))
    with open(os.path.join(path, "shape.json"), "w") as f:
        json.dump({"rows": p.rows(), "cols": p.cols(), "nnz": p.a.nonzeros()}, f)


def load_problem(path: str) -> LpProblem:
    """Memory-mapped, read-only arrays (the solver only reads its inputs)."""
    import json
    import os
    with open(os.path.join(path, "shape.json")) as f:
        shape = json.load(f)
    a = {name: np.load(os.path.join(path, name + ".npy"), mmap_mode="r") for name in _ARRAYS}
    return LpProblem(
        SparseMatrix(shape["rows"], shape["cols"],
                     CompressedLayout(a["row_start"], a["row_index"], a["row_value"]),
                     CompressedLayout(a["col_start"], a["col_index"], a["col_value"])),
        a["objective"], a["con_lower"], a["con_upper"], a["var_lower"], a["var_upper"])
