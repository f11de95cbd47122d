"""MPS reader / writer (the reference's parse_mps / read_mps_file / write_mps,
proj/include/pdhglp/mps.hpp:87-535) over the C-ABI.

    model = parse_mps(text)          # or read_mps(path)
    model.problem                    # LpProblem, minimization form
    model.maximize                   # OBJSENSE MAX was declared (objective negated)
    text = write_mps(problem, "name", maximize=False)

Parse errors raise ValueError with the reference's message ("line N: ..." or
"invalid model: ...").
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .problem import CompressedLayout, LpProblem, SparseMatrix


@dataclass
class MpsModel:
    problem: LpProblem
    maximize: bool = False
    name: str = ""
    objective_name: str = ""
    row_names: list = field(default_factory=list)
    col_names: list = field(default_factory=list)


def _arr(ptr, n, dtype):
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def _layout(v) -> CompressedLayout:
    return CompressedLayout(_arr(v.start, v.primary_dim + 1, np.int64) if v.start else
                            np.zeros(v.primary_dim + 1, np.int64),
                            _arr(v.index, v.nnz, np.int64), _arr(v.value, v.nnz, np.float64))


def model_from_handle(lib, prefix: str, handle) -> MpsModel:
    """Copies a parsed model out of a `<prefix>view`-style handle (used for
    this library and, in the tests, for the reference's parser)."""
    view = N.ProblemView()
    getattr(lib, prefix + "view")(handle, C.byref(view))
    m, n = view.rows, view.cols
    a = SparseMatrix(m, n, _layout(view.by_row), _layout(view.by_col))
    p = LpProblem(a, _arr(view.objective, n, np.float64), _arr(view.con_lower, m, np.float64),
                  _arr(view.con_upper, m, np.float64), _arr(view.var_lower, n, np.float64),
                  _arr(view.var_upper, n, np.float64))
    s = lambda b: b.decode() if b is not None else ""  # noqa: E731
    return MpsModel(p, bool(getattr(lib, prefix + "maximize")(handle)),
                    s(getattr(lib, prefix + "name")(handle)),
                    s(getattr(lib, prefix + "objective_name")(handle)),
                    [s(getattr(lib, prefix + "row_name")(handle, j)) for j in range(m)],
                    [s(getattr(lib, prefix + "col_name")(handle, i)) for i in range(n)])


def parse_mps(text: str | bytes) -> MpsModel:
    lib = N.lib()
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    rc = lib.pdlp_mps_parse(data, len(data), C.byref(h))
    if rc != N.PDLP_OK:
        raise ValueError(N.last_error())
    try:
        return model_from_handle(lib, "pdlp_mps_", h)
    finally:
        lib.pdlp_mps_free(h)


def read_mps(path: str) -> MpsModel:
    lib = N.lib()
    h = C.c_void_p()
    rc = lib.pdlp_mps_read_file(str(path).encode(), C.byref(h))
    if rc != N.PDLP_OK:
        raise ValueError(N.last_error())
    try:
        return model_from_handle(lib, "pdlp_mps_", h)
    finally:
        lib.pdlp_mps_free(h)


def write_text(lib, fn: str, free_fn: str, problem: LpProblem, name: str, maximize: bool) -> str:
    buf, n = C.c_void_p(), C.c_size_t()
    rc = getattr(lib, fn)(C.byref(problem.view()), name.encode(), 1 if maximize else 0,
                          C.byref(buf), C.byref(n))
    if rc != N.PDLP_OK:
        raise RuntimeError(f"{fn} error {rc}")
    try:
        return C.string_at(buf, n.value).decode()
    finally:
        getattr(lib, free_fn)(buf)


def write_mps(problem: LpProblem, name: str = "", maximize: bool = False) -> str:
    """write_mps: a minimization-form problem as free MPS (OBJ / R# / C#
    names; with maximize the file declares OBJSENSE MAX and stores -c)."""
    return write_text(N.lib(), "pdlp_mps_write", "pdlp_mps_free_text", problem, name, maximize)


def write_mps_file(path: str, problem: LpProblem, name: str = "", maximize: bool = False) -> None:
    with open(path, "w") as f:
        f.write(write_mps(problem, name, maximize))
