"""TEST INFRASTRUCTURE — the bench's reference arm (bench.py --impl reference
and the cpu_baseline leg).  Loaded by file path (not through oracle/__init__),
so the process that runs it maps exactly one native library of this repo:
oracle/_ref/libpdhglp_ref.so, the unmodified reference compiled by
oracle/Makefile.  It imports numpy and ctypes only — no module of the product
package, no product library.

The instance comes from a directory written by problem.save_problem (the
seeded generator runs in a separate process); the arrays are memory-mapped.
The solve is the reference's own pdhglp::solve with tolerances unreachable
and a timestamp-only iteration observer (oracle/ref_capi.cpp
ref_time_window; the observer hook is proj/include/pdhglp/solver.hpp:521-529).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref", "libpdhglp_ref.so")

_ARRAYS = ("row_start", "row_index", "row_value", "col_start", "col_index", "col_value",
           "objective", "con_lower", "con_upper", "var_lower", "var_upper")


class CsrView(C.Structure):
    """include/pdlp_b200.h pdlp_csr_view (the shim's input struct)."""
    _fields_ = [("primary_dim", C.c_int64), ("nnz", C.c_int64),
                ("start", C.POINTER(C.c_int64)), ("index", C.POINTER(C.c_int64)),
                ("value", C.POINTER(C.c_double))]


class ProblemView(C.Structure):
    """include/pdlp_b200.h pdlp_problem_view."""
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("by_row", CsrView),
                ("by_col", CsrView), ("objective", C.POINTER(C.c_double)),
                ("con_lower", C.POINTER(C.c_double)), ("con_upper", C.POINTER(C.c_double)),
                ("var_lower", C.POINTER(C.c_double)), ("var_upper", C.POINTER(C.c_double))]


def load_arrays(path: str) -> dict:
    with open(os.path.join(path, "shape.json")) as f:
        d = dict(json.load(f))
    for name in _ARRAYS:
        d[name] = np.load(os.path.join(path, name + ".npy"), mmap_mode="r")
    return d


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def view(d: dict) -> ProblemView:
    v = ProblemView()
    v.rows, v.cols = int(d["rows"]), int(d["cols"])
    for lay, pre in (("by_row", "row"), ("by_col", "col")):
        cv = getattr(v, lay)
        st, ix, va = d[pre + "_start"], d[pre + "_index"], d[pre + "_value"]
        cv.primary_dim = st.shape[0] - 1
        cv.nnz = va.shape[0]
        cv.start = _ptr(st, C.c_int64)
        cv.index = _ptr(ix, C.c_int64)
        cv.value = _ptr(va, C.c_double)
    for name in ("objective", "con_lower", "con_upper", "var_lower", "var_upper"):
        setattr(v, name, _ptr(d[name], C.c_double))
    return v


def _lib() -> C.CDLL:
    if not os.path.exists(REF_PATH):
        raise FileNotFoundError(f"{REF_PATH} not built (make -C oracle ref)")
    lib = C.CDLL(REF_PATH)
    lib.ref_time_window.restype = C.c_int
    lib.ref_time_window.argtypes = [C.POINTER(ProblemView), C.c_int32, C.c_int32, C.c_int64,
                                    C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.c_int64]
    lib.ref_last_error.restype = C.c_char_p
    return lib


def time_window(d: dict, threads: int, warmup: int, steps: int, shards_per_thread: int = 4) -> dict:
    """The reference solve over iterations (warmup, warmup + steps] plus the
    budget-hit cadence that ends it: iterations/s over that window."""
    lib = _lib()
    v = view(d)
    out = (C.c_double * 6)()
    rc = lib.ref_time_window(C.byref(v), threads, shards_per_thread, warmup, steps, out, None, 0)
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib.ref_last_error().decode()}")
    window, iters, pre, total, restarts, retries = list(out)
    return {"value": iters / window if window > 0 else 0.0, "window_seconds": window,
            "iterations": int(iters), "setup_and_warmup_seconds": pre, "total_seconds": total,
            "restarts": int(restarts), "step_retries": int(retries), "threads": threads}


def load_module_by_path():
    """For callers: import this file without executing oracle/__init__.py."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("pdlp_ref_arm", os.path.abspath(__file__))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
