"""TEST INFRASTRUCTURE — the CPU parity checkers.  Never imported by the
product package; only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference arm use it.

Two checkers with one C-ABI (``ref_*`` symbols, include/pdlp_b200.h structs):

  REF   oracle/_ref/libpdhglp_ref.so — the UNMODIFIED reference library
        (/root/reference/proj/include, header-only C++20) compiled in place by
        oracle/Makefile behind ref_capi.cpp.  Travels to the GPU box prebuilt.
  PORT  oracle/_build/libpdlp_oracle.so — the CPU restatement in
        oracle/pdlp_oracle.cpp (same algorithm, written independently, pinned
        bit-for-bit against REF and the reference's known-answer tests).

``get()`` returns REF when it is built, else PORT.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from paper_2501_07018_b200 import _native as N
from paper_2501_07018_b200.problem import LpProblem, _pd, _wrap
from paper_2501_07018_b200 import solver as S

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref", "libpdhglp_ref.so")
PORT_PATH = os.path.join(HERE, "_build", "libpdlp_oracle.so")

P = C.POINTER(N.ProblemView)
D = N.c_double_p
_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_default_options": (None, [C.POINTER(N.Options)]),
    "ref_solve": (C.c_int, [P, C.POINTER(N.Options), C.POINTER(N.Result)]),
    "ref_pdhg_step": (C.c_int, [P, D, D, C.c_double, C.c_double, D, D, N.c_int32_p]),
    "ref_adaptive_step": (C.c_int, [P, D, D, D, D, C.c_int32, C.c_int32, D, D, D, N.c_int32_p]),
    "ref_spmv": (C.c_int, [P, D, D, C.c_int32, C.c_int32]),
    "ref_spmv_transpose": (C.c_int, [P, D, D, C.c_int32, C.c_int32]),
    "ref_apply_rescaling": (C.c_int, [P, C.c_int32, C.c_int32] + [D] * 9),
    "ref_normalized_duality_gap": (C.c_int, [P, D, D, D, D, C.c_double, C.c_double, D]),
    "ref_kkt_residuals": (C.c_int, [P, D, D, C.c_int32, D, C.POINTER(N.ResidualSummary)]),
    "ref_step_size_rules": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int64,
                                      D, D]),
    "ref_initialize_primal_weight": (C.c_double, [P]),
    "ref_initial_step_size": (C.c_double, [P]),
    "ref_validate": (C.c_int, [P, C.c_char_p, C.c_int32]),
    "ref_feasibility_run": (C.c_int, [P, D, D, C.c_double, C.c_int64, C.c_int32, D, D,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
}
_REF_ONLY = {
    "ref_generate": (C.c_void_p, [C.c_int32, C.c_int64, C.c_int64, C.c_double, C.c_uint64]),
    "ref_from_triplets": (C.c_void_p, [C.c_int64, C.c_int64, C.c_int64, N.c_int64_p, N.c_int64_p,
                                       D] + [D] * 5),
    "ref_instance_view": (None, [C.c_void_p, P]),
    "ref_instance_optimal_objective": (C.c_double, [C.c_void_p]),
    "ref_instance_free": (None, [C.c_void_p]),
    "ref_instance_feasible_point": (None, [C.c_void_p, D]),
    "ref_mps_parse": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "ref_mps_view": (None, [C.c_void_p, P]),
    "ref_mps_maximize": (C.c_int32, [C.c_void_p]),
    "ref_mps_name": (C.c_char_p, [C.c_void_p]),
    "ref_mps_objective_name": (C.c_char_p, [C.c_void_p]),
    "ref_mps_row_name": (C.c_char_p, [C.c_void_p, C.c_int64]),
    "ref_mps_col_name": (C.c_char_p, [C.c_void_p, C.c_int64]),
    "ref_mps_free": (None, [C.c_void_p]),
    "ref_mps_write": (C.c_int, [P, C.c_char_p, C.c_int32, C.POINTER(C.c_void_p),
                                C.POINTER(C.c_size_t)]),
    "ref_mps_free_text": (None, [C.c_void_p]),
}

KIND = {"random-feasible": 0, "random-infeasible": 1, "transport": 2, "feasibility-system": 3}


class Oracle:
    def __init__(self, path: str, name: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.name = name
        self.path = path
        self.lib = C.CDLL(path)
        sigs = dict(_SIGS)
        if name == "reference":
            sigs.update(_REF_ONLY)
        for fn, (res, args) in sigs.items():
            f = getattr(self.lib, fn)
            f.restype = res
            f.argtypes = args

    def _check(self, rc):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            if rc == N.PDLP_ERR_INVALID_PROBLEM:
                raise ValueError(msg)
            raise RuntimeError(f"{self.name} oracle error {rc}: {msg}")

    def options(self, o: S.SolverOptions) -> N.Options:
        c = N.Options()
        self.lib.ref_default_options(C.byref(c))
        d = S.to_c_options(o)
        for f, _ in N.Options._fields_:
            if f not in ("observer", "observer_user"):
                setattr(c, f, getattr(d, f))
        return c

    def solve(self, p: LpProblem, o: S.SolverOptions | None = None) -> S.SolveResult:
        o = o or S.SolverOptions()
        lib = self.lib

        class _Shim:
            ref_solve = lib.ref_solve
            ref_last_error = lib.ref_last_error

        return S.run_solve(_Shim, "ref_solve", p, o, self.options(o))

    # reference MPS reader / writer (mps.hpp), compiled reference only
    def parse_mps(self, text):
        from paper_2501_07018_b200.mps import model_from_handle
        data = text.encode() if isinstance(text, str) else bytes(text)
        h = C.c_void_p()
        self._check(self.lib.ref_mps_parse(data, len(data), C.byref(h)))
        try:
            return model_from_handle(self.lib, "ref_mps_", h)
        finally:
            self.lib.ref_mps_free(h)

    def write_mps(self, p, name="", maximize=False):
        from paper_2501_07018_b200.mps import write_text
        return write_text(self.lib, "ref_mps_write", "ref_mps_free_text", p, name, maximize)

    def pdhg_step(self, p, x, y, omega, eta):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        xo, yo = np.zeros(p.cols()), np.zeros(p.rows())
        fin = C.c_int32(0)
        self._check(self.lib.ref_pdhg_step(C.byref(p.view()), _pd(x), _pd(y), omega, eta, _pd(xo),
                                           _pd(yo), C.byref(fin)))
        return (xo, yo) if fin.value else None

    def adaptive_step(self, p, x, y, aty, eta_hat, k=0, omega=1.0, max_retries=60, threads=1,
                      spt=4):
        x = np.array(x, np.float64)
        y = np.array(y, np.float64)
        aty = np.array(aty, np.float64)
        st = np.array([eta_hat, float(k), float(max_retries), omega])
        px, py = np.zeros(p.cols()), np.zeros(p.rows())
        stats = np.zeros(4)
        out = C.c_int32(0)
        self._check(self.lib.ref_adaptive_step(C.byref(p.view()), _pd(x), _pd(y), _pd(aty), _pd(st),
                                               threads, spt, _pd(px), _pd(py), _pd(stats),
                                               C.byref(out)))
        return dict(accepted=out.value == 0, x=x, y=y, aty=aty, prev_x=px, prev_y=py,
                    eta_hat=st[0], k=int(st[1]), accepted_steps=int(stats[0]),
                    retries=int(stats[1]), min_eta_bar=stats[2], eta_used=stats[3])

    def spmv(self, p, x, threads=1, spt=4):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(p.rows())
        self._check(self.lib.ref_spmv(C.byref(p.view()), _pd(x), _pd(out), threads, spt))
        return out

    def spmv_transpose(self, p, y, threads=1, spt=4):
        y = np.ascontiguousarray(y, np.float64)
        out = np.zeros(p.cols())
        self._check(self.lib.ref_spmv_transpose(C.byref(p.view()), _pd(y), _pd(out), threads, spt))
        return out

    def apply_rescaling(self, p, ruiz_passes=10, pock_chambolle=True):
        nnz, m, n = p.a.nonzeros(), p.rows(), p.cols()
        keys = ("row_values", "col_values", "objective", "con_lower", "con_upper", "var_lower",
                "var_upper", "row_scale", "col_scale")
        sizes = (nnz, nnz, n, m, m, n, n, m, n)
        out = {k: np.zeros(s) for k, s in zip(keys, sizes)}
        self._check(self.lib.ref_apply_rescaling(C.byref(p.view()), ruiz_passes, int(pock_chambolle),
                                                 *[_pd(out[k]) for k in keys]))
        return out

    def normalized_duality_gap(self, p, x, y, ax, aty, omega, r):
        arrs = [np.ascontiguousarray(a, np.float64) for a in (x, y, ax, aty)]
        g = C.c_double(0.0)
        self._check(self.lib.ref_normalized_duality_gap(C.byref(p.view()), *[_pd(a) for a in arrs],
                                                        omega, r, C.byref(g)))
        return g.value

    def kkt_residuals(self, p, x, y, rc_mode=0):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        r = np.zeros(p.cols())
        s = N.ResidualSummary()
        self._check(self.lib.ref_kkt_residuals(C.byref(p.view()), _pd(x), _pd(y), rc_mode, _pd(r),
                                               C.byref(s)))
        return r, S.ResidualSummary(s.primal_residual_inf, s.dual_residual_inf, s.primal_objective,
                                    s.dual_objective, s.abs_gap, s.rel_gap)

    def step_size_rules(self, movement, curvature, eta_bar, eta, k):
        a, b = C.c_double(0.0), C.c_double(0.0)
        self._check(self.lib.ref_step_size_rules(movement, curvature, eta_bar, eta, k, C.byref(a),
                                                 C.byref(b)))
        return a.value, b.value

    def initialize_primal_weight(self, p):
        return self.lib.ref_initialize_primal_weight(C.byref(p.view()))

    def initial_step_size(self, p):
        return self.lib.ref_initial_step_size(C.byref(p.view()))

    def validate(self, p):
        buf = C.create_string_buffer(256)
        bad = self.lib.ref_validate(C.byref(p.view()), buf, 256)
        return buf.value.decode() if bad else None

    # Appendix-B harness (tests/feasibility_method.hpp:60-85)
    def feasibility_run(self, p, b, x0, eta: float, restart_length: int, rounds: int):
        """(restart points [k, n], residuals [k], finite) like FeasibilityRun."""
        n = p.cols()
        pts = np.zeros((rounds + 1, n))
        res = np.zeros(rounds + 1)
        rec, fin = C.c_int32(0), C.c_int32(0)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        self._check(self.lib.ref_feasibility_run(C.byref(p.view()), _pd(b), _pd(x0), eta,
                                                 restart_length, rounds, _pd(pts), _pd(res),
                                                 C.byref(rec), C.byref(fin)))
        return pts[:rec.value].copy(), res[:rec.value].copy(), bool(fin.value)

    def generate_feasibility_system(self, rows: int, cols: int, density: float, seed: int):
        """The reference's FeasibilitySystem instance and its positive point."""
        h = self.lib.ref_generate(KIND["feasibility-system"], rows, cols, density, seed)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        inst = _RefInstance(self, h)
        p = inst.problem()
        pt = np.zeros(p.cols())
        self.lib.ref_instance_feasible_point(h, _pd(pt))
        return p, pt

    # reference generator (generator.hpp:347-374), reference oracle only
    def generate(self, kind: str, rows: int, cols: int, density: float, seed: int):
        h = self.lib.ref_generate(KIND[kind], rows, cols, density, seed)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return _RefInstance(self, h).problem()


class _RefInstance:
    def __init__(self, oracle: Oracle, h):
        self.o = oracle
        self.h = h

    def problem(self) -> LpProblem:
        v = N.ProblemView()
        self.o.lib.ref_instance_view(self.h, C.byref(v))
        from paper_2501_07018_b200.problem import CompressedLayout, SparseMatrix, _as_array
        lay = lambda L: CompressedLayout(_as_array(L.start, L.primary_dim + 1, np.int64).copy(),
                                         _as_array(L.index, L.nnz, np.int64).copy(),
                                         _as_array(L.value, L.nnz, np.float64).copy())
        m, n = v.rows, v.cols
        p = LpProblem(SparseMatrix(m, n, lay(v.by_row), lay(v.by_col)),
                      _as_array(v.objective, n, np.float64).copy(),
                      _as_array(v.con_lower, m, np.float64).copy(),
                      _as_array(v.con_upper, m, np.float64).copy(),
                      _as_array(v.var_lower, n, np.float64).copy(),
                      _as_array(v.var_upper, n, np.float64).copy())
        p.optimal_objective = self.o.lib.ref_instance_optimal_objective(self.h)
        return p

    def __del__(self):
        if self.h:
            self.o.lib.ref_instance_free(self.h)
            self.h = None


_cache: dict[str, Oracle] = {}


def reference() -> Oracle:
    if "reference" not in _cache:
        _cache["reference"] = Oracle(REF_PATH, "reference")
    return _cache["reference"]


def port() -> Oracle:
    if "port" not in _cache:
        _cache["port"] = Oracle(PORT_PATH, "port")
    return _cache["port"]


def have_reference() -> bool:
    return os.path.exists(REF_PATH)


def have_port() -> bool:
    return os.path.exists(PORT_PATH)


def get() -> Oracle:
    return reference() if have_reference() else port()


def build(with_reference: bool | None = None) -> None:
    """make -C oracle (the restatement always; the reference when its sources
    are present, i.e. in the build container — the GPU box uses prebuilt .so)."""
    import subprocess
    targets = ["oracle"] if os.path.exists(os.path.join(HERE, "pdlp_oracle.cpp")) else []
    if with_reference is None:
        with_reference = os.path.isdir("/root/reference/proj/include")
    if with_reference:
        targets.append("ref")
        lib = os.path.join(os.path.dirname(HERE), "paper_2501_07018_b200", "libpdlp_b200.so")
        if os.path.exists(lib):
            targets.append("acceptance")
    if targets:
        subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)
