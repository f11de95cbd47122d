"""Reference-shaped Python API over the C-ABI (libpdlp_b200.so).

    SolverOptions, TerminationTolerances, RestartThresholds
        <- solver.hpp:69-90, residuals.hpp:187-191, restarts.hpp:235-239
    SolveStatus, SolveResult, ResidualSummary, InfeasibilityCertificate
        <- solver.hpp:35-54, 92-108, residuals.hpp:66-73, 200-210
    solve(problem, options)          <- pdhglp::solve (solver.hpp:535-608)

Plus the single-component entry points the parity tests use (pdhg_step,
adaptive_step, spmv, ... ; see include/pdlp_b200.h).  Every call runs CUDA
kernels; errors raise (ValueError for an invalid problem, as the reference's
std::invalid_argument; RuntimeError for device failures).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import sys
import time
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N
from .problem import LpProblem, _pd

INF = math.inf


class SolveStatus(enum.IntEnum):
    OPTIMAL = 0
    PRIMAL_INFEASIBLE = 1
    DUAL_INFEASIBLE = 2
    ITERATION_LIMIT = 3
    TIME_LIMIT = 4
    NUMERICAL_ERROR = 5


STATUS_NAMES = ["optimal", "primal_infeasible", "dual_infeasible", "iteration_limit",
                "time_limit", "numerical_error"]


def solve_status_name(s: int) -> str:
    return STATUS_NAMES[int(s)] if 0 <= int(s) < 6 else "numerical_error"


class CertificateKind(enum.IntEnum):
    PRIMAL_INFEASIBLE = 0
    DUAL_INFEASIBLE = 1


@dataclass
class TerminationTolerances:
    eps_primal: float = 1e-8
    eps_dual: float = 1e-8
    eps_rel_gap: float = 1e-2


@dataclass
class RestartThresholds:
    sufficient: float = 0.1
    necessary: float = 0.9
    artificial: float = 0.5


@dataclass
class IterationRecord:
    iteration: int
    x: np.ndarray
    y: np.ndarray
    eta: float
    omega: float


@dataclass
class SolverOptions:
    tolerances: TerminationTolerances = field(default_factory=TerminationTolerances)
    iteration_limit: int = 200000
    time_limit_seconds: float = INF
    threads: int = 1
    shards_per_thread: int = 4
    enable_scaling: bool = True
    ruiz_passes: int = 10
    pock_chambolle: bool = True
    enable_polish: bool = True
    enable_restarts: bool = True
    detect_infeasibility: bool = True
    eps_ray: float = 1e-12
    check_interval: int = 64
    restart_thresholds: RestartThresholds = field(default_factory=RestartThresholds)
    fixed_step_size: Optional[float] = None
    fixed_primal_weight: Optional[float] = None
    logging: bool = False
    observer: Optional[Callable[[IterationRecord], None]] = None
    # B200 extensions (additive)
    mode: str = "perf"  # "perf" | "parity"
    device: int = 0
    profile_kernels: bool = False
    timing_warmup_iterations: int = 0


@dataclass
class ResidualSummary:
    primal_residual_inf: float = INF
    dual_residual_inf: float = INF
    primal_objective: float = 0.0
    dual_objective: float = 0.0
    abs_gap: float = INF
    rel_gap: float = INF


@dataclass
class InfeasibilityCertificate:
    kind: CertificateKind
    ray_x: np.ndarray
    ray_y: np.ndarray
    ray_r: np.ndarray
    residual_inf: float
    objective: float
    source: str


@dataclass
class SolveResult:
    status: SolveStatus = SolveStatus.NUMERICAL_ERROR
    x: np.ndarray = None
    y: np.ndarray = None
    reduced_costs: np.ndarray = None
    summary: ResidualSummary = field(default_factory=ResidualSummary)
    certificate: Optional[InfeasibilityCertificate] = None
    iterations: int = 0
    polish_iterations: int = 0
    restarts: int = 0
    step_retries: int = 0
    final_step_size: float = 0.0
    final_primal_weight: float = 1.0
    min_step_size_limit: float = INF
    solve_seconds: float = 0.0
    termination_detail: str = ""
    # B200 extensions
    attempts: int = 0
    upload_seconds: float = 0.0
    precondition_seconds: float = 0.0
    loop_seconds: float = 0.0
    step_seconds: float = 0.0
    timed_seconds: float = 0.0
    timed_iterations: int = 0
    timed_attempts: int = 0
    kernel_seconds: list = field(default_factory=lambda: [0.0] * 4)
    kernel_launches: list = field(default_factory=lambda: [0] * 4)


def _mode(m) -> int:
    if isinstance(m, int):
        return m
    return N.MODE_PARITY if str(m).lower() == "parity" else N.MODE_PERF


def to_c_options(o: SolverOptions) -> N.Options:
    c = N.Options()
    N.lib().pdlp_default_options(C.byref(c))
    c.eps_primal = o.tolerances.eps_primal
    c.eps_dual = o.tolerances.eps_dual
    c.eps_rel_gap = o.tolerances.eps_rel_gap
    c.iteration_limit = int(o.iteration_limit)
    c.time_limit_seconds = float(o.time_limit_seconds)
    c.threads = int(o.threads)
    c.shards_per_thread = int(o.shards_per_thread)
    c.enable_scaling = int(bool(o.enable_scaling))
    c.ruiz_passes = int(o.ruiz_passes)
    c.pock_chambolle = int(bool(o.pock_chambolle))
    c.enable_polish = int(bool(o.enable_polish))
    c.enable_restarts = int(bool(o.enable_restarts))
    c.detect_infeasibility = int(bool(o.detect_infeasibility))
    c.eps_ray = float(o.eps_ray)
    c.check_interval = int(o.check_interval)
    c.restart_sufficient = o.restart_thresholds.sufficient
    c.restart_necessary = o.restart_thresholds.necessary
    c.restart_artificial = o.restart_thresholds.artificial
    if o.fixed_step_size is not None:
        c.has_fixed_step_size = 1
        c.fixed_step_size = float(o.fixed_step_size)
    if o.fixed_primal_weight is not None:
        c.has_fixed_primal_weight = 1
        c.fixed_primal_weight = float(o.fixed_primal_weight)
    c.logging = int(bool(o.logging))
    c.mode = _mode(o.mode)
    c.device = int(o.device)
    c.profile_kernels = int(bool(o.profile_kernels))
    c.timing_warmup_iterations = int(o.timing_warmup_iterations)
    return c


def _observer_thunk(fn):
    def cb(_user, rec_p):
        rec = rec_p.contents
        x = np.ctypeslib.as_array(rec.x, shape=(rec.x_len,)).copy() if rec.x_len else np.zeros(0)
        y = np.ctypeslib.as_array(rec.y, shape=(rec.y_len,)).copy() if rec.y_len else np.zeros(0)
        fn(IterationRecord(int(rec.iteration), x, y, float(rec.eta), float(rec.omega)))
    return N.OBSERVER_FN(cb)


def _check(rc: int) -> None:
    if rc == N.PDLP_OK:
        return
    msg = N.last_error()
    if rc == N.PDLP_ERR_INVALID_PROBLEM:
        raise ValueError(msg)
    raise RuntimeError(f"pdlp error {rc}: {msg}")


def run_solve(lib, fn_name: str, p: LpProblem | None, options: SolverOptions, c_opts: N.Options,
              extra: tuple = (), first_arg=None, dims: tuple | None = None,
              out: dict | None = None) -> SolveResult:
    """Shared marshalling for pdlp_solve, the sharded solves (extra = the
    arguments between options and result) and the oracle's ref_solve.  The
    shard-local solves pass no problem: first_arg is their shard argument
    and dims = (rows, cols) of the whole problem.  out: caller buffers for
    x / y / reduced_costs (float64, contiguous; e.g. registered with
    `pinned`, so the results come back by DMA)."""
    t_prep = time.perf_counter()
    if p is not None:
        view = p.view()
        first_arg = C.byref(view)
        m, n = p.rows(), p.cols()
    else:
        m, n = dims

    def buf(name, size):
        a = (out or {}).get(name)
        if a is None:
            return np.zeros(size)
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
                and a.shape == (size,)):
            raise ValueError(f"out[{name!r}] must be a contiguous float64 array of {size}")
        return a

    x = buf("x", n)
    y = buf("y", m)
    r = buf("reduced_costs", n)
    rx = np.zeros(n)
    ry = np.zeros(m)
    rr = np.zeros(n)
    res = N.Result()
    res.x, res.y, res.reduced_costs = _pd(x), _pd(y), _pd(r)
    res.cert_ray_x, res.cert_ray_y, res.cert_ray_r = _pd(rx), _pd(ry), _pd(rr)
    thunk = None
    if options.observer is not None:
        thunk = _observer_thunk(options.observer)
        c_opts.observer = thunk
    t_call = time.perf_counter()
    rc = getattr(lib, fn_name)(first_arg, C.byref(c_opts), *extra, C.byref(res))
    if os.environ.get("PDLP_TIMING"):
        print(f"phase=python event=timing call={time.perf_counter() - t_call:.4f} "
              f"native_solve={res.solve_seconds:.4f} prep={t_call - t_prep:.4f}", file=sys.stderr)
    if rc != 0:
        err = lib.pdlp_last_error() if hasattr(lib, "pdlp_last_error") else lib.ref_last_error()
        msg = err.decode()
        if rc == N.PDLP_ERR_INVALID_PROBLEM:
            raise ValueError(msg)
        raise RuntimeError(f"{fn_name} error {rc}: {msg}")
    s = res.summary
    cert = None
    if res.has_certificate:
        cert = InfeasibilityCertificate(
            CertificateKind(res.cert_kind),
            rx if res.cert_kind == 1 else np.zeros(0),
            ry if res.cert_kind == 0 else np.zeros(0),
            rr if res.cert_kind == 0 else np.zeros(0),
            res.cert_residual_inf, res.cert_objective, res.cert_source.decode())
    return SolveResult(
        status=SolveStatus(res.status), x=x, y=y, reduced_costs=r,
        summary=ResidualSummary(s.primal_residual_inf, s.dual_residual_inf, s.primal_objective,
                                s.dual_objective, s.abs_gap, s.rel_gap),
        certificate=cert, iterations=res.iterations, polish_iterations=res.polish_iterations,
        restarts=res.restarts, step_retries=res.step_retries,
        final_step_size=res.final_step_size, final_primal_weight=res.final_primal_weight,
        min_step_size_limit=res.min_step_size_limit, solve_seconds=res.solve_seconds,
        termination_detail=res.termination_detail.decode(), attempts=res.attempts,
        upload_seconds=res.upload_seconds, precondition_seconds=res.precondition_seconds,
        loop_seconds=res.loop_seconds, step_seconds=res.step_seconds,
        timed_seconds=getattr(res, "timed_seconds", 0.0),
        timed_iterations=getattr(res, "timed_iterations", 0),
        timed_attempts=getattr(res, "timed_attempts", 0),
        kernel_seconds=list(res.kernel_seconds), kernel_launches=list(res.kernel_launches))


def solve(problem: LpProblem, options: SolverOptions | None = None,
          out: dict | None = None) -> SolveResult:
    """pdhglp::solve on the GPU (solver.hpp:535-608).  out: optional caller
    buffers {"x", "y", "reduced_costs"} the result is written into."""
    options = options or SolverOptions()
    return run_solve(N.lib(), "pdlp_solve", problem, options, to_c_options(options), out=out)


class _PinnedBlock:
    """One pdlp_host_alloc block; freed when the last array over it dies."""

    def __init__(self, nbytes: int):
        self.ptr = C.c_void_p()
        _check(N.lib().pdlp_host_alloc(max(int(nbytes), 1), C.byref(self.ptr)))

    def __del__(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            N.lib().pdlp_host_free(self.ptr)
            self.ptr = None


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """An uninitialised numpy array in page-locked host memory
    (pdlp_host_alloc): solves read it / write it by DMA."""
    dt = np.dtype(dtype)
    count = int(np.prod(shape)) if np.ndim(shape) else int(shape)
    blk = _PinnedBlock(count * dt.itemsize)
    buf = (C.c_char * max(count * dt.itemsize, 1)).from_address(blk.ptr.value)
    buf._pinned_block = blk  # the array keeps buf alive, buf keeps the block
    return np.frombuffer(buf, dtype=dt, count=count).reshape(shape)


def pinned_copy(problem: LpProblem) -> LpProblem:
    """The same LP with every array copied into page-locked host memory:
    solves of the copy upload by DMA (64-bit indices narrowed on the
    device) instead of through the pinned staging ring's host copies."""
    from .problem import CompressedLayout, SparseMatrix

    def cp(a):
        out = pinned_empty(a.shape, a.dtype)
        np.copyto(out, a)
        return out

    a = problem.a
    lay = lambda L: CompressedLayout(cp(L.start), cp(L.index), cp(L.value))  # noqa: E731
    problem.view()  # normalises the vectors to contiguous float64 first
    return LpProblem(SparseMatrix(a.rows, a.cols, lay(a.by_row), lay(a.by_col)),
                     cp(problem.objective), cp(problem.con_lower), cp(problem.con_upper),
                     cp(problem.var_lower), cp(problem.var_upper))


class pinned:
    """Page-lock host arrays for the solves inside the block (B200 extension,
    pdlp_host_register): a problem registered this way uploads with one DMA
    per array (64-bit indices narrowed on the device) instead of through the
    pinned staging ring's host copies, and registered result buffers (solve's
    `out`) are filled by DMA.  Accepts LpProblem and numpy arrays.

        with P.pinned(problem, x, y, r):
            P.solve(problem, options, out={"x": x, "y": y, "reduced_costs": r})
    """

    def __init__(self, *objs):
        self._arrays = []
        for o in objs:
            if isinstance(o, LpProblem):
                for lay in (o.a.by_row, o.a.by_col):
                    self._arrays += [lay.start, lay.index, lay.value]
                o.view()  # normalises the vectors to contiguous float64 first
                self._arrays += [o.objective, o.con_lower, o.con_upper, o.var_lower, o.var_upper]
            else:
                self._arrays.append(o)
        self._done = []

    def __enter__(self):
        lib = N.lib()
        for a in self._arrays:
            if isinstance(a, np.ndarray) and a.nbytes > 0 and a.flags.c_contiguous:
                _check(lib.pdlp_host_register(a.ctypes.data, a.nbytes))
                self._done.append(a)
        return self

    def __exit__(self, *exc):
        lib = N.lib()
        for a in self._done:
            lib.pdlp_host_unregister(a.ctypes.data)
        self._done = []
        return False


# ------------------------------------------------------ component entries ---
def pdhg_step(p: LpProblem, x, y, omega: float, eta: float, mode="parity", shards: int = 4):
    """reference pdhg_step (step.hpp:100-115); None when non-finite."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    xo, yo = np.zeros(p.cols()), np.zeros(p.rows())
    fin = C.c_int32(0)
    _check(N.lib().pdlp_pdhg_step(C.byref(p.view()), _pd(x), _pd(y), omega, eta, _mode(mode),
                                  shards, _pd(xo), _pd(yo), C.byref(fin)))
    return (xo, yo) if fin.value else None


def adaptive_step(p: LpProblem, x, y, aty, eta_hat: float, k: int = 0, omega: float = 1.0,
                  max_retries: int = 60, mode="parity", shards: int = 4) -> dict:
    """reference adaptive_step (step.hpp:161-193) from (x, y, aty)."""
    x = np.array(x, np.float64)
    y = np.array(y, np.float64)
    aty = np.array(aty, np.float64)
    st = np.array([eta_hat, float(k), float(max_retries), omega])
    px, py = np.zeros(p.cols()), np.zeros(p.rows())
    stats = np.zeros(4)
    out = C.c_int32(0)
    _check(N.lib().pdlp_adaptive_step(C.byref(p.view()), _pd(x), _pd(y), _pd(aty), _pd(st),
                                      _mode(mode), shards, _pd(px), _pd(py), _pd(stats),
                                      C.byref(out)))
    return dict(accepted=out.value == 0, x=x, y=y, aty=aty, prev_x=px, prev_y=py,
                eta_hat=st[0], k=int(st[1]), accepted_steps=int(stats[0]),
                retries=int(stats[1]), min_eta_bar=stats[2], eta_used=stats[3])


def spmv(p: LpProblem, x, mode="parity") -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(p.rows())
    _check(N.lib().pdlp_spmv(C.byref(p.view()), _pd(x), _pd(out), _mode(mode)))
    return out


def spmv_transpose(p: LpProblem, y, mode="parity") -> np.ndarray:
    y = np.ascontiguousarray(y, np.float64)
    out = np.zeros(p.cols())
    _check(N.lib().pdlp_spmv_transpose(C.byref(p.view()), _pd(y), _pd(out), _mode(mode)))
    return out


def apply_rescaling(p: LpProblem, ruiz_passes: int = 10, pock_chambolle: bool = True) -> dict:
    nnz, m, n = p.a.nonzeros(), p.rows(), p.cols()
    out = {k: np.zeros(s) for k, s in (("row_values", nnz), ("col_values", nnz), ("objective", n),
                                       ("con_lower", m), ("con_upper", m), ("var_lower", n),
                                       ("var_upper", n), ("row_scale", m), ("col_scale", n))}
    _check(N.lib().pdlp_apply_rescaling(C.byref(p.view()), ruiz_passes, int(pock_chambolle),
                                        *[_pd(out[k]) for k in ("row_values", "col_values",
                                                                "objective", "con_lower",
                                                                "con_upper", "var_lower",
                                                                "var_upper", "row_scale",
                                                                "col_scale")]))
    return out


def normalized_duality_gap(p: LpProblem, x, y, ax, aty, omega: float, r: float,
                           mode="parity") -> float:
    arrs = [np.ascontiguousarray(a, np.float64) for a in (x, y, ax, aty)]
    g = C.c_double(0.0)
    _check(N.lib().pdlp_normalized_duality_gap(C.byref(p.view()), *[_pd(a) for a in arrs], omega,
                                               r, _mode(mode), C.byref(g)))
    return g.value


def kkt_residuals(p: LpProblem, x, y, rc_mode: int = 0, mode="parity"):
    """recover_reduced_costs + kkt_residuals (residuals.hpp:49-64, 135-158)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    r = np.zeros(p.cols())
    s = N.ResidualSummary()
    _check(N.lib().pdlp_kkt_residuals(C.byref(p.view()), _pd(x), _pd(y), rc_mode, _mode(mode),
                                      _pd(r), C.byref(s)))
    return r, ResidualSummary(s.primal_residual_inf, s.dual_residual_inf, s.primal_objective,
                              s.dual_objective, s.abs_gap, s.rel_gap)


def kkt_residuals_given(p: LpProblem, x, y, r, mode="perf") -> ResidualSummary:
    """kkt_residuals(p, x, y, r) with the given reduced costs (residuals.hpp:
    135-158), original space, on the device (the `check` command)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    r = np.array(r, np.float64)
    s = N.ResidualSummary()
    _check(N.lib().pdlp_kkt_residuals(C.byref(p.view()), _pd(x), _pd(y), 2, _mode(mode), _pd(r),
                                      C.byref(s)))
    return ResidualSummary(s.primal_residual_inf, s.dual_residual_inf, s.primal_objective,
                           s.dual_objective, s.abs_gap, s.rel_gap)


def check_certificate(p: LpProblem, kind, ray, eps_ray: float = 1e-12):
    """try_primal_infeasibility / try_dual_infeasibility (residuals.hpp:222-299)
    on the original data, on the device.  Returns (verified, residual, objective)."""
    ray = np.ascontiguousarray(ray, np.float64)
    ok, res, obj = C.c_int32(0), C.c_double(0.0), C.c_double(0.0)
    _check(N.lib().pdlp_check_certificate(C.byref(p.view()), int(kind), _pd(ray), eps_ray,
                                          C.byref(ok), C.byref(res), C.byref(obj)))
    return bool(ok.value), res.value, obj.value


def step_size_rules(movement: float, curvature: float, eta_bar: float, eta: float, k: int):
    lim, nxt = C.c_double(0.0), C.c_double(0.0)
    _check(N.lib().pdlp_step_size_rules(movement, curvature, eta_bar, eta, k, C.byref(lim),
                                        C.byref(nxt)))
    return lim.value, nxt.value


def device_count() -> int:
    return int(N.lib().pdlp_device_count())
