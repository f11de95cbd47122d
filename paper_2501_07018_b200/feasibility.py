"""The reference's Appendix-B fixed-restart feasibility harness on the GPU.

Reference: proj/tests/feasibility_method.hpp:40-85
(``testharness::fixed_restart_feasibility``), the iteration behind acceptance
criterion 10 (proj/tests/acceptance.cpp:700-795): find x >= 0 with A x = b by
primal-dual steps of a fixed size; each round runs ``restart_length`` steps
from the previous restart point with the duals reset to zero, averages the
primal iterates and adopts the average as the next restart point.

On the device (``pdlp_feasibility_run``) a step is the SpMV kernels (A^T y by
columns, A x by rows) plus two elementwise kernels; rounds replay captured
CUDA graphs of up to 64 steps.  ``mode="parity"`` reproduces the reference's
arithmetic bit for bit (sequential line sums, row-order residual sums);
``mode="perf"`` uses the tiled SpMV and tree reductions.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .problem import LpProblem, _pd
from .solver import _check, _mode


@dataclass
class FeasibilityRun:
    """FeasibilityRun (feasibility_method.hpp:19-23)."""
    restart_points: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))  # [k, n]
    residuals: np.ndarray = field(default_factory=lambda: np.zeros(0))  # ||A x - b||_2 per point
    finite: bool = True


def feasibility_residual(p: LpProblem, x, b) -> float:
    """||A x - b||_2 (feasibility_method.hpp:26-34), on the device."""
    run = fixed_restart_feasibility(p, b, x, 1.0, 1, 0)
    return float(run.residuals[0])


def fixed_restart_feasibility(p: LpProblem, b, x0, eta: float, restart_length: int, rounds: int,
                              mode: str = "parity", device: int = 0) -> FeasibilityRun:
    """testharness::fixed_restart_feasibility(a, b, x0, eta, restart_length,
    rounds) with a = p's constraint matrix (its other data is not read)."""
    if restart_length < 1 or rounds < 0:
        raise ValueError("restart_length must be >= 1 and rounds >= 0")
    n = p.cols()
    b = np.ascontiguousarray(b, np.float64)
    x0 = np.ascontiguousarray(x0, np.float64)
    if b.shape != (p.rows(),) or x0.shape != (n,):
        raise ValueError("b must have one entry per row and x0 one per column")
    pts = np.zeros((rounds + 1, n))
    res = np.zeros(rounds + 1)
    rec, fin = C.c_int32(0), C.c_int32(0)
    _check(N.lib().pdlp_feasibility_run(C.byref(p.view()), _pd(b), _pd(x0), float(eta),
                                        int(restart_length), int(rounds), _mode(mode), int(device),
                                        _pd(pts), _pd(res), C.byref(rec), C.byref(fin)))
    k = rec.value
    return FeasibilityRun(pts[:k].copy(), res[:k].copy(), bool(fin.value))
