"""Small LP fixtures restated from the reference's tests (file:line cited)."""
from __future__ import annotations

import numpy as np

from paper_2501_07018_b200 import problem

INF = float("inf")


def tiny_lp():
    """min -x1 - 2x2, x1 + x2 <= 1, x >= 0 (test_util.hpp:91-102)."""
    return problem(1, 2, [(0, 0, 1.0), (0, 1, 1.0)], [-1.0, -2.0], [-INF], [1.0], [0.0, 0.0],
                   [INF, INF])


def one_var_equality():
    """min x, x = 1, x >= 0 (test_step.cpp:116-130)."""
    return problem(1, 1, [(0, 0, 1.0)], [1.0], [1.0], [1.0], [0.0], [INF])


def clamp_free_row():
    """x <= 2 with a free row (test_step.cpp:132-148)."""
    return problem(2, 1, [(0, 0, 1.0)], [0.0], [-INF, -INF], [2.0, INF], [-INF], [INF])


def rejection_lp():
    """x = 10, free x, zero objective (test_step.cpp:255-270)."""
    return problem(1, 1, [(0, 0, 1.0)], [0.0], [10.0], [10.0], [-INF], [INF])


def overflow_lp():
    """test_step.cpp:327-345."""
    return problem(1, 1, [(0, 0, 1.0)], [1e308], [0.0], [0.0], [-INF], [INF])


def contradictory_rows():
    """x1 + x2 <= 1 and >= 3 (test_solver.cpp:120-130)."""
    t = [(0, 0, 1.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 1.0)]
    return problem(2, 2, t, [0.0, 0.0], [-INF, 3.0], [1.0, INF], [0.0, 0.0], [INF, INF])


def unbounded_lp():
    """min -x1 - x2, x1 + x2 >= 1 (test_solver.cpp:143-152)."""
    return problem(1, 2, [(0, 0, 1.0), (0, 1, 1.0)], [-1.0, -1.0], [1.0], [INF], [0.0, 0.0],
                   [INF, INF])


def random_matrix_triplets(rng, rows, cols, density, lo=-1.0, hi=1.0):
    mask = rng.random((rows, cols)) < density
    r, c = np.nonzero(mask)
    v = rng.uniform(lo, hi, size=r.shape[0])
    return list(zip(r.tolist(), c.tolist(), v.tolist()))


def random_box_lp(rng, rows, cols):
    """Mixed row/column bound types (test_step.cpp:63-93)."""
    t = random_matrix_triplets(rng, rows, cols, 0.6)
    obj = rng.uniform(-2.0, 2.0, cols)
    lc, uc = np.empty(rows), np.empty(rows)
    for j in range(rows):
        kind = rng.integers(4)
        b = rng.uniform(-1.0, 1.0)
        lc[j], uc[j] = [(b, b), (-INF, b), (b, INF), (b - 0.5, b + 0.5)][kind]
    lv, uv = np.empty(cols), np.empty(cols)
    for i in range(cols):
        kind = rng.integers(4)
        lv[i], uv[i] = [(0.0, INF), (-INF, INF), (-1.0, 1.0), (-INF, 0.5)][kind]
    return problem(rows, cols, t, obj, lc, uc, lv, uv)


def box_interior_point(rng, p):
    lo = np.maximum(p.var_lower, -2.0)
    hi = np.minimum(p.var_upper, 2.0)
    return rng.uniform(lo, hi)


def equality_lp(rng, rows, cols):
    """Feasible equality LP around an interior point (test_solver.cpp:38-50)."""
    t = random_matrix_triplets(rng, rows, cols, 0.4)
    p = problem(rows, cols, t, rng.uniform(-1, 1, cols), np.zeros(rows), np.zeros(rows),
                np.zeros(cols), np.full(cols, 2.0))
    xhat = rng.uniform(0.5, 1.5, cols)
    A = dense(p)
    b = np.array([sum(p.a.by_row.value[k] * xhat[p.a.by_row.index[k]]
                      for k in range(p.a.by_row.start[r], p.a.by_row.start[r + 1]))
                  for r in range(rows)])
    p.con_lower = b.copy()
    p.con_upper = b.copy()
    del A
    return p


def slack_row_box_lp(rng, rows, cols):
    """test_solver.cpp:17-27; optimum is the separable box corner."""
    t = random_matrix_triplets(rng, rows, cols, 0.6)
    return problem(rows, cols, t, rng.uniform(-2, 2, cols), np.full(rows, -cols - 10.0),
                   np.full(rows, cols + 10.0), rng.uniform(-1.0, -0.1, cols),
                   rng.uniform(0.1, 1.0, cols))


def dense(p):
    A = np.zeros((p.rows(), p.cols()))
    L = p.a.by_row
    for r in range(p.rows()):
        for k in range(L.start[r], L.start[r + 1]):
            A[r, L.index[k]] += L.value[k]
    return A


def same_bits(a, b) -> bool:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return a.shape == b.shape and bool(np.all(a.view(np.int64) == b.view(np.int64)))


def max_rel(a, b) -> float:
    """Largest relative discrepancy between iterates: for each iterate (a row
    of a 2-D array) ||a_k - b_k||_inf / max(||a_k||_inf, ||b_k||_inf) -- a
    scale-free measure (no absolute floor); 0 when both are zero."""
    a = np.atleast_2d(np.asarray(a, np.float64))
    b = np.atleast_2d(np.asarray(b, np.float64))
    if a.size == 0:
        return 0.0
    num = np.max(np.abs(a - b), axis=1)
    den = np.maximum(np.max(np.abs(a), axis=1), np.max(np.abs(b), axis=1))
    rel = np.where(den > 0.0, num / np.where(den > 0.0, den, 1.0), 0.0)
    return float(np.max(rel))


def max_rel_elem(a, b, floor: float = 0.0) -> float:
    """Elementwise relative discrepancy |a-b| / max(|a|, |b|, floor)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    d = np.where(den > 0.0, np.abs(a - b) / np.where(den > 0.0, den, 1.0), 0.0)
    return float(np.max(d))
