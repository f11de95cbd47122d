"""bench.py's algorithmic byte model and its uniform-vector
rule: the roofline is computed on what the step kernels must move."""
from __future__ import annotations

import numpy as np

import bench
import paper_2501_07018_b200 as P


def test_step_bytes_c1_formula():
    m, n, nnz = 4000, 4_000_000, 8_000_000
    kb = bench.step_kernel_bytes(m, n, nnz)
    assert kb["primal_pass"] == 72 * n
    assert kb["row_pass"] == 12 * nnz + 4 * (m + 1) + 8 * n + 56 * m
    assert kb["col_pass"] == 12 * nnz + 4 * (n + 1) + 8 * m + 32 * n
    # x >= 0 everywhere: l_v and u_v are read as scalars
    assert bench.step_kernel_bytes(m, n, nnz, 2)["primal_pass"] == 56 * n


def test_uniform_vectors_rule():
    p = P.generate("c1", 0, sources=20, sinks=30)       # l_v = 0, u_v = inf
    assert bench.uniform_vectors(p) == 2
    q = P.generate("c0", 0, rows=50, cols=80)           # l_v = 0, u_v = 10 (scaled: not uniform)
    assert bench.uniform_vectors(q) == 1
    q.var_lower[3] = -0.0                                # bitwise different from +0.0
    assert bench.uniform_vectors(q) == 0
    r = P.generate("c1", 0, sources=20, sinks=30)
    r.objective[:] = 0.0                                 # zero objective: uniform too
    assert bench.uniform_vectors(r) == 3
    assert np.all(r.objective == 0.0)
