"""Window sort of the normalized duality gap's breakpoints (perf mode).

The gap (restarts.hpp:107-220) sweeps the breakpoint events in descending
lambda to the first crossing.  k_gap.cu's window path sorts only the events at
depth fractions [qa, qb] and enters the sweep with the summed masses of the
events above; it either decides (crossing inside) or falls back to the full
sort.  Either way the value must equal the full sort's to rounding: the only
difference is the summation order of the masses above the window.  The same
holds for the estimated window of a first evaluation.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2501_07018_b200 as P

# (-2, -2): the window estimated from a mass-carrying key sample (the first
# evaluation of a restart query)
WINDOWS = [(0.0, 0.1), (0.0, 0.45), (0.05, 0.3), (0.25, 0.5), (0.4, 0.6), (0.45, 0.55),
           (0.55, 0.8), (0.7, 0.99), (0.6, 1.0), (0.9995, 1.0), (-2.0, -2.0)]


@pytest.mark.gpu
def test_window_sort_matches_full_sort(gpu, monkeypatch):
    p = P.generate("c1", 0, sources=1100, sinks=1000)  # > 2^20 events
    rng = np.random.default_rng(7)
    x = np.clip(rng.uniform(-1, 3, p.cols()), p.var_lower, p.var_upper)
    y = rng.normal(size=p.rows())
    ax, aty = P.spmv(p, x, mode="perf"), P.spmv_transpose(p, y, mode="perf")
    for omega in (0.3, 2.0):
        for r in (1e-2, 1.0, 30.0, 1e3, 1e6):  # 1e6: no crossing
            monkeypatch.delenv("PDLP_GAP_WINDOW", raising=False)
            full = P.normalized_duality_gap(p, x, y, ax, aty, omega, r, mode="perf")
            for qa, qb in WINDOWS:
                monkeypatch.setenv("PDLP_GAP_WINDOW", f"{qa}:{qb}")
                g = P.normalized_duality_gap(p, x, y, ax, aty, omega, r, mode="perf")
                assert g == pytest.approx(full, rel=1e-12, abs=1e-300), (omega, r, qa, qb)
