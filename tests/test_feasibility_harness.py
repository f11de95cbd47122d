"""Appendix-B fixed-restart feasibility harness.

The reference's harness is proj/tests/feasibility_method.hpp:40-85
(testharness::fixed_restart_feasibility), exercised by acceptance criterion 10
(proj/tests/acceptance.cpp:700-795).  The restatement in oracle/pdlp_oracle.cpp
is pinned bit for bit to the reference's own harness (compiled in oracle/_ref);
the device harness (pdlp_feasibility_run) is pinned bit for bit to the oracle
in parity mode and reproduces criterion 10's properties: geometric decay of
the restart residuals (log-linear fit, slope < 0, R^2 > 0.9) and restart
excursions within 14x the distance from x0 to {x : A x = b}.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2501_07018_b200 as P
from tests.helpers import dense, random_matrix_triplets, same_bits


def _system(seed: int, rows: int = 20, cols: int = 40, density: float = 0.25):
    """A consistent system A x = b with a strictly positive solution, and a
    start within 0.01 of it (criterion 10's setup, own generator)."""
    rng = np.random.default_rng(seed)
    t = random_matrix_triplets(rng, rows, cols, density)
    xs = rng.uniform(0.1, 1.1, cols)
    p = P.problem(rows, cols, t, np.zeros(cols), np.zeros(rows), np.zeros(rows),
                  np.zeros(cols), np.full(cols, np.inf))
    b = dense(p) @ xs
    p.con_lower[:] = b
    p.con_upper[:] = b
    x0 = xs + rng.uniform(-0.01, 0.01, cols)
    return p, b, x0


def _eta(p) -> float:
    """1 / (2 sigma_max(A)) (criterion 10 uses a power-iteration lower bound
    of sigma_max; the exact value keeps eta * sigma <= 1/2)."""
    s = np.linalg.svd(dense(p), compute_uv=False)
    return 1.0 / (2.0 * float(s[0])) if s.size and s[0] > 0 else 1.0


@pytest.fixture(scope="module")
def refimpl():
    import oracle
    try:
        return oracle.reference()
    except FileNotFoundError:
        pytest.skip("compiled reference (oracle/_ref) not built")


@pytest.fixture(scope="module")
def port():
    import oracle
    return oracle.port()


def _ref_systems(refimpl, seeds=range(1, 21)):
    """Criterion 10's instances: the reference's FeasibilitySystem kind at
    20 x 40, density 0.25, x0 = the planted point + U(-0.01, 0.01)."""
    for seed in seeds:
        p, pt = refimpl.generate_feasibility_system(20, 40, 0.25, seed)
        rng = np.random.default_rng(seed)
        yield p, p.con_lower.copy(), pt + rng.uniform(-0.01, 0.01, pt.shape[0])


# ----------------------------------------------------------------- CPU ---
def test_restatement_matches_reference_harness(refimpl, port):
    for p, b, x0 in _ref_systems(refimpl, range(1, 9)):
        eta = _eta(p)
        a = refimpl.feasibility_run(p, b, x0, eta, 500, 25)
        c = port.feasibility_run(p, b, x0, eta, 500, 25)
        assert a[2] and c[2]
        assert same_bits(a[0], c[0]) and same_bits(a[1], c[1])


@pytest.mark.parametrize("case", ["diverges", "one-step-rounds", "no-rounds", "ragged"])
def test_restatement_edge_cases(refimpl, port, case):
    if case == "ragged":
        p, b, x0 = _system(3, rows=7, cols=31, density=0.4)
    else:
        p, b, x0 = _system(4)
    eta, length, rounds = _eta(p), 500, 6
    if case == "diverges":
        eta *= 400.0  # far past 1/sigma: the averages blow up to inf / nan
        rounds = 60
    elif case == "one-step-rounds":
        length = 1
    elif case == "no-rounds":
        rounds = 0
    a = refimpl.feasibility_run(p, b, x0, eta, length, rounds)
    c = port.feasibility_run(p, b, x0, eta, length, rounds)
    assert a[2] == c[2] and a[0].shape == c[0].shape
    assert same_bits(a[0], c[0]) and same_bits(a[1], c[1])
    if case == "diverges":
        assert not a[2]


# ----------------------------------------------------------------- GPU ---
@pytest.mark.gpu
def test_device_harness_is_bit_exact(gpu, ref):
    cases = [_system(s) for s in (1, 2)] + [_system(5, rows=7, cols=31, density=0.4)]
    cases.append(_system(6, rows=300, cols=700, density=0.02))
    for p, b, x0 in cases:
        eta = _eta(p)
        want = ref.feasibility_run(p, b, x0, eta, 500, 8)
        got = P.fixed_restart_feasibility(p, b, x0, eta, 500, 8)
        assert got.finite == want[2]
        assert same_bits(got.restart_points, want[0])
        assert same_bits(got.residuals, want[1])


@pytest.mark.gpu
@pytest.mark.parametrize("length,rounds,scale", [(1, 5, 1.0), (65, 3, 1.0), (130, 2, 1.0),
                                                 (500, 0, 1.0), (50, 40, 400.0)])
def test_device_harness_edges(gpu, ref, length, rounds, scale):
    """Graph chunking (64-step bodies + tails), zero rounds, and a diverging
    run that stops at the first non-finite restart point."""
    p, b, x0 = _system(7)
    eta = _eta(p) * scale
    want = ref.feasibility_run(p, b, x0, eta, length, rounds)
    got = P.fixed_restart_feasibility(p, b, x0, eta, length, rounds)
    assert got.finite == want[2] and got.restart_points.shape == want[0].shape
    assert same_bits(got.restart_points, want[0]) and same_bits(got.residuals, want[1])


@pytest.mark.gpu
def test_device_harness_perf_mode_tracks_parity(gpu):
    p, b, x0 = _system(8, rows=400, cols=900, density=0.02)
    eta = _eta(p)
    a = P.fixed_restart_feasibility(p, b, x0, eta, 200, 6, mode="parity")
    c = P.fixed_restart_feasibility(p, b, x0, eta, 200, 6, mode="perf")
    scale = np.max(np.abs(a.restart_points))
    assert np.max(np.abs(a.restart_points - c.restart_points)) <= 1e-9 * scale
    np.testing.assert_allclose(c.residuals, a.residuals, rtol=1e-6, atol=1e-12 * (1 + np.linalg.norm(b)))


def _fit(logs):
    t = np.arange(len(logs), dtype=float)
    slope, icpt = np.polyfit(t, logs, 1)
    pred = slope * t + icpt
    ss_res = float(np.sum((logs - pred) ** 2))
    ss_tot = float(np.sum((logs - np.mean(logs)) ** 2))
    return slope, (1.0 - ss_res / ss_tot) if ss_tot > 0 else 1.0


@pytest.mark.gpu
def test_criterion10_properties_on_device(gpu):
    """Acceptance criterion 10 (acceptance.cpp:700-795) on the device harness:
    20 consistent 20 x 40 systems, eta = 1/(2 sigma), 25 rounds of 500 steps."""
    try:
        import oracle
        systems = list(_ref_systems(oracle.reference()))
    except FileNotFoundError:
        systems = [_system(s) for s in range(1, 21)]
    for p, b, x0 in systems:
        A = dense(p)
        eta = _eta(p)
        run = P.fixed_restart_feasibility(p, b, x0, eta, 500, 25)
        assert run.finite
        # distance oracle: projection of x0 onto {x : A x = b} (interior here)
        u = np.linalg.solve(A @ A.T, A @ x0 - b)
        xp = x0 - A.T @ u
        assert np.max(np.abs(A @ xp - b)) <= 1e-9 and xp.min() >= 0.0
        dist = np.linalg.norm(x0 - xp)
        ratios = [np.linalg.norm(pt - x0) / dist for pt in run.restart_points]
        assert max(ratios) <= 14.0 * (1 + 1e-4)
        floor = 1e-12 * (1.0 + np.linalg.norm(b))
        logs = []
        for r in run.residuals:
            logs.append(np.log10(max(r, 1e-300)))
            if r <= floor:
                break
        if len(logs) < 3:
            assert run.residuals[len(logs) - 1] <= floor  # too fast to fit
            continue
        slope, r2 = _fit(np.array(logs))
        assert slope < 0.0 and r2 > 0.9
