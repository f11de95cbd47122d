#!/usr/bin/env python3
"""Measure the solver on BASELINE.json's larger configs at full size (one GPU).

  python tools/bench_configs.py [c2] [c3] [--steps K] [--warmup W] [--ttt-limit S]

For each config: seeded instance (csrc/gen/instances.cpp, host), then
  value        iterations/s over K timed iterations (tolerances unreachable,
               CUDA-event timed region of the main loop, inputs resident)
  per_kernel   CUDA-event mean per step kernel vs its algorithmic bytes
               (SURVEY 8(d)), against MEASURED_PEAKS.json hbm_gbs
  time_to_tol  solve to the 1e-4 relative KKT mapping, capped at --ttt-limit s
One JSON line per config on stdout.  bench.py stays the C1 contract line;
these are supporting measurements.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (step_kernel_bytes, peaks, options)
import paper_2501_07018_b200 as P  # noqa: E402


def measure(cfg: str, steps: int, warmup: int, ttt_limit: float) -> dict:
    t0 = time.perf_counter()
    extra = {}
    if cfg == "c4w":
        # C4 recipe, 1/8 row shard as a standalone LP (SURVEY 8(d) C4 row:
        # 18.75M x 300M, ~375M entries on one GPU); polishing off so the
        # polishing states of 300M columns are not reserved
        p = P.generate("c4", 0, row_window=(0, 150_000_000 // 8))
        extra = {"enable_polish": False}
    else:
        p = P.generate(cfg, 0)
    gen_s = time.perf_counter() - t0
    m, n, nnz = p.rows(), p.cols(), p.a.nonzeros()
    P.solve(p, bench._options(P, 8, 0, **extra))  # warm-up (module, pool, staging)
    res = P.solve(p, bench._options(P, steps, warmup, **extra))
    value = res.timed_iterations / res.timed_seconds
    prof = P.solve(p, bench._options(P, steps, warmup, profile_kernels=True, **extra))
    kb = bench.step_kernel_bytes(m, n, nnz, bench.uniform_vectors(p))
    peak, peak_src = bench._peaks()
    per = {}
    for q, nm in enumerate(["primal_pass", "row_pass", "col_pass"]):
        mean_s = prof.kernel_seconds[q] / max(prof.kernel_launches[q], 1)
        per[nm] = {"mean_us": mean_s * 1e6, "bytes": kb[nm], "gbs": kb[nm] / mean_s / 1e9,
                   "frac": kb[nm] / mean_s / 1e9 / peak}
    att_s = sum(prof.kernel_seconds[:3]) / max(prof.kernel_launches[0], 1)
    step_bytes = sum(kb.values())
    tol = P.relative_tolerances(p)
    ttt = P.solve(p, P.SolverOptions(tolerances=P.TerminationTolerances(*tol),
                                     iteration_limit=1_000_000, time_limit_seconds=ttt_limit,
                                     **extra))
    return {
        "config": cfg, "m": m, "n": n, "nnz": nnz, "generate_seconds": gen_s,
        "value": value, "unit": "iters/s", "steps": steps, "warmup": warmup,
        "ms_per_iteration": 1e3 / value, "timed_attempts": res.timed_attempts,
        "upload_seconds": res.upload_seconds, "precondition_seconds": res.precondition_seconds,
        "per_kernel": per,
        "step": {"bytes_per_attempt": step_bytes, "kernel_time_us_per_attempt": att_s * 1e6,
                 "gbs": step_bytes / att_s / 1e9, "frac": step_bytes / att_s / 1e9 / peak},
        "peak_gbs": peak, "peak_source": peak_src,
        "time_to_tol": {"status": P.solve_status_name(ttt.status), "seconds": ttt.solve_seconds,
                        "iterations": ttt.iterations, "polish_iterations": ttt.polish_iterations,
                        "restarts": ttt.restarts, "limit_seconds": ttt_limit,
                        "primal_residual": ttt.summary.primal_residual_inf,
                        "dual_residual": ttt.summary.dual_residual_inf,
                        "rel_gap": ttt.summary.rel_gap, "tolerances": list(tol)},
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c3"])
    ap.add_argument("--steps", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--ttt-limit", type=float, default=120.0)
    a = ap.parse_args()
    for cfg in a.configs:
        print(json.dumps(measure(cfg, a.steps, a.warmup, a.ttt_limit)), flush=True)


if __name__ == "__main__":
    main()
