#!/usr/bin/env python3
"""Benchmark: PDHG iterations/sec of the B200 solver on BASELINE.json configs[1]
(C1: 2000x2000 transportation LP, m=4,000, n=4M, nnz=8M, fp64).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one accepted PDHG iteration of the reference loop
(proj/include/pdhglp/solver.hpp:475-529) including its share of the 64-step
cadence (restart tests, residual screens, ray checks).  Tolerances are set
unreachable so every run does identical work; W untimed iterations, then
exactly K timed iterations, timed on the device with CUDA events (the
solver's timed region).  Every iteration streams ~656 MB (> 126 MB L2), so
no L2 flush is needed between iterations.

Line keys beyond the base contract:
  e2e          same metric through the C-ABI pdlp_solve() from host buffers
               (H2D of the problem, preconditioning, K iterations, D2H of x/y/r)
  roofline     dominant step kernel: algorithmic bytes per launch / mean CUDA-
               event launch time vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline the compiled reference (oracle/_ref) on this host's cores
  time_to_tol  C1 solved to BASELINE's 1e-4 relative KKT (SURVEY §8(d) mapping)
Multi-GPU (torchrun, N > 1): ONE C1 solve row-sharded over the N GPUs
(paper_2501_07018_b200.sharded): rank g owns rows
[g*mb, (g+1)*mb) of A in both layouts and the column block [g*nb, (g+1)*nb);
per attempt x-bar is all-gathered, K_g^T dy reduce-scattered and 5 step
scalars all-gathered over NCCL.  Total work is fixed, so scaling = "strong"
and value = iterations/s of that one solve, timed as the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# stdout carries exactly one JSON line: NCCL prints its version banner (and
# any log) at every NCCL_DEBUG level from VERSION up, so its output goes to
# stderr instead; the level itself is left as the environment sets it.
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

METRIC = "PDHG iters/sec, time to 1e-4 rel. KKT, achieved HBM GB/s vs peak"
UNIT = "iters/s"
WORKLOAD = "C1 transport 2000x2000 (m=4000, n=4,000,000, nnz=8,000,000), fp64"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def uniform_vectors(p) -> int:
    """How many of c, l_v, u_v the solver reads as a scalar: bitwise uniform
    and 0 or +-inf (the only uniform values column scaling keeps uniform)."""
    import numpy as np
    k = 0
    for v in (p.objective, p.var_lower, p.var_upper):
        b = v.view(np.int64)
        if b.size and np.all(b == b[0]) and (v[0] == 0.0 or np.isinf(v[0])):
            k += 1
    return k


def step_kernel_bytes(m: int, n: int, nnz: int, uniform: int = 0) -> dict:
    """Algorithmic bytes per launch of each perf-mode step kernel (SURVEY.md
    §8(d) dataflow: every array touched once; int32 indices/row pointers).
    uniform: vectors among c, l_v, u_v the primal pass takes as a scalar."""
    return {
        # R x, c, aty, l_v, u_v; W x', xbar; R+W sum_x (deferred average)
        "primal_pass": 8 * (9 - uniform) * n,
        # CSR(K) 12 nnz + 4(m+1); gather xbar once (8n); R y, l_c, u_c; W y', dy; R+W sum_y
        "row_pass": 12 * nnz + 4 * (m + 1) + 8 * n + 8 * 7 * m,
        # CSR(K^T) 12 nnz + 4(n+1); gather dy once (8m); R aty, x, x'; W aty'
        "col_pass": 12 * nnz + 4 * (n + 1) + 8 * m + 8 * 4 * n,
    }


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed work."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, under_load_mhz: float = 900.0) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                s = float(parts[0])
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            if s >= under_load_mhz:
                sm.append(s)
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(self.lines),
                "samples_under_load": len(sm)}


def _options(P, k: int, w: int, **kw):
    o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0), iteration_limit=w + k,
                        timing_warmup_iterations=w, mode="perf")
    for key, val in kw.items():
        setattr(o, key, val)
    return o


def problem_bytes(p) -> int:
    a = p.a
    b = 0
    for L in (a.by_row, a.by_col):
        b += L.start.nbytes + L.index.nbytes + L.value.nbytes
    return b + sum(v.nbytes for v in (p.objective, p.con_lower, p.con_upper, p.var_lower, p.var_upper))


def cpu_reference_rate(p, iterations: int, threads: int) -> dict:
    """Reference (oracle/_ref, else the restatement) on the host cores:
    iterations/sec between the first and last observed iteration (excludes
    its setup and rescaling, like the GPU value)."""
    import oracle
    import paper_2501_07018_b200 as P
    R = oracle.get()
    stamps = []
    o = P.SolverOptions(tolerances=P.TerminationTolerances(0.0, 0.0, 0.0),
                        iteration_limit=iterations, threads=threads, shards_per_thread=4)
    o.observer = lambda rec: stamps.append((rec.iteration, time.perf_counter()))
    t0 = time.perf_counter()
    R.solve(p, o)
    wall = time.perf_counter() - t0
    (k0, t_0), (k1, t_1) = stamps[0], stamps[-1]
    rate = (k1 - k0) / (t_1 - t_0) if t_1 > t_0 else 0.0
    return {"value": rate, "unit": UNIT, "cores": threads,
            "kind": "reference" if R.name == "reference" else "port",
            "sample": f"C1 full size, iterations {k0}..{k1} of a {iterations}-iteration run "
                      f"(tolerances unreachable), threads={threads} x 4 shards; "
                      f"whole call incl. setup {wall:.1f}s"}


def run_ours(args) -> None:
    import paper_2501_07018_b200 as P

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local if world > 1 else 0

    # every rank builds the same instance; the sharded solve keeps its shard
    p = P.generate("c1", 0, sources=args.sources, sinks=args.sinks)
    m, n, nnz = p.rows(), p.cols(), p.a.nonzeros()
    K, W = args.steps, args.warmup
    if world > 1 or args.sharded:
        from paper_2501_07018_b200 import sharded as S
        if dist is None:  # --sharded at N=1: the same path over a 1-rank NCCL communicator
            solve = lambda o: S.solve_sharded(p, o, 0, 1, S.nccl_unique_id())  # noqa: E731
        else:
            solve = lambda o: S.solve_distributed(p, o)  # noqa: E731
    else:
        solve = lambda o: P.solve(p, o)  # noqa: E731

    # untimed warm-up solve (context, module load, allocator, NCCL init)
    solve(_options(P, 64, 0, device=device))

    if dist is not None:
        dist.barrier()
    with ClockSampler(device) as clocks:
        res = solve(_options(P, K, W, device=device))
    timed = res.timed_seconds
    if dist is not None:
        import torch
        t = torch.tensor([timed], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        timed = float(t.item())
    value = res.timed_iterations / timed  # one solve (sharded when N > 1)

    # e2e: through the C-ABI from host buffers, K iterations, wall clock
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_res = solve(_options(P, K, 0, device=device))
    e2e_wall = time.perf_counter() - t0
    if dist is not None:
        import torch
        t = torch.tensor([e2e_wall], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_wall = float(t.item())
    e2e_value = e2e_res.iterations / e2e_wall

    kb = step_kernel_bytes(m, n, nnz, uniform_vectors(p))
    names = ["primal_pass", "row_pass", "col_pass"]
    per = {}
    if world == 1 and not args.sharded:
        # kernel roofline from an instrumented run (CUDA events per launch)
        prof = P.solve(p, _options(P, K, W, device=device, profile_kernels=True))
        for q, nm in enumerate(names):
            launches = max(prof.kernel_launches[q], 1)
            mean_s = prof.kernel_seconds[q] / launches
            per[nm] = {"mean_us": mean_s * 1e6, "bytes": kb[nm],
                       "gbs": kb[nm] / mean_s / 1e9 if mean_s > 0 else 0.0}
        total_kernel_s = sum(prof.kernel_seconds[:3])
        dom = max(names, key=lambda nm: prof.kernel_seconds[names.index(nm)])
        attempts_prof = max(prof.kernel_launches[0], 1)
    else:
        # sharded: per-GPU share of the algorithmic step bytes over the
        # measured time per attempt (collectives included in the time)
        t_att = timed / max(res.timed_attempts, 1)
        share = sum(kb.values()) / world
        per["sharded_attempt"] = {"mean_us": t_att * 1e6, "bytes": share, "gbs": share / t_att / 1e9}
        total_kernel_s, dom, attempts_prof = t_att, "sharded_attempt", 1
    peak, peak_src = _peaks()
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_json):
        try:
            traffic = json.load(open(prof_json)).get(dom)
        except Exception:
            traffic = None
    step_bytes = sum(kb.values()) / world
    attempt_s = total_kernel_s / attempts_prof

    # time to BASELINE's 1e-4 relative KKT (SURVEY §8(d) mapping), polishing on
    # Run twice: the first solve in a process that polishes maps the polishing
    # states' memory (0.01-0.3 s on a freshly acquired box); the second is
    # the warm number reported, the first is kept as cold_seconds.
    tol = P.relative_tolerances(p)
    ttt_opts = P.SolverOptions(tolerances=P.TerminationTolerances(*tol), iteration_limit=100000,
                               device=device)
    ttt_cold = solve(ttt_opts)
    ttt = solve(ttt_opts)

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_rate(p, args.cpu_iterations, os.cpu_count() or 1)
        except Exception as e:  # the checker is optional on the box; say why
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    # primal, row, column passes per attempt (one GPU); sharded attempts add
    # the partial product, column epilogue, totals and decision kernels
    launches = res.timed_attempts * (3 if (world == 1 and not args.sharded) else 6)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": 1e3 * timed / max(res.timed_iterations, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C1 transportation recipe of BASELINE.json configs[1])",
        "config": {"workload": WORKLOAD, "m": m, "n": n, "nnz": nnz, "mode": "perf",
                   "parallelism": f"rowshard{world}" if (world > 1 or args.sharded) else "single",
                   "l2": "inputs larger than L2 (656 MB streamed per iteration)",
                   "tolerances": "unreachable (fixed-work window)",
                   "timed_attempts": res.timed_attempts, "restarts": res.restarts},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": problem_bytes(p) / K,
                "d2h_bytes_per_step": 8 * (2 * n + m) / K,
                "note": f"pdlp_solve() wall time from host buffers for K={K} iterations: "
                        f"wall {e2e_wall:.3f}s = upload+validation {e2e_res.upload_seconds:.3f}s + "
                        f"preconditioning {e2e_res.precondition_seconds:.3f}s + loop "
                        f"{e2e_res.loop_seconds:.3f}s + rest (init, result copy, teardown)"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": per[dom]["gbs"], "peak": peak,
                     "unit": "GB/s", "frac": per[dom]["gbs"] / peak, "traffic": traffic,
                     "peak_source": peak_src, "per_kernel": per,
                     "step": {"bytes_per_attempt": step_bytes,
                              "kernel_time_us_per_attempt": attempt_s * 1e6,
                              "gbs": step_bytes / attempt_s / 1e9 if attempt_s > 0 else 0.0,
                              "frac": step_bytes / attempt_s / 1e9 / peak if attempt_s > 0 else 0.0}},
        "time_to_tol": {"status": P.solve_status_name(ttt.status), "seconds": ttt.solve_seconds,
                        "loop_seconds": ttt.loop_seconds, "step_seconds": ttt.step_seconds,
                        "upload_seconds": ttt.upload_seconds, "iterations": ttt.iterations,
                        "polish_iterations": ttt.polish_iterations,
                        "cold_seconds": ttt_cold.solve_seconds,
                        "tolerance": "1e-4 relative (eps_p=1e-4(1+|b|inf), eps_d=1e-4(1+|c|inf))"},
        "gpu_launches": launches,
        "gpu_launches_note": (f"the step kernels only ({launches // max(res.timed_attempts, 1)} per "
                              "attempt, counted exactly); the cadence's "
                              "reductions, products, gap and CUB sort/scan kernels add about 0.6 "
                              "launches per step kernel (profiles/r1_launches_v6.md)"),
        "clocks": clocks.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    emit(line)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args) -> None:
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    compiled from /root/reference) on this host's cores, same config/metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2501_07018_b200 as P
    p = P.generate("c1", 0, sources=args.sources, sinks=args.sinks)
    threads = os.cpu_count() or 1
    iters = max(args.warmup, 3) + min(args.steps, args.ref_iterations)
    cpu = cpu_reference_rate(p, iters, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": UNIT,
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded C1 transportation recipe of BASELINE.json configs[1])",
        "config": {"workload": WORKLOAD, "bounded_sample_iterations": iters},
        "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


# stdout carries exactly one JSON line.  Libraries print on the C-level
# stdout too (NCCL's version banner at NCCL_DEBUG=VERSION/WARN goes there
# whatever NCCL_DEBUG_FILE says), so fd 1 points at stderr for the whole run
# and is restored only to print the line.
_REAL_STDOUT = None


def _stdout_to_stderr() -> None:
    global _REAL_STDOUT
    sys.stdout.flush()
    _REAL_STDOUT = os.dup(1)
    os.dup2(2, 1)


def emit(line: dict) -> None:
    sys.stdout.flush()
    if _REAL_STDOUT is not None:
        os.dup2(_REAL_STDOUT, 1)
    print(json.dumps(line), flush=True)


def main():
    _stdout_to_stderr()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2048)
    ap.add_argument("--warmup", type=int, default=64)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--sources", type=int, default=2000)
    ap.add_argument("--sinks", type=int, default=2000)
    ap.add_argument("--cpu-iterations", type=int, default=96)
    ap.add_argument("--ref-iterations", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the row-sharded solve even at N=1 (1-rank NCCL communicator)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
