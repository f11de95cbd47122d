"""Command line front end (the reference's tools/main.cpp):

    python -m paper_2501_07018_b200 solve model.mps [--out result.json] ...
    python -m paper_2501_07018_b200 check model.mps result.json
    python -m paper_2501_07018_b200 generate --kind c0 --seed 1 [--out model.mps]

`solve` and `check` take the reference's options and keep its output (the
JSON document of solution_io.hpp, the check report lines) and exit codes:
solve 0 optimal, 2 infeasible or unbounded, 3 iteration/time limit,
4 numerical failure, 5 input error; check 0 all verified, 1 a verification
failed, 5 input error.  The solve runs on the GPU; `check` recomputes the
residuals and re-tests certificates on the GPU (original space).  `generate`
emits this repo's seeded BASELINE recipes (c0..c4, transport,
unit-commitment) rather than the reference's test-instance kinds.
"""
from __future__ import annotations

import argparse
import math
import sys

from .problem import generate as _generate
from .mps import read_mps, write_mps
from .solution_io import make_document, solution_from_json, solution_to_json
from .solver import (SolveStatus, SolverOptions, TerminationTolerances, check_certificate,
                     kkt_residuals_given, solve)

EXIT_OPTIMAL, EXIT_VERIFY_FAIL, EXIT_INFEASIBLE, EXIT_LIMIT, EXIT_NUMERICAL, EXIT_INPUT = 0, 1, 2, 3, 4, 5


def exit_code_for(status: SolveStatus) -> int:
    if status == SolveStatus.OPTIMAL:
        return EXIT_OPTIMAL
    if status in (SolveStatus.PRIMAL_INFEASIBLE, SolveStatus.DUAL_INFEASIBLE):
        return EXIT_INFEASIBLE
    if status in (SolveStatus.ITERATION_LIMIT, SolveStatus.TIME_LIMIT):
        return EXIT_LIMIT
    return EXIT_NUMERICAL


def _g(v: float) -> str:
    """C++ ostream default formatting (6 significant digits)."""
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%g" % v


def run_solve(a) -> int:
    try:
        model = read_mps(a.input)
    except ValueError as e:
        print(f"error: {a.input}: {e}", file=sys.stderr)
        return EXIT_INPUT
    o = SolverOptions(tolerances=TerminationTolerances(a.eps_primal, a.eps_dual, a.rel_gap),
                      iteration_limit=a.iters, threads=a.threads, enable_polish=not a.no_polish,
                      enable_scaling=not a.no_scaling, enable_restarts=not a.no_restarts,
                      detect_infeasibility=not a.no_detect, logging=not a.quiet,
                      mode=a.mode, device=a.device)
    if a.time_limit > 0.0:
        o.time_limit_seconds = a.time_limit
    if a.fixed_step is not None:
        o.fixed_step_size = a.fixed_step
    if a.fixed_weight is not None:
        o.fixed_primal_weight = a.fixed_weight
    try:
        result = solve(model.problem, o)
    except Exception as e:  # noqa: BLE001 - the reference reports any failure the same way
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    doc = make_document(result, model.maximize, not a.no_solution)
    text = solution_to_json(doc)
    if a.out:
        try:
            with open(a.out, "w") as f:
                f.write(text)
        except OSError:
            print(f"error: cannot write '{a.out}'", file=sys.stderr)
            return EXIT_INPUT
    else:
        sys.stdout.write(text)
    if not a.quiet:
        print(f"status={doc['status']} objective={doc['objective']['primal']:.12g} "
              f"iterations={result.iterations} seconds={result.solve_seconds:.3f}", file=sys.stderr)
    return exit_code_for(result.status)


def _close(got: float, want: float, rel: float) -> bool:
    if not (math.isfinite(got) and math.isfinite(want)):
        return (math.isnan(got) and math.isnan(want)) or got == want
    return abs(got - want) <= rel * max(1.0, abs(want))


def run_check(a) -> int:
    try:
        model = read_mps(a.input)
    except ValueError as e:
        print(f"error: {a.input}: {e}", file=sys.stderr)
        return EXIT_INPUT
    try:
        with open(a.solution) as f:
            text = f.read()
    except OSError:
        print(f"error: cannot open '{a.solution}'", file=sys.stderr)
        return EXIT_INPUT
    try:
        doc = solution_from_json(text)
    except (ValueError, KeyError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    p = model.problem
    state = {"ok": True, "any": False}

    def report(what: str, ok: bool, detail: str) -> None:
        print(f"{what}: {'ok' if ok else 'FAIL'}{' ' if detail else ''}{detail}")
        state["ok"] = state["ok"] and ok
        state["any"] = True

    if doc["maximize"] != model.maximize:
        report("objective sense matches the model", False,
               "(solution says max, model says min)" if doc["maximize"]
               else "(solution says min, model says max)")
    if doc["has_solution"]:
        if len(doc["x"]) != p.cols() or len(doc["y"]) != p.rows() or len(doc["reduced_costs"]) != p.cols():
            print("error: solution array sizes do not match the model", file=sys.stderr)
            return EXIT_INPUT
        s = kkt_residuals_given(p, doc["x"], doc["y"], doc["reduced_costs"])
        sign = -1.0 if model.maximize else 1.0
        report("reported primal residual matches",
               _close(s.primal_residual_inf, doc["primal_residual_inf"], a.consistency),
               f"(reported {_g(doc['primal_residual_inf'])}, recomputed {_g(s.primal_residual_inf)})")
        report("reported dual residual matches",
               _close(s.dual_residual_inf, doc["dual_residual_inf"], a.consistency),
               f"(reported {_g(doc['dual_residual_inf'])}, recomputed {_g(s.dual_residual_inf)})")
        report("reported objective matches",
               _close(sign * s.primal_objective, doc["objective_primal"], a.consistency),
               f"(reported {_g(doc['objective_primal'])}, recomputed {_g(sign * s.primal_objective)})")
        if doc["status"] == "optimal":
            ok = (s.primal_residual_inf <= a.eps_primal and s.dual_residual_inf <= a.eps_dual
                  and s.rel_gap <= a.rel_gap)
            report("point satisfies the optimality tolerances", ok,
                   f"(primal {_g(s.primal_residual_inf)}, dual {_g(s.dual_residual_inf)}, "
                   f"rel_gap {_g(s.rel_gap)})")
    if doc["has_certificate"]:
        kind = doc["certificate_kind"]
        if kind not in ("primal_infeasible", "dual_infeasible"):
            print(f"error: unknown certificate kind '{kind}'", file=sys.stderr)
            return EXIT_INPUT
        primal = kind == "primal_infeasible"
        ray = doc["ray_y"] if primal else doc["ray_x"]
        if len(ray) != (p.rows() if primal else p.cols()):
            print("error: certificate ray size does not match the model", file=sys.stderr)
            return EXIT_INPUT
        ok, res, obj = check_certificate(p, 0 if primal else 1, ray, a.eps_ray)
        report(f"{'primal' if primal else 'dual'} infeasibility certificate verifies", ok,
               f"(ray objective {_g(obj)}, residual {_g(res)})" if ok else "")
    if not state["any"]:
        print("error: solution file carries neither arrays nor a certificate", file=sys.stderr)
        return EXIT_INPUT
    return 0 if state["ok"] else EXIT_VERIFY_FAIL


def run_generate(a) -> int:
    kw = {}
    if a.kind in ("c0", "c2", "c4"):
        if a.rows:
            kw["rows"] = a.rows
        if a.cols:
            kw["cols"] = a.cols
    elif a.kind == "transport":
        kw = {"sources": a.rows or 50, "sinks": a.cols or 100}
    elif a.kind == "unit-commitment":
        kw = {"periods": a.rows or 24, "generators": a.cols or 10}
    cfg = {"transport": "c1", "unit-commitment": "c3"}.get(a.kind, a.kind)
    try:
        p = _generate(cfg, a.seed, **kw)
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    text = write_mps(p, f"{a.kind}-{p.rows()}x{p.cols()}-s{a.seed}")
    if a.out:
        try:
            with open(a.out, "w") as f:
                f.write(text)
        except OSError:
            print(f"error: cannot write '{a.out}'", file=sys.stderr)
            return EXIT_INPUT
    else:
        sys.stdout.write(text)
    return 0


def parser() -> argparse.ArgumentParser:
    d = TerminationTolerances()
    ap = argparse.ArgumentParser(prog="python -m paper_2501_07018_b200",
                                 description="B200 PDLP solver (drop-in for the reference CLI)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="Solve an MPS model and emit JSON")
    s.add_argument("input")
    s.add_argument("--eps-primal", type=float, default=d.eps_primal)
    s.add_argument("--eps-dual", type=float, default=d.eps_dual)
    s.add_argument("--rel-gap", type=float, default=d.eps_rel_gap)
    s.add_argument("--iters", type=int, default=SolverOptions().iteration_limit)
    s.add_argument("--time-limit", type=float, default=0.0)
    s.add_argument("--threads", type=int, default=1)
    for flag in ("--no-polish", "--no-scaling", "--no-restarts", "--no-detect", "--no-solution",
                 "--quiet"):
        s.add_argument(flag, action="store_true")
    s.add_argument("--out", default="")
    s.add_argument("--fixed-step", type=float, default=None)
    s.add_argument("--fixed-weight", type=float, default=None)
    s.add_argument("--mode", choices=["perf", "parity"], default="perf")
    s.add_argument("--device", type=int, default=0)
    c = sub.add_parser("check", help="Verify a solution file against its model")
    c.add_argument("input")
    c.add_argument("solution")
    c.add_argument("--eps-primal", type=float, default=d.eps_primal)
    c.add_argument("--eps-dual", type=float, default=d.eps_dual)
    c.add_argument("--rel-gap", type=float, default=d.eps_rel_gap)
    c.add_argument("--consistency", type=float, default=1e-6)
    c.add_argument("--eps-ray", type=float, default=1e-12)
    g = sub.add_parser("generate", help="Emit a seeded benchmark instance as MPS")
    g.add_argument("--kind", default="c0",
                   choices=["c0", "c2", "c4", "transport", "unit-commitment"])
    g.add_argument("--rows", type=int, default=0)
    g.add_argument("--cols", type=int, default=0)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--out", default="")
    return ap


def main(argv=None) -> int:
    a = parser().parse_args(argv)
    return {"solve": run_solve, "check": run_check, "generate": run_generate}[a.cmd](a)
