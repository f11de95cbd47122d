"""JSON result documents (the reference's make_document / solution_to_json /
solution_from_json, proj/include/pdhglp/solution_io.hpp:93-236).

The same ordered schema (schema_version 1): status, termination_detail,
sense, objective{primal, dual} in the user's sense, residuals, statistics,
optional certificate and solution arrays in minimization form; non-finite
numbers as the strings "inf" / "-inf" / "nan"; shortest round-trip floats.
"""
from __future__ import annotations

import json
import math

import numpy as np

from .solver import CertificateKind, SolveResult, solve_status_name

SCHEMA_VERSION = 1


def _enc(v: float):
    v = float(v)
    if math.isfinite(v):
        return v
    if math.isnan(v):
        return "nan"
    return "inf" if v > 0 else "-inf"


def _dec(v, where: str) -> float:
    if isinstance(v, bool):
        raise ValueError(f"solution file: bad number in {where}")
    if isinstance(v, (int, float)):
        return float(v)
    if v == "inf":
        return math.inf
    if v == "-inf":
        return -math.inf
    if v == "nan":
        return math.nan
    raise ValueError(f"solution file: bad number in {where}")


def _dec_vec(v, where: str) -> np.ndarray:
    if not isinstance(v, list):
        raise ValueError(f"solution file: {where} is not an array")
    return np.array([_dec(e, where) for e in v], dtype=np.float64)


def make_document(result: SolveResult, maximize: bool, include_solution: bool) -> dict:
    """solution_io.hpp:93-131: objectives in the stated sense, the rest in
    minimization form."""
    sign = -1.0 if maximize else 1.0
    s = result.summary
    doc = {
        "schema_version": SCHEMA_VERSION,
        "status": solve_status_name(result.status),
        "termination_detail": result.termination_detail,
        "sense": "max" if maximize else "min",
        "objective": {"primal": _enc(sign * s.primal_objective), "dual": _enc(sign * s.dual_objective)},
        "residuals": {"primal_inf": _enc(s.primal_residual_inf), "dual_inf": _enc(s.dual_residual_inf),
                      "abs_gap": _enc(s.abs_gap), "rel_gap": _enc(s.rel_gap)},
        "statistics": {"iterations": int(result.iterations),
                       "polish_iterations": int(result.polish_iterations),
                       "restarts": int(result.restarts), "step_retries": int(result.step_retries),
                       "solve_seconds": float(result.solve_seconds),
                       "final_step_size": _enc(result.final_step_size),
                       "final_primal_weight": _enc(result.final_primal_weight)},
    }
    c = result.certificate
    if c is not None:
        doc["certificate"] = {
            "kind": "primal_infeasible" if c.kind == CertificateKind.PRIMAL_INFEASIBLE
            else "dual_infeasible",
            "residual_inf": _enc(c.residual_inf), "objective": _enc(c.objective),
            "ray_x": [_enc(v) for v in c.ray_x], "ray_y": [_enc(v) for v in c.ray_y],
            "ray_r": [_enc(v) for v in c.ray_r]}
    if include_solution:
        doc["solution"] = {"x": [_enc(v) for v in result.x], "y": [_enc(v) for v in result.y],
                           "reduced_costs": [_enc(v) for v in result.reduced_costs]}
    return doc


def solution_to_json(doc: dict, indent: int = 2) -> str:
    return json.dumps(doc, indent=indent) + "\n"


def solution_from_json(text: str) -> dict:
    """solution_io.hpp:171-236, with its error messages.  Returns the document
    with numbers decoded (arrays as numpy)."""
    try:
        j = json.loads(text)
    except ValueError as e:
        raise ValueError(f"solution file: {e}") from None
    if not isinstance(j, dict):
        raise ValueError("solution file: top level is not an object")
    if j.get("schema_version", 0) != SCHEMA_VERSION:
        raise ValueError("solution file: unsupported schema_version")
    if not isinstance(j.get("status"), str):
        raise ValueError("solution file: missing status")
    d = {"schema_version": SCHEMA_VERSION, "status": j["status"],
         "termination_detail": j.get("termination_detail", ""),
         "maximize": j.get("sense", "min") == "max",
         "objective_primal": 0.0, "objective_dual": 0.0, "primal_residual_inf": 0.0,
         "dual_residual_inf": 0.0, "abs_gap": 0.0, "rel_gap": 0.0,
         "has_solution": False, "has_certificate": False}
    if "objective" in j:
        d["objective_primal"] = _dec(j["objective"]["primal"], "objective.primal")
        d["objective_dual"] = _dec(j["objective"]["dual"], "objective.dual")
    if "residuals" in j:
        r = j["residuals"]
        for k in ("primal_inf", "dual_inf"):
            d[f"{k.split('_')[0]}_residual_inf"] = _dec(r[k], f"residuals.{k}")
        d["abs_gap"] = _dec(r["abs_gap"], "residuals.abs_gap")
        d["rel_gap"] = _dec(r["rel_gap"], "residuals.rel_gap")
    if "statistics" in j:
        st = j["statistics"]
        for k in ("iterations", "polish_iterations", "restarts", "step_retries"):
            d[k] = int(st.get(k, 0))
        d["solve_seconds"] = float(st.get("solve_seconds", 0.0))
        if "final_step_size" in st:
            d["final_step_size"] = _dec(st["final_step_size"], "statistics.final_step_size")
        if "final_primal_weight" in st:
            d["final_primal_weight"] = _dec(st["final_primal_weight"],
                                            "statistics.final_primal_weight")
    if "certificate" in j:
        c = j["certificate"]
        d["has_certificate"] = True
        d["certificate_kind"] = c.get("kind", "")
        d["certificate_residual"] = _dec(c["residual_inf"], "certificate.residual_inf")
        d["certificate_objective"] = _dec(c["objective"], "certificate.objective")
        for k in ("ray_x", "ray_y", "ray_r"):
            d[k] = _dec_vec(c[k], f"certificate.{k}")
    if "solution" in j:
        s = j["solution"]
        d["has_solution"] = True
        d["x"] = _dec_vec(s["x"], "solution.x")
        d["y"] = _dec_vec(s["y"], "solution.y")
        d["reduced_costs"] = _dec_vec(s["reduced_costs"], "solution.reduced_costs")
    return d
