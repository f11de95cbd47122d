"""ctypes mirror of include/pdlp_b200.h and include/pdlp_gen.h.

Loads the in-tree libpdlp_b200.so / libpdlp_gen.so (built by build.py).  A
missing library is an ImportError-grade failure: there is no Python or CPU
fallback for the solver path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PDLP_LIB: an alternative build of the same library (tuning sweeps only)
LIB_PATH = os.environ.get("PDLP_LIB") or os.path.join(HERE, "libpdlp_b200.so")
GEN_LIB_PATH = os.path.join(HERE, "libpdlp_gen.so")

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)
c_int32_p = C.POINTER(C.c_int32)

PDLP_OK = 0
PDLP_ERR_INVALID_PROBLEM = -1
PDLP_ERR_INVALID_ARGUMENT = -2
PDLP_ERR_CUDA = -3
PDLP_ERR_OUT_OF_MEMORY = -4
PDLP_ERR_INTERNAL = -5

MODE_PERF = 0
MODE_PARITY = 1


class CsrView(C.Structure):
    _fields_ = [
        ("primary_dim", C.c_int64),
        ("nnz", C.c_int64),
        ("start", c_int64_p),
        ("index", c_int64_p),
        ("value", c_double_p),
    ]


class ProblemView(C.Structure):
    _fields_ = [
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("by_row", CsrView),
        ("by_col", CsrView),
        ("objective", c_double_p),
        ("con_lower", c_double_p),
        ("con_upper", c_double_p),
        ("var_lower", c_double_p),
        ("var_upper", c_double_p),
    ]


class IterationRecord(C.Structure):
    _fields_ = [
        ("iteration", C.c_int64),
        ("x", c_double_p),
        ("x_len", C.c_int64),
        ("y", c_double_p),
        ("y_len", C.c_int64),
        ("eta", C.c_double),
        ("omega", C.c_double),
    ]


OBSERVER_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(IterationRecord))


class Options(C.Structure):
    _fields_ = [
        ("eps_primal", C.c_double),
        ("eps_dual", C.c_double),
        ("eps_rel_gap", C.c_double),
        ("iteration_limit", C.c_int64),
        ("time_limit_seconds", C.c_double),
        ("threads", C.c_int32),
        ("shards_per_thread", C.c_int32),
        ("enable_scaling", C.c_int32),
        ("ruiz_passes", C.c_int32),
        ("pock_chambolle", C.c_int32),
        ("enable_polish", C.c_int32),
        ("enable_restarts", C.c_int32),
        ("detect_infeasibility", C.c_int32),
        ("eps_ray", C.c_double),
        ("check_interval", C.c_int64),
        ("restart_sufficient", C.c_double),
        ("restart_necessary", C.c_double),
        ("restart_artificial", C.c_double),
        ("has_fixed_step_size", C.c_int32),
        ("has_fixed_primal_weight", C.c_int32),
        ("fixed_step_size", C.c_double),
        ("fixed_primal_weight", C.c_double),
        ("logging", C.c_int32),
        ("_pad0", C.c_int32),
        ("observer", OBSERVER_FN),
        ("observer_user", C.c_void_p),
        ("mode", C.c_int32),
        ("device", C.c_int32),
        ("reserved0", C.c_int32),
        ("profile_kernels", C.c_int32),
        ("timing_warmup_iterations", C.c_int64),
    ]


class ResidualSummary(C.Structure):
    _fields_ = [
        ("primal_residual_inf", C.c_double),
        ("dual_residual_inf", C.c_double),
        ("primal_objective", C.c_double),
        ("dual_objective", C.c_double),
        ("abs_gap", C.c_double),
        ("rel_gap", C.c_double),
    ]


class Result(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("has_certificate", C.c_int32),
        ("x", c_double_p),
        ("y", c_double_p),
        ("reduced_costs", c_double_p),
        ("summary", ResidualSummary),
        ("cert_kind", C.c_int32),
        ("_pad0", C.c_int32),
        ("cert_ray_x", c_double_p),
        ("cert_ray_y", c_double_p),
        ("cert_ray_r", c_double_p),
        ("cert_residual_inf", C.c_double),
        ("cert_objective", C.c_double),
        ("cert_source", C.c_char * 32),
        ("iterations", C.c_int64),
        ("polish_iterations", C.c_int64),
        ("restarts", C.c_int64),
        ("step_retries", C.c_int64),
        ("final_step_size", C.c_double),
        ("final_primal_weight", C.c_double),
        ("min_step_size_limit", C.c_double),
        ("solve_seconds", C.c_double),
        ("termination_detail", C.c_char * 256),
        ("attempts", C.c_int64),
        ("upload_seconds", C.c_double),
        ("precondition_seconds", C.c_double),
        ("loop_seconds", C.c_double),
        ("step_seconds", C.c_double),
        ("timed_seconds", C.c_double),
        ("timed_iterations", C.c_int64),
        ("timed_attempts", C.c_int64),
        ("kernel_seconds", C.c_double * 4),
        ("kernel_launches", C.c_int64 * 4),
    ]


class GenParams(C.Structure):
    _fields_ = [
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("count_kind", C.c_int32),
        ("value_kind", C.c_int32),
        ("count_fixed", C.c_int64),
        ("alpha", C.c_double),
        ("kmin", C.c_int64),
        ("kmax", C.c_int64),
        ("value_lo", C.c_double),
        ("value_hi", C.c_double),
        ("eq_frac", C.c_double),
        ("eq_rows_first", C.c_int32),
        ("bound_kind", C.c_int32),
        ("box_hi", C.c_double),
        ("slack_hi", C.c_double),
        ("seed", C.c_uint64),
    ]


class ShardPlan(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("row_block", C.c_int64),
        ("col_block", C.c_int64),
        ("row_begin", C.c_int64),
        ("row_end", C.c_int64),
        ("col_begin", C.c_int64),
        ("col_end", C.c_int64),
        ("cut", C.c_int32),
        ("_pad", C.c_int32),
    ]


class ShardView(C.Structure):
    _fields_ = [
        ("plan", ShardPlan),
        ("rows", CsrView),
        ("cols", CsrView),
        ("objective", c_double_p),
        ("var_lower", c_double_p),
        ("var_upper", c_double_p),
        ("con_lower", c_double_p),
        ("con_upper", c_double_p),
        ("entry_offset", C.c_int64),
        ("row_entry_offset", C.POINTER(C.c_int64)),
    ]


# Every symbol include/pdlp_b200.h declares, with its ctypes signature.
SOLVER_SIGNATURES = {
    "pdlp_default_options": (None, [C.POINTER(Options)]),
    "pdlp_solve": (C.c_int, [C.POINTER(ProblemView), C.POINTER(Options), C.POINTER(Result)]),
    "pdlp_last_error": (C.c_char_p, []),
    "pdlp_abi_version": (C.c_int, []),
    "pdlp_device_count": (C.c_int, []),
    "pdlp_trim_device_memory": (C.c_int, [C.c_int]),
    "pdlp_host_register": (C.c_int, [C.c_void_p, C.c_size_t]),
    "pdlp_host_unregister": (C.c_int, [C.c_void_p]),
    "pdlp_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "pdlp_host_free": (C.c_int, [C.c_void_p]),
    "pdlp_gap_dist_stats": (None, [C.POINTER(C.c_int64), c_double_p, C.c_int32]),
    "pdlp_shard_plan_for": (C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                      C.POINTER(ShardPlan)]),
    "pdlp_shard_extract": (C.c_int, [C.POINTER(ProblemView), C.c_int32, C.c_int32,
                                     C.POINTER(ShardView), C.POINTER(C.c_void_p)]),
    "pdlp_shard_extract_cut": (C.c_int, [C.POINTER(ProblemView), C.c_int32, C.c_int32, C.c_int32,
                                         C.POINTER(ShardView), C.POINTER(C.c_void_p)]),
    "pdlp_shard_free": (None, [C.c_void_p]),
    "pdlp_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "pdlp_check_certificate": (C.c_int, [C.POINTER(ProblemView), C.c_int32, c_double_p, C.c_double,
                                         C.POINTER(C.c_int32), c_double_p, c_double_p]),
    "pdlp_feasibility_run": (C.c_int, [C.POINTER(ProblemView), c_double_p, c_double_p, C.c_double,
                                       C.c_int64, C.c_int32, C.c_int32, C.c_int32, c_double_p,
                                       c_double_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "pdlp_mps_parse": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "pdlp_mps_read_file": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "pdlp_mps_view": (None, [C.c_void_p, C.POINTER(ProblemView)]),
    "pdlp_mps_maximize": (C.c_int32, [C.c_void_p]),
    "pdlp_mps_name": (C.c_char_p, [C.c_void_p]),
    "pdlp_mps_objective_name": (C.c_char_p, [C.c_void_p]),
    "pdlp_mps_row_name": (C.c_char_p, [C.c_void_p, C.c_int64]),
    "pdlp_mps_col_name": (C.c_char_p, [C.c_void_p, C.c_int64]),
    "pdlp_mps_free": (None, [C.c_void_p]),
    "pdlp_mps_write": (C.c_int, [C.POINTER(ProblemView), C.c_char_p, C.c_int32,
                                 C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "pdlp_mps_free_text": (None, [C.c_void_p]),
    "pdlp_solve_sharded": (C.c_int, [C.POINTER(ProblemView), C.POINTER(Options), C.c_int32,
                                     C.c_int32, C.c_char_p, C.POINTER(Result)]),
    "pdlp_solve_sharded_emulated": (C.c_int, [C.POINTER(ProblemView), C.POINTER(Options),
                                              C.c_int32, C.POINTER(Result)]),
    "pdlp_solve_sharded_local": (C.c_int, [C.POINTER(ShardView), C.POINTER(Options), C.c_int32,
                                           C.c_int32, C.c_char_p, C.POINTER(Result)]),
    "pdlp_solve_sharded_local_emulated": (C.c_int, [C.POINTER(C.POINTER(ShardView)),
                                                    C.POINTER(Options), C.c_int32,
                                                    C.POINTER(Result)]),
    "pdlp_pdhg_step": (C.c_int, [C.POINTER(ProblemView), c_double_p, c_double_p, C.c_double,
                                 C.c_double, C.c_int32, C.c_int32, c_double_p, c_double_p,
                                 c_int32_p]),
    "pdlp_adaptive_step": (C.c_int, [C.POINTER(ProblemView), c_double_p, c_double_p, c_double_p,
                                     c_double_p, C.c_int32, C.c_int32, c_double_p, c_double_p,
                                     c_double_p, c_int32_p]),
    "pdlp_spmv": (C.c_int, [C.POINTER(ProblemView), c_double_p, c_double_p, C.c_int32]),
    "pdlp_spmv_transpose": (C.c_int, [C.POINTER(ProblemView), c_double_p, c_double_p, C.c_int32]),
    "pdlp_apply_rescaling": (C.c_int, [C.POINTER(ProblemView), C.c_int32, C.c_int32] + [c_double_p] * 9),
    "pdlp_normalized_duality_gap": (C.c_int, [C.POINTER(ProblemView), c_double_p, c_double_p,
                                              c_double_p, c_double_p, C.c_double, C.c_double,
                                              C.c_int32, c_double_p]),
    "pdlp_kkt_residuals": (C.c_int, [C.POINTER(ProblemView), c_double_p, c_double_p, C.c_int32,
                                     C.c_int32, c_double_p, C.POINTER(ResidualSummary)]),
    "pdlp_step_size_rules": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int64,
                                       c_double_p, c_double_p]),
}

GEN_SIGNATURES = {
    "pdlp_gen_c0_params": (None, [C.POINTER(GenParams), C.c_uint64]),
    "pdlp_gen_c2_params": (None, [C.POINTER(GenParams), C.c_uint64]),
    "pdlp_gen_c4_params": (None, [C.POINTER(GenParams), C.c_uint64]),
    "pdlp_gen_random_lp": (C.c_void_p, [C.POINTER(GenParams)]),
    "pdlp_gen_random_lp_window": (C.c_void_p, [C.POINTER(GenParams), C.c_int64, C.c_int64]),
    "pdlp_gen_transport": (C.c_void_p, [C.c_int64, C.c_int64, C.c_uint64]),
    "pdlp_gen_unit_commitment": (C.c_void_p, [C.c_int64, C.c_int64, C.c_uint64]),
    "pdlp_instance_from_triplets": (C.c_void_p, [C.c_int64, C.c_int64, C.c_int64, c_int64_p,
                                                 c_int64_p, c_double_p] + [c_double_p] * 5),
    "pdlp_instance_view": (None, [C.c_void_p, C.POINTER(ProblemView)]),
    "pdlp_instance_feasible_point": (c_double_p, [C.c_void_p]),
    "pdlp_instance_free": (None, [C.c_void_p]),
    "pdlp_gen_random_lp_shard": (C.c_void_p, [C.POINTER(GenParams), C.c_int64, C.c_int64,
                                               C.c_int64, C.c_int64]),
    "pdlp_gen_random_lp_colshard": (C.c_void_p, [C.POINTER(GenParams), C.c_int64, C.c_int64,
                                               C.c_int64, C.c_int64]),
    "pdlp_gen_shard_view": (None, [C.c_void_p, C.POINTER(ShardView)]),
    "pdlp_gen_shard_free": (None, [C.c_void_p]),
}


def _bind(lib: C.CDLL, sigs: dict) -> C.CDLL:
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None
_gen = None


def lib() -> C.CDLL:
    """The solver library.  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -m paper_2501_07018_b200.build` "
                "(there is no CPU fallback)")
        _lib = _bind(C.CDLL(LIB_PATH), SOLVER_SIGNATURES)
    return _lib


def gen() -> C.CDLL:
    global _gen
    if _gen is None:
        if not os.path.exists(GEN_LIB_PATH):
            raise ImportError(f"{GEN_LIB_PATH} is missing: run `python -m paper_2501_07018_b200.build`")
        _gen = _bind(C.CDLL(GEN_LIB_PATH), GEN_SIGNATURES)
    return _gen


def last_error() -> str:
    return lib().pdlp_last_error().decode()
