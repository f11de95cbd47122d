"""B200-native PDLP/PDHG solver: a drop-in for the reference's pdhglp::solve.

Native code: libpdlp_b200.so (sm_100a kernels + C++ driver, C-ABI in
include/pdlp_b200.h) and libpdlp_gen.so (seeded BASELINE instances).  This
package is the Python mirror of the reference interface over that C-ABI.
"""
from .problem import (CompressedLayout, LpProblem, SparseMatrix, generate, generate_with_point,
                      problem, relative_tolerances)
from .solver import (CertificateKind, InfeasibilityCertificate, IterationRecord, ResidualSummary,
                     RestartThresholds, SolveResult, SolverOptions, SolveStatus,
                     TerminationTolerances, adaptive_step, apply_rescaling, device_count,
                     kkt_residuals, normalized_duality_gap, pdhg_step, pinned, pinned_copy,
                     pinned_empty, solve,
                     solve_status_name,
                     spmv, spmv_transpose, step_size_rules)

from .mps import MpsModel, parse_mps, read_mps, write_mps, write_mps_file
from .feasibility import FeasibilityRun, feasibility_residual, fixed_restart_feasibility

__all__ = [
    "FeasibilityRun", "feasibility_residual", "fixed_restart_feasibility",
    "MpsModel", "parse_mps", "read_mps", "write_mps", "write_mps_file",
    "CompressedLayout", "LpProblem", "SparseMatrix", "generate", "generate_with_point", "problem",
    "relative_tolerances", "CertificateKind", "InfeasibilityCertificate", "IterationRecord",
    "ResidualSummary", "RestartThresholds", "SolveResult", "SolverOptions", "SolveStatus",
    "TerminationTolerances", "adaptive_step", "apply_rescaling", "device_count", "kkt_residuals",
    "normalized_duality_gap", "pdhg_step", "solve", "solve_status_name", "spmv",
    "spmv_transpose", "step_size_rules",
]
