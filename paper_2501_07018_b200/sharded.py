"""Row-sharded multi-GPU solve over the C-ABI.

One process per GPU (torchrun).  Rank g owns rows [row_begin, row_end) of A
in both layouts (K_g, and K_g^T = those rows' entries of every column) plus
the primal block [col_begin, col_end).  Per PDHG attempt the ranks exchange
x-bar (all-gather), the partial K_g^T dy (reduce-scatter to the column
owners) and 5 step scalars (all-gather); every rank takes the same
accept/reject, restart and termination decisions.  The reference solve is
single-process (solver.hpp:535-608); this is the B200 extension of it.

    solve_distributed(problem, options)   under torch.distributed (NCCL)
    solve_sharded(problem, options, rank, world, nccl_id)
    solve_sharded_emulated(problem, options, world)
        the same sharded program with `world` ranks as threads sharing this
        process's GPU (collectives = host barriers + device copies): checks
        the sharded path where fewer GPUs than ranks exist.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .problem import LpProblem
from .solver import SolveResult, SolverOptions, _check, run_solve, to_c_options


@dataclass
class ShardPlan:
    rank: int
    world: int
    rows: int
    cols: int
    row_block: int
    col_block: int
    row_begin: int
    row_end: int
    col_begin: int
    col_end: int


def _plan(p: N.ShardPlan) -> ShardPlan:
    return ShardPlan(p.rank, p.world, p.rows, p.cols, p.row_block, p.col_block, p.row_begin,
                     p.row_end, p.col_begin, p.col_end)


def shard_plan(rows: int, cols: int, rank: int, world: int) -> ShardPlan:
    out = N.ShardPlan()
    _check(N.lib().pdlp_shard_plan_for(rows, cols, rank, world, C.byref(out)))
    return _plan(out)


def _arr(ptr, n: int, dtype) -> np.ndarray:
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def extract_shard(problem: LpProblem, rank: int, world: int) -> dict:
    """Host-side shard of one rank (copies): K_g and K_g^T in CSR form plus
    the rank's vector blocks.  CPU only."""
    view = problem.view()
    out = N.ShardView()
    owner = C.c_void_p()
    _check(N.lib().pdlp_shard_extract(C.byref(view), rank, world, C.byref(out), C.byref(owner)))
    try:
        pl = _plan(out.plan)
        ml, nl = pl.row_end - pl.row_begin, pl.col_end - pl.col_begin

        def csr(v):
            return {"dim": v.primary_dim, "nnz": v.nnz,
                    "start": _arr(v.start, v.primary_dim + 1, np.int64),
                    "index": _arr(v.index, v.nnz, np.int64),
                    "value": _arr(v.value, v.nnz, np.float64)}

        return {"plan": pl, "rows": csr(out.rows), "cols": csr(out.cols),
                "objective": _arr(out.objective, nl, np.float64),
                "var_lower": _arr(out.var_lower, nl, np.float64),
                "var_upper": _arr(out.var_upper, nl, np.float64),
                "con_lower": _arr(out.con_lower, ml, np.float64),
                "con_upper": _arr(out.con_upper, ml, np.float64),
                "entry_offset": out.entry_offset}
    finally:
        N.lib().pdlp_shard_free(owner)


def _quiet_nccl() -> None:
    # NCCL prints its version banner (and logs) on stdout at every NCCL_DEBUG
    # level from VERSION up: send them to stderr, keep the level
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


def nccl_unique_id() -> bytes:
    _quiet_nccl()
    buf = C.create_string_buffer(128)
    _check(N.lib().pdlp_nccl_unique_id(buf))
    return buf.raw


def solve_sharded(problem: LpProblem, options: SolverOptions | None, rank: int, world: int,
                  nccl_id: bytes) -> SolveResult:
    """This process's rank of a `world`-GPU sharded solve (NCCL).  Every
    rank gets the whole result."""
    options = options or SolverOptions(mode="perf")
    _quiet_nccl()
    if len(nccl_id) != 128:
        raise ValueError("nccl_id must be the 128-byte ncclUniqueId")
    return run_solve(N.lib(), "pdlp_solve_sharded", problem, options, to_c_options(options),
                     extra=(rank, world, C.c_char_p(nccl_id)))


def solve_sharded_emulated(problem: LpProblem, options: SolverOptions | None,
                           world: int) -> SolveResult:
    options = options or SolverOptions(mode="perf")
    return run_solve(N.lib(), "pdlp_solve_sharded_emulated", problem, options,
                     to_c_options(options), extra=(world,))


def solve_distributed(problem: LpProblem, options: SolverOptions | None = None,
                      group=None) -> SolveResult:
    """Sharded solve across the ranks of torch.distributed (one GPU each,
    device = LOCAL_RANK).  torch.distributed only carries the ncclUniqueId;
    the solver's collectives run on its own NCCL communicator."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    options = options or SolverOptions(mode="perf")
    options.device = int(os.environ.get("LOCAL_RANK", options.device))
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return solve_sharded(problem, options, rank, world, obj[0])
