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

Shard-local ingest (no host holds the whole problem):
    generate_shard(config, seed, rank, world)   one rank's shard of the
        counter-based random-LP instance (libpdlp_gen pdlp_gen_random_lp_shard)
    solve_distributed_local(shard, options)     under torch.distributed
    solve_sharded_local(shard, options, rank, world, nccl_id)
    solve_sharded_local_emulated(shards, options)
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
    cut: str = "rows"  # "rows": K_g = the rank's rows; "cols": its columns


CUTS = {"rows": 0, "cols": 1}


def _plan(p: N.ShardPlan) -> ShardPlan:
    return ShardPlan(p.rank, p.world, p.rows, p.cols, p.row_block, p.col_block, p.row_begin,
                     p.row_end, p.col_begin, p.col_end, "cols" if p.cut == 1 else "rows")


def shard_plan(rows: int, cols: int, rank: int, world: int) -> ShardPlan:
    out = N.ShardPlan()
    _check(N.lib().pdlp_shard_plan_for(rows, cols, rank, world, C.byref(out)))
    return _plan(out)


def _arr(ptr, n: int, dtype) -> np.ndarray:
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def extract_shard(problem: LpProblem, rank: int, world: int, cut: str | None = None) -> dict:
    """Host-side shard of one rank (copies): the rows / cols layouts in CSR
    form plus the rank's vector blocks; cut "rows" / "cols" (default: the
    one pdlp_shard_plan_for picks).  CPU only."""
    view = problem.view()
    out = N.ShardView()
    owner = C.c_void_p()
    if cut is None:
        _check(N.lib().pdlp_shard_extract(C.byref(view), rank, world, C.byref(out), C.byref(owner)))
    else:
        _check(N.lib().pdlp_shard_extract_cut(C.byref(view), rank, world, CUTS[cut], C.byref(out),
                                              C.byref(owner)))
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
                "entry_offset": out.entry_offset,
                "row_entry_offset": _arr(out.row_entry_offset,
                                         out.rows.primary_dim if pl.cut == "cols" else 0, np.int64)}
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


def gap_dist_stats(reset: bool = False) -> dict:
    """Counters of the distributed normalized gap (process-wide): evaluations,
    bracket-search rounds, events swept after the search, evaluations
    compared with the gathered gap (PDLP_GAPD_CHECK=1) and the largest
    relative difference seen there."""
    out = (C.c_int64 * 4)()
    mx = (C.c_double * 2)()
    N.lib().pdlp_gap_dist_stats(out, mx, 1 if reset else 0)
    return {"evals": out[0], "rounds": out[1], "final_events": out[2], "checked": out[3],
            "max_rel": mx[0], "max_rel_lambda": mx[1]}


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


# ------------------------------------------------------ shard-local ingest ---
class LocalShard:
    """One rank's shard, owned by the generator library: K_g (global column
    indices), K_g^T (all columns, local rows), the row bounds and the column
    block's objective and bounds (kernels.h / pdlp_b200.h pdlp_shard_view)."""

    def __init__(self, handle, plan: N.ShardPlan):
        self._h = handle
        self.view = N.ShardView()
        N.gen().pdlp_gen_shard_view(handle, C.byref(self.view))
        self.view.plan = plan
        self.plan = _plan(plan)

    def __del__(self):
        if getattr(self, "_h", None):
            N.gen().pdlp_gen_shard_free(self._h)
            self._h = None

    def vectors(self) -> dict:
        """Copies of the shard's vectors (no layouts)."""
        v, pl = self.view, self.plan
        ml, nl = pl.row_end - pl.row_begin, pl.col_end - pl.col_begin
        return {"objective": _arr(v.objective, nl, np.float64),
                "var_lower": _arr(v.var_lower, nl, np.float64),
                "var_upper": _arr(v.var_upper, nl, np.float64),
                "con_lower": _arr(v.con_lower, ml, np.float64),
                "con_upper": _arr(v.con_upper, ml, np.float64)}

    def as_dict(self) -> dict:
        """Copies of the shard's arrays (the layout of extract_shard)."""
        v, pl = self.view, self.plan
        ml, nl = pl.row_end - pl.row_begin, pl.col_end - pl.col_begin

        def csr(c):
            return {"dim": c.primary_dim, "nnz": c.nnz,
                    "start": _arr(c.start, c.primary_dim + 1, np.int64),
                    "index": _arr(c.index, c.nnz, np.int64),
                    "value": _arr(c.value, c.nnz, np.float64)}

        return {"plan": pl, "rows": csr(v.rows), "cols": csr(v.cols),
                "objective": _arr(v.objective, nl, np.float64),
                "var_lower": _arr(v.var_lower, nl, np.float64),
                "var_upper": _arr(v.var_upper, nl, np.float64),
                "con_lower": _arr(v.con_lower, ml, np.float64),
                "con_upper": _arr(v.con_upper, ml, np.float64),
                "entry_offset": v.entry_offset}


def generate_shard(config: str, seed: int, rank: int, world: int, cut: str = "rows",
                   **overrides) -> LocalShard:
    """Rank `rank` of `world`'s shard of the counter-based instance
    generate(config, seed, row_window=(0, rows), **overrides) -- built without
    the rest of the instance (C0 / C2 / C4 recipes); cut "rows" (K_g = the
    rank's rows) or "cols" (the rank's columns), "auto" = pdlp_shard_plan_for's."""
    cfg = config.lower()
    if cfg not in ("c0", "c2", "c4"):
        raise ValueError("shard-local generation exists for the random-LP recipes c0, c2, c4")
    prm = N.GenParams()
    getattr(N.gen(), f"pdlp_gen_{cfg}_params")(C.byref(prm), seed)
    for k, val in overrides.items():
        setattr(prm, k, val)
    plan = N.ShardPlan()
    _check(N.lib().pdlp_shard_plan_for(prm.rows, prm.cols, rank, world, C.byref(plan)))
    if cut != "auto":
        plan.cut = CUTS[cut]
    fn = N.gen().pdlp_gen_random_lp_colshard if plan.cut == CUTS["cols"] else \
        N.gen().pdlp_gen_random_lp_shard
    h = fn(C.byref(prm), plan.row_begin, plan.row_end, plan.col_begin, plan.col_end)
    if not h:
        raise ValueError("bad shard ranges")
    return LocalShard(h, plan)


def solve_sharded_local(shard: LocalShard, options: SolverOptions | None, rank: int, world: int,
                        nccl_id: bytes) -> SolveResult:
    options = options or SolverOptions(mode="perf")
    _quiet_nccl()
    if len(nccl_id) != 128:
        raise ValueError("nccl_id must be the 128-byte ncclUniqueId")
    return run_solve(N.lib(), "pdlp_solve_sharded_local", None, options, to_c_options(options),
                     extra=(rank, world, C.c_char_p(nccl_id)), first_arg=C.byref(shard.view),
                     dims=(shard.plan.rows, shard.plan.cols))


def solve_sharded_local_emulated(shards: list, options: SolverOptions | None) -> SolveResult:
    options = options or SolverOptions(mode="perf")
    arr = (C.POINTER(N.ShardView) * len(shards))(*[C.pointer(sh.view) for sh in shards])
    return run_solve(N.lib(), "pdlp_solve_sharded_local_emulated", None, options,
                     to_c_options(options), extra=(len(shards),), first_arg=arr,
                     dims=(shards[0].plan.rows, shards[0].plan.cols))


def solve_distributed_local(shard: LocalShard, options: SolverOptions | None = None,
                            group=None) -> SolveResult:
    """solve_distributed with each rank passing only its own shard."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    options = options or SolverOptions(mode="perf")
    options.device = int(os.environ.get("LOCAL_RANK", options.device))
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return solve_sharded_local(shard, options, rank, world, obj[0])
