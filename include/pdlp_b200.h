/*
 * pdlp_b200.h — C-ABI of the B200-native PDLP/PDHG solver (libpdlp_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (`pdhglp`, header-only C++20) has no FFI of its own; its entry point is
 *
 *     pdhglp::SolveResult pdhglp::solve(const LpProblem&, const SolverOptions&)
 *         (reference: proj/include/pdhglp/solver.hpp:535-608)
 *
 * and every struct below mirrors one of the reference's structs field for
 * field, with plain pointers and sizes instead of std::vector:
 *
 *   pdlp_csr_view            <- pdhglp::CompressedLayout      sparse.hpp:21-28
 *   pdlp_problem_view        <- pdhglp::LpProblem + SparseMatrix problem.hpp:15-25, sparse.hpp:33-42
 *   pdlp_options             <- pdhglp::SolverOptions          solver.hpp:69-90
 *                               (+ TerminationTolerances residuals.hpp:187-191,
 *                                  RestartThresholds restarts.hpp:235-239)
 *   pdlp_iteration_record    <- pdhglp::IterationRecord        solver.hpp:59-65
 *   pdlp_residual_summary    <- pdhglp::ResidualSummary        residuals.hpp:66-73
 *   pdlp_result              <- pdhglp::SolveResult            solver.hpp:92-108
 *                               (+ InfeasibilityCertificate residuals.hpp:202-210)
 *
 * The C++ drop-in (include/pdhglp_b200/solver.hpp) marshals the reference's
 * own structs onto these and calls pdlp_solve(); see INTEGRATION.md.
 *
 * Conventions: 0 = OK, negative = error (pdlp_last_error() has the text).
 * No C++ exception crosses this boundary.  Host arrays are borrowed for the
 * duration of the call only.  All indices are int64 on the host side (as in
 * the reference); the device copy uses int32 column indices.
 *
 * There is NO CPU fallback: every entry point that computes runs CUDA
 * kernels on the selected device and fails with PDLP_ERR_CUDA when no
 * device is usable.
 */
#ifndef PDLP_B200_H_
#define PDLP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDLP_ABI_VERSION 1

/* Error codes. */
#define PDLP_OK 0
#define PDLP_ERR_INVALID_PROBLEM -1 /* reference: std::invalid_argument, solver.hpp:538-541 */
#define PDLP_ERR_INVALID_ARGUMENT -2
#define PDLP_ERR_CUDA -3
#define PDLP_ERR_OUT_OF_MEMORY -4
#define PDLP_ERR_INTERNAL -5

/* SolveStatus, same order as reference solver.hpp:35-42. */
#define PDLP_STATUS_OPTIMAL 0
#define PDLP_STATUS_PRIMAL_INFEASIBLE 1
#define PDLP_STATUS_DUAL_INFEASIBLE 2
#define PDLP_STATUS_ITERATION_LIMIT 3
#define PDLP_STATUS_TIME_LIMIT 4
#define PDLP_STATUS_NUMERICAL_ERROR 5

/* CertificateKind, reference residuals.hpp:200. */
#define PDLP_CERT_PRIMAL_INFEASIBLE 0
#define PDLP_CERT_DUAL_INFEASIBLE 1

/* Execution modes (B200 extension, additive to SolverOptions). */
#define PDLP_MODE_PERF 0   /* load-balanced SpMV + tree reductions (deterministic) */
#define PDLP_MODE_PARITY 1 /* bit-exact emulation of the reference's shard plan   */

/* One compressed orientation (reference CompressedLayout, sparse.hpp:21-28). */
typedef struct pdlp_csr_view {
  int64_t primary_dim; /* rows for by_row, cols for by_col */
  int64_t nnz;
  const int64_t* start; /* primary_dim + 1 */
  const int64_t* index; /* nnz, sorted within each line */
  const double* value;  /* nnz */
} pdlp_csr_view;

/* min c'x  s.t.  con_lower <= A x <= con_upper, var_lower <= x <= var_upper
 * (reference LpProblem, problem.hpp:15-25; matrix held in both layouts as in
 * SparseMatrix, sparse.hpp:33-42). */
typedef struct pdlp_problem_view {
  int64_t rows;
  int64_t cols;
  pdlp_csr_view by_row;
  pdlp_csr_view by_col;
  const double* objective; /* cols */
  const double* con_lower; /* rows */
  const double* con_upper; /* rows */
  const double* var_lower; /* cols */
  const double* var_upper; /* cols */
} pdlp_problem_view;

/* Reference IterationRecord (solver.hpp:59-65).  x/y are host copies of the
 * scaled-space iterate, valid only during the callback. */
typedef struct pdlp_iteration_record {
  int64_t iteration;
  const double* x;
  int64_t x_len;
  const double* y;
  int64_t y_len;
  double eta;
  double omega;
} pdlp_iteration_record;

typedef void (*pdlp_observer_fn)(void* user, const pdlp_iteration_record* rec);

/* Reference SolverOptions (solver.hpp:69-90) flattened; defaults via
 * pdlp_default_options(). */
typedef struct pdlp_options {
  /* TerminationTolerances, residuals.hpp:187-191 */
  double eps_primal;
  double eps_dual;
  double eps_rel_gap;
  int64_t iteration_limit;
  double time_limit_seconds; /* +inf = none */
  int32_t threads;
  int32_t shards_per_thread;
  int32_t enable_scaling;
  int32_t ruiz_passes;
  int32_t pock_chambolle;
  int32_t enable_polish;
  int32_t enable_restarts;
  int32_t detect_infeasibility;
  double eps_ray;
  int64_t check_interval;
  /* RestartThresholds, restarts.hpp:235-239 */
  double restart_sufficient;
  double restart_necessary;
  double restart_artificial;
  int32_t has_fixed_step_size;
  int32_t has_fixed_primal_weight;
  double fixed_step_size;
  double fixed_primal_weight;
  int32_t logging;
  int32_t _pad0;
  pdlp_observer_fn observer;
  void* observer_user;
  /* ---- B200 extensions (additive; the reference fields above are unchanged) */
  int32_t mode;   /* PDLP_MODE_PERF (default) or PDLP_MODE_PARITY */
  int32_t device; /* CUDA device ordinal */
  int32_t reserved0; /* reserved, must be 0 (keeps the struct layout) */
  int32_t profile_kernels; /* CUDA events around every step kernel (bench roofline) */
  /* Timed region of the main loop starts once this many iterations are done
   * (right after that cadence); see pdlp_result.timed_*.  0 = whole loop. */
  int64_t timing_warmup_iterations;
} pdlp_options;

/* Reference ResidualSummary, residuals.hpp:66-73. */
typedef struct pdlp_residual_summary {
  double primal_residual_inf;
  double dual_residual_inf;
  double primal_objective;
  double dual_objective;
  double abs_gap;
  double rel_gap;
} pdlp_residual_summary;

/* Reference SolveResult (solver.hpp:92-108) + InfeasibilityCertificate
 * (residuals.hpp:202-210).  Vector outputs go to caller-owned buffers; any of
 * them may be NULL to skip the copy. */
typedef struct pdlp_result {
  int32_t status;
  int32_t has_certificate;
  double* x;             /* cols */
  double* y;             /* rows */
  double* reduced_costs; /* cols */
  pdlp_residual_summary summary;
  /* certificate */
  int32_t cert_kind;
  int32_t _pad0;
  double* cert_ray_x; /* cols (dual infeasible) */
  double* cert_ray_y; /* rows (primal infeasible) */
  double* cert_ray_r; /* cols (primal infeasible) */
  double cert_residual_inf;
  double cert_objective;
  char cert_source[32];
  /* statistics */
  int64_t iterations;
  int64_t polish_iterations;
  int64_t restarts;
  int64_t step_retries;
  double final_step_size;
  double final_primal_weight;
  double min_step_size_limit;
  double solve_seconds;
  char termination_detail[256];
  /* B200 extensions: timing breakdown */
  int64_t attempts;           /* step attempts (accepted + retries), main + polish */
  double upload_seconds;      /* host->device copy of the problem */
  double precondition_seconds;
  double loop_seconds;        /* wall time inside run_inner (main loop) */
  double step_seconds;        /* device time of the step kernels only (CUDA events) */
  double timed_seconds;       /* CUDA-event time of the timed region (main loop) */
  int64_t timed_iterations;   /* accepted main-loop steps inside it */
  int64_t timed_attempts;     /* step attempts inside it */
  /* profile_kernels: summed device time and launch count per step kernel:
   * [0] primal pass, [1] row pass (+dual update), [2] column pass (+decision),
   * [3] parity-mode reductions/decision */
  double kernel_seconds[4];
  int64_t kernel_launches[4];
} pdlp_result;

/* ---------------------------------------------------------------- solve --- */

/* Defaults equal to the reference's SolverOptions{} (solver.hpp:69-90). */
void pdlp_default_options(pdlp_options* opt);

/* The drop-in: reference pdhglp::solve (solver.hpp:535-608). */
int pdlp_solve(const pdlp_problem_view* problem, const pdlp_options* options,
               pdlp_result* result);

const char* pdlp_last_error(void);
int pdlp_abi_version(void);
/* Number of CUDA devices visible, or a negative error code. */
int pdlp_device_count(void);
/* B200 extension.  Solves allocate from the device's stream-ordered memory
 * pool and keep it between calls (no map/unmap per solve); this returns the
 * pool's unused memory on `device` to the driver.  0 or a negative error. */
int pdlp_trim_device_memory(int device);
/* B200 extension.  Page-lock caller memory (cudaHostRegister, portable) for
 * the solves that read or write it: a problem's arrays registered this way
 * upload with one DMA each (64-bit indices narrowed on the device) instead of
 * through the pinned staging ring's host copies; registered result buffers
 * are filled by DMA.  Unregister before freeing the memory. */
int pdlp_host_register(void* ptr, size_t bytes);
int pdlp_host_unregister(void* ptr);
/* B200 extension.  Page-locked host allocation (cudaHostAlloc, portable) for
 * a caller that builds its problem or result buffers in pinned memory
 * directly (where registering existing pages is not permitted). */
int pdlp_host_alloc(size_t bytes, void** out);
int pdlp_host_free(void* ptr);
/* B200 extension.  Counters of the sharded solves' distributed normalized
 * gap (restarts.hpp:107-220 evaluated without gathering a vector, DESIGN.md
 * §8): out[0..3] = evaluations, bracket-search rounds, events swept after
 * the search, evaluations compared with the gathered one (PDLP_GAPD_CHECK=1);
 * max_rel[0] / max_rel[1] = the largest relative difference seen there in
 * the gap value / in lambda* (max_rel holds 2 doubles).  reset != 0 zeroes
 * them after reading.  Process-wide. */
void pdlp_gap_dist_stats(int64_t* out, double* max_rel, int32_t reset);

/* Original-space re-verification of an infeasibility certificate (the `check`
 * command, tools/main.cpp:199-311 -> residuals.hpp:222-299): kind 0 tests a
 * primal-infeasibility ray y (rows), kind 1 a dual-infeasibility ray x
 * (columns), at relative tolerance eps_ray.  *verified = 1 when it holds;
 * residual / objective as the reference's try_*_infeasibility reports them. */
int pdlp_check_certificate(const pdlp_problem_view* problem, int32_t kind, const double* ray,
                           double eps_ray, int32_t* verified, double* residual,
                           double* objective);

/* ---------------------------------------------- feasibility harness --- *
 * The reference's Appendix-B fixed-restart feasibility iteration
 * (proj/tests/feasibility_method.hpp:40-85, testharness::
 * fixed_restart_feasibility; acceptance criterion 10) on the device: find
 * x >= 0 with A x = b by primal-dual steps of fixed size eta; each round runs
 * restart_length steps from the last restart point with y = 0, averages the
 * primal iterates and adopts the average.  Only A (both layouts) of `a` is
 * read.  restart_points ((rounds+1) * cols, may be NULL) and residuals
 * (rounds+1, ||A x - b||_2) receive x0 and every finite restart point;
 * *recorded = how many; *finite = 0 if a round produced a non-finite point
 * (the run stops there, like FeasibilityRun::finite).  PARITY mode
 * reproduces the reference bit for bit. */
int pdlp_feasibility_run(const pdlp_problem_view* a, const double* b, const double* x0,
                         double eta, int64_t restart_length, int32_t rounds, int32_t mode,
                         int32_t device, double* restart_points, double* residuals,
                         int32_t* recorded, int32_t* finite);

/* ------------------------------------------------------------- MPS --- *
 * Free-format MPS reader / writer with the reference's behaviour
 * (proj/include/pdhglp/mps.hpp:87-535: parse_mps, read_mps_file, write_mps).
 * The parsed model is in minimization form (OBJSENSE MAX negates the
 * objective; pdlp_mps_maximize reports it).  Parse errors return
 * PDLP_ERR_INVALID_PROBLEM with the reference's message ("line N: ...", or
 * "invalid model: ..." for a model that fails validation). */
typedef struct pdlp_mps pdlp_mps;
int pdlp_mps_parse(const char* text, size_t len, pdlp_mps** out);
int pdlp_mps_read_file(const char* path, pdlp_mps** out);
/* Borrowed view, valid until pdlp_mps_free. */
void pdlp_mps_view(const pdlp_mps* model, pdlp_problem_view* view);
int32_t pdlp_mps_maximize(const pdlp_mps* model);
const char* pdlp_mps_name(const pdlp_mps* model);
const char* pdlp_mps_objective_name(const pdlp_mps* model);
const char* pdlp_mps_row_name(const pdlp_mps* model, int64_t row);
const char* pdlp_mps_col_name(const pdlp_mps* model, int64_t col);
void pdlp_mps_free(pdlp_mps* model);
/* write_mps text (generated names OBJ / R# / C#); free with pdlp_mps_free_text. */
int pdlp_mps_write(const pdlp_problem_view* problem, const char* name, int32_t maximize,
                   char** text, size_t* len);
void pdlp_mps_free_text(char* text);

/* ----------------------------------------------------- sharded solve --- *
 * B200 extension (the reference solve is single-process).
 * `world` ranks, one GPU each.  Every rank owns a row block
 * [row_begin,row_end) (y, A x, row bounds) and a column block
 * [col_begin,col_end) (x, A'y, c, variable bounds); the matrix is cut one of
 * two ways:
 *   PDLP_CUT_ROWS  rank g holds its rows of A in both layouts: K_g (its
 *                  rows, global column indices) and K_g^T (all n columns,
 *                  its rows' entries).  Per attempt: x-bar all-gather, local
 *                  K_g x-bar + dual update, partial K_g^T dy reduce-scattered
 *                  to the column owners -- two n-vectors exchanged.
 *   PDLP_CUT_COLS  rank g holds its columns of A in both layouts: K_g^T
 *                  (its columns, global row indices) and K_g (all m rows,
 *                  its columns' entries).  Per attempt: partial K_g x-bar
 *                  reduce-scattered to the row owners + dual update, dy
 *                  all-gathered, local K_g^T dy -- two m-vectors exchanged.
 * plus one all-gather of 5 step scalars; every rank takes the same
 * decisions.  Blocks are equal-sized (NCCL all-gather / reduce-scatter);
 * both are even. */
#define PDLP_CUT_ROWS 0
#define PDLP_CUT_COLS 1
typedef struct pdlp_shard_plan {
  int32_t rank;
  int32_t world;
  int64_t rows, cols;           /* m, n of the whole problem */
  int64_t row_block, col_block; /* mb, nb */
  int64_t row_begin, row_end;
  int64_t col_begin, col_end;
  int32_t cut; /* PDLP_CUT_ROWS / PDLP_CUT_COLS */
  int32_t _pad;
} pdlp_shard_plan;

/* One rank's shard, host side.  PDLP_CUT_ROWS: rows = K_g (lines local,
 * global column indices, pointing into the caller's by_row arrays), cols =
 * K_g^T (all n columns, local row indices, owned by the shard).
 * PDLP_CUT_COLS: rows = all m rows restricted to the column block (local
 * column indices, owned by the shard), cols = the block's columns (global
 * row indices, pointing into the caller's by_col arrays). */
typedef struct pdlp_shard_view {
  pdlp_shard_plan plan;
  pdlp_csr_view rows;
  pdlp_csr_view cols;
  const double* objective; /* col_end - col_begin */
  const double* var_lower;
  const double* var_upper;
  const double* con_lower; /* row_end - row_begin */
  const double* con_upper;
  int64_t entry_offset; /* PDLP_CUT_ROWS: by_row position of K_g's first entry */
  /* PDLP_CUT_COLS: per row r (m entries), by_row position of the row's first
   * shard entry minus rows.start[r] (validation messages carry whole-problem
   * entry indices); NULL when unknown (messages then carry shard indices). */
  const int64_t* row_entry_offset;
} pdlp_shard_view;

/* The shard of `rank`: equal even blocks; the cut exchanges the smaller
 * dimension (PDLP_CUT_COLS when rows < cols; PDLP_SHARD_CUT=rows|cols in the
 * environment overrides). */
int pdlp_shard_plan_for(int64_t rows, int64_t cols, int32_t rank, int32_t world,
                        pdlp_shard_plan* out);
/* CPU only.  *owner keeps the shard's arrays alive; release with
 * pdlp_shard_free.  Structural layout errors -> PDLP_ERR_INVALID_PROBLEM. */
int pdlp_shard_extract(const pdlp_problem_view* problem, int32_t rank, int32_t world,
                       pdlp_shard_view* out, void** owner);
/* The same with an explicit cut (PDLP_CUT_ROWS / PDLP_CUT_COLS). */
int pdlp_shard_extract_cut(const pdlp_problem_view* problem, int32_t rank, int32_t world,
                           int32_t cut, pdlp_shard_view* out, void** owner);
void pdlp_shard_free(void* owner);

/* 128-byte ncclUniqueId for pdlp_solve_sharded (rank 0 creates it, the
 * launcher shares it); 0 or PDLP_ERR_CUDA when libnccl is unavailable. */
int pdlp_nccl_unique_id(unsigned char out[128]);
/* Collective over `world` processes, one GPU each (options->device).  Every
 * rank passes the whole problem and receives the whole result (x, y and
 * reduced costs gathered).  Perf mode only; no observer. */
int pdlp_solve_sharded(const pdlp_problem_view* problem, const pdlp_options* options,
                       int32_t rank, int32_t world, const unsigned char nccl_id[128],
                       pdlp_result* result);
/* The same sharded program with `world` ranks as threads of this process on
 * one GPU (collectives = host barriers + device copies, no cross-kernel
 * waits): validates the sharded path where fewer GPUs than ranks exist.
 * Fills `result` from rank 0. */
int pdlp_solve_sharded_emulated(const pdlp_problem_view* problem, const pdlp_options* options,
                                int32_t world, pdlp_result* result);

/* Shard-local ingest: each rank passes only its own shard (its rows in both
 * layouts, its column block's objective and bounds; e.g. built by
 * pdlp_gen_random_lp_shard), so no host ever holds the whole problem.
 * The shard plan (rows, cols, row and column ranges) must be pdlp_shard_plan_for's for
 * (rank, world).  Results as pdlp_solve_sharded (whole x, y, r per rank). */
int pdlp_solve_sharded_local(const pdlp_shard_view* shard, const pdlp_options* options,
                             int32_t rank, int32_t world, const unsigned char nccl_id[128],
                             pdlp_result* result);
/* The same with `world` ranks as threads on this process's GPU (tests). */
int pdlp_solve_sharded_local_emulated(const pdlp_shard_view* const* shards,
                                      const pdlp_options* options, int32_t world,
                                      pdlp_result* result);

/* ------------------------------------------------------ component entry --- *
 * Single-component entry points used by the parity tests (each runs the same
 * device kernels the solver uses; host arrays in, host arrays out). */

/* reference pdhg_step (step.hpp:100-115): one step at (omega, eta) from (x, y)
 * with aty = A'y computed on device.  Returns 1 in *finite when every output
 * entry is finite. */
int pdlp_pdhg_step(const pdlp_problem_view* problem, const double* x, const double* y,
                   double omega, double eta, int32_t mode, int32_t shards, double* x_out,
                   double* y_out, int32_t* finite);

/* reference adaptive_step (step.hpp:161-193) on the iterate (x, y, aty).
 * io_state = {eta_hat, k, max_retries(as double), omega}; on return the
 * iterate arrays hold the new iterate, prev_* the previous one (the trial
 * buffers), stats = {accepted, retries, min_eta_bar, eta_used}.
 * Returns outcome 0 = accepted, 1 = numerical error in *outcome. */
int pdlp_adaptive_step(const pdlp_problem_view* problem, double* x, double* y, double* aty,
                       double* io_state, int32_t mode, int32_t shards, double* prev_x,
                       double* prev_y, double* stats, int32_t* outcome);

/* kernels::spmv / spmv_transpose (kernels.hpp:30-59). */
int pdlp_spmv(const pdlp_problem_view* problem, const double* x, double* out, int32_t mode);
int pdlp_spmv_transpose(const pdlp_problem_view* problem, const double* y, double* out,
                        int32_t mode);

/* apply_rescaling (rescaling.hpp:137-143).  Outputs: scaled by_row/by_col
 * values (nnz each), scaled objective/bounds, row_scale (rows), col_scale
 * (cols). */
int pdlp_apply_rescaling(const pdlp_problem_view* problem, int32_t ruiz_passes,
                         int32_t pock_chambolle, double* row_values, double* col_values,
                         double* objective, double* con_lower, double* con_upper,
                         double* var_lower, double* var_upper, double* row_scale,
                         double* col_scale);

/* normalized_duality_gap (restarts.hpp:107-220) with ax = A x, aty = A'y. */
int pdlp_normalized_duality_gap(const pdlp_problem_view* problem, const double* x,
                                const double* y, const double* ax, const double* aty,
                                double omega, double r, int32_t mode, double* gap);

/* recover_reduced_costs (residuals.hpp:49-64) + kkt_residuals
 * (residuals.hpp:135-158) on the given problem.  rc_mode 0 = Natural,
 * 1 = BoundRobust (r_out, may be NULL, receives them); 2 = use the reduced
 * costs passed in r_out (kkt_residuals(p, x, y, r), the `check` command). */
int pdlp_kkt_residuals(const pdlp_problem_view* problem, const double* x, const double* y,
                       int32_t rc_mode, int32_t mode, double* r_out,
                       pdlp_residual_summary* summary);

/* Scalar step-size rules (step.hpp:126-141), evaluated by the same device code
 * the decision kernel uses (schedule factors from the host table). */
int pdlp_step_size_rules(double movement, double curvature, double eta_bar, double eta,
                         int64_t k, double* limit_out, double* next_out);

#ifdef __cplusplus
}
#endif

#endif /* PDLP_B200_H_ */
