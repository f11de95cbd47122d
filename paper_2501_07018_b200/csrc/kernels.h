// kernels.h — the thin internal C-ABI between the host C++ driver
// (solver.cpp) and the hand-written sm_100a kernels (k_*.cu).
//
// Plain structs of device pointers and sizes; every launcher is extern "C",
// enqueues on the given stream and never synchronises.  Scalars that the
// host needs come back through a small device "slot" array that the driver
// copies in one batch (pdlpk_slots_*).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Reduction orders.  PARITY reproduces the reference's arithmetic order:
 *   SEQ   — one sequential chain in index order (the reference's plain loops)
 *   SHARD — make_shard_plan(dim, 1, S) chains + ascending combine
 *           (kernels.hpp:69-97, shard.hpp:24-40)
 * PERF maps both onto TREE (fixed block tree; deterministic run to run). */
#define PDLPK_RED_TREE 0
#define PDLPK_RED_SEQ 1
#define PDLPK_RED_SHARD 2

/* Device CSR for one orientation (int32 secondary indices, fp64 values;
 * row pointers int32 when nnz < 2^31, else int64) plus the perf-mode
 * load-balancing schedule built at upload time. */
typedef struct pdlpk_csr {
  int64_t dim;
  int64_t nnz;
  const void* start; /* dim+1 entries, int32 or int64 */
  int32_t wide;      /* 1: start is int64 */
  int32_t tile_blocks; /* CTAs for the tiled short-line segment */
  const int32_t* index;
  const double* value;      /* scaled values (the iteration matrix) */
  const double* value_orig; /* original values (verification products) */
  /* Lines longer than PDLPK_SHORT_MAX are cut into chunks of at most
   * PDLPK_CHUNK entries, one warp each.  A line's chunks are consecutive;
   * the last-arriving warp of a multi-chunk line sums the chunk partials in
   * chunk order and writes the line's epilogue contributions to its slot in
   * line_acc (kept out of the per-CTA partials so the totals stay
   * deterministic). */
  const int32_t* chunk_row;  /* line of each chunk */
  const int64_t* chunk_beg;  /* first entry of each chunk */
  const int32_t* chunk_len;  /* entries of each chunk */
  const int32_t* chunk_pos;  /* index in line | (chunks in line << 16) */
  const int32_t* chunk_slot; /* multi-chunk line slot, -1 for single-chunk lines */
  int64_t n_chunks;     /* warp chunks first, then n_cta_chunks CTA chunks */
  int64_t n_cta_chunks; /* chunks of lines > PDLPK_WARP_LINE_MAX, one CTA each */
  int64_t n_multi;      /* multi-chunk lines */
  double* chunk_part;  /* n_chunks partial sums */
  unsigned* chunk_cnt; /* arrival counters, at each line's first chunk */
  double* line_acc;    /* n_multi * PDLPK_LINE_ACC epilogue contributions */
  const int32_t* tile_row0; /* first line of each warp tile of short lines */
  const int32_t* tile_rows; /* lines | (entries << 8) of each tile */
  const int64_t* tile_nnz0; /* first entry of each tile (= start[tile_row0]) */
  int64_t n_tiles;
  /* Row-sharded solves (solver.cpp): how a product with this
   * layout crosses ranks.  PDLPK_DIST_GATHER: lines are local, entries index
   * the all-gathered column-side operand.  PDLPK_DIST_PARTIAL: lines are all
   * n columns, entries index local rows; the output is reduce-scattered to
   * the column owners.  PDLPK_DIST_NONE on one GPU. */
  int32_t dist_kind;
  int32_t tile_direct; /* 1: tiles are direct (thread per line, spmv.cuh) */
  int32_t tile_lines_cap;   /* staged tile shape of this layout: lines and */
  int32_t tile_nnz_cap;     /* entries per tile ... */
  int32_t tile_stage_bytes; /* ... and the bytes of one ring stage */
  /* Segmented spans (spmv.cuh seg_spans), an alternative schedule for
   * skewed layouts: seg_mode = 1 replaces every other segment.  Span
   * {r0, nl > 0, e0, len}: whole non-empty lines r0 .. r0+nl-1; span
   * {r, -1-c, e0, len}: chunk c of a line longer than a span (or an empty
   * line), seg_aux = {first partial slot, chunks, line_acc slot or -1, 0}.
   * Per 256-entry step of a line run, 8 words of line-start bits and 8 of
   * line-end bits (seg_masks, from seg_step0[span]). */
  int32_t seg_mode;
  const int4* seg_spans;
  const int4* seg_aux;
  const int32_t* seg_step0;
  const uint32_t* seg_masks;
  int64_t n_seg_spans;
  /* 1: a column pass over this layout (the dual polishing subproblem's K^T
   * is the row layout) takes the split form, whose partials follow the line
   * index: set on row layouts whose warp lines may run interleaved
   * (solver.cpp build_schedule), so results do not depend on the order. */
  int32_t col_split;
} pdlpk_csr;

#define PDLPK_DIST_NONE 0
#define PDLPK_DIST_GATHER 1
#define PDLPK_DIST_PARTIAL 2

/* Schedule limits (spmv.cuh) the host planner must respect. */
#ifndef PDLPK_SHORT_MAX
#define PDLPK_SHORT_MAX 32 /* longest line of a staged tile */
#endif
#ifndef PDLPK_CHUNK
#define PDLPK_CHUNK 2048 /* entries per CTA chunk: 8 warps x one 256-entry batch */
#endif
#ifndef PDLPK_WARP_LINE_MAX
#define PDLPK_WARP_LINE_MAX 2048 /* longer lines are processed by CTA chunks */
#endif
#define PDLPK_LINE_ACC 4
#ifndef PDLPK_TILE_NNZ
#define PDLPK_TILE_NNZ 896 /* entries of the default stage budget (with PDLPK_TILE_ROWS lines) */
#endif
#ifndef PDLPK_TILE_ROWS
#define PDLPK_TILE_ROWS 448 /* most lines per staged tile (7 consumer warps x 32 x 2 lines/lane) */
#endif
#ifndef PDLPK_XBAR_KEEP
#define PDLPK_XBAR_KEEP 1
#endif
#ifndef PDLPK_PDL
#define PDLPK_PDL 1
#endif
#ifndef PDLPK_PDL_TRIGGER
#define PDLPK_PDL_TRIGGER 0
#endif
#ifndef PDLPK_PDL_CADENCE
#define PDLPK_PDL_CADENCE 1
#endif
#ifndef PDLPK_DY_KEEP
#define PDLPK_DY_KEEP 0
#endif
#ifndef PDLPK_XN_STREAM
#define PDLPK_XN_STREAM 1
#endif
#ifndef PDLPK_MATRIX_EVICT_FIRST
#define PDLPK_MATRIX_EVICT_FIRST 1
#endif
#ifndef PDLPK_XBAR_KEEP_MB
#define PDLPK_XBAR_KEEP_MB 48
#endif
#ifndef PDLPK_TILE_STAGES
#define PDLPK_TILE_STAGES 2 /* staged tiles in flight per CTA */
#endif

/* Device-resident step controller: one per inner loop (main / polish). */
typedef struct pdlpk_step_state {
  double eta;      /* trial step size for the next attempt */
  double omega;    /* primal weight */
  double eta_used; /* step size of the last accepted attempt */
  double min_eta_bar;
  double avg_weight; /* AverageState::weight */
  double avg_w;      /* pending average weight (deferred add) */
  double dx2, dy2, curv, eta_bar, inf_x, inf_y; /* last attempt */
  int64_t k;        /* accepted steps in this inner loop (st.k == ctrl.k) */
  int64_t k_target; /* halt when k reaches this */
  int64_t accepted;
  int64_t retries;
  int64_t attempts;
  int64_t avg_count;
  int32_t cur;    /* ping-pong index of the current iterate */
  int32_t halt;   /* 1: every step kernel returns immediately */
  int32_t status; /* 0 running, 1 numerical error */
  int32_t attempt_in_step;
  int32_t max_retries;
  int32_t avg_pending;
  int32_t fixed; /* fixed-step mode (solver.hpp:477-491) */
  int32_t table_short; /* schedule table exhausted */
  uint32_t ticket;     /* last-CTA election */
  uint32_t _pad;
} pdlpk_step_state;

typedef struct pdlpk_problem {
  int64_t m;
  int64_t n;
  pdlpk_csr K;  /* row layout of A   */
  pdlpk_csr KT; /* column layout of A */
  const double *c, *lc, *uc, *lv, *uv;           /* scaled */
  const double *c_o, *lc_o, *uc_o, *lv_o, *uv_o; /* original */
  const double *row_scale, *col_scale;           /* m, n */
  /* Bitwise-uniform scaled vectors (bit 0 c, 1 l_v, 2 u_v) and their value:
   * the primal pass then uses the scalar instead of streaming the vector
   * (x >= 0 problems, the zero objective of the polishing subproblems).
   * 0 = no assumption. */
  uint32_t uniform;
  uint32_t _pad_uniform;
  double c_u, lv_u, uv_u;
} pdlpk_problem;

/* or_and[0] |= OR of v's 64-bit patterns, or_and[1] &= AND (caller seeds 0 /
 * all-ones): v is bitwise uniform iff they are equal. */
int pdlpk_uniform_bits(const double* v, int64_t n, unsigned long long* or_and, cudaStream_t s);

typedef struct pdlpk_step_args {
  pdlpk_problem P;
  double* x[2];
  double* y[2];
  double* aty[2];
  double* xbar;     /* n: 2x' - x */
  double* dy;       /* m: y' - y */
  double* aty_diff; /* n: A'(y'-y) (parity path) */
  double* sum_x;    /* n */
  double* sum_y;    /* m */
  pdlpk_step_state* state;
  const double* f_down; /* 1 - (max(k,1)+1)^-0.3, host libm */
  const double* f_up;   /* 1 + (max(k,1)+1)^-0.6 */
  int64_t table_len;
  double* part2; /* per-CTA partials of the row pass */
  double* part3; /* per-CTA partials of the column pass */
  int32_t mode;  /* PDLP_MODE_PERF / PDLP_MODE_PARITY */
  int32_t shards;
  double* shard_part; /* parity: 4*shards partials */
  /* 1: the row pass writes each line's |dy|^2 and |y'| terms to part2[r],
   * part2[m + r] and the decision sums them in line order, so the step's
   * reductions do not depend on the SpMV schedule (perf mode, one GPU,
   * m <= PDLPK_LINE_PARTIALS_MAX). */
  int32_t line_partials;
  /* Column panels of the row pass (perf mode, one GPU, large n): the row
   * layout re-laid out as n_row_panels CSR matrices over consecutive column
   * ranges (host array row_panels, each a full m-line layout).  The row pass
   * then runs one launch per panel, carrying each line's running sum in
   * carry[] from panel to panel (rows are sorted by column, so the chained
   * sum adds the line's products in storage order); only the last launch
   * runs the dual-update epilogue.  The x-bar range a launch gathers from
   * then stays in L2.  panel_phase (set per launch): 0 no panels, 1 first,
   * 2 middle, 3 last. */
  int32_t n_row_panels;
  int32_t panel_phase;
  int32_t _pad_panel;
  const pdlpk_csr* row_panels; /* host pointer: read by the launch code only */
  double* carry;               /* m */
  /* Sliced-ELL copy of the row layout (measurement knob PDLP_ROW_SELL=1,
   * perf mode, one GPU): rows in slices of 32 in their natural order, entry
   * k of the slice's lane l at off[g] + 32 k + l, so a warp's index and value
   * loads are coalesced without staging and each lane sums its own row in
   * storage order.  off == NULL: not built.  blocks = CTAs of the pass (its
   * per-CTA partials). */
  struct {
    const int64_t* off; /* ng + 1 */
    const int32_t* sidx;
    const double* sval;
    int64_t ng;
    int32_t blocks;
    int32_t _pad;
  } sell;
} pdlpk_step_args;

/* SELL build (k_step.cu): slice offsets from the row layout's line lengths
 * (tmp == NULL: only *tmp_bytes is set), then the scatter of its entries. */
int pdlpk_sell_plan(const pdlpk_csr* K, int64_t* w32, int64_t* off, void* tmp, size_t* tmp_bytes,
                    cudaStream_t s);
int pdlpk_sell_fill(const pdlpk_csr* K, const int64_t* off, int32_t* sidx, double* sval, cudaStream_t s);
#define PDLPK_MAX_ROW_PANELS 8

/* Device pointers of the column panels (k_vec.cu pdlpk_panel_scatter). */
typedef struct pdlpk_panel_ptrs {
  int32_t np;
  int32_t _pad;
  const int32_t* start[PDLPK_MAX_ROW_PANELS]; /* m+1 each, panel-local positions */
  int32_t* idx[PDLPK_MAX_ROW_PANELS];
  double* val[PDLPK_MAX_ROW_PANELS];
} pdlpk_panel_ptrs;
int pdlpk_panel_scatter(const pdlpk_csr* K, const pdlpk_panel_ptrs* pp, cudaStream_t s);

/* Multi-vector products on a segmented-span layout (k_multi.cu, perf mode):
 * out.v[q] = A in.v[q] for q < vec (2 or 4) in one pass; pack = scratch of
 * vec * operand_len doubles, part = scratch of vec * A->n_chunks doubles. */
typedef struct pdlpk_multi_vecs {
  double* v[4];
} pdlpk_multi_vecs;
int pdlpk_spmv_multi(const pdlpk_csr* A, int32_t orig, int32_t vec, const pdlpk_multi_vecs* in,
                     int64_t operand_len, double* pack, const pdlpk_multi_vecs* out, double* part,
                     cudaStream_t s);
#define PDLPK_LINE_PARTIALS_MAX 65536 /* the decision reads 2m terms serially in one CTA: bounded to 1 MB */

/* Reduction context for cadence operations. */
typedef struct pdlpk_red {
  int32_t order;  /* PDLPK_RED_* for sequential-loop sums (SEQ in parity, TREE in perf) */
  int32_t shards; /* S for sharded reductions (parity) */
  int32_t parity;
  int32_t _pad;
  double* scratch; /* >= pdlpk_red_scratch_doubles() */
} pdlpk_red;

int64_t pdlpk_red_scratch_doubles(void);
int64_t pdlpk_step_partials(const pdlpk_problem* P);
/* Staged-tile shape for a layout whose short lines average `avg_len`
 * entries: the most lines (<= PDLPK_TILE_ROWS) whose entries still fit one
 * ring stage, and the entry cap for that line count. */
void pdlpk_tile_shape(double avg_len, int32_t budget, int32_t* lines, int32_t* nnz,
                      int32_t* stage_bytes, int32_t staged);
/* Ring-stage bytes of a PDLPK_TILE_ROWS x nnz tile (budgets for tile_shape). */
int32_t pdlpk_stage_budget(int32_t nnz);
/* SMs x resident CTAs of the staged-tile kernels with this ring. */
int64_t pdlpk_tile_resident_ctas(int32_t stage_bytes);
int64_t pdlpk_seg_resident_ctas(void);

/* ---- row-sharded attempt pieces (the host interleaves the collectives) ----
 * primal:     primal_pass; xbar is written at a->xbar
 * row_fused:  K xbar + dual update, operand a->xbar, dy written at a->dy
 * row_epi:    dual update from reduce-scattered sums acc[m]
 * col_fused:  K^T dy + column epilogue (no decision), operand a->dy
 * col_epi:    column epilogue from reduce-scattered sums d[n]
 * totals:     this rank's [dy2, infy, dx2, curv, infx] from the partials
 *             (g2 / g3 CTAs; *_acc: add the multi-chunk line slots)
 * decide:     combine world x 8 gathered totals in rank order, then the
 *             accept/reject rule.  Every piece is a no-op once halted. */
int64_t pdlpk_dist_ew_grid(int64_t n);
int64_t pdlpk_dist_sched_grid(const pdlpk_csr* A);
int pdlpk_dist_primal(const pdlpk_step_args* a, cudaStream_t s);
int pdlpk_dist_row_fused(const pdlpk_step_args* a, cudaStream_t s);
// Reduce-scatter folded into the epilogue: the line sums are read straight
// from every rank's partial product over NVLink P2P (rank order, so the sum
// is deterministic); world == 0 means `acc` already holds them.
#define PDLPK_MAX_PEERS 8
typedef struct {
  const double* p[PDLPK_MAX_PEERS];
  int32_t world;
  int64_t offset;  // this rank's block within each partial product
} pdlpk_peer_sum;
int pdlpk_dist_row_epi_peers(const pdlpk_step_args* a, const pdlpk_peer_sum* ps, cudaStream_t s);
int pdlpk_dist_col_epi_peers(const pdlpk_step_args* a, const pdlpk_peer_sum* ps, cudaStream_t s);
// primal pass that also stores x-bar into every peer's gathered vector
// (dst.p[r] + dst.offset; null entries are skipped): all-gather folded in.
int pdlpk_dist_primal_push(const pdlpk_step_args* a, const pdlpk_peer_sum* dst, cudaStream_t s);
// out[i] = sum over ranks (rank order) of p[r][offset + i], i < count.
int pdlpk_peer_reduce(double* out, const pdlpk_peer_sum* ps, int64_t count, cudaStream_t s);
int pdlpk_dist_row_epi(const pdlpk_step_args* a, const double* acc, cudaStream_t s);
int pdlpk_dist_col_fused(const pdlpk_step_args* a, cudaStream_t s);
int pdlpk_dist_col_epi(const pdlpk_step_args* a, const double* d, cudaStream_t s);
int pdlpk_dist_totals(const pdlpk_step_args* a, int64_t g2, int64_t g3, int32_t k_acc,
                      int32_t kt_acc, double* out8, cudaStream_t s);
int pdlpk_dist_decide(const pdlpk_step_args* a, const double* all8, int32_t world,
                      cudaStream_t s);

/* ---- cross-rank combines ----
 * Reductions launched while a log is set on this host thread record their
 * output (count, sum/max mask) so the engine can combine them across ranks
 * before the host reads them. */
typedef struct pdlpk_red_log {
  int32_t count;
  int32_t k[48];
  uint32_t maxmask[48];
  double* out[48];
} pdlpk_red_log;
void pdlpk_set_red_log(pdlpk_red_log* log);
/* slots[i] for bit i of `marked` = rank-ordered sum (or max, bit i of
 * `maxbits`) of all[r * stride + i], r < world. */
int pdlpk_combine_slots(const double* all, int32_t world, int32_t stride, uint64_t marked,
                        uint64_t maxbits, double* slots, cudaStream_t s);
/* out[i] = out[i] + in[i] (or max) */
int pdlpk_accumulate(double* out, const double* in, int64_t n, int32_t use_max, cudaStream_t s);
/* f = sqrt(norm) where norm > 0, else 1 (rescaling.hpp:90,98,115,123) */
int pdlpk_norm_to_factor(double* f, int64_t n, cudaStream_t s);
/* acc[line] += sequential sum of |a| over the layout's entries of each line */
int pdlpk_line_onenorm_continue(const pdlpk_csr* A, double* acc, cudaStream_t s);
/* raw line norms (inf or 1) of a layout into `norm` */
int pdlpk_line_norms(const pdlpk_csr* A, const int32_t* line_of, int32_t one_norm, double* norm,
                     unsigned long long* bits, cudaStream_t s);

/* ---------------------------------------------------------------- setup --- */
int pdlpk_index_to_i32(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t s);
int pdlpk_start_to_i32(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t s);

/* Validation (k_valid.cu; reference problem.hpp:119-154, sparse.hpp:118-133).
 * keys[0..3] receive (first failing index << 3 | condition) for objective,
 * variable bounds, constraint bounds and matrix values (all ones = none).
 * Layout checks OR bits into *bad: 1 row pointers, 2 index range, 4 row line
 * order, 8 column entry without an equal row entry, 16 per-row counts. */
int pdlpk_validate_vectors(const double* c, const double* lv, const double* uv, int64_t n,
                           const double* lc, const double* uc, int64_t m,
                           const double* row_values, int64_t nnz, unsigned long long* keys,
                           cudaStream_t s);
int pdlpk_validate_raw_layout(const int64_t* start, int64_t dim, const int64_t* idx,
                              int64_t count, int64_t nnz, int64_t bound, unsigned* bad,
                              cudaStream_t s);
/* Same on 32-bit arrays (narrowed on the host with saturation, so an
 * out-of-range 64-bit value stays out of range). */
int pdlpk_validate_raw_layout32(const int32_t* start, int64_t dim, const int32_t* idx,
                                int64_t count, int64_t nnz, int64_t bound, unsigned* bad,
                                cudaStream_t s);
int pdlpk_validate_consistency(const pdlpk_csr* R, const int32_t* row_of, const pdlpk_csr* C,
                               const int32_t* col_of, int* row_count, unsigned* bad,
                               cudaStream_t s);

/* ----------------------------------------------------------------- step --- */
/* Arm the controller for a run: k_target, halt = 0. */
int pdlpk_arm(pdlpk_step_state* st, int64_t k_target, cudaStream_t s);
/* One step attempt (primal pass, row pass + dual update, column pass +
 * decision).  Every kernel is a no-op once state->halt is set. */
int pdlpk_attempt(const pdlpk_step_args* a, cudaStream_t s);
/* Same, recording ev[0..3] around the launches (primal | row | column[+reduce]). */
int pdlpk_attempt_timed(const pdlpk_step_args* a, cudaEvent_t* ev, cudaStream_t s);
/* Apply a pending deferred average add (AverageState::add, step.hpp:209-216). */
int pdlpk_flush_average(const pdlpk_step_args* a, cudaStream_t s);

/* ------------------------------------- feasibility harness (k_feas.cu) --- */
/* Appendix-B fixed-restart feasibility iteration
 * (tests/feasibility_method.hpp:40-85), per-entry parts. */
int pdlpk_feas_primal(double* x, const double* aty, double* scratch, double* x_sum, double eta,
                      int64_t n, cudaStream_t s);
int pdlpk_feas_dual(double* y, const double* b, const double* ax_mid, double eta, int64_t m,
                    cudaStream_t s);
int pdlpk_feas_average(double* x_start, double* x, double* x_sum, double len, int64_t n,
                       int32_t* finite, cudaStream_t s);

/* ------------------------------------------------------------- cadence --- */
/* out = A v with the given layout; orig != 0 uses the original values.
 * cond (device scalar, may be NULL): the product is skipped when *cond == 0. */
int pdlpk_spmv(const pdlpk_csr* A, int32_t orig, const double* v, double* out, int32_t parity,
               cudaStream_t s);
int pdlpk_spmv_cond(const pdlpk_csr* A, int32_t orig, const double* v, double* out,
                    int32_t parity, const double* cond, cudaStream_t s);

/* slot = sum_i (a_i - b_i)^2 over dim n (sharded in parity). */
int pdlpk_diff_norm_sq(const double* a, const double* b, int64_t n, const pdlpk_red* red,
                       double* slot, cudaStream_t s);
/* out = a - b */
int pdlpk_fill(double* x, double v, int64_t n, cudaStream_t s);
int pdlpk_sub(const double* a, const double* b, double* out, int64_t n, cudaStream_t s);
/* out = sum * (1/weight), weight read from the state (average_into, step.hpp:219-227). */
int pdlpk_average_into(const pdlpk_step_state* st, const double* sum_x, const double* sum_y,
                       double* x, double* y, int64_t n, int64_t m, cudaStream_t s);
/* out = scale .* v (unscale_primal / unscale_dual, rescaling.hpp:145-153). */
/* out = v / scale (perf mode: an original-space product from a scaled one) */
int pdlpk_scale_div(const double* scale, const double* v, double* out, int64_t n, cudaStream_t s);
int pdlpk_scale_mul(const double* scale, const double* v, double* out, int64_t n,
                    cudaStream_t s);

/* Residual screen (recover_reduced_costs_from + residuals_from_scaled /
 * kkt_residuals_from, residuals.hpp:29-47, 98-133, 165-185).  Uses the scaled
 * (orig = 0) or original (orig = 1, unit scales) data.  slots[0..3] =
 * primal_inf, dual_inf, pobj, penalty (dobj = -penalty).  r_out (n) may be NULL. */
int pdlpk_screen(const pdlpk_problem* P, int32_t orig, const double* x, const double* y,
                 const double* ax, const double* aty, int32_t rc_mode, const pdlpk_red* red,
                 double* r_out, double* slots, cudaStream_t s);

/* Ray tests (residuals.hpp:222-299), split around their matrix product:
 *  primal: prep writes ray = proj_cone(yc), slots[0] = |ray|_inf,
 *          slots[1] = number of coordinates the projection changed;
 *          finish (after aty = A'ray) writes rhat, slots[0] = residual,
 *          slots[1] = penalty of (ray, rhat) (objective = -penalty).  When
 *          aty_alt and changed are given and *changed == 0 the ray equals yc
 *          and aty_alt (= A'yc, same kernel) is used instead of aty.
 *  dual:   prep: slots[0] = |xc|_inf, slots[1] = box residual, slots[2] = c'xc;
 *          finish (after ax = A xc): slots[0] = row residual. */
int pdlpk_ray_primal_prep(const pdlpk_problem* P, int32_t orig, const double* yc, double* ray,
                          const pdlpk_red* red, double* slots, cudaStream_t s);
int pdlpk_ray_primal_finish(const pdlpk_problem* P, int32_t orig, const double* ray,
                            const double* aty, const double* aty_alt, const double* changed,
                            double* rhat, const pdlpk_red* red, double* slots, cudaStream_t s);
int pdlpk_ray_dual_prep(const pdlpk_problem* P, int32_t orig, const double* xc,
                        const pdlpk_red* red, double* slots, cudaStream_t s);
int pdlpk_ray_dual_finish(const pdlpk_problem* P, int32_t orig, const double* ax,
                          const pdlpk_red* red, double* slots, cudaStream_t s);

/* Normalized duality gap (restarts.hpp:107-220), k_gap.cu.  prepare computes
 * the lam->inf masses and compacts the breakpoint events (their count goes to
 * *count_out, a device int); finish sorts the E events the host read back,
 * sweeps, assembles the candidate and writes the gap to *gap_slot.  r read
 * from r_slot (radius) unless r_slot == NULL (then r_value).  work must hold
 * pdlpk_gap_work_bytes(n, m) bytes and stay untouched between the two calls. */
size_t pdlpk_gap_work_bytes(int64_t n, int64_t m);
int pdlpk_gap_prepare(const pdlpk_problem* P, const double* x, const double* y, const double* ax,
                      const double* aty, double omega, const pdlpk_red* red, void* work,
                      int* count_out, cudaStream_t s);
/* gap_slot[0] = the gap, gap_slot[2] = the first crossing's position as a
 * fraction of E (1 if none).  0 <= qa < qb, qb - qa < 0.5: perf mode first
 * sorts only the events at depth fractions [qa, qb] of the descending order
 * (exact when the crossing lies inside; else the full sort runs). */
int pdlpk_gap_finish(const pdlpk_problem* P, const double* x, const double* y, const double* ax,
                     const double* aty, double omega, const double* r_slot, double r_value,
                     int64_t E, const pdlpk_red* red, void* work, double* gap_slot, double qa,
                     double qb, cudaStream_t s);
/* Window sorts tried / decided on this host thread (cumulative). */
void pdlpk_gap_window_stats(int64_t* tried, int64_t* decided);

/* Distributed gap (row-sharded solves, k_gap.cu; the host drives the bracket
 * search, solver.cpp Engine::gap_dist).  After pdlpk_gap_prepare on the
 * rank's local views (work sized for the local n, m):
 *   stage    dst[0..2] = local b_inf, c_inf, event count
 *   keys     the E local events' order keys into list 0 (keys0 / slots0)
 *   lists    the two ping-pong bracket lists (keys, event slots) inside work
 *   sample   out[0..S) = S strided keys of a list (bit patterns), out[S] = taken
 *   split    out[0..4] = masses (c, b) of list events with key > s_key, with
 *            key >= s_key, and the count with key < s_key (TREE order)
 *   compact  the list events with lo <= key <= hi into the other list
 *   pack     dst[0..3K) = keys | d_const | d_inverse of a list, zero padded
 *   final    rank-ordered concatenation of `world` packed blocks (counts[q]
 *            events each), stable descending sort, sweep from the masses
 *            (c0, b0) above the bracket and hi0 = lambda of the group above
 *            it; lower_bounded: the bracket's lowest group is known to cross.
 *            *lambda_star -> the device scalar.  fwork holds
 *            pdlpk_gapd_final_bytes(cap) bytes, cap >= total events.
 *   value    this rank's partial of gap_value_at at *lambda_star (TREE). */
#define PDLPK_GAPD_MAX_RANKS 64
int pdlpk_gapd_stage(void* work, int64_t n, int64_t m, double* dst, cudaStream_t s);
int pdlpk_gapd_keys(void* work, int64_t n, int64_t m, int64_t E, cudaStream_t s);
int pdlpk_gapd_lists(void* work, int64_t n, int64_t m, uint64_t** keys0, int32_t** slots0,
                     uint64_t** keys1, int32_t** slots1);
int pdlpk_gapd_sample(const uint64_t* keys, int64_t A, int S, double* out, cudaStream_t s);
int pdlpk_gapd_split(void* work, int64_t n, int64_t m, const uint64_t* keys, const int32_t* slots,
                     int64_t A, uint64_t s_key, const pdlpk_red* red, double* out, cudaStream_t s);
int pdlpk_gapd_compact(void* work, int64_t n, int64_t m, const uint64_t* keys_in,
                       const int32_t* slots_in, int64_t A, uint64_t lo, uint64_t hi,
                       uint64_t* keys_out, int32_t* slots_out, cudaStream_t s);
int pdlpk_gapd_pack(void* work, int64_t n, int64_t m, const uint64_t* keys, const int32_t* slots,
                    int64_t A, int64_t K, double* dst, cudaStream_t s);
size_t pdlpk_gapd_final_bytes(int64_t T);
/* *dst (device) = lambda* of the last gap evaluated in `work` (checks). */
int pdlpk_gap_lambda_star(void* work, int64_t n, int64_t m, double* dst, cudaStream_t s);
int pdlpk_gapd_final(void* fwork, int64_t cap, const double* all, int world, int64_t K,
                     const int64_t* counts, double c0, double b0, double hi0, int lower_bounded,
                     double r, double** lambda_star, cudaStream_t s);
int pdlpk_gapd_value(const pdlpk_problem* P, const double* x, const double* y, const double* ax,
                     const double* aty, double omega, const double* lambda_star,
                     const pdlpk_red* red, double* out, cudaStream_t s);
/* slot = sqrt(omega*dx2 + dy2/omega) from two slots (restart_progress_metric). */
int pdlpk_radius(const double* dx2, const double* dy2, double omega, double* out,
                 cudaStream_t s);

/* ------------------------------------------------------- preconditioning --- */
/* dst[k] = src[k] narrowed to int32 with the host stager's saturation
 * (x < 0 -> -1, x > INT32_MAX -> INT32_MAX), for uploads from pinned memory. */
int pdlpk_narrow_i64(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t s);
/* line_of[k] = line owning entry k (max-scan over line heads; k_scale.cu). */
size_t pdlpk_line_of_work_bytes(int64_t nnz);
int pdlpk_line_of(const pdlpk_csr* A, int32_t* line_of, void* work, size_t work_bytes,
                  cudaStream_t s);
/* f[line] = sqrt(max|v|) or 1 (ruiz) / sqrt(sum|v|) or 1 (pock-chambolle),
 * per line of the layout (rescaling.hpp:80-127).  bits: dim scratch words. */
int pdlpk_line_factors(const pdlpk_csr* A, const int32_t* line_of, int32_t one_norm, double* f,
                       unsigned long long* bits, cudaStream_t s);
/* value /= f_primary[line] * f_secondary[index] for one layout. */
int pdlpk_apply_factors(const pdlpk_csr* A, const int32_t* line_of, double* value,
                        const double* f_primary, const double* f_secondary, cudaStream_t s);
/* Ruiz passes on one GPU: bits[line] = max |v| of the layout's lines
 * (order-free, exact); f = sqrt(max) or 1 from them; the division of
 * apply_factors fused with the next pass's bits of the result
 * (bits_next == NULL: the division alone). */
int pdlpk_line_absmax(const pdlpk_csr* A, const int32_t* line_of, unsigned long long* bits,
                      cudaStream_t s);
int pdlpk_factors_from_bits(const unsigned long long* bits, int64_t dim, double* f, cudaStream_t s);
int pdlpk_apply_factors_max(const pdlpk_csr* A, const int32_t* line_of, double* value,
                            const double* f_primary, const double* f_secondary,
                            unsigned long long* bits_next, cudaStream_t s);
/* Vector part of apply_factors (rescaling.hpp:61-73). */
int pdlpk_apply_vec_factors(double* lc, double* uc, double* row_scale, const double* fr,
                            int64_t m, double* c, double* lv, double* uv, double* col_scale,
                            const double* fc, int64_t n, cudaStream_t s);
/* slot = max |v| (initial_step_size, step.hpp:14-18). */
int pdlpk_abs_max(const double* v, int64_t n, const pdlpk_red* red, double* slot,
                  cudaStream_t s);
/* slots[0] = sum c^2, slots[1] = sum mag(lc,uc)^2 (initialize_primal_weight,
 * restarts.hpp:278-294). */
int pdlpk_primal_weight_sums(const double* c, int64_t n, const double* lc, const double* uc,
                             int64_t m, const pdlpk_red* red, double* slots, cudaStream_t s);
/* x0 = clamp(0, lv, uv) (initial_point, solver.hpp:196-202). */
int pdlpk_initial_point(const double* lv, const double* uv, double* x, int64_t n,
                        cudaStream_t s);
/* Dual-feasibility subproblem bounds (problem.hpp:181-238):
 * con bounds (n) from the parent objective and variable cones, variable
 * bounds (m) from the parent constraint cones. */
int pdlpk_dual_feas_bounds(const double* c, const double* lv, const double* uv, int64_t n,
                           const double* lc, const double* uc, int64_t m, double* sub_lc,
                           double* sub_uc, double* sub_lv, double* sub_uv, cudaStream_t s);
/* Validation scan (problem.hpp:119-154 minus layouts_consistent):
 * slot[0] = first failing check code (0 = ok), slot[1] = index. */
int pdlpk_check_finite(const double* v, int64_t n, int32_t code, int32_t* first, cudaStream_t s);

#ifdef __cplusplus
}
#endif
