/*
 * pdlp_gen.h — seeded synthetic LP instances for the BASELINE.json configs
 * (libpdlp_gen.so; host-only data plumbing, not part of the solve path).
 *
 * The reference's own generator (proj/include/pdhglp/generator.hpp:96-104)
 * samples an m×n Bernoulli mask and cannot build the BASELINE configs, so
 * these are new recipes in the same splitmix64 style (generator.hpp:75-94),
 * restated from BASELINE.json configs[0..4] / SURVEY.md §8(d):
 *
 *   C0  pdlp_gen_random_lp with params from pdlp_gen_c0_params()
 *   C1  pdlp_gen_transport(2000, 2000, seed)
 *   C2  pdlp_gen_random_lp with params from pdlp_gen_c2_params()
 *   C3  pdlp_gen_unit_commitment(8760, 1000, seed)
 *   C4  pdlp_gen_random_lp with params from pdlp_gen_c4_params()
 *
 * Instances own their arrays; pdlp_instance_view() exposes them as the
 * solver's pdlp_problem_view.
 */
#ifndef PDLP_GEN_H_
#define PDLP_GEN_H_

#include <stdint.h>

#include "pdlp_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pdlp_instance pdlp_instance;

typedef struct pdlp_gen_params {
  int64_t rows;
  int64_t cols;
  /* per-column entry counts: 0 = fixed (count_fixed), 1 = discrete power law
   * P(k) ~ k^-alpha on [kmin, kmax] (inverse-CDF sampling, rejection above kmax) */
  int32_t count_kind;
  int32_t value_kind; /* 0 = magnitude uniform [lo, hi], 1 = log-uniform [lo, hi]; random sign */
  int64_t count_fixed;
  double alpha;
  int64_t kmin;
  int64_t kmax;
  double value_lo;
  double value_hi;
  /* row types: the first round(eq_frac*rows) rows are equalities when
   * eq_rows_first != 0, else each row is an equality with prob. eq_frac;
   * the others are <= rows with slack U[0, slack_hi]. */
  double eq_frac;
  int32_t eq_rows_first;
  /* variable bounds: 0 = all [0, box_hi] (C0); 1 = mix [0,inf) 60 % / [l,u] 30 % / free 10 % (C2) */
  int32_t bound_kind;
  double box_hi;
  double slack_hi;
  uint64_t seed;
} pdlp_gen_params;

void pdlp_gen_c0_params(pdlp_gen_params* p, uint64_t seed);
void pdlp_gen_c2_params(pdlp_gen_params* p, uint64_t seed);
void pdlp_gen_c4_params(pdlp_gen_params* p, uint64_t seed);

/* Random sparse LP constructed feasible and bounded (C0/C2/C4 recipes). */
pdlp_instance* pdlp_gen_random_lp(const pdlp_gen_params* params);
/* Rows [r0, r1) of the random-LP family as a standalone LP (a row shard of a
 * large instance without building the whole; per-column / per-row
 * counter-based streams, multi-threaded).  NULL on bad arguments. */
pdlp_instance* pdlp_gen_random_lp_window(const pdlp_gen_params* params, int64_t r0, int64_t r1);

/* One rank's shard of the counter-based instance pdlp_gen_random_lp_window
 * (params, 0, rows) (every rank builds only its part):
 * rows [r0, r1) in both layouts -- K_g with global column indices and K_g^T
 * over all cols with local row indices, exactly the window's -- the row
 * bounds, and for the column block [c0, c1) the variable bounds and the
 * GLOBAL objective c = A'y* + r* (all rows of the block's columns).  With
 * [r0,r1) x [c0,c1) from pdlp_shard_plan_for it equals pdlp_shard_extract of
 * the whole instance.  NULL on bad ranges. */
typedef struct pdlp_gen_shard pdlp_gen_shard;
pdlp_gen_shard* pdlp_gen_random_lp_shard(const pdlp_gen_params* params, int64_t r0, int64_t r1,
                                         int64_t c0, int64_t c1);
/* The same instance's shard under PDLP_CUT_COLS: the block's columns
 * [c0, c1) in both layouts -- K_g^T with global row indices, exactly the
 * instance's columns, and K_g over all rows with local column indices --
 * their variable bounds and objective, and the row bounds of [r0, r1) (from
 * the row window, which draws every column's stream once).  Equals
 * pdlp_shard_extract_cut(..., PDLP_CUT_COLS) of the whole instance except
 * row_entry_offset (NULL: not known without the rest of the rows). */
pdlp_gen_shard* pdlp_gen_random_lp_colshard(const pdlp_gen_params* params, int64_t r0, int64_t r1,
                                            int64_t c0, int64_t c1);
/* The shard as the solver's pdlp_shard_view (plan.rank / world / blocks left
 * 0 for the caller to fill; plan.cut set; arrays owned by the shard). */
void pdlp_gen_shard_view(const pdlp_gen_shard* shard, pdlp_shard_view* out);
void pdlp_gen_shard_free(pdlp_gen_shard* shard);

/* Transportation LP (C1): `sources` supply rows sum_d x_sd <= s_s (s integer
 * U[50,150]), `sinks` demand rows sum_s x_sd >= d_d (d scaled to 95 % of total
 * supply), n = sources*sinks flows x >= 0, all coefficients +1, costs U[1,100]. */
pdlp_instance* pdlp_gen_transport(int64_t sources, int64_t sinks, uint64_t seed);

/* Unit-commitment-style staircase LP relaxation (C3).  Variables p_gt >= 0,
 * u_gt in [0,1]; rows: demand balance per period, ramp rows linking adjacent
 * periods, capacity rows p_gt - P_g u_gt <= 0. */
pdlp_instance* pdlp_gen_unit_commitment(int64_t periods, int64_t generators, uint64_t seed);

/* Build an instance from triplets with the reference's from_triplets
 * semantics (sparse.hpp:48-115): counting sort by line, stable sort by
 * secondary index, duplicates summed in input order.  Vectors are copied. */
pdlp_instance* pdlp_instance_from_triplets(int64_t rows, int64_t cols, int64_t count,
                                           const int64_t* r, const int64_t* c,
                                           const double* v, const double* objective,
                                           const double* con_lower, const double* con_upper,
                                           const double* var_lower, const double* var_upper);

void pdlp_instance_view(const pdlp_instance* inst, pdlp_problem_view* view);
/* Known feasible primal point (length cols) or NULL. */
const double* pdlp_instance_feasible_point(const pdlp_instance* inst);
void pdlp_instance_free(pdlp_instance* inst);

#ifdef __cplusplus
}
#endif

#endif /* PDLP_GEN_H_ */
