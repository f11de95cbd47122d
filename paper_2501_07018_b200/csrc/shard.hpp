// Sharded partition of an LP, host side.  Two cuts
// (pdlp_b200.h): PDLP_CUT_ROWS below, and PDLP_CUT_COLS, its transpose --
// rank g holds its columns in both layouts (K_g^T: the block's columns with
// global row indices; K_g: all m rows, only the block's entries, local
// column indices) and the same row / column blocks of the vectors.
//
// PDLP_CUT_ROWS: rank g of `world` owns
//   rows    [g*mb, min(m, (g+1)*mb))   of A, both layouts restricted to them:
//           K_g   = those rows of CSR(A)      (lines local, global columns)
//           K_g^T = CSR(A^T) over all n columns, only entries of those rows,
//                   row indices made local
//   columns [g*nb, min(n, (g+1)*nb))   the primal block: x, c, l_v, u_v, A'y.
// Blocks are equal-sized (nb, mb even, so every rank's block of a gathered
// vector starts 16-byte aligned) because NCCL all-gather / reduce-scatter
// exchange equal blocks; only the last blocks may be short or empty.
#pragma once

#include <cstdint>
#include <vector>

#include "pdlp_b200.h"

namespace pdlp_host {

pdlp_shard_plan shard_plan(int64_t m, int64_t n, int rank, int world, int cut);
// The cut pdlp_shard_plan_for picks: the one exchanging the smaller
// dimension (PDLP_SHARD_CUT=rows|cols overrides).
int auto_cut(int64_t m, int64_t n);

// Owned arrays behind a pdlp_shard_view.  PDLP_CUT_ROWS: index/value of K_g
// point into the caller's by_row arrays, K_g^T is rebuilt here.
// PDLP_CUT_COLS: index/value of K_g^T point into the caller's by_col arrays,
// K_g (all rows, the block's columns) is rebuilt here.
struct ShardData {
  pdlp_shard_view view{};
  std::vector<int64_t> row_start;
  std::vector<int64_t> col_start, col_index;
  std::vector<double> col_value;
  std::vector<int64_t> row_index, row_entry_offset;
  std::vector<double> row_value;
};

// Throws InvalidProblem-style std::invalid_argument on a structurally broken
// layout (non-monotone line pointers, an index out of range or unsorted
// within a line); the per-value checks run on device after upload.
void extract_shard(const pdlp_problem_view& p, int rank, int world, int cut, ShardData& out);

}  // namespace pdlp_host
