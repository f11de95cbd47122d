// Row-sharded partition of an LP, host side.
//
// Rank g of `world` owns
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

pdlp_shard_plan shard_plan(int64_t m, int64_t n, int rank, int world);

// Owned arrays behind a pdlp_shard_view (index/value of K_g point into the
// caller's by_row arrays; K_g^T is rebuilt here).
struct ShardData {
  pdlp_shard_view view{};
  std::vector<int64_t> row_start;
  std::vector<int64_t> col_start, col_index;
  std::vector<double> col_value;
};

// Throws InvalidProblem-style std::invalid_argument on a structurally broken
// layout (non-monotone line pointers, a row index out of range or unsorted
// within a column); the per-value checks run on device after upload.
void extract_shard(const pdlp_problem_view& p, int rank, int world, ShardData& out);

}  // namespace pdlp_host
