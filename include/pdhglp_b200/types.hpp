// Standalone definitions of the reference structs the solve() boundary uses,
// for builds without the reference headers (define PDHGLP_B200_STANDALONE).
// Field names, order and defaults follow the reference:
//   Scalar/Index/Vector/kInf           core.hpp:10-14
//   CompressedLayout, SparseMatrix     sparse.hpp:21-42
//   LpProblem                          problem.hpp:15-25
//   ResidualSummary, TerminationTolerances,
//   CertificateKind, InfeasibilityCertificate   residuals.hpp:66-73, 187-210
//   RestartThresholds                  restarts.hpp:235-239
#pragma once

#include <algorithm>
#include <cstdint>
#include <limits>
#include <utility>
#include <vector>

namespace pdhglp {

using Scalar = double;
using Index = std::int64_t;
using Vector = std::vector<Scalar>;
inline constexpr Scalar kInf = std::numeric_limits<Scalar>::infinity();

struct Triplet {
  Index row = 0;
  Index col = 0;
  Scalar value = 0.0;
};

struct CompressedLayout {
  std::vector<Index> start;
  std::vector<Index> index;
  std::vector<Scalar> value;
  Index primary_dim() const { return static_cast<Index>(start.size()) - 1; }
  Index nonzeros() const { return static_cast<Index>(value.size()); }
};

struct SparseMatrix {
  Index rows = 0;
  Index cols = 0;
  CompressedLayout by_row;
  CompressedLayout by_col;
  Index nonzeros() const { return by_row.nonzeros(); }

  // Lines sorted by secondary index, duplicates summed in input order.
  static SparseMatrix from_triplets(Index rows, Index cols, const std::vector<Triplet>& t) {
    SparseMatrix a;
    a.rows = rows;
    a.cols = cols;
    a.by_row = orient(rows, t, true);
    a.by_col = orient(cols, t, false);
    return a;
  }

 private:
  static CompressedLayout orient(Index dim, const std::vector<Triplet>& t, bool by_row) {
    std::vector<std::vector<std::pair<Index, Scalar>>> lines(static_cast<size_t>(dim));
    for (const Triplet& e : t) {
      lines[static_cast<size_t>(by_row ? e.row : e.col)].push_back({by_row ? e.col : e.row, e.value});
    }
    CompressedLayout out;
    out.start.push_back(0);
    for (auto& line : lines) {
      std::stable_sort(line.begin(), line.end(),
                       [](const auto& x, const auto& y) { return x.first < y.first; });
      for (size_t i = 0; i < line.size();) {
        Scalar s = line[i].second;
        size_t j = i + 1;
        for (; j < line.size() && line[j].first == line[i].first; ++j) s += line[j].second;
        out.index.push_back(line[i].first);
        out.value.push_back(s);
        i = j;
      }
      out.start.push_back(static_cast<Index>(out.index.size()));
    }
    return out;
  }
};

struct LpProblem {
  SparseMatrix a;
  Vector objective;
  Vector con_lower;
  Vector con_upper;
  Vector var_lower;
  Vector var_upper;
  Index rows() const { return a.rows; }
  Index cols() const { return a.cols; }
};

struct ResidualSummary {
  Scalar primal_residual_inf = kInf;
  Scalar dual_residual_inf = kInf;
  Scalar primal_objective = 0.0;
  Scalar dual_objective = 0.0;
  Scalar abs_gap = kInf;
  Scalar rel_gap = kInf;
};

struct TerminationTolerances {
  Scalar eps_primal = 1e-8;
  Scalar eps_dual = 1e-8;
  Scalar eps_rel_gap = 1e-2;
};

enum class CertificateKind { PrimalInfeasible, DualInfeasible };

struct InfeasibilityCertificate {
  CertificateKind kind = CertificateKind::PrimalInfeasible;
  Vector ray_x;
  Vector ray_y;
  Vector ray_r;
  Scalar residual_inf = kInf;
  Scalar objective = 0.0;
  const char* source = "";
};

struct RestartThresholds {
  Scalar sufficient = 0.1;
  Scalar necessary = 0.9;
  Scalar artificial = 0.5;
};

}  // namespace pdhglp
