// The paper's step-selection rule (§2.1.2), evaluated on the host in double.
//
// Bit-exact schedule parity with the reference requires every floating-point
// expression below to be evaluated in the same operation order as
// cost_model.hpp:67-250 of the reference (ExpMark, the four single-step
// costs, the DFS-tail predictions, the greedy exception and the fixed
// tie order).  The host is compiled with -ffp-contract=off and no -march so
// no FMA contraction changes a rounding.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <optional>

#include "common.hpp"

namespace synchro {

enum class StepKind { BFS = 0, BFS_NH = 1, IBFS = 2, IBFS_NH = 3, DFS = 4 };

inline const char* step_kind_name(StepKind k) {
  static constexpr const char* kNames[] = {"BFS", "BFS_NH", "IBFS", "IBFS_NH", "DFS"};
  const int i = static_cast<int>(k);
  return (i >= 0 && i < 5) ? kNames[i] : "?";
}

struct TuningParams {
  double set_cost = 512.0;
  std::optional<double> dfs_reduction_of_reduction;  // 1/k when unset
  double dfs_set_cost_weight = 0.25;
  double dfs_check_cost_weight = 0.25;
  double reduction_of_reduction(double k) const {
    return dfs_reduction_of_reduction ? *dfs_reduction_of_reduction : 1.0 / k;
  }
};

struct SideStats {
  double list_size = 0, list_density = 0;
  double hist_size = 0, hist_density = 0;
  double r_dupl = 0, r_self = 0, r_hist = 0;
  bool hist_dropped = false;
  bool step_feasible = true;
  bool nh_feasible = true;
};

struct SearchStats {
  SideStats bfs, ibfs;
  double k = 2;
  double r = 0;
  double R = 1;
  bool dfs_feasible = true;
};

inline constexpr double kDensityEps = 1e-6;

// ExpMark(|A|, |B|, d_A, d_B): expected subset checks of MarkSupersets.
inline double exp_mark(double a_s, double b_s, double a_d, double b_d) {
  if (a_s <= 0 || b_s <= 0) return 0.0;
  a_d = std::clamp(a_d, kDensityEps, 1.0 - kDensityEps);
  b_d = std::clamp(b_d, kDensityEps, 1.0 - kDensityEps);
  const double base = (1.0 + b_d) / (1.0 + a_d * b_d - a_d);
  const double expo = std::log(1.0 + b_d) / std::log(base);
  return b_s * ((1.0 + b_d) / b_d + 1.0 / (a_d - a_d * b_d)) * std::pow(a_s, expo);
}

inline double dfs_branching_factor(const SearchStats& s, const TuningParams& p) {
  return s.k * (1.0 - s.ibfs.r_dupl * p.reduction_of_reduction(s.k));
}

inline double geometric_levels(double f, double m) {
  if (m <= 0) return 0.0;
  if (f == 1.0) return m;
  return f * (std::pow(f, m) - 1.0) / (f - 1.0);
}

namespace cost_detail {
// Expected list sizes after each reduction, multiplied in the reference's order:
// k*(1-r_dupl)*L, k*(1-r_dupl)*(1-r_self)*L, k*(1-r_dupl)*(1-r_self)*(1-r_hist)*L.
inline double after_dupl(double k, const SideStats& s) { return k * (1 - s.r_dupl) * s.list_size; }
inline double after_self(double k, const SideStats& s) {
  return k * (1 - s.r_dupl) * (1 - s.r_self) * s.list_size;
}
inline double after_hist(double k, const SideStats& s) {
  return k * (1 - s.r_dupl) * (1 - s.r_self) * (1 - s.r_hist) * s.list_size;
}
// Meet-check ExpMark after a step of `kind` (BFS side is always the A list).
inline double meet_term(StepKind kind, double k, const SideStats& B, const SideStats& I) {
  switch (kind) {
    case StepKind::BFS: return exp_mark(after_hist(k, B), I.list_size, B.list_density, I.list_density);
    case StepKind::BFS_NH: return exp_mark(after_self(k, B), I.list_size, B.list_density, I.list_density);
    case StepKind::IBFS: return exp_mark(B.list_size, after_hist(k, I), B.list_density, I.list_density);
    default: return exp_mark(B.list_size, after_self(k, I), B.list_density, I.list_density);
  }
}
}  // namespace cost_detail

// Single-step cost: expansion + self-reduction [+ history] + meet check.
// IBFS reductions run on complements (density 1-d).
inline double step_cost(StepKind kind, const SearchStats& s, const TuningParams& p) {
  using namespace cost_detail;
  const double k = s.k;
  const SideStats& B = s.bfs;
  const SideStats& I = s.ibfs;
  switch (kind) {
    case StepKind::BFS:
      return p.set_cost * k * B.list_size +
             exp_mark(after_dupl(k, B), after_dupl(k, B), B.list_density, B.list_density) +
             exp_mark(B.hist_size, after_self(k, B), B.hist_density, B.list_density) +
             meet_term(kind, k, B, I);
    case StepKind::BFS_NH:
      return p.set_cost * k * B.list_size +
             exp_mark(after_dupl(k, B), after_dupl(k, B), B.list_density, B.list_density) +
             meet_term(kind, k, B, I);
    case StepKind::IBFS:
      return p.set_cost * k * I.list_size +
             exp_mark(after_dupl(k, I), after_dupl(k, I), 1 - I.list_density, 1 - I.list_density) +
             exp_mark(I.hist_size, after_self(k, I), 1 - I.hist_density, 1 - I.list_density) +
             meet_term(kind, k, B, I);
    case StepKind::IBFS_NH:
      return p.set_cost * k * I.list_size +
             exp_mark(after_dupl(k, I), after_dupl(k, I), 1 - I.list_density, 1 - I.list_density) +
             meet_term(kind, k, B, I);
    case StepKind::DFS: break;
  }
  throw std::logic_error("step_cost: DFS has no single-step cost");
}

// Step cost plus the DFS tail over the remaining horizon.
inline double predicted_cost(StepKind kind, const SearchStats& s, const TuningParams& p) {
  const double k = s.k;
  const double f = dfs_branching_factor(s, p);
  const double set_term = p.set_cost * p.dfs_set_cost_weight * k / f;
  if (kind == StepKind::DFS)
    return geometric_levels(f, s.R - s.r) *
           (set_term + p.dfs_check_cost_weight * exp_mark(s.bfs.list_size, s.ibfs.list_size,
                                                          s.bfs.list_density, s.ibfs.list_density));
  const double tail = geometric_levels(f, s.R - s.r - 1);
  const double check = cost_detail::meet_term(kind, k, s.bfs, s.ibfs);
  return step_cost(kind, s, p) + tail * (set_term + p.dfs_check_cost_weight * check);
}

struct StepCosts {
  std::array<double, 5> step{};
  std::array<double, 5> pred{};
  std::array<bool, 5> feasible{};
};

inline StepCosts compute_step_costs(const SearchStats& s, const TuningParams& p) {
  constexpr double inf = std::numeric_limits<double>::infinity();
  const bool gate[5] = {s.bfs.step_feasible && !s.bfs.hist_dropped, s.bfs.nh_feasible,
                        s.ibfs.step_feasible && !s.ibfs.hist_dropped, s.ibfs.nh_feasible,
                        s.dfs_feasible};
  StepCosts c;
  for (int i = 0; i < 4; ++i) {
    c.feasible[i] = gate[i];
    c.step[i] = gate[i] ? step_cost(static_cast<StepKind>(i), s, p) : inf;
    c.pred[i] = gate[i] ? predicted_cost(static_cast<StepKind>(i), s, p) : inf;
  }
  c.step[4] = inf;
  c.feasible[4] = gate[4];
  c.pred[4] = gate[4] ? predicted_cost(StepKind::DFS, s, p) : inf;
  return c;
}

// Greedy BFS/IBFS by step cost while both history-free variants are dearer;
// otherwise minimal predicted cost, ties in order BFS, IBFS, BFS_NH, IBFS_NH, DFS.
inline StepKind select_step(const StepCosts& c) {
  if (std::none_of(c.feasible.begin(), c.feasible.end(), [](bool f) { return f; }))
    throw OutOfMemoryError("no feasible search step");
  if (c.step[1] > c.step[0] && c.step[3] > c.step[2])
    return c.step[0] <= c.step[2] ? StepKind::BFS : StepKind::IBFS;
  static constexpr int kOrder[5] = {0, 2, 1, 3, 4};
  int best = -1;
  for (int i : kOrder)
    if (c.feasible[i] && (best < 0 || c.pred[i] < c.pred[best])) best = i;
  return static_cast<StepKind>(best);
}

}  // namespace synchro
