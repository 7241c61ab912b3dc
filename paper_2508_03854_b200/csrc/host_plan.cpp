// Host-side mesh planning: Topology, plan_greedy, validate_plan, owner_of,
// imbalance_ratio, effective_lr.  Same semantics and error behaviour as the
// reference planner (src/planner.cpp:20-143, src/topology.cpp:7-17,
// src/optimizer.cpp:19-23,61-63); pure host logic, no device work.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "common.h"

namespace s2d {

void check_optimizer(const s2d_optimizer_config& c) {
  // OptimizerConfig::validate (optimizer.cpp:19-23): NaN fails every test.
  if (!(c.eta > 0)) throw Error(S2D_EINVAL, "optimizer.eta must be > 0");
  if (!(c.eps > 0)) throw Error(S2D_EINVAL, "optimizer.eps must be > 0");
  if (!(c.c > 0)) throw Error(S2D_EINVAL, "optimizer.c must be > 0");
  if (c.variant != S2D_ROWWISE_ADAGRAD && c.variant != S2D_SGD)
    throw Error(S2D_EINVAL, "unknown optimizer variant " + std::to_string(c.variant));
}

s2d_topology make_topology(uint32_t total, uint32_t groups) {
  if (total == 0) throw Error(S2D_EINVAL, "total_ranks must be >= 1");
  if (groups == 0) throw Error(S2D_EINVAL, "groups must be >= 1");
  if (total % groups)
    throw Error(S2D_EINVAL, "groups (" + std::to_string(groups) + ") must divide total_ranks (" +
                                std::to_string(total) + ")");
  return s2d_topology{total, groups, total / groups};
}

std::vector<s2d_plan_entry> plan_greedy(const std::vector<s2d_table_load_profile>& profiles,
                                        uint32_t n, int strategy) {
  if (n < 1) throw Error(S2D_EINVAL, "ranks per group must be >= 1");
  if (profiles.empty()) throw Error(S2D_EINVAL, "no table profiles");
  std::vector<s2d_plan_entry> plan;
  if (strategy == S2D_ROW_WISE) {
    // N near-equal contiguous ranges [R*j/N, R*(j+1)/N), range j -> local j;
    // empty ranges are dropped.
    for (const auto& p : profiles) {
      for (uint32_t j = 0; j < n; ++j) {
        const uint64_t lo = p.num_rows * j / n, hi = p.num_rows * (j + 1) / n;
        if (hi > lo) plan.push_back({p.table_id, (uint32_t)lo, (uint32_t)hi, j});
      }
    }
    return plan;
  }
  if (strategy != S2D_TABLE_WISE) throw Error(S2D_EINVAL, "unknown sharding strategy");
  // Longest-processing-time greedy: heaviest expected load first (ties:
  // lower table id first) into the least-loaded rank (ties: lower rank).
  std::vector<size_t> order(profiles.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    const auto &x = profiles[a], &y = profiles[b];
    if (x.expected_lookups_per_batch != y.expected_lookups_per_batch)
      return x.expected_lookups_per_batch > y.expected_lookups_per_batch;
    return x.table_id < y.table_id;
  });
  std::vector<double> load(n, 0.0);
  for (size_t i : order) {
    const auto& p = profiles[i];
    const uint32_t best = (uint32_t)(std::min_element(load.begin(), load.end()) - load.begin());
    load[best] += p.expected_lookups_per_batch;
    plan.push_back({p.table_id, 0u, (uint32_t)p.num_rows, best});
  }
  std::sort(plan.begin(), plan.end(),
            [](const s2d_plan_entry& a, const s2d_plan_entry& b) { return a.table_id < b.table_id; });
  return plan;
}

void validate_plan(const std::vector<s2d_plan_entry>& plan, uint32_t ranks_per_group,
                   const std::vector<s2d_table_load_profile>& profiles) {
  for (const auto& e : plan)
    if (e.local_rank >= ranks_per_group)
      throw Error(S2D_EINVAL, "plan entry names local rank " + std::to_string(e.local_rank) +
                                  " >= N=" + std::to_string(ranks_per_group));
  for (const auto& p : profiles) {
    std::vector<s2d_plan_entry> mine;
    for (const auto& e : plan)
      if (e.table_id == p.table_id) mine.push_back(e);
    std::sort(mine.begin(), mine.end(),
              [](const s2d_plan_entry& a, const s2d_plan_entry& b) { return a.row_lo < b.row_lo; });
    uint64_t next = 0;
    for (const auto& e : mine) {
      if (e.row_lo != next)
        throw Error(S2D_EINVAL, "table " + std::to_string(p.table_id) + " rows [" +
                                    std::to_string(next) + "," + std::to_string(e.row_lo) +
                                    ") uncovered or overlapping");
      next = e.row_hi;
    }
    if (next != p.num_rows)
      throw Error(S2D_EINVAL, "table " + std::to_string(p.table_id) + " covered to row " +
                                  std::to_string(next) + " of " + std::to_string(p.num_rows));
  }
}

uint32_t plan_owner_of(const s2d_plan_entry* plan, uint32_t n, uint32_t table, uint32_t row) {
  for (uint32_t i = 0; i < n; ++i)
    if (plan[i].table_id == table && row >= plan[i].row_lo && row < plan[i].row_hi)
      return plan[i].local_rank;
  throw Error(S2D_ERANGE, "row " + std::to_string(row) + " of table " + std::to_string(table) +
                              " not covered by plan");
}

double imbalance_ratio(const double* v, uint32_t n) {
  if (n == 0) throw Error(S2D_EINVAL, "imbalance_ratio over empty list");
  double sum = 0.0, mx = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    if (v[i] < 0.0) throw Error(S2D_EINVAL, "imbalance_ratio needs nonnegative values");
    sum += v[i];
    mx = std::max(mx, v[i]);
  }
  if (sum == 0.0) throw Error(S2D_EINVAL, "imbalance_ratio undefined for all-zero loads");
  return mx / (sum / (double)n);
}

double effective_lr(double v, const s2d_optimizer_config& c) {
  return c.eta / (std::sqrt(v / c.c) + c.eps);
}

}  // namespace s2d
