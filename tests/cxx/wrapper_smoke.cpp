// Host-only checks of include/sparse2d_b200.hpp (no GPU): the reference's
// C++ API shape and exception types over the C ABI.  Known answers from the
// reference's tests (tests/python/test_smoke.py:47-53, test_planner.cpp).
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "sparse2d_b200.hpp"

namespace b = sparse2d_b200;

#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                    \
    }                                                              \
  } while (0)

template <typename E, typename F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  const s2d_topology t = b::make_topology(8, 2);
  EXPECT(t.total_ranks == 8 && t.groups == 2 && t.ranks_per_group == 4);
  EXPECT(throws<std::invalid_argument>([] { b::make_topology(8, 3); }));

  const std::vector<s2d_table_load_profile> prof = {
      {0, 640, 7.0, 10}, {1, 640, 5.0, 10}, {2, 640, 4.0, 10}, {3, 640, 3.0, 10}, {4, 640, 1.0, 10}};
  const auto plan = b::plan_greedy(prof, 2, b::ShardingStrategy::kTableWise);
  EXPECT(plan.size() == 5);
  const uint32_t want[5] = {0, 1, 1, 0, 1};
  for (const auto& e : plan) EXPECT(e.local_rank == want[e.table_id]);
  b::validate_plan(plan, 2, prof);
  EXPECT(b::owner_of(plan, 3, 7) == 0);
  EXPECT(throws<std::out_of_range>([&] { b::owner_of(plan, 3, 10); }));
  const std::vector<s2d_plan_entry> bad = {{0, 0, 5, 0}};
  EXPECT(throws<std::invalid_argument>([&] { b::validate_plan(bad, 2, {{0, 40, 1.0, 10}}); }));

  const auto rw = b::plan_greedy({{0, 400, 1.0, 10}}, 4, b::ShardingStrategy::kRowWise);
  EXPECT(rw.size() == 4 && rw[1].row_lo == 2 && rw[1].row_hi == 5);  // [R*j/N, R*(j+1)/N)

  EXPECT(b::imbalance_ratio({10.0, 10.0, 10.0, 50.0}) == 2.5);
  EXPECT(throws<std::invalid_argument>([] { b::imbalance_ratio({}); }));

  const s2d_optimizer_config cfg{0.1, 1e-8, 4.0, S2D_ROWWISE_ADAGRAD};
  EXPECT(b::effective_lr(16.0, cfg) == 0.1 / (std::sqrt(16.0 / 4.0) + 1e-8));
  const s2d_optimizer_config badc{0.1, 1e-8, 0.0, S2D_ROWWISE_ADAGRAD};
  EXPECT(throws<std::invalid_argument>([&] { b::effective_lr(1.0, badc); }));
  std::printf("WRAPPER OK\n");
  EXPECT(b::memory_overhead(1700.0, 1, 1024) == 0.0);
  EXPECT(std::fabs(b::memory_overhead(1700.0, 4, 1024) - 4.98046875) < 1e-12);
  EXPECT(b::closed_form_ratio(0.0, 1.0, 16, 32, 4) == 4.0);
  EXPECT(std::fabs(b::recommend_c(1.0, 0.5, 4, 1, 4) - 1.6) < 1e-12);
  EXPECT(throws<std::invalid_argument>([] { b::qps_scaling_factor(1.0, 4, 2.0, 4); }));
  return 0;
}
