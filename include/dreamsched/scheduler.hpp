// dreamsched/scheduler.hpp — Algorithm 2 (pruned DFS) + bubble fill (Eq. 10).
// Drop-in for the reference's scheduler.hpp:30-78; output must match the
// reference bit-for-bit for identical profiles (tests/test_scheduler_parity.py).
#ifndef DREAMSCHED_SCHEDULER_HPP_
#define DREAMSCHED_SCHEDULER_HPP_

#include <cstdint>
#include <optional>
#include <vector>

#include "dreamsched/cost_model.hpp"
#include "dreamsched/profile.hpp"
#include "dreamsched/schedule.hpp"

namespace dreamsched {

enum class Assignment { kCommunicationHide, kCommunicationOverflow };

struct AssignmentState {
  std::vector<std::vector<int>> sets;
  int next_layer = 0;
  int iteration = 1;
};

Assignment classify_assignment(const AssignmentState& state, int layer,
                               const ModelProfile& profile);

enum class AssignRule { kAtLeastOne, kOptimalHiding, kDelayedCo, kDfsBranch };

struct AssignmentDecision {
  int layer = 0;
  int iteration = 0;
  AssignRule rule = AssignRule::kAtLeastOne;
};

struct SearchReport {
  Schedule best;
  double best_cost = 0.0;
  std::uint64_t solutions_explored = 0;
  std::optional<double> oracle_cost;
  std::vector<AssignmentDecision> classification_log;
};

SearchReport schedule_dfs(const ModelProfile& profile, int period);
SearchReport schedule_brute_force(const ModelProfile& profile, int period,
                                  std::optional<std::uint64_t> limit = {});
std::uint64_t brute_force_candidate_count(int layer_count, int period);
Schedule bubble_fill(const Schedule& schedule, const ModelProfile& profile);

}  // namespace dreamsched

#endif  // DREAMSCHED_SCHEDULER_HPP_
