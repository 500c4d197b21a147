// planner.h — internal interface of the C++ planner (see planner.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/slip.h"

namespace slip {

struct Cluster {
  int N = 0, DP = 0, m = 0;
  std::vector<uint8_t> live;  // [N*DP]
  bool is_live(int i, int k) const { return live[static_cast<size_t>(i) * DP + k] != 0; }
};

struct Plan {
  std::vector<int> exec;  // [(i*m + j)*DP + k] -> k_s
  std::vector<slip_op> ops;
  std::vector<int64_t> makespans;
  int64_t period = 0;
};

bool recoverable(const Cluster& c);
bool assign(const Cluster& c, std::vector<int>& exec);
slip_status plan(const Cluster& c, const slip_costs& costs, const slip_plan_opts& opts, Plan& out);
uint64_t plan_hash(const slip_op* ops, int64_t n);
slip_status read_cluster(const slip_cluster* c, Cluster& out);

}  // namespace slip
