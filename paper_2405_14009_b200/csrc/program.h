// program.h — per-rank programs derived from the plan (see program.cpp).
#pragma once
#include <vector>

#include "planner.h"

namespace slip {

inline int rank_of_worker(int N, int i, int k) { return k * N + i; }

slip_status build_program(const Cluster& cl, const Plan& plan, int H, int rank, std::vector<slip_action>& out,
                          int& n_slots);

// True iff, for every directed pair (involving only_rank, or all pairs if < 0), the
// receiver's receive order equals the sender's send order.
bool check_fifo(const Cluster& cl, const std::vector<std::vector<slip_action>>& progs, int only_rank);

}  // namespace slip
