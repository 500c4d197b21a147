// normalize.cpp — Phase 1 of the Planner (§4.2.1): Algorithm 1
// over a cost table, the heuristic cost table built from the list scheduler of
// planner.cpp, the placement of R, and the minimum migration swaps.  Host only;
// bit-exact with oracle/normalize.py (readings R26-R29 in DESIGN.md).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.h"
#include "planner.h"

using namespace slip;

namespace {

constexpr int64_t kInf = SLIP_COST_INF;

Cluster full_cluster(int N, int DP, int m) {
  Cluster c;
  c.N = N;
  c.DP = DP;
  c.m = m;
  c.live.assign(static_cast<size_t>(N) * DP, 1);
  return c;
}

int failed_at(const std::vector<uint8_t>& live, int DP, int i) {
  int n = 0;
  for (int k = 0; k < DP; ++k) n += live[static_cast<size_t>(i) * DP + k] == 0;
  return n;
}

}  // namespace

extern "C" {

slip_status slip_normalize_costs(const slip_cluster* c, const slip_costs* costs, const slip_plan_opts* opts,
                                 int32_t F, int64_t* out_cost) {
  SLIP_CHECK(c && costs && opts && out_cost && F >= 0, SLIP_EINVAL, "normalize_costs: bad argument");
  SLIP_CHECK(c->num_stages >= 1 && c->num_pipelines >= 1 && c->num_microbatches >= 1, SLIP_EINVAL,
             "normalize_costs: N, DP and m must be >= 1");
  const int N = c->num_stages, DP = c->num_pipelines, m = c->num_microbatches;
  Plan base;
  SLIP_TRY(plan(full_cluster(N, DP, m), *costs, *opts, base));
  for (int i = 0; i < N; ++i)
    for (int x = 0; x <= F; ++x) {
      int64_t& out = out_cost[static_cast<size_t>(i) * (F + 1) + x];
      if (x == 0) {
        out = 0;
      } else if (x > DP - 1) {
        out = kInf;
      } else {
        Cluster cl = full_cluster(N, DP, m);
        for (int q = 0; q < x; ++q) cl.live[static_cast<size_t>(i) * DP + (DP - 1 - q)] = 0;
        Plan p;
        SLIP_TRY(plan(cl, *costs, *opts, p));
        out = p.period - base.period;
      }
    }
  return SLIP_OK;
}

slip_status slip_normalize(int32_t N, int32_t DP, int32_t F, const int64_t* cost, int64_t* out_C, int32_t* out_R) {
  SLIP_CHECK(cost && out_R && N >= 1 && DP >= 1 && F >= 0, SLIP_EINVAL, "normalize: bad argument");
  if (static_cast<int64_t>(F) > static_cast<int64_t>(N) * (DP - 1)) {
    set_error("normalize: F exceeds N (DP - 1); some stage would lose every worker");
    return SLIP_EUNRECOVERABLE;
  }
  const int W = F + 1;
  auto cst = [&](int i, int x) { return cost[static_cast<size_t>(i) * W + x]; };
  std::vector<int64_t> C(static_cast<size_t>(N) * W, kInf);
  std::vector<int> X(static_cast<size_t>(N) * W, -1);  // argmin x of A[i][f] (A = concat(A[i-1][f-x], x))
  for (int i = 0; i < N; ++i)
    for (int f = 0; f <= F; ++f) {
      if (i == 0) {
        if (f <= DP - 1) {  // cap, reading R26
          C[f] = cst(0, f);
          X[f] = f;
        }
        continue;
      }
      int64_t best = kInf;
      int bx = -1;
      for (int x = 0; x <= std::min(f, DP - 1); ++x) {
        const int64_t prev = C[static_cast<size_t>(i - 1) * W + (f - x)];
        if (prev == kInf) continue;
        const int64_t v = prev + cst(i, x);
        if (bx < 0 || v <= best) {  // ties -> larger x at the later stage (R27)
          best = v;
          bx = x;
        }
      }
      if (bx >= 0) {
        C[static_cast<size_t>(i) * W + f] = best;
        X[static_cast<size_t>(i) * W + f] = bx;
      }
    }
  // R = A[N-1][F], unrolled backwards through the argmins
  int f = F;
  for (int i = N - 1; i >= 0; --i) {
    const int x = X[static_cast<size_t>(i) * W + f];
    SLIP_CHECK(x >= 0, SLIP_ESTATE, "normalize: no assignment (internal)");
    out_R[i] = x;
    f -= x;
  }
  if (out_C) std::copy(C.begin(), C.end(), out_C);
  return SLIP_OK;
}

slip_status slip_normalized_live(int32_t N, int32_t DP, const int32_t* R, uint8_t* out_live) {
  SLIP_CHECK(R && out_live && N >= 1 && DP >= 1, SLIP_EINVAL, "normalized_live: bad argument");
  for (int i = 0; i < N; ++i)
    SLIP_CHECK(R[i] >= 0 && R[i] <= DP - 1, SLIP_EINVAL, "normalized_live: R[i] must be in [0, DP-1]");
  std::fill(out_live, out_live + static_cast<size_t>(N) * DP, 1);
  int c = 0;
  for (int i = N - 1; i >= 0; --i)
    for (int q = 0; q < R[i]; ++q, ++c) out_live[static_cast<size_t>(i) * DP + (DP - 1 - c % DP)] = 0;
  return SLIP_OK;
}

slip_status slip_migration_plan(const slip_cluster* c, const int32_t* R, slip_swap* out, int32_t cap,
                                int32_t* n_swaps, uint8_t* out_live) {
  Cluster cl;
  SLIP_TRY(read_cluster(c, cl));
  SLIP_CHECK(R && n_swaps, SLIP_EINVAL, "migration_plan: NULL argument");
  const int N = cl.N, DP = cl.DP;
  int F = 0, sumR = 0;
  for (int i = 0; i < N; ++i) {
    F += failed_at(cl.live, DP, i);
    SLIP_CHECK(R[i] >= 0, SLIP_EINVAL, "migration_plan: negative R");
    sumR += R[i];
  }
  SLIP_CHECK(sumR == F, SLIP_EINVAL, "migration_plan: sum(R) differs from the number of failed workers");
  bool ok = recoverable(cl);
  for (int i = 0; i < N; ++i) ok = ok && R[i] <= DP - 1;
  if (!ok) {
    set_error("migration_plan: actual set or target R leaves a stage without a live worker");
    return SLIP_EUNRECOVERABLE;
  }
  // excess failures leave their stage highest k first; deficit stages filled from the last back (R29)
  std::vector<std::pair<int, int>> movers;
  for (int i = 0; i < N; ++i) {
    int excess = failed_at(cl.live, DP, i) - R[i];
    for (int k = DP - 1; k >= 0 && excess > 0; --k)
      if (!cl.is_live(i, k)) {
        movers.push_back({i, k});
        --excess;
      }
  }
  std::vector<int> holes;
  for (int i = N - 1; i >= 0; --i)
    for (int d = R[i] - failed_at(cl.live, DP, i); d > 0; --d) holes.push_back(i);
  SLIP_CHECK(movers.size() == holes.size(), SLIP_ESTATE, "migration_plan: internal count mismatch");
  std::vector<uint8_t> cur = cl.live;
  auto at = [&](int i, int k) -> uint8_t& { return cur[static_cast<size_t>(i) * DP + k]; };
  std::vector<slip_swap> swaps;
  for (size_t s = 0; s < movers.size(); ++s) {
    const int i = movers[s].first, k = movers[s].second, i2 = holes[s];
    int src = -1;
    for (int kk = 0; kk < DP && src < 0; ++kk)
      if (at(i, kk)) src = kk;
    at(i, k) = 1;
    int k2 = -1, best = 0;
    for (int kk = DP - 1; kk >= 0; --kk) {  // fewest failures in the pipeline, ties -> highest k
      if (!at(i2, kk)) continue;
      int pf = 0;
      for (int ii = 0; ii < N; ++ii) pf += at(ii, kk) == 0;
      if (k2 < 0 || pf < best) {
        k2 = kk;
        best = pf;
      }
    }
    SLIP_CHECK(src >= 0 && k2 >= 0, SLIP_ESTATE, "migration_plan: no source or target (internal)");
    at(i2, k2) = 0;
    swaps.push_back({i, k, i2, k2, src});
  }
  *n_swaps = static_cast<int32_t>(swaps.size());
  if (out && cap > 0) std::copy(swaps.begin(), swaps.begin() + std::min<size_t>(cap, swaps.size()), out);
  if (out_live) std::copy(cur.begin(), cur.end(), out_live);
  return SLIP_OK;
}

}  // extern "C"
