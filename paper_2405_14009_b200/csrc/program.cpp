// program.cpp — per-rank programs derived from the plan (host logic, no GPU).
//
// Worker (i, k) = rank k*N + i walks its ops in planned start order (the AR op of each
// iteration right after its last W / BC of that iteration) and emits, per op:
//   F  : LOAD_X (stage 0) | RECV_X from exec(i-1, j, k); F; SEND_Y to exec(i+1, j, k)
//   B  : LOSS (last stage) | RECV_DY from exec(i+1, j, k); B; SEND_DX to exec(i-1, j, k)
//   W  : W (releases the slot)        BC: like B, then W semantics
//   AR, OPT
// These are the ReRouteAct / ReRouteGrad pipeline instructions of PAPER.md line 554 in
// explicit form.  check_fifo() verifies that every directed pair receives in send order.
#include <algorithm>
#include <map>
#include <vector>

#include "common.h"
#include "planner.h"
#include "program.h"

namespace slip {

slip_status build_program(const Cluster& cl, const Plan& plan, int H, int rank, std::vector<slip_action>& out,
                          int& n_slots) {
  out.clear();
  n_slots = 0;
  const int N = cl.N, DP = cl.DP, m = cl.m;
  const int me_i = rank % N, me_k = rank / N;
  if (rank < 0 || rank >= N * DP) {
    set_error("rank_program: rank out of range");
    return SLIP_EINVAL;
  }
  if (!cl.is_live(me_i, me_k)) return SLIP_OK;
  auto exec_of = [&](int i, int j, int k) { return plan.exec[(static_cast<size_t>(i) * m + j) * DP + k]; };
  std::vector<slip_op> mine;
  for (const slip_op& o : plan.ops)
    if (o.phase != SLIP_AR && o.stage == me_i && o.exec == me_k) mine.push_back(o);
  std::vector<int> last_w(H, -1);
  for (size_t q = 0; q < mine.size(); ++q)
    if (mine[q].phase == SLIP_W || mine[q].phase == SLIP_BC) last_w[mine[q].iter] = static_cast<int>(q);
  std::vector<char> used;  // slot occupancy
  std::map<int64_t, int> slot_of;
  std::vector<char> first_b(H, 1), first_w(H, 1);
  auto key = [&](const slip_op& o) { return (static_cast<int64_t>(o.iter) * m + o.mb) * DP + o.origin; };
  auto act = [&](int kind, const slip_op& o, int peer, int slot, int acc) {
    out.push_back({kind, o.iter, o.mb, o.origin, peer, slot, acc});
  };
  for (size_t q = 0; q < mine.size(); ++q) {
    const slip_op& o = mine[q];
    if (o.phase == SLIP_F) {
      int slot = 0;
      while (slot < static_cast<int>(used.size()) && used[slot]) ++slot;
      if (slot == static_cast<int>(used.size())) used.push_back(0);
      used[slot] = 1;
      n_slots = std::max(n_slots, slot + 1);
      slot_of[key(o)] = slot;
      if (me_i == 0) act(SLIP_ACT_LOAD_X, o, -1, slot, 0);
      else act(SLIP_ACT_RECV_X, o, rank_of_worker(N, me_i - 1, exec_of(me_i - 1, o.mb, o.origin)), slot, 0);
      act(SLIP_ACT_F, o, -1, slot, 0);
      if (me_i + 1 < N) act(SLIP_ACT_SEND_Y, o, rank_of_worker(N, me_i + 1, exec_of(me_i + 1, o.mb, o.origin)), slot, 0);
    } else if (o.phase == SLIP_B || o.phase == SLIP_BC) {
      auto it = slot_of.find(key(o));
      if (it == slot_of.end()) {
        set_error("rank_program: B before F in the plan");
        return SLIP_ESTATE;
      }
      const int slot = it->second;
      int acc = first_b[o.iter] ? 0 : 1;
      // the LOSS head's B-side gradients (final LayerNorm) accumulate like B's
      if (me_i + 1 == N) act(SLIP_ACT_LOSS, o, -1, slot, acc);
      else act(SLIP_ACT_RECV_DY, o, rank_of_worker(N, me_i + 1, exec_of(me_i + 1, o.mb, o.origin)), slot, 0);
      first_b[o.iter] = 0;
      if (o.phase == SLIP_BC) {
        acc |= (first_w[o.iter] ? 0 : 2);
        first_w[o.iter] = 0;
      }
      act(o.phase == SLIP_BC ? SLIP_ACT_BC : SLIP_ACT_B, o, -1, slot, acc);
      if (me_i > 0) act(SLIP_ACT_SEND_DX, o, rank_of_worker(N, me_i - 1, exec_of(me_i - 1, o.mb, o.origin)), slot, 0);
      if (o.phase == SLIP_BC) {
        used[slot] = 0;
        slot_of.erase(it);
      }
    } else if (o.phase == SLIP_W) {
      auto it = slot_of.find(key(o));
      if (it == slot_of.end()) {
        set_error("rank_program: W before F in the plan");
        return SLIP_ESTATE;
      }
      const int acc = first_w[o.iter] ? 0 : 1;
      first_w[o.iter] = 0;
      act(SLIP_ACT_W, o, -1, it->second, acc);
      used[it->second] = 0;
      slot_of.erase(it);
    } else if (o.phase == SLIP_OPT) {
      act(SLIP_ACT_OPT, o, -1, -1, 0);
    }
    for (int t = 0; t < H; ++t)
      if (last_w[t] == static_cast<int>(q)) out.push_back({SLIP_ACT_AR, t, -1, -1, -1, -1, 0});
  }
  return SLIP_OK;
}

bool check_fifo(const Cluster& cl, const std::vector<std::vector<slip_action>>& progs, int only_rank) {
  // (src, dst, kind 0 = act / 1 = grad) -> sequence of (iter, mb, origin)
  std::map<std::tuple<int, int, int>, std::vector<std::tuple<int, int, int>>> snd, rcv;
  const int W = cl.N * cl.DP;
  for (int r = 0; r < W; ++r)
    for (const slip_action& a : progs[r]) {
      const auto id = std::make_tuple(a.iter, a.mb, a.origin);
      if (a.kind == SLIP_ACT_SEND_Y) snd[{r, a.peer, 0}].push_back(id);
      if (a.kind == SLIP_ACT_SEND_DX) snd[{r, a.peer, 1}].push_back(id);
      if (a.kind == SLIP_ACT_RECV_X) rcv[{a.peer, r, 0}].push_back(id);
      if (a.kind == SLIP_ACT_RECV_DY) rcv[{a.peer, r, 1}].push_back(id);
    }
  if (only_rank < 0) return snd == rcv;
  for (const auto& kv : rcv)
    if (std::get<1>(kv.first) == only_rank || std::get<0>(kv.first) == only_rank) {
      auto it = snd.find(kv.first);
      if (it == snd.end() || it->second != kv.second) return false;
    }
  for (const auto& kv : snd)
    if (std::get<1>(kv.first) == only_rank || std::get<0>(kv.first) == only_rank) {
      auto it = rcv.find(kv.first);
      if (it == rcv.end() || it->second != kv.second) return false;
    }
  return true;
}

}  // namespace slip

using namespace slip;

extern "C" slip_status slip_rank_program(const slip_cluster* c, const slip_costs* costs, const slip_plan_opts* opts,
                                         int32_t rank, slip_action* out, int64_t cap, int64_t* n, int32_t* n_slots) {
  Cluster cl;
  SLIP_TRY(read_cluster(c, cl));
  SLIP_CHECK(costs && opts && n, SLIP_EINVAL, "rank_program: NULL argument");
  Plan plan;
  SLIP_TRY(slip::plan(cl, *costs, *opts, plan));
  std::vector<slip_action> prog;
  int ns = 0;
  SLIP_TRY(build_program(cl, plan, opts->horizon < 1 ? 1 : opts->horizon, rank, prog, ns));
  *n = static_cast<int64_t>(prog.size());
  if (out && cap > 0) std::copy(prog.begin(), prog.begin() + std::min<int64_t>(cap, *n), out);
  if (n_slots) *n_slots = ns;
  return SLIP_OK;
}
