// planner.cpp — deterministic CPU planner: recoverability, round-robin re-route
// assignment and the heuristic list schedule (Adaptive Pipelining + Decoupled BackProp +
// Staggered Optimizer).  Algorithm and tie-breaks: DESIGN.md "Planner reading"
// (§3.1-3.4, §4.2 lines 426-430 heuristic, Eqs. 2-6 dependencies).  The
// Python oracle (oracle/planner.py) is an independent transcription of the same
// algorithm; tests/test_planner_parity.py checks the two op lists for equality.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "common.h"
#include "planner.h"

namespace slip {

namespace {
constexpr int64_t kUnknown = std::numeric_limits<int64_t>::min();
}

bool recoverable(const Cluster& c) {
  for (int i = 0; i < c.N; ++i) {
    bool any = false;
    for (int k = 0; k < c.DP; ++k) any |= c.live[i * c.DP + k] != 0;
    if (!any) return false;
  }
  return true;
}

// exec[(i*m + j)*DP + k] = k_s
bool assign(const Cluster& c, std::vector<int>& ex) {
  if (!recoverable(c)) return false;
  ex.assign(static_cast<size_t>(c.N) * c.m * c.DP, -1);
  for (int i = 0; i < c.N; ++i) {
    std::vector<int> surv;
    for (int k = 0; k < c.DP; ++k)
      if (c.live[i * c.DP + k]) surv.push_back(k);
    int r = 0;
    for (int k = 0; k < c.DP; ++k)
      if (c.live[i * c.DP + k])
        for (int j = 0; j < c.m; ++j) ex[(static_cast<size_t>(i) * c.m + j) * c.DP + k] = k;
    for (int k = 0; k < c.DP; ++k) {
      if (c.live[i * c.DP + k]) continue;
      for (int j = 0; j < c.m; ++j) {
        ex[(static_cast<size_t>(i) * c.m + j) * c.DP + k] = surv[r % surv.size()];
        ++r;
      }
    }
  }
  return true;
}

namespace {

struct Task {
  int ph, t, i, j, k;  // OPT: j = -1, k = exec
};

class Scheduler {
 public:
  Scheduler(const Cluster& c, const slip_costs& co, const slip_plan_opts& op, const std::vector<int>& ex)
      : c_(c), co_(co), ex_(ex) {
    N = c.N;
    DP = c.DP;
    m = c.m;
    H = op.horizon < 1 ? 1 : op.horizon;
    dec = op.decoupled != 0;
    stag = op.staggered != 0;
    bwd = dec ? SLIP_B : SLIP_BC;
    lastw = dec ? SLIP_W : SLIP_BC;
    lim = co.m_limit > 0 ? co.m_limit : -1;
    const size_t nt = static_cast<size_t>(H) * N * m * DP;
    for (int p = 0; p < 4; ++p) end_[p].assign(nt, kUnknown);
    opt_end_.assign(static_cast<size_t>(H) * N * DP, kUnknown);
    ar_end_.assign(static_cast<size_t>(H) * N, kUnknown);
    for (int i = 0; i < N; ++i)
      for (int ks = 0; ks < DP; ++ks)
        if (c.live[i * DP + ks]) workers.push_back({i, ks});
    const size_t nw = workers.size();
    busy.assign(nw, 0);
    mem.assign(nw, 0);
    inflight.assign(nw, 0);
    pending.resize(nw);
    n_w.assign(nw, 0);
    for (size_t w = 0; w < nw; ++w) {
      const int i = workers[w].first, ks = workers[w].second;
      std::vector<char> origins(DP, 0);
      for (int j = 0; j < m; ++j)
        for (int k = 0; k < DP; ++k)
          if (exec(i, j, k) == ks) origins[k] = 1;
      for (int k = 0; k < DP; ++k) n_w[w] += origins[k];
      for (int t = 0; t < H; ++t) {
        for (int k = 0; k < DP; ++k)
          for (int j = 0; j < m; ++j) {
            if (exec(i, j, k) != ks) continue;
            pending[w].push_back({SLIP_F, t, i, j, k});
            if (dec) {
              pending[w].push_back({SLIP_B, t, i, j, k});
              pending[w].push_back({SLIP_W, t, i, j, k});
            } else {
              pending[w].push_back({SLIP_BC, t, i, j, k});
            }
          }
        pending[w].push_back({SLIP_OPT, t, i, -1, ks});
      }
    }
  }

  slip_status run(std::vector<slip_op>& out, std::vector<int64_t>& makespans, int64_t& period) {
    int64_t now = 0;
    auto any_pending = [&] {
      for (auto& p : pending)
        if (!p.empty()) return true;
      return false;
    };
    while (any_pending()) {
      bool progress = true;
      while (progress) {
        progress = false;
        update_ar();
        for (size_t w = 0; w < workers.size(); ++w)
          if (busy[w] <= now && dispatch(w, now)) progress = true;
      }
      update_ar();
      int64_t nxt = kUnknown;
      auto consider = [&](int64_t v) {
        if (v > now && (nxt == kUnknown || v < nxt)) nxt = v;
      };
      for (size_t w = 0; w < workers.size(); ++w) {
        consider(busy[w]);
        for (const Task& tk : pending[w]) {
          const int64_t rt = ready_time(tk);
          if (rt != kUnknown) consider(rt);
        }
      }
      if (nxt == kUnknown) {
        if (any_pending()) {
          set_error("planner: memory limit admits no further forward (Eq. 6 infeasible)");
          return SLIP_EINFEASIBLE_MEMORY;
        }
        break;
      }
      now = nxt;
    }
    update_ar();
    // canonical order: compute ops by (stage, exec, start) — stable — then AR by (iter, stage)
    std::vector<slip_op> comp, ars;
    for (const slip_op& o : ops)
      (o.phase == SLIP_AR ? ars : comp).push_back(o);
    std::stable_sort(comp.begin(), comp.end(), [](const slip_op& a, const slip_op& b) {
      if (a.stage != b.stage) return a.stage < b.stage;
      if (a.exec != b.exec) return a.exec < b.exec;
      return a.start < b.start;
    });
    std::stable_sort(ars.begin(), ars.end(), [](const slip_op& a, const slip_op& b) {
      if (a.iter != b.iter) return a.iter < b.iter;
      return a.stage < b.stage;
    });
    out = comp;
    out.insert(out.end(), ars.begin(), ars.end());
    makespans.assign(H, 0);
    for (int t = 0; t < H; ++t) {
      int64_t mx = kUnknown;
      for (const slip_op& o : out)
        if (o.iter == t) mx = std::max(mx, o.end);
      makespans[t] = mx;
    }
    period = H >= 2 ? makespans[H - 1] - makespans[H - 2] : makespans[0];
    return SLIP_OK;
  }

 private:
  int exec(int i, int j, int k) const { return ex_[(static_cast<size_t>(i) * m + j) * DP + k]; }
  size_t tid(int t, int i, int j, int k) const { return ((static_cast<size_t>(t) * N + i) * m + j) * DP + k; }
  int64_t& E(int ph, int t, int i, int j, int k) { return end_[ph][tid(t, i, j, k)]; }
  int64_t& OPTE(int t, int i, int ks) { return opt_end_[(static_cast<size_t>(t) * N + i) * DP + ks]; }
  int64_t dur(int ph) const {
    switch (ph) {
      case SLIP_F: return co_.t_f;
      case SLIP_B: return co_.t_b;
      case SLIP_W: return co_.t_w;
      case SLIP_BC: return co_.t_b + co_.t_w;
      default: return co_.t_opt;
    }
  }

  void update_ar() {
    for (int t = 0; t < H; ++t)
      for (int i = 0; i < N; ++i) {
        int64_t& a = ar_end_[static_cast<size_t>(t) * N + i];
        if (a != kUnknown) continue;
        int64_t mx = 0;
        bool done = true;
        for (int k = 0; k < DP && done; ++k)
          for (int j = 0; j < m; ++j) {
            const int64_t e = E(lastw, t, i, j, k);
            if (e == kUnknown) {
              done = false;
              break;
            }
            mx = std::max(mx, e);
          }
        if (!done) continue;
        a = mx + co_.t_ar;
        ops.push_back({i, -1, -1, SLIP_AR, -1, t, mx, mx + co_.t_ar});
      }
  }

  int64_t opt_dep(int t, int i, int ks) {
    if (t == 0) return 0;
    if (stag) return OPTE(t - 1, i, ks);
    int64_t mx = 0;
    for (auto& w : workers) {
      const int64_t e = OPTE(t - 1, w.first, w.second);
      if (e == kUnknown) return kUnknown;
      mx = std::max(mx, e);
    }
    return mx;
  }

  int64_t ready_time(const Task& x) {
    if (x.ph == SLIP_OPT) {
      if (stag) return ar_end_[static_cast<size_t>(x.t) * N + x.i];
      int64_t mx = 0;
      for (int ii = 0; ii < N; ++ii) {
        const int64_t e = ar_end_[static_cast<size_t>(x.t) * N + ii];
        if (e == kUnknown) return kUnknown;
        mx = std::max(mx, e);
      }
      return mx;
    }
    if (x.ph == SLIP_F) {
      const int64_t od = opt_dep(x.t, x.i, exec(x.i, x.j, x.k));
      if (od == kUnknown) return kUnknown;
      if (x.i == 0) return od;
      const int64_t up = E(SLIP_F, x.t, x.i - 1, x.j, x.k);
      return up == kUnknown ? kUnknown : std::max(od, up + co_.t_comm);
    }
    if (x.ph == SLIP_B || x.ph == SLIP_BC) {
      const int64_t fe = E(SLIP_F, x.t, x.i, x.j, x.k);
      if (fe == kUnknown) return kUnknown;
      if (x.i == N - 1) return fe;
      const int64_t dn = E(bwd, x.t, x.i + 1, x.j, x.k);
      return dn == kUnknown ? kUnknown : std::max(fe, dn + co_.t_comm);
    }
    return E(SLIP_B, x.t, x.i, x.j, x.k);  // W
  }

  int64_t arrival(const Task& x) {
    if (x.ph == SLIP_F) return x.i == 0 ? 0 : E(SLIP_F, x.t, x.i - 1, x.j, x.k) + co_.t_comm;
    if (x.i == N - 1) return E(SLIP_F, x.t, x.i, x.j, x.k);
    return E(bwd, x.t, x.i + 1, x.j, x.k) + co_.t_comm;
  }

  bool dispatch(size_t w, int64_t now) {
    const int i = workers[w].first, ks = workers[w].second;
    int best_opt = -1, best_b = -1, best_f = -1, best_w = -1;
    int64_t kb[5] = {0}, kf[4] = {0}, kw[4] = {0};
    std::vector<Task>& pend = pending[w];
    for (size_t q = 0; q < pend.size(); ++q) {
      const Task& x = pend[q];
      const int64_t rt = ready_time(x);
      if (rt == kUnknown || rt > now) continue;
      if (x.ph == SLIP_OPT) {
        if (best_opt < 0 || x.t < pend[best_opt].t) best_opt = static_cast<int>(q);
      } else if (x.ph == SLIP_B || x.ph == SLIP_BC) {
        const int64_t key[5] = {arrival(x), E(SLIP_F, x.t, x.i, x.j, x.k), x.t, x.k, x.j};
        if (best_b < 0 || std::lexicographical_compare(key, key + 5, kb, kb + 5)) {
          best_b = static_cast<int>(q);
          std::memcpy(kb, key, sizeof key);
        }
      } else if (x.ph == SLIP_F) {
        const int64_t key[4] = {arrival(x), x.t, x.k, x.j};
        if (best_f < 0 || std::lexicographical_compare(key, key + 4, kf, kf + 4)) {
          best_f = static_cast<int>(q);
          std::memcpy(kf, key, sizeof key);
        }
      } else {  // W
        const int64_t key[4] = {E(SLIP_B, x.t, x.i, x.j, x.k), x.t, x.k, x.j};
        if (best_w < 0 || std::lexicographical_compare(key, key + 4, kw, kw + 4)) {
          best_w = static_cast<int>(q);
          std::memcpy(kw, key, sizeof key);
        }
      }
    }
    int pick = -1;
    if (best_opt >= 0) {
      pick = best_opt;
    } else if (best_b >= 0) {
      pick = best_b;
    } else {
      const bool f_ok = best_f >= 0 && inflight[w] < static_cast<int64_t>(N - i) * n_w[w] &&
                        (lim < 0 || mem[w] + co_.a_f <= lim);
      if (f_ok) pick = best_f;
      else if (best_w >= 0) pick = best_w;
    }
    if (pick < 0) return false;
    const Task x = pend[pick];
    pend.erase(pend.begin() + pick);
    const int64_t s = now, e = now + dur(x.ph);
    busy[w] = e;
    switch (x.ph) {
      case SLIP_F:
        inflight[w] += 1;
        mem[w] += co_.a_f;
        break;
      case SLIP_B:
        inflight[w] -= 1;
        mem[w] -= co_.a_f - co_.a_w;
        break;
      case SLIP_W:
        mem[w] -= co_.a_w;
        break;
      case SLIP_BC:
        inflight[w] -= 1;
        mem[w] -= co_.a_f;
        break;
      default:
        break;
    }
    if (x.ph == SLIP_OPT) {
      OPTE(x.t, i, ks) = e;
      ops.push_back({i, -1, -1, SLIP_OPT, ks, x.t, s, e});
    } else {
      E(x.ph, x.t, x.i, x.j, x.k) = e;
      ops.push_back({i, x.j, x.k, x.ph, ks, x.t, s, e});
    }
    return true;
  }

  const Cluster& c_;
  const slip_costs& co_;
  const std::vector<int>& ex_;
  int N, DP, m, H;
  bool dec, stag;
  int bwd, lastw;
  int64_t lim;
  std::vector<int64_t> end_[4];  // indexed by phase F, B, W, BC
  std::vector<int64_t> opt_end_, ar_end_;
  std::vector<std::pair<int, int>> workers;
  std::vector<int64_t> busy, mem, inflight, n_w;
  std::vector<std::vector<Task>> pending;
  std::vector<slip_op> ops;
};

}  // namespace

slip_status plan(const Cluster& c, const slip_costs& costs, const slip_plan_opts& opts, Plan& out) {
  if (!assign(c, out.exec)) {
    set_error("planner: some stage has no live worker (unrecoverable, PAPER.md §3.4)");
    return SLIP_EUNRECOVERABLE;
  }
  if (opts.decoupled == 2) {
    // selective decoupling (§3.2, reading R32): plan with and
    // without Decoupled BackProp, keep the shorter steady-state period (ties: decoupled)
    slip_plan_opts od = opts, oc = opts;
    od.decoupled = 1;
    oc.decoupled = 0;
    Plan pd, pc;
    SLIP_TRY(plan(c, costs, od, pd));
    SLIP_TRY(plan(c, costs, oc, pc));
    out = pc.period < pd.period ? std::move(pc) : std::move(pd);
    return SLIP_OK;
  }
  Scheduler sch(c, costs, opts, out.exec);
  return sch.run(out.ops, out.makespans, out.period);
}

uint64_t plan_hash(const slip_op* ops, int64_t n) {
  uint64_t h = 0xCBF29CE484222325ULL;
  auto mix = [&](int64_t v) {
    for (int b = 0; b < 8; ++b) {
      h ^= static_cast<uint64_t>((static_cast<uint64_t>(v) >> (8 * b)) & 0xFF);
      h *= 0x100000001B3ULL;
    }
  };
  for (int64_t q = 0; q < n; ++q) {
    const slip_op& o = ops[q];
    mix(o.stage);
    mix(o.mb);
    mix(o.origin);
    mix(o.phase);
    mix(o.exec);
    mix(o.iter);
    mix(o.start);
    mix(o.end);
  }
  return h;
}

slip_status read_cluster(const slip_cluster* c, Cluster& out) {
  SLIP_CHECK(c && c->live, SLIP_EINVAL, "cluster or cluster->live is NULL");
  SLIP_CHECK(c->num_stages >= 1 && c->num_pipelines >= 1 && c->num_microbatches >= 1, SLIP_EINVAL,
             "cluster: N, DP and m must be >= 1");
  out.N = c->num_stages;
  out.DP = c->num_pipelines;
  out.m = c->num_microbatches;
  out.live.assign(c->live, c->live + static_cast<size_t>(out.N) * out.DP);
  return SLIP_OK;
}

}  // namespace slip

using namespace slip;

extern "C" {

slip_status slip_recoverable(const slip_cluster* c, int32_t* out) {
  Cluster cl;
  SLIP_TRY(read_cluster(c, cl));
  SLIP_CHECK(out, SLIP_EINVAL, "recoverable: out is NULL");
  *out = recoverable(cl) ? 1 : 0;
  return SLIP_OK;
}

slip_status slip_assign(const slip_cluster* c, int32_t* out_exec) {
  Cluster cl;
  SLIP_TRY(read_cluster(c, cl));
  SLIP_CHECK(out_exec, SLIP_EINVAL, "assign: out is NULL");
  std::vector<int> ex;
  if (!assign(cl, ex)) {
    set_error("assign: some stage has no live worker");
    return SLIP_EUNRECOVERABLE;
  }
  std::copy(ex.begin(), ex.end(), out_exec);
  return SLIP_OK;
}

slip_status slip_plan_schedule(const slip_cluster* c, const slip_costs* costs, const slip_plan_opts* opts,
                               slip_op* out_ops, int64_t cap, int64_t* n_ops, int64_t* out_makespans,
                               int64_t* out_period) {
  Cluster cl;
  SLIP_TRY(read_cluster(c, cl));
  SLIP_CHECK(costs && opts && n_ops, SLIP_EINVAL, "plan_schedule: NULL argument");
  SLIP_CHECK(costs->t_f >= 0 && costs->t_b >= 0 && costs->t_w >= 0 && costs->t_comm >= 0 && costs->t_ar >= 0 &&
                 costs->t_opt >= 0,
             SLIP_EINVAL, "plan_schedule: negative duration");
  Plan p;
  SLIP_TRY(plan(cl, *costs, *opts, p));
  *n_ops = static_cast<int64_t>(p.ops.size());
  if (out_ops && cap > 0) std::copy(p.ops.begin(), p.ops.begin() + std::min<int64_t>(cap, *n_ops), out_ops);
  if (out_makespans) std::copy(p.makespans.begin(), p.makespans.end(), out_makespans);
  if (out_period) *out_period = p.period;
  return SLIP_OK;
}

uint64_t slip_plan_hash(const slip_op* ops, int64_t n) { return plan_hash(ops, n); }

}  // extern "C"
