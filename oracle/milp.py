"""Exact single-iteration schedule by the paper's MILP — TEST INFRASTRUCTURE.

PAPER.md §4.2.2 (lines 438-546): minimise the makespan max E over B_Weight ends (Eq. 1)
subject to the cross-stage dependencies of the forward (Eq. 2) and backward (Eq. 3), the
same-stage B_Input -> B_Weight dependency (Eq. 4), no two operations of one worker
overlapping (Eq. 5, ordering binaries O and a big-M), and the memory limit (Eq. 6, the
activation deltas Delta M of the operations ordered before each operation).  The
micro-batch -> worker assignment S is an input (the Planner's round-robin re-route, here
taken from oracle/planner.assign).

Used to pin the heuristic schedules of oracle/planner.py against an exact optimum on
small instances (SURVEY.md §8(c.9) "HiGHS MILP of Eqs. 1-6 on tiny instances") and to
settle the running example's "36 time steps" (reading R17).

Modes:
  * coupled (``decoupled=False``): one backward task of length t_b + t_w per micro-batch
    (the paper's pre-SlipStream backward; "adaptive pipelining alone");
  * decoupled: B_Input and B_Weight as separate tasks (Eq. 4).
Memory (Eq. 6): Delta M = +1 for F, -1 for the (coupled) backward / -(1 - a_w) and -a_w
for B_Input / B_Weight with unit activations, limit = the 1F1B in-flight cap
(N - i) * n_w of the list scheduler (oracle/planner.py step 5), or None for no limit.
T_comm is added on cross-stage edges between different workers (Eqs. 2-3).

Solved with scipy.optimize.milp (HiGHS).
"""
from __future__ import annotations

import numpy as np
from scipy.optimize import Bounds, LinearConstraint, milp

from . import planner as PL


def solve(live, m, t_f=1, t_b=1, t_w=1, t_comm=0, decoupled=False, mem_cap=True, time_limit=600.0,
          symmetry=True):
    """Returns dict(makespan, status, ends {(i, j, k, c): E}, gap).  c in 'F', 'B', 'W'
    (coupled: 'B' is the whole backward of length t_b + t_w)."""
    N, DP = len(live), len(live[0])
    ex = PL.assign(live, m)  # {(i, j, k): k_s}
    kinds = ("F", "B", "W") if decoupled else ("F", "B")
    dur = {"F": t_f, "B": t_b if decoupled else t_b + t_w, "W": t_w}
    ops = [(i, j, k, c) for i in range(N) for k in range(DP) for j in range(m) for c in kinds]
    idx = {o: n for n, o in enumerate(ops)}
    nE = len(ops)
    worker = {o: (o[0], ex[(o[0], o[1], o[2])]) for o in ops}
    by_worker = {}
    for o in ops:
        by_worker.setdefault(worker[o], []).append(o)
    # horizon (big-M): a serial schedule of everything
    H = float(sum(dur[o[3]] for o in ops) + t_comm * 2 * N * m * DP + 1)
    pairs = []
    for w, lst in by_worker.items():
        for a in range(len(lst)):
            for b in range(a + 1, len(lst)):
                pairs.append((lst[a], lst[b]))
    nO = len(pairs)
    nv = nE + nO + 1  # E..., O..., C (makespan)
    iC = nE + nO
    rows, lo, hi = [], [], []

    def add(coef, l, h):
        rows.append(coef)
        lo.append(l)
        hi.append(h)

    def row():
        return {}

    # every end >= its duration
    lb = np.zeros(nv)
    for o in ops:
        lb[idx[o]] = dur[o[3]]
    # Eq. 2: F(i) >= F(i-1) + comm + t_f ; Eq. 3: B(i) >= B(i+1) + comm + t_b ; B(N-1) after F(N-1)
    for (i, j, k, c) in ops:
        e = idx[(i, j, k, c)]
        if c == "F" and i > 0:
            p = (i - 1, j, k, "F")
            comm = t_comm if worker[p][1] != worker[(i, j, k, c)][1] else 0
            add({e: 1.0, idx[p]: -1.0}, comm + dur["F"], np.inf)
        if c == "B":
            if i + 1 < N:
                p = (i + 1, j, k, "B")
                comm = t_comm if worker[p][1] != worker[(i, j, k, c)][1] else 0
                add({e: 1.0, idx[p]: -1.0}, comm + dur["B"], np.inf)
            add({e: 1.0, idx[(i, j, k, "F")]: -1.0}, dur["B"], np.inf)
        if c == "W":  # Eq. 4
            add({e: 1.0, idx[(i, j, k, "B")]: -1.0}, dur["W"], np.inf)
        last = "W" if decoupled else "B"
        if c == last:  # Eq. 1: C >= every last task's end
            add({iC: 1.0, e: -1.0}, 0.0, np.inf)
    # Eq. 5: no overlap on a worker, O = 1: a before b
    for n, (a, b) in enumerate(pairs):
        o = nE + n
        # E_b >= E_a + d_b - H (1 - O)   ->  E_b - E_a - H O >= d_b - H
        add({idx[b]: 1.0, idx[a]: -1.0, o: -H}, dur[b[3]] - H, np.inf)
        # E_a >= E_b + d_a - H O          ->  E_a - E_b + H O >= d_a
        add({idx[a]: 1.0, idx[b]: -1.0, o: H}, dur[a[3]], np.inf)
    # Eq. 6: memory, with unit activations: in flight (F started, backward not done) before
    # every F stays below the 1F1B cap (N - i) * n_w of the list scheduler
    if mem_cap:
        pos = {p: n for n, p in enumerate(pairs)}
        n_w = {w: len({o[2] for o in lst}) for w, lst in by_worker.items()}
        free = "B" if not decoupled else "W"
        for w, lst in by_worker.items():
            cap = (N - w[0]) * n_w[w]
            for b in lst:
                if b[3] != "F":
                    continue
                coef = {}
                for a in lst:
                    if a == b or a[3] not in ("F", free):
                        continue
                    delta = 1.0 if a[3] == "F" else -1.0
                    # before(a, b) = O if (a, b) is stored in that order, else 1 - O
                    if (a, b) in pos:
                        v = nE + pos[(a, b)]
                        coef[v] = coef.get(v, 0.0) + delta
                        const = 0.0
                    else:
                        v = nE + pos[(b, a)]
                        coef[v] = coef.get(v, 0.0) - delta
                        const = delta
                    coef.setdefault("_c", 0.0)
                    coef["_c"] += const
                c0 = coef.pop("_c", 0.0)
                # 1 (b itself) + c0 + sum coef * O <= cap
                add(coef, -np.inf, cap - 1.0 - c0)
    # symmetry: the micro-batches of one origin pipeline are interchangeable — relabel so
    # that they enter stage 0 in index order
    if symmetry:
        for k in range(DP):
            for j in range(m - 1):
                add({idx[(0, j + 1, k, "F")]: 1.0, idx[(0, j, k, "F")]: -1.0}, dur["F"], np.inf)
    A = np.zeros((len(rows), nv))
    for r, coef in enumerate(rows):
        for v, c in coef.items():
            A[r, v] = c
    cobj = np.zeros(nv)
    cobj[iC] = 1.0
    integrality = np.zeros(nv)
    integrality[nE:nE + nO] = 1
    ub = np.full(nv, H)
    ub[nE:nE + nO] = 1.0
    res = milp(cobj, constraints=LinearConstraint(A, lo, hi), integrality=integrality, bounds=Bounds(lb, ub),
               options={"time_limit": time_limit, "disp": False})
    out = {"status": res.status, "message": res.message, "makespan": None, "ends": None,
           "gap": getattr(res, "mip_gap", None), "bound": getattr(res, "mip_dual_bound", None)}
    if res.x is not None:
        out["makespan"] = float(res.x[iC])
        out["ends"] = {o: float(res.x[idx[o]]) for o in ops}
    return out


def solve_time_indexed(live, m, horizon, t_f=1, t_b=1, t_w=1, t_comm=0, decoupled=False, mem_cap=True,
                       time_limit=600.0, symmetry=True):
    """The same problem (Eqs. 1-6) in a time-indexed form, for integer costs: x[o, t] = 1 if
    operation o starts at slot t < horizon.  Eq. 5 becomes "at most one operation of a
    worker covers each slot", Eqs. 2-4 the disaggregated precedences "b has started by t
    only if a started by t - d_a - comm", Eq. 6 "in flight (F started, its last backward
    task not finished) <= cap at every slot".  Its LP relaxation is far tighter than the
    big-M form, so HiGHS proves optima on instances of the running example's size.
    Returns dict(makespan, status, starts {(i, j, k, c): t}); makespan None = infeasible
    within the horizon."""
    N, DP = len(live), len(live[0])
    ex = PL.assign(live, m)
    kinds = ("F", "B", "W") if decoupled else ("F", "B")
    dur = {"F": t_f, "B": t_b if decoupled else t_b + t_w, "W": t_w}
    last = "W" if decoupled else "B"
    ops = [(i, j, k, c) for i in range(N) for k in range(DP) for j in range(m) for c in kinds]
    worker = {o: (o[0], ex[(o[0], o[1], o[2])]) for o in ops}
    Tm = int(horizon)
    nvar = {}
    for o in ops:
        for t in range(Tm - dur[o[3]] + 1):
            nvar[(o, t)] = len(nvar)
    iC = len(nvar)
    nv = iC + 1
    rows_i, rows_j, rows_v, lo, hi = [], [], [], [], []
    r = [0]

    def add(coef, l, h):
        for v, c in coef.items():
            rows_i.append(r[0])
            rows_j.append(v)
            rows_v.append(c)
        lo.append(l)
        hi.append(h)
        r[0] += 1

    def starts(o, upto):  # variables "o started at a slot <= upto"
        return [nvar[(o, t)] for t in range(0, min(upto, Tm - dur[o[3]]) + 1)]

    for o in ops:  # every operation starts exactly once
        add({v: 1.0 for v in starts(o, Tm)}, 1.0, 1.0)

    def prec(a, b, gap):  # start(b) >= start(a) + gap, disaggregated over slots
        for t in range(Tm - dur[b[3]] + 1):
            cb = {v: 1.0 for v in starts(b, t)}
            for v in starts(a, t - gap):
                cb[v] = cb.get(v, 0.0) - 1.0
            add(cb, -np.inf, 0.0)

    for (i, j, k, c) in ops:
        o = (i, j, k, c)
        if c == "F" and i > 0:
            p = (i - 1, j, k, "F")
            prec(p, o, dur["F"] + (t_comm if worker[p][1] != worker[o][1] else 0))
        if c == "B":
            if i + 1 < N:
                p = (i + 1, j, k, "B")
                prec(p, o, dur["B"] + (t_comm if worker[p][1] != worker[o][1] else 0))
            else:
                prec((i, j, k, "F"), o, dur["F"])
        if c == "W":
            prec((i, j, k, "B"), o, dur["B"])
        if c == last:  # C >= start + dur
            add({**{nvar[(o, t)]: -float(t + dur[c]) for t in range(Tm - dur[c] + 1)}, iC: 1.0}, 0.0, np.inf)
    by_worker = {}
    for o in ops:
        by_worker.setdefault(worker[o], []).append(o)
    for w, lst in by_worker.items():
        for s in range(Tm):  # one operation covers slot s
            coef = {}
            for o in lst:
                for t in range(max(0, s - dur[o[3]] + 1), min(s, Tm - dur[o[3]]) + 1):
                    coef[nvar[(o, t)]] = 1.0
            if coef:
                add(coef, -np.inf, 1.0)
        if mem_cap:
            cap = (N - w[0]) * len({o[2] for o in lst})
            free = last
            for s in range(Tm):  # F started by s minus last-backward finished by s
                coef = {}
                for o in lst:
                    if o[3] == "F":
                        for v in starts(o, s):
                            coef[v] = coef.get(v, 0.0) + 1.0
                    elif o[3] == free:
                        for v in starts(o, s - dur[free]):
                            coef[v] = coef.get(v, 0.0) - 1.0
                add(coef, -np.inf, float(cap))
    if symmetry:
        for k in range(DP):
            for j in range(m - 1):
                prec((0, j, k, "F"), (0, j + 1, k, "F"), dur["F"])
    from scipy.sparse import csr_matrix
    A = csr_matrix((rows_v, (rows_i, rows_j)), shape=(r[0], nv))
    cobj = np.zeros(nv)
    cobj[iC] = 1.0
    integ = np.ones(nv)
    integ[iC] = 0
    ub = np.ones(nv)
    ub[iC] = Tm
    res = milp(cobj, constraints=LinearConstraint(A, lo, hi), integrality=integ, bounds=Bounds(np.zeros(nv), ub),
               options={"time_limit": time_limit, "disp": False})
    out = {"status": res.status, "message": res.message, "makespan": None, "starts": None}
    if res.x is not None and res.status in (0, 1):
        out["makespan"] = int(round(res.x[iC]))
        out["starts"] = {o: t for (o, t), v in nvar.items() if res.x[v] > 0.5}
    return out
