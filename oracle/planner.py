"""Planner oracle: recoverability, re-route assignment, list scheduler and
validator, in integer time — TEST INFRASTRUCTURE (see oracle/__init__.py).

Follows the algorithm step by step in the paper's notation (DESIGN.md "Planner
reading"):

  1. Recoverability (§3.4): RECOVERABLE iff every stage
     keeps at least one functional worker.
  2. Assignment S^{k_s}_{i,j,k} (§4.2; §3.1
     "evenly distribute micro-batches across all functional peers"; §4.3 line
     554 "round-robin"): survivors S_i = ascending live k; the failed workers'
     micro-batches, enumerated in (k, j) order, go to S_i[r mod |S_i|].  This
     reproduces the Fig. 5b anchors (mb 7 -> W_{0_2}, mb 10 -> W_{2_2},
     PAPER.md lines 211-214).  Reading R14.
  3. Tasks per iteration t: F, B (=B_input), W (=B_weight) per (i, j, k), or
     F, BC (coupled) when Decoupled BackProp is off; AR(t, i) per stage (the
     DP all-reduce, runs on the comm stream); OPT(t, i, k_s) per live worker.
  4. Dependencies: Eq. 2 (F after upstream F + T_comm), Eq. 3 (B after
     downstream B + T_comm), Eq. 4 (W after B), F after own F before B, AR
     after every W of the stage, OPT after AR; staggered (§3.3): F of
     iteration t+1 on worker (i, k_s) waits only for OPT(t, i, k_s); not
     staggered: OPT waits for all stages' AR and F(t+1) for every OPT(t).
  5. Dispatch: event-driven over integer time.  At each event time the idle
     workers, in (i, k_s) order, pick the best ready task: OPT; then B
     (earliest arrival, then earliest F end, then (t, k, j)); then F if
     admissible (in-flight F without B < (N - i) * n_w and memory + a_f <=
     m_limit; earliest arrival, then (t, k, j)); then W (earliest B end, then
     (t, k, j)).  "B_weight operations are scheduled opportunistically" when
     a gap exists (§4.2).  Memory is applied with the
     net deltas F +a_f, B -(a_f - a_w), W -a_w (reading R18).
  6. Outputs: per-worker op lists with integer (start, end); makespan of each
     iteration; period = M_{H-1} - M_{H-2} (steady state).
  7. Validator: Eqs. 2-6 plus COVERAGE / ASSIGNMENT / OPT ordering.
"""
from __future__ import annotations

from dataclasses import dataclass, field

# phases (values fixed by include/slip.h, slip_phase)
F, B, W, BC, OPT, AR = 0, 1, 2, 3, 4, 5
PHASE_NAMES = {F: "F", B: "B", W: "W", BC: "BC", OPT: "OPT", AR: "AR"}


@dataclass(frozen=True)
class Costs:
    t_f: int = 1
    t_b: int = 1
    t_w: int = 1
    t_comm: int = 0
    t_ar: int = 0
    t_opt: int = 0
    a_f: int = 0
    a_w: int = 0
    m_limit: int = 0  # <= 0: unlimited


@dataclass(frozen=True)
class Opts:
    decoupled: int = True  # True / False, or 2 = selective (the better of both)
    staggered: bool = True
    horizon: int = 3


@dataclass
class Op:
    stage: int
    mb: int        # j, -1 for OPT / AR
    origin: int    # k, -1 for OPT / AR
    phase: int
    exec: int      # k_s, -1 for AR
    it: int        # iteration t
    start: int
    end: int

    def key(self):
        return (self.stage, self.mb, self.origin, self.phase, self.exec, self.it, self.start, self.end)


@dataclass
class Plan:
    ops: list = field(default_factory=list)        # sorted: (exec-worker, start) then AR
    assignment: dict = field(default_factory=dict)  # (i, j, k) -> k_s
    makespans: list = field(default_factory=list)   # per iteration
    period: int = 0
    peak_mem: dict = field(default_factory=dict)    # (i, k_s) -> bytes


class Unrecoverable(Exception):
    pass


# ---------------------------------------------------------------- step 1, 2
def peers(live, i):
    """Live workers of stage i in ascending k (SPEC core_model.peers)."""
    return [k for k in range(len(live[i])) if live[i][k]]


def recoverable(live) -> bool:
    return all(any(row) for row in live)


def assign(live, m):
    """exec[(i, j, k)] = k_s (step 2)."""
    N, DP = len(live), len(live[0])
    if not recoverable(live):
        raise Unrecoverable("some stage has no functional worker")
    ex = {}
    for i in range(N):
        surv = peers(live, i)
        r = 0
        for k in range(DP):
            for j in range(m):
                if live[i][k]:
                    ex[(i, j, k)] = k
        for k in range(DP):
            if live[i][k]:
                continue
            for j in range(m):
                ex[(i, j, k)] = surv[r % len(surv)]
                r += 1
    return ex


def comm_edges(ex, N, DP, m):
    """ACT edges exec(i,j,k) -> exec(i+1,j,k) and GRAD edges in reverse
    (ReRouteAct / ReRouteGrad, §4.3)."""
    edges = []
    for k in range(DP):
        for j in range(m):
            for i in range(N - 1):
                edges.append(("ACT", (i, ex[(i, j, k)]), (i + 1, ex[(i + 1, j, k)]), j, k, i))
                edges.append(("GRAD", (i + 1, ex[(i + 1, j, k)]), (i, ex[(i, j, k)]), j, k, i))
    return edges


# ---------------------------------------------------------------- step 3-6
def schedule(live, m, costs: Costs, opts: Opts) -> Plan:
    if opts.decoupled == 2:
        # selective decoupling (§3.2; R32): both plans,
        # the shorter steady-state period wins, ties to Decoupled BackProp
        pd = schedule(live, m, costs, Opts(True, opts.staggered, opts.horizon))
        pc = schedule(live, m, costs, Opts(False, opts.staggered, opts.horizon))
        return pc if pc.period < pd.period else pd
    N, DP = len(live), len(live[0])
    H = max(1, int(opts.horizon))
    ex = assign(live, m)
    c = costs
    tbc = c.t_b + c.t_w
    lim = c.m_limit if c.m_limit > 0 else None
    workers = [(i, ks) for i in range(N) for ks in range(DP) if live[i][ks]]
    # origin pipelines routed to each worker (n_w)
    n_w = {w: len({k for (i, j, k), ks in ex.items() if (i, ks) == w}) for w in workers}
    # task bookkeeping: end times of scheduled compute tasks
    end = {}          # (phase, t, i, j, k) -> end ; (OPT, t, i, ks) -> end
    ar_end = {}       # (t, i) -> end
    busy = {w: 0 for w in workers}
    mem = {w: 0 for w in workers}
    peak = {w: 0 for w in workers}
    inflight = {w: 0 for w in workers}
    pending = {w: [] for w in workers}  # list of task keys
    for w in workers:
        i, ks = w
        for t in range(H):
            for k in range(DP):
                for j in range(m):
                    if ex[(i, j, k)] != ks:
                        continue
                    pending[w].append((F, t, i, j, k))
                    if opts.decoupled:
                        pending[w].append((B, t, i, j, k))
                        pending[w].append((W, t, i, j, k))
                    else:
                        pending[w].append((BC, t, i, j, k))
            pending[w].append((OPT, t, i, -1, ks))
    ops = []
    bwd = B if opts.decoupled else BC
    last_w = W if opts.decoupled else BC

    def dur(ph):
        return {F: c.t_f, B: c.t_b, W: c.t_w, BC: tbc, OPT: c.t_opt}[ph]

    def stage_tasks_done(t, i):
        """All W (or BC) of stage i, iteration t scheduled -> max end, else None."""
        mx = 0
        for k in range(DP):
            for j in range(m):
                e = end.get((last_w, t, i, j, k))
                if e is None:
                    return None
                mx = max(mx, e)
        return mx

    def update_ar():
        for t in range(H):
            for i in range(N):
                if (t, i) in ar_end:
                    continue
                mx = stage_tasks_done(t, i)
                if mx is not None:
                    ar_end[(t, i)] = mx + c.t_ar
                    ops.append(Op(i, -1, -1, AR, -1, t, mx, mx + c.t_ar))

    def opt_dep(t, i, ks):
        """Earliest time F of iteration t may start on worker (i, ks), None if unknown."""
        if t == 0:
            return 0
        if opts.staggered:
            return end.get((OPT, t - 1, i, -1, ks))
        mx = 0
        for (ii, kk) in workers:
            e = end.get((OPT, t - 1, ii, -1, kk))
            if e is None:
                return None
            mx = max(mx, e)
        return mx

    def ready_time(task):
        """Time the task's dependencies are satisfied, or None if not yet known."""
        ph, t, i, j, k = task
        if ph == OPT:
            if opts.staggered:
                return ar_end.get((t, i))
            mx = 0
            for ii in range(N):
                e = ar_end.get((t, ii))
                if e is None:
                    return None
                mx = max(mx, e)
            return mx
        if ph == F:
            od = opt_dep(t, i, ex[(i, j, k)])
            if od is None:
                return None
            if i == 0:
                return od
            up = end.get((F, t, i - 1, j, k))
            return None if up is None else max(od, up + c.t_comm)
        if ph in (B, BC):
            fe = end.get((F, t, i, j, k))
            if fe is None:
                return None
            if i == N - 1:
                return fe
            dn = end.get((bwd, t, i + 1, j, k))
            return None if dn is None else max(fe, dn + c.t_comm)
        if ph == W:
            return end.get((B, t, i, j, k))
        raise AssertionError(ph)

    def arrival(task):
        """Arrival of the task's cross-stage input (tie-break key)."""
        ph, t, i, j, k = task
        if ph == F:
            if i == 0:
                return 0
            return end[(F, t, i - 1, j, k)] + c.t_comm
        if i == N - 1:
            return end[(F, t, i, j, k)]
        return end[(bwd, t, i + 1, j, k)] + c.t_comm

    def dispatch(w, now):
        """Pick and place the best ready task for idle worker w at time now."""
        i, ks = w
        cands = [x for x in pending[w] if (lambda rt: rt is not None and rt <= now)(ready_time(x))]
        if not cands:
            return False
        opt_c = [x for x in cands if x[0] == OPT]
        b_c = [x for x in cands if x[0] in (B, BC)]
        f_c = [x for x in cands if x[0] == F]
        w_c = [x for x in cands if x[0] == W]
        pick = None
        if opt_c:
            pick = min(opt_c, key=lambda x: x[1])
        elif b_c:
            pick = min(b_c, key=lambda x: (arrival(x), end[(F, x[1], x[2], x[3], x[4])], x[1], x[4], x[3]))
        else:
            f_ok = bool(f_c) and inflight[w] < (N - i) * n_w[w] and (lim is None or mem[w] + c.a_f <= lim)
            if f_ok:
                pick = min(f_c, key=lambda x: (arrival(x), x[1], x[4], x[3]))
            elif w_c:
                pick = min(w_c, key=lambda x: (end[(B, x[1], x[2], x[3], x[4])], x[1], x[4], x[3]))
        if pick is None:
            return False
        ph, t, _, j, k = pick
        s, e = now, now + dur(ph)
        end[pick] = e
        busy[w] = e
        pending[w].remove(pick)
        if ph == F:
            inflight[w] += 1
            mem[w] += c.a_f
        elif ph == B:
            inflight[w] -= 1
            mem[w] -= c.a_f - c.a_w
        elif ph == W:
            mem[w] -= c.a_w
        elif ph == BC:
            inflight[w] -= 1
            mem[w] -= c.a_f
        peak[w] = max(peak[w], mem[w])
        if ph == OPT:
            ops.append(Op(i, -1, -1, OPT, ks, t, s, e))
        else:
            ops.append(Op(i, j, k, ph, ks, t, s, e))
        return True

    now = 0
    while any(pending[w] for w in workers):
        # repeat passes at the same instant: zero-length tasks (t_opt = 0,
        # t_ar = 0) can make further tasks ready at `now`
        progress = True
        while progress:
            progress = False
            update_ar()
            for w in workers:
                if busy[w] <= now and dispatch(w, now):
                    progress = True
        update_ar()
        # next event: a worker becoming free, or a pending task becoming ready
        nxt = None
        for w in workers:
            if busy[w] > now:
                nxt = busy[w] if nxt is None else min(nxt, busy[w])
            for task in pending[w]:
                rt = ready_time(task)
                if rt is not None and rt > now:
                    nxt = rt if nxt is None else min(nxt, rt)
        if nxt is None:
            if any(pending[w] for w in workers):
                # all workers idle and nothing becomes ready: only admissibility blocks
                raise RuntimeError("infeasible: memory limit admits no further forward")
            break
        now = nxt
    update_ar()
    plan = Plan()
    plan.assignment = ex
    plan.ops = sort_ops(ops, N, DP)
    plan.makespans = [max(o.end for o in ops if o.it == t) for t in range(H)]
    plan.period = plan.makespans[-1] - plan.makespans[-2] if H >= 2 else plan.makespans[0]
    plan.peak_mem = peak
    return plan


def sort_ops(ops, N, DP):
    """Canonical op-list order: compute ops by worker (stage, exec) then start;
    AR ops last by (iteration, stage)."""
    comp = sorted((o for o in ops if o.phase != AR), key=lambda o: (o.stage, o.exec, o.start))
    ars = sorted((o for o in ops if o.phase == AR), key=lambda o: (o.it, o.stage))
    return comp + ars


def worker_ops(plan, i, ks):
    return [o for o in plan.ops if o.phase != AR and o.stage == i and o.exec == ks]


def count_bubbles(plan, i, ks, it=0):
    """Idle time of worker (i, ks) inside [first start of stage 0 in iteration it,
    makespan of iteration it] (SPEC baseline_schedule.count_bubbles)."""
    s0 = min(o.start for o in plan.ops if o.it == it and o.stage == 0 and o.phase != AR)
    M = plan.makespans[it]
    busy = sum(min(o.end, M) - max(o.start, s0) for o in worker_ops(plan, i, ks)
               if o.it == it and o.end > s0 and o.start < M)
    return (M - s0) - busy


# ---------------------------------------------------------------- step 7
def validate(plan, live, m, costs: Costs, opts: Opts):
    """Returns a list of (kind, detail) violations; empty = valid.  Kinds:
    CROSS_STAGE_DEP (Eqs. 2-3), SAME_STAGE_DEP (Eq. 4 and F->B), OVERLAP
    (Eq. 5), MEMORY (Eq. 6), ASSIGNMENT, COVERAGE, OPT_ORDER."""
    N, DP = len(live), len(live[0])
    H = max(1, int(opts.horizon))
    c = costs
    ex = assign(live, m)
    v = []
    comp = [o for o in plan.ops if o.phase != AR]
    idx = {}
    for o in comp:
        key = (o.phase, o.it, o.stage, o.mb, o.origin) if o.phase != OPT else (OPT, o.it, o.stage, -1, o.exec)
        if key in idx:
            v.append(("COVERAGE", f"duplicate {key}"))
        idx[key] = o
        dd = {F: c.t_f, B: c.t_b, W: c.t_w, BC: c.t_b + c.t_w, OPT: c.t_opt}[o.phase]
        if o.end - o.start != dd:
            v.append(("COVERAGE", f"duration {key}"))
    phases = (F, B, W) if opts.decoupled else (F, BC)
    bwd = B if opts.decoupled else BC
    for t in range(H):
        for i in range(N):
            for k in range(DP):
                for j in range(m):
                    for ph in phases:
                        o = idx.get((ph, t, i, j, k))
                        if o is None:
                            v.append(("COVERAGE", f"missing {(ph, t, i, j, k)}"))
                        elif o.exec != ex[(i, j, k)]:
                            v.append(("ASSIGNMENT", f"{(ph, t, i, j, k)} on {o.exec}"))
            for ks in range(DP):
                if live[i][ks] and (OPT, t, i, -1, ks) not in idx:
                    v.append(("COVERAGE", f"missing OPT {(t, i, ks)}"))
    if v:
        return v
    for t in range(H):
        for i in range(N):
            for k in range(DP):
                for j in range(m):
                    f = idx[(F, t, i, j, k)]
                    b = idx[(bwd, t, i, j, k)]
                    if i > 0 and f.start < idx[(F, t, i - 1, j, k)].end + c.t_comm:
                        v.append(("CROSS_STAGE_DEP", f"Eq2 {(t, i, j, k)}"))
                    if i < N - 1 and b.start < idx[(bwd, t, i + 1, j, k)].end + c.t_comm:
                        v.append(("CROSS_STAGE_DEP", f"Eq3 {(t, i, j, k)}"))
                    if b.start < f.end:
                        v.append(("SAME_STAGE_DEP", f"B before F {(t, i, j, k)}"))
                    if opts.decoupled and idx[(W, t, i, j, k)].start < b.end:
                        v.append(("SAME_STAGE_DEP", f"Eq4 {(t, i, j, k)}"))
    # AR / OPT ordering
    ars = {(o.it, o.stage): o for o in plan.ops if o.phase == AR}
    last = W if opts.decoupled else BC
    for t in range(H):
        for i in range(N):
            a = ars.get((t, i))
            mx = max(idx[(last, t, i, j, k)].end for k in range(DP) for j in range(m))
            if a is None or a.start < mx or a.end - a.start != c.t_ar:
                v.append(("OPT_ORDER", f"AR {(t, i)}"))
                continue
            for ks in range(DP):
                if not live[i][ks]:
                    continue
                op = idx[(OPT, t, i, -1, ks)]
                need = a.end if opts.staggered else max(ars[(t, ii)].end for ii in range(N))
                if op.start < need:
                    v.append(("OPT_ORDER", f"OPT {(t, i, ks)}"))
                if t + 1 < H:
                    for k in range(DP):
                        for j in range(m):
                            if ex[(i, j, k)] != ks:
                                continue
                            f = idx[(F, t + 1, i, j, k)]
                            if opts.staggered:
                                if f.start < op.end:
                                    v.append(("OPT_ORDER", f"F after OPT {(t, i, j, k)}"))
    if not opts.staggered:
        for t in range(H - 1):
            bar = max(idx[(OPT, t, i, -1, ks)].end for i in range(N) for ks in range(DP) if live[i][ks])
            for o in comp:
                if o.it == t + 1 and o.phase == F and o.start < bar:
                    v.append(("OPT_ORDER", f"F before barrier {(o.it, o.stage, o.mb, o.origin)}"))
    # Eq. 5 overlap and Eq. 6 memory, per worker
    lim = c.m_limit if c.m_limit > 0 else None
    for i in range(N):
        for ks in range(DP):
            if not live[i][ks]:
                if any(o.stage == i and o.exec == ks for o in comp):
                    v.append(("ASSIGNMENT", f"ops on failed worker {(i, ks)}"))
                continue
            lst = sorted((o for o in comp if o.stage == i and o.exec == ks), key=lambda o: o.start)
            for a, b in zip(lst, lst[1:]):
                if b.start < a.end:
                    v.append(("OVERLAP", f"{(i, ks)} {a.key()} {b.key()}"))
            memv = 0
            for o in sorted(lst, key=lambda o: o.end):
                memv += {F: c.a_f, B: -(c.a_f - c.a_w), W: -c.a_w, BC: -c.a_f, OPT: 0}[o.phase]
                if lim is not None and memv > lim:
                    v.append(("MEMORY", f"{(i, ks)} at {o.end}: {memv}"))
    return v


def pair_fifo_ok(plan, live, m):
    """Per directed worker pair, the receiver consumes messages in the sender's
    send order (needed by per-pair NCCL channels)."""
    ex = plan.assignment
    N = len(live)
    comp = [o for o in plan.ops if o.phase in (F, B, BC)]
    by = {(o.phase, o.it, o.stage, o.mb, o.origin): o for o in comp}
    sends, recvs = {}, {}
    for o in sorted(comp, key=lambda o: o.end):
        if o.phase == F and o.stage < N - 1:
            dst = (o.stage + 1, ex[(o.stage + 1, o.mb, o.origin)])
            sends.setdefault(((o.stage, o.exec), dst), []).append((o.it, o.mb, o.origin))
        if o.phase in (B, BC) and o.stage > 0:
            dst = (o.stage - 1, ex[(o.stage - 1, o.mb, o.origin)])
            sends.setdefault(((o.stage, o.exec), dst, "g"), []).append((o.it, o.mb, o.origin))
    for o in sorted(comp, key=lambda o: o.start):
        if o.phase == F and o.stage > 0:
            src = (o.stage - 1, ex[(o.stage - 1, o.mb, o.origin)])
            recvs.setdefault((src, (o.stage, o.exec)), []).append((o.it, o.mb, o.origin))
        if o.phase in (B, BC) and o.stage < N - 1:
            src = (o.stage + 1, ex[(o.stage + 1, o.mb, o.origin)])
            recvs.setdefault((src, (o.stage, o.exec), "g"), []).append((o.it, o.mb, o.origin))
    del by
    return sends == recvs


def plan_hash(ops) -> int:
    """FNV-1a 64 over the op tuples (int64 little-endian), in list order."""
    h = 0xCBF29CE484222325
    for o in ops:
        for x in o.key():
            for byte in int(x).to_bytes(8, "little", signed=True):
                h ^= byte
                h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h
