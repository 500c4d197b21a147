"""Normalization phase of the Planner — TEST
INFRASTRUCTURE (see oracle/__init__.py).

Follows PAPER.md §4.2.1 "Normalization Phase" (lines 382-430) step by step:

  * normalize(): Algorithm 1 (lines 391-414) — the tables C[N x (F+1)] (cost) and
    A[N x (F+1)] (assignment lists), recurrence
        C[i][f] = min_{x <= f} (C[i-1][f-x] + cost(i, x)),
        A[i][f] = concat(A[i-1][f-x], x),
    R = A[N-1][F] with sum(R) = F (lines 417-424).  Two readings (R26, R27):
    the minimum also caps x <= DP-1 (a stage may not lose its whole peer group,
    §3.4), and ties take the LARGEST x at the current (later) stage
    ("move failures to later pipeline stages with more bubbles", line 383).
  * heuristic_cost(): cost(i, x) = "the extra bubbles used to handle the extra
    micro-batches from x failures in the i-th stage" (lines 421-430), estimated
    with the heuristic schedule the paper describes there — 1F1B-like, B only
    schedules B_input, B_weight opportunistically in gaps of time and memory —
    which is oracle.planner.schedule (decoupled, staggered).  Reading R28: the
    extra bubbles are measured as the increase of the steady-state iteration
    period over the fault-free one, in the planner's integer time units.
  * normalized_live(): one concrete placement of R ("the specific pipeline
    assignment does not affect performance and can be arbitrary", line 418).
  * migration_plan(): the point-to-point swaps that move an actual failure set
    to R (lines 377-379: "swap the location of two workers in the pipeline for
    each failure").  Failures already at a stage with remaining quota stay put,
    so the number of swaps is sum_i max(0, actual[i] - R[i]) (reading R29).
"""
from __future__ import annotations

import itertools

from . import planner as P

INF = float("inf")


class Infeasible(Exception):
    pass


def normalize(N: int, DP: int, F: int, cost):
    """Algorithm 1.  cost(i, x) -> number for 0 <= x <= min(F, DP-1).
    Returns (R, C, A): R the per-stage failure counts, C and A the tables."""
    if F < 0 or F > N * (DP - 1):
        raise Infeasible(f"F={F} failures cannot leave a live worker in each of {N} stages of {DP}")
    C = [[INF] * (F + 1) for _ in range(N)]
    A = [[None] * (F + 1) for _ in range(N)]
    for i in range(N):
        for f in range(F + 1):
            if i == 0:
                if f <= DP - 1:                      # cap (R26)
                    C[i][f] = cost(i, f)
                    A[i][f] = [f]
            else:
                best, bx = INF, None
                for x in range(min(f, DP - 1) + 1):  # x <= f, x <= DP-1 (R26)
                    if C[i - 1][f - x] == INF:
                        continue
                    v = C[i - 1][f - x] + cost(i, x)
                    if v <= best:                    # ties -> larger x at the later stage (R27)
                        best, bx = v, x
                if bx is not None:
                    C[i][f] = best
                    A[i][f] = A[i - 1][f - bx] + [bx]
    R = A[N - 1][F]
    return R, C, A


def brute_force(N: int, DP: int, F: int, cost):
    """Exhaustive minimum over every composition of F into N parts, each <= DP-1;
    ties broken to the composition that is largest read from the last stage back
    (the order R27 induces).  Test pin for normalize()."""
    best, bestR = INF, None
    for R in itertools.product(range(min(F, DP - 1) + 1), repeat=N):
        if sum(R) != F:
            continue
        v = sum(cost(i, R[i]) for i in range(N))
        if v < best or (v == best and tuple(reversed(R)) > tuple(reversed(bestR))):
            best, bestR = v, list(R)
    return bestR, best


def failed_positions(N: int, DP: int, R):
    """normalized_live placement: stages from the last to the first, failure c
    (counted over all stages) at pipeline (DP-1-c) mod DP — failures of one stage
    sit in distinct pipelines, consecutive stages alternate pipelines."""
    out, c = [], 0
    for i in range(N - 1, -1, -1):
        for _ in range(R[i]):
            out.append((i, (DP - 1 - c) % DP))
            c += 1
    return out


def normalized_live(N: int, DP: int, R):
    live = [[1] * DP for _ in range(N)]
    for (i, k) in failed_positions(N, DP, R):
        live[i][k] = 0
    return live


def heuristic_cost(N: int, DP: int, m: int, costs: P.Costs, opts: P.Opts = P.Opts()):
    """cost(i, x) of R28, memoised: period(x failures at stage i) - period(none).
    The x failures of stage i sit at pipelines DP-1, DP-2, ..., DP-x."""
    base = P.schedule([[1] * DP for _ in range(N)], m, costs, opts).period
    memo = {}

    def cost(i, x):
        if x == 0:
            return 0
        if (i, x) not in memo:
            live = [[1] * DP for _ in range(N)]
            for c in range(x):
                live[i][DP - 1 - c] = 0
            memo[(i, x)] = P.schedule(live, m, costs, opts).period - base
        return memo[(i, x)]

    return cost


def migration_plan(live, R):
    """Swaps (failed (i, k), target (i2, k2), source k_src) moving the failures of
    `live` to the per-stage counts R.  After a swap the GPU that sat at the live
    target (i2, k2) takes over the failed position (i, k), receiving stage i's state
    from the live peer (i, k_src); (i2, k2) becomes the hole.

    Order (R29): excess failures leave their stage highest k first; deficit stages
    are filled from the last stage back; a hole goes to the live pipeline of that
    stage with the fewest failures so far (ties: highest k); the source is the
    lowest live k of the failed worker's stage."""
    N, DP = len(live), len(live[0])
    F = sum(1 for i in range(N) for k in range(DP) if not live[i][k])
    if sum(R) != F or len(R) != N:
        raise ValueError("R does not describe the actual failure count")
    if any(r > DP - 1 for r in R) or not P.recoverable(live):
        raise P.Unrecoverable("normalization target or actual set leaves a stage empty")
    cur = [list(row) for row in live]
    movers = []
    for i in range(N):
        fk = [k for k in range(DP) if not live[i][k]]
        excess = len(fk) - R[i]
        if excess > 0:
            movers += [(i, k) for k in sorted(fk, reverse=True)[:excess]]
    holes_needed = []
    for i in range(N - 1, -1, -1):
        deficit = R[i] - sum(1 for k in range(DP) if not live[i][k])
        holes_needed += [i] * max(0, deficit)
    assert len(movers) == len(holes_needed)
    swaps = []
    for (i, k), i2 in zip(movers, holes_needed):
        src = min(kk for kk in range(DP) if cur[i][kk])
        cur[i][k] = 1
        pipe_fail = [sum(1 for ii in range(N) if not cur[ii][kk]) for kk in range(DP)]
        cands = [kk for kk in range(DP) if cur[i2][kk]]
        k2 = min(cands, key=lambda kk: (pipe_fail[kk], -kk))
        cur[i2][k2] = 0
        swaps.append(((i, k), (i2, k2), src))
    return swaps, cur
