"""Pins of oracle/normalize.py (Algorithm 1, §4.2.1) against
sources other than itself: exhaustive enumeration of compositions, the paper's
worked examples, closed forms for the swap count, and invariants."""
import itertools
import random

import pytest

from oracle import normalize as NZ
from oracle import planner as P


def table_cost(tab):
    return lambda i, x: tab[i][x]


def random_table(rng, N, F, lo=-3, hi=9):
    return [[0] + [rng.randint(lo, hi) for _ in range(F)] for _ in range(N)]


def test_alg1_equals_brute_force_on_random_tables():
    """DP optimality: N <= 4, DP <= 3, F <= 4, any cost table —
    same cost AND the same composition under the R27 tie order."""
    rng = random.Random(2405)
    n = 0
    for N in range(1, 5):
        for DP in range(2, 4):
            for F in range(0, min(4, N * (DP - 1)) + 1):
                for _ in range(12):
                    tab = random_table(rng, N, F, 0 if _ % 2 else -3, 3 if _ % 3 == 0 else 9)
                    R, C, A = NZ.normalize(N, DP, F, table_cost(tab))
                    Rb, cb = NZ.brute_force(N, DP, F, table_cost(tab))
                    assert C[N - 1][F] == cb and R == Rb, (N, DP, F, tab)
                    assert sum(R) == F and all(0 <= r <= DP - 1 for r in R)
                    assert len(A[N - 1][F]) == N
                    n += 1
    assert n > 200


def test_tables_are_prefix_optimal():
    """C[i][f] is the brute-force optimum of the first i+1 stages, and A[i][f] has
    length i+1 and sums to f."""
    rng = random.Random(7)
    N, DP, F = 4, 3, 4
    tab = random_table(rng, N, F)
    _, C, A = NZ.normalize(N, DP, F, table_cost(tab))
    for i in range(N):
        for f in range(F + 1):
            sub = [row for row in tab[:i + 1]]
            if f > (i + 1) * (DP - 1):
                assert C[i][f] == NZ.INF and A[i][f] is None
                continue
            _, cb = NZ.brute_force(i + 1, DP, f, table_cost(sub))
            assert C[i][f] == cb
            assert len(A[i][f]) == i + 1 and sum(A[i][f]) == f


def test_trivial_and_infeasible():
    R, C, _ = NZ.normalize(4, 3, 0, lambda i, x: 5 * x)
    assert R == [0, 0, 0, 0] and C[3][0] == 0
    with pytest.raises(NZ.Infeasible):
        NZ.normalize(2, 2, 3, lambda i, x: 0)  # 3 > N (DP-1) = 2
    R, _, _ = NZ.normalize(2, 2, 2, lambda i, x: 0)
    assert R == [1, 1]  # forced: one per stage (cap R26)


def test_later_stage_preferred_on_ties_and_cheapest_stage_chosen():
    # equal costs everywhere: the failure goes to the last stage (line 383, R27)
    R, _, _ = NZ.normalize(4, 3, 1, lambda i, x: x)
    assert R == [0, 0, 0, 1]
    # a strictly cheaper middle stage wins
    tab = [[0, 5, 9], [0, 1, 9], [0, 5, 9], [0, 5, 9]]
    R, _, _ = NZ.normalize(4, 3, 1, table_cost(tab))
    assert R == [0, 1, 0, 0]
    # convex per-stage cost spreads failures across peer groups (line 383 a)
    R, _, _ = NZ.normalize(4, 3, 3, lambda i, x: x * x)
    assert R == [0, 1, 1, 1]


def test_monotone_in_f_for_nondecreasing_costs():
    """C[N-1][f] non-decreasing in f for non-negative costs that are
    non-decreasing in x (adding a failure never removes work)."""
    rng = random.Random(11)
    for _ in range(50):
        N, DP = rng.randint(1, 5), rng.randint(2, 4)
        F = N * (DP - 1)
        tab = []
        for i in range(N):
            row, v = [0], 0
            for x in range(F):
                v += rng.randint(0, 4)
                row.append(v)
            tab.append(row)
        _, C, _ = NZ.normalize(N, DP, F, table_cost(tab))
        col = [C[N - 1][f] for f in range(F + 1)]
        assert all(a <= b for a, b in zip(col, col[1:]))


def test_heuristic_cost_running_example():
    """Running example (§3, Figs. 5-7: N=4, DP=3, m=6, unit F/B/W, no comm):
    with Decoupled BackProp + Staggered Optimizer one failure at stage 2 brings the
    period to 27, the fault-free COUPLED 1F1B period (§3.3 "zero overhead over the
    fault-free 1F1B").  cost() measures against the fault-free period of the same
    (decoupled, staggered) plan, so cost(2, 1) = 27 - that period.  With equal costs
    at every stage the failure goes to the last stage (line 383, R27)."""
    costs = P.Costs(t_f=1, t_b=1, t_w=1)
    cost = NZ.heuristic_cost(4, 3, 6, costs)
    base = P.schedule([[1] * 3 for _ in range(4)], 6, costs, P.Opts()).period
    assert cost(2, 1) == 27 - base and cost(2, 1) > 0
    R, C, _ = NZ.normalize(4, 3, 1, cost)
    assert C[3][1] == min(cost(i, 1) for i in range(4))
    if len({cost(i, 1) for i in range(4)}) == 1:
        assert R == [0, 0, 0, 1]


def test_heuristic_cost_is_period_delta():
    """cost(i, x) is literally period(x failures at stage i) - period(fault free)
    of the heuristic schedule (R28) — checked against a schedule built by hand."""
    costs = P.Costs(t_f=2, t_b=2, t_w=1, t_comm=1, t_opt=1, t_ar=1)
    N, DP, m = 3, 3, 4
    cost = NZ.heuristic_cost(N, DP, m, costs)
    base = P.schedule([[1] * DP for _ in range(N)], m, costs, P.Opts()).period
    live = [[1, 1, 1], [1, 1, 1], [1, 0, 0]]
    assert cost(2, 2) == P.schedule(live, m, costs, P.Opts()).period - base
    assert cost(1, 0) == 0


def test_normalized_live_matches_R():
    rng = random.Random(3)
    for _ in range(100):
        N, DP = rng.randint(1, 6), rng.randint(2, 5)
        R = [rng.randint(0, DP - 1) for _ in range(N)]
        live = NZ.normalized_live(N, DP, R)
        for i in range(N):
            assert sum(1 - v for v in live[i]) == R[i]
        assert P.recoverable(live)
    # DP = 2: consecutive failed stages alternate pipelines (bench placement, R20)
    assert NZ.failed_positions(4, 2, [0, 0, 1, 1]) == [(3, 1), (2, 0)]


def brute_min_swaps(live, R):
    """Minimum number of single-failure relocations turning the per-stage failure
    counts of `live` into R, by breadth-first search over count vectors."""
    N = len(live)
    start = tuple(sum(1 - v for v in row) for row in live)
    goal = tuple(R)
    frontier, seen, d = {start}, {start}, 0
    while goal not in frontier:
        nxt = set()
        for s in frontier:
            for a in range(N):
                for b in range(N):
                    if a != b and s[a] > 0:
                        t = list(s)
                        t[a] -= 1
                        t[b] += 1
                        t = tuple(t)
                        if t not in seen:
                            seen.add(t)
                            nxt.add(t)
        frontier, d = nxt, d + 1
    return d


def test_migration_plan_is_minimal_and_lands_on_R():
    """Swap count = sum max(0, actual - R) = BFS minimum; targets
    live, sources live peers of the failed stage, result has counts R and stays
    recoverable; failures at stages with quota stay put."""
    rng = random.Random(17)
    for _ in range(300):
        N, DP = rng.randint(1, 4), rng.randint(2, 4)
        F = rng.randint(0, N * (DP - 1))
        # random recoverable actual failure set of size F
        while True:
            cells = rng.sample([(i, k) for i in range(N) for k in range(DP)], F)
            live = [[1] * DP for _ in range(N)]
            for (i, k) in cells:
                live[i][k] = 0
            if P.recoverable(live):
                break
        R = [0] * N
        for _f in range(F):
            i = rng.choice([i for i in range(N) if R[i] < DP - 1])
            R[i] += 1
        swaps, after = NZ.migration_plan(live, R)
        actual = [sum(1 - v for v in row) for row in live]
        assert len(swaps) == sum(max(0, a - r) for a, r in zip(actual, R)) == brute_min_swaps(live, R)
        assert [sum(1 - v for v in row) for row in after] == R and P.recoverable(after)
        cur = [list(r) for r in live]
        for (i, k), (i2, k2), src in swaps:
            assert not cur[i][k] and cur[i2][k2] and cur[i][src] and src != k and R[i] < actual[i]
            cur[i][k], cur[i2][k2] = 1, 0
        assert cur == after
        for i in range(N):  # untouched failures stay
            if actual[i] <= R[i]:
                assert all(after[i][k] == 0 for k in range(DP) if not live[i][k])


def test_migration_paper_examples():
    # a single failure at stage 0, R = [0,0,0,1]: one swap to a stage-3 worker (line 378, "W_{2_3}")
    live = [[0, 1, 1], [1, 1, 1], [1, 1, 1], [1, 1, 1]]
    swaps, after = NZ.migration_plan(live, [0, 0, 0, 1])
    assert len(swaps) == 1 and swaps[0][0] == (0, 0) and swaps[0][1][0] == 3 and swaps[0][2] == 1
    # already normalized: no swap
    swaps, after = NZ.migration_plan(after, [0, 0, 0, 1])
    assert swaps == []
    # three failures at stage 1 of DP=4, R=[0,1,1,1]: 2 swaps
    live = [[1, 1, 1, 1], [0, 0, 0, 1], [1, 1, 1, 1], [1, 1, 1, 1]]
    swaps, after = NZ.migration_plan(live, [0, 1, 1, 1])
    assert len(swaps) == 2
    # the two holes land in distinct pipelines, both differing from the stay-put failure
    pipes = [k for i in range(4) for k in range(4) if not after[i][k]]
    assert len(set(pipes)) == 3


def test_all_failure_counts_end_to_end_small():
    """Every F up to N(DP-1) on a small cluster: heuristic cost + Alg. 1 give a
    recoverable normalized placement whose period equals what the planner gives
    for that placement, and no placement of F failures found by enumeration is
    recoverable-and-cheaper under the same additive cost."""
    costs = P.Costs(t_f=2, t_b=2, t_w=1, t_comm=1)
    N, DP, m = 3, 2, 3
    cost = NZ.heuristic_cost(N, DP, m, costs)
    for F in range(N * (DP - 1) + 1):
        R, C, _ = NZ.normalize(N, DP, F, cost)
        live = NZ.normalized_live(N, DP, R)
        assert P.recoverable(live)
        best = min(sum(cost(i, r[i]) for i in range(N))
                   for r in itertools.product(range(DP), repeat=N) if sum(r) == F)
        assert C[N - 1][F] == best
