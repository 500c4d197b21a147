"""C++ normalization (csrc/normalize.cpp, through the C-ABI) vs oracle/normalize.py:
bit-exact R, C tables, heuristic cost tables, placements and migration swaps."""
import random

import pytest

from oracle import normalize as NZ
from oracle import planner as P


@pytest.fixture(scope="module")
def rt():
    from paper_2405_14009_b200 import runtime
    return runtime


def test_alg1_tables_bit_exact(rt):
    rng = random.Random(99)
    for _ in range(300):
        N, DP = rng.randint(1, 6), rng.randint(1, 5)
        F = rng.randint(0, N * max(0, DP - 1))
        tab = {(i, x): (0 if x == 0 else rng.randint(-5, 20)) for i in range(N) for x in range(F + 1)}
        R, C = rt.normalize(N, DP, F, tab)
        Ro, Co, _ = NZ.normalize(N, DP, F, lambda i, x: tab[(i, x)])
        assert R == Ro
        assert C == [[None if v == NZ.INF else v for v in row] for row in Co]


def test_infeasible_F_is_rejected(rt):
    from paper_2405_14009_b200._binding import SlipError
    with pytest.raises(SlipError):
        rt.normalize(2, 2, 3, {(i, x): 0 for i in range(2) for x in range(4)})


def test_heuristic_cost_tables_bit_exact(rt):
    rng = random.Random(5)
    for _ in range(25):
        N, DP, m = rng.randint(1, 4), rng.randint(2, 4), rng.randint(1, 6)
        F = rng.randint(1, N * (DP - 1))
        c = dict(t_f=rng.randint(1, 4), t_b=rng.randint(1, 4), t_w=rng.randint(1, 3), t_comm=rng.randint(0, 2),
                 t_ar=rng.randint(0, 2), t_opt=rng.randint(0, 2))
        dec = rng.random() < 0.8
        stag = dec and rng.random() < 0.8
        tab = rt.normalize_costs(N, DP, m, rt.make_costs(**c), F, dec, stag)
        cost = NZ.heuristic_cost(N, DP, m, P.Costs(**c), P.Opts(dec, stag, 3))
        for i in range(N):
            for x in range(F + 1):
                assert tab[(i, x)] == (cost(i, x) if x <= DP - 1 else None), (i, x)
        R, _ = rt.normalize(N, DP, F, tab)
        Ro, _, _ = NZ.normalize(N, DP, F, cost)
        assert R == Ro
        assert rt.normalized_live(N, DP, R) == NZ.normalized_live(N, DP, Ro)


def test_migration_plans_bit_exact(rt):
    rng = random.Random(23)
    for _ in range(300):
        N, DP = rng.randint(1, 5), rng.randint(2, 4)
        F = rng.randint(0, N * (DP - 1))
        while True:
            cells = rng.sample([(i, k) for i in range(N) for k in range(DP)], F)
            live = [[1] * DP for _ in range(N)]
            for (i, k) in cells:
                live[i][k] = 0
            if P.recoverable(live):
                break
        R = [0] * N
        for _f in range(F):
            R[rng.choice([i for i in range(N) if R[i] < DP - 1])] += 1
        sw, after = rt.migration_plan(N, DP, live, R)
        swo, aftero = NZ.migration_plan(live, R)
        assert sw == swo and after == aftero
