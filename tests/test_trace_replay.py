"""tools/trace_replay.py (§5.2 Fig. 9 methodology; SPEC
S:384-439): closed forms and invariants on hand-built traces."""
import math
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import trace_replay as TR  # noqa: E402

P = [0.080, 0.160, 0.170]  # s per iteration with 0 / 1 / 2 failures
TOK = 8192.0


def test_empty_trace_is_fault_free():
    r = TR.replay(P, TOK, [], 1000 * P[0])
    assert r["iterations_completed"] == 1000
    assert r["average_normalized_throughput"] == pytest.approx(1.0, abs=1e-12)
    assert r["fault_scaled_reference"] == pytest.approx(1.0)


def test_single_permanent_failure_from_t0():
    H = 600 * P[1]
    r = TR.replay(P, TOK, [(0.0, +1)], H, total_workers=4)
    assert r["iterations_completed"] == 600
    assert r["average_normalized_throughput"] == pytest.approx(P[0] / P[1], rel=1e-12)
    assert r["fault_scaled_reference"] == pytest.approx(0.75)


def test_staircase_closed_form():
    """fail at t1, again at t2, one rejoin at t3, a migration stall s per swap: the
    iterations are the floor of each segment's usable time over its plan's period (the
    in-flight iteration at every event is discarded)."""
    t1, t2, t3, H, s = 10.0, 25.0, 40.0, 60.0, 0.5
    ev = [(t1, +1), (t2, +1), (t3, -1)]
    r = TR.replay(P, TOK, ev, H, migration_s=s, total_workers=8)
    n = (math.floor(t1 / P[0]) + math.floor((t2 - t1 - s) / P[1] + 1e-12) + math.floor((t3 - t2 - s) / P[2] + 1e-12)
         + math.floor((H - t3 - s) / P[1] + 1e-12))
    assert r["iterations_completed"] == n
    assert r["average_normalized_throughput"] == pytest.approx(n * TOK / H / (TOK / P[0]), rel=1e-12)
    assert [x["cause"] for x in r["stall_log"]] == ["MIGRATION"] * 3
    live = (t1 * 8 + (t2 - t1) * 7 + (t3 - t2) * 6 + (H - t3) * 7) / (8 * H)
    assert r["fault_scaled_reference"] == pytest.approx(live, rel=1e-12)


def test_invariants_on_a_random_trace():
    ev = TR.poisson_trace(mtbf_h=0.5, repair_h=0.3, hours=6, seed=3, max_failed=2)
    assert ev == TR.poisson_trace(mtbf_h=0.5, repair_h=0.3, hours=6, seed=3, max_failed=2)  # deterministic
    assert ev == sorted(ev)
    down = 0
    for _, d in ev:
        down += d
        assert 0 <= down <= 2
    r = TR.replay(P, TOK, ev, 6 * 3600.0, migration_s=0.011, total_workers=8)
    assert r["average_normalized_throughput"] <= 1.0 + 1e-9
    assert r["tokens"] == r["iterations_completed"] * TOK
    assert sum(x["iterations"] for x in r["samples"]) == r["iterations_completed"]
    spans = sorted([(x["t0"], x["t1"]) for x in r["samples"]] +
                   [(x["time_s"], x["time_s"] + x["duration_s"]) for x in r["stall_log"]])
    assert all(a[1] <= b[0] + 1e-9 for a, b in zip(spans, spans[1:]))  # stalls never overlap iterations


def test_more_failures_than_plans_stalls_until_rejoin():
    r = TR.replay(P[:2], TOK, [(1.0, +1), (2.0, +1), (5.0, -1)], 10.0)
    assert any(x["cause"] == "NO_PLAN" and x["duration_s"] == pytest.approx(3.0) for x in r["stall_log"])
    with pytest.raises(ValueError):
        TR.replay(P, TOK, [(2.0, +1), (1.0, -1)], 10.0)
