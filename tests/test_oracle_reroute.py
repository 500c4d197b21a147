"""Re-route invariant (BJ): a re-routed micro-batch yields the same summed DP
gradient as the fault-free run.  Forms (i)-(iii) of SURVEY §8(c.9)."""
import numpy as np
import pytest

import slipdata as sd
from oracle import pipeline as PPL
from oracle import planner as PL
from oracle.adam import AdamCfg, adamw_step_layer

CFG = sd.ModelCfg(hidden=32, heads=2, ffn=128, seq=8, micro_batch=2, layers=1)


def _data(N, DP, m):
    stages = [sd.stage_params(CFG, i, 1) for i in range(N)]
    xs = {(k, j): sd.stage_input(CFG, k, j) for k in range(DP) for j in range(m)}
    rs = {(k, j): sd.stage_target(CFG, k, j) for k in range(DP) for j in range(m)}
    return stages, xs, rs


@pytest.mark.parametrize("N,DP,m,failed", [(2, 2, 2, [(1, 1)]), (2, 2, 2, [(0, 0)]),
                                           (2, 3, 4, [(1, 1)]), (2, 3, 4, [(0, 2), (1, 0)]),
                                           (2, 3, 4, [(1, 0), (1, 2)])])
def test_reroute_invariant(N, DP, m, failed):
    stages, xs, rs = _data(N, DP, m)
    delta, _ = PPL.contributions(stages, CFG, DP, m, xs, rs)
    live_ff = [[1] * DP for _ in range(N)]
    live = [[1] * DP for _ in range(N)]
    for (i, k) in failed:
        live[i][k] = 0
    costs = PL.Costs(t_f=1, t_b=1, t_w=1, t_comm=1)
    opts = PL.Opts(decoupled=True, staggered=True, horizon=1)
    plan_ff = PL.schedule(live_ff, m, costs, opts)
    plan = PL.schedule(live, m, costs, opts)
    for i in range(N):
        ref = PPL.canonical_sum(delta, i, DP, m)
        # (i) canonical order: executor identity does not touch the numbers
        assert all(np.array_equal(a[n], b[n]) for a, b in zip(ref, PPL.canonical_sum(delta, i, DP, m)) for n in a)
        # (ii) per-worker accumulation in plan order + live-peer sum
        got = PPL.per_worker_sum(delta, plan, live, i)
        got_ff = PPL.per_worker_sum(delta, plan_ff, live_ff, i)
        for a, b, c in zip(got, ref, got_ff):
            for n in a:
                scale = np.max(np.abs(b[n]))
                assert np.max(np.abs(a[n] - b[n])) <= 1e-12 * scale, n
                assert np.max(np.abs(a[n] - c[n])) <= 1e-12 * scale, n
    # (iii) work conservation, exact
    assert PPL.w_partition(plan, N, DP, m)
    # no op on a failed worker
    assert not any(o.stage == i and o.exec == k for (i, k) in failed for o in plan.ops)


def test_peers_identical_after_adam():
    """Peers of a stage apply the same all-reduced gradient and stay identical."""
    N, DP, m = 2, 2, 2
    stages, xs, rs = _data(N, DP, m)
    delta, _ = PPL.contributions(stages, CFG, DP, m, xs, rs)
    g = PPL.canonical_sum(delta, 1, DP, m)[0]
    P = stages[1][0]
    z = {k: np.zeros_like(v) for k, v in P.items()}
    a = adamw_step_layer(P, z, z, g, 1, AdamCfg(), grad_scale=1.0 / (DP * m))
    b = adamw_step_layer({k: v.copy() for k, v in P.items()}, z, z, g, 1, AdamCfg(), grad_scale=1.0 / (DP * m))
    for n in P:
        assert np.array_equal(a[0][n], b[0][n])
