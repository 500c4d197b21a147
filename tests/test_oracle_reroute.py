"""Re-route invariant (BJ): a re-routed micro-batch yields the same summed DP
gradient as the fault-free run.  Forms (ii)-(iii) of SURVEY §8(c.9) (form (i), the
canonical-order sum, is the reference the others are compared with), and the pins
of oracle/pipeline.py's per-micro-batch pass: torch fp64 autograd through a 2-stage
stack with the MSE head, and the (j, k) bookkeeping of `contributions`."""
import numpy as np
import pytest
import torch
import torch.nn.functional as Fn
from test_oracle_layer import _torch_layer

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


def _torch_stack_grads(stages, cfg, x, r):
    """Library pin: torch fp64 forward through every stage's layers (F.layer_norm,
    F.linear, SDPA, F.gelu), loss = 1/2 F.mse_loss(mean) = 1/2 ||Out - R||^2 / (T h),
    autograd for every parameter of every stage."""
    tp = [[{n: torch.tensor(v, requires_grad=True) for n, v in P.items()} for P in layers] for layers in stages]
    y = torch.tensor(x)
    for layers in tp:
        for P in layers:
            y = _torch_layer(P, y, cfg)
    loss = 0.5 * Fn.mse_loss(y, torch.tensor(r), reduction="mean")
    loss.backward()
    return loss.item(), [[{n: t.grad.numpy() for n, t in P.items()} for P in layers] for layers in tp]


def test_microbatch_pass_matches_autograd():
    """oracle/pipeline.py microbatch_pass (stage order, MSE head, dy hand-off between
    stages, B + W merge) against torch fp64 autograd of the whole 2-stage stack."""
    cfg = sd.ModelCfg(hidden=32, heads=2, ffn=128, seq=8, micro_batch=2, layers=3)
    stages = [sd.stage_params(cfg, 0, 2, total_layers=3), sd.stage_params(cfg, 1, 1, total_layers=3)]
    x, r = sd.stage_input(cfg, 1, 2), sd.stage_target(cfg, 1, 2)
    loss, grads = PPL.microbatch_pass(stages, cfg, x, r)
    lref, gref = _torch_stack_grads(stages, cfg, x, r)
    assert abs(loss - lref) <= 1e-12 * abs(lref)
    for i in range(len(stages)):
        for l in range(len(stages[i])):
            for n in sd.PARAM_ORDER:
                a, b = grads[i][l][n], gref[i][l][n]
                assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b)), (i, l, n)


def test_contributions_key_micro_batches_by_j_and_k():
    """Delta[(i, j, k)] is micro-batch j of pipeline k (inputs X_{k,j}, targets R_{k,j}):
    checked against autograd for an entry with j != k, so a (j, k) swap fails."""
    cfg = CFG
    N, DP, m = 2, 2, 3
    stages, xs, rs = _data(N, DP, m)
    delta, losses = PPL.contributions(stages, cfg, DP, m, xs, rs)
    assert sorted(delta) == sorted((i, j, k) for i in range(N) for j in range(m) for k in range(DP))
    j, k = 2, 1
    lref, gref = _torch_stack_grads(stages, cfg, sd.stage_input(cfg, k, j), sd.stage_target(cfg, k, j))
    assert abs(losses[(j, k)] - lref) <= 1e-12 * abs(lref)
    for i in range(N):
        for n in sd.PARAM_ORDER:
            a, b = delta[(i, j, k)][0][n], gref[i][0][n]
            assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b)), (i, n)
