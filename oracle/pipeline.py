"""DP x PP numerics with Adaptive Pipelining re-routes — TEST INFRASTRUCTURE.

PAPER.md §3.1 (line 215): "The overall mathematical computation remains
unchanged from the fault-free 1F1B schedule"; §3.4 / §5 (line 802):
"operations are mathematically consistent regardless of the number of
failures".  The stage-i gradient is the sum over every (j, k) micro-batch of
its per-micro-batch contribution Delta_{i,j,k}; a failure only changes which
worker (i, k_s) computes it.

Three forms (SURVEY.md §8(c.9) "Re-route"):
  (i)   canonical-order sum over (k asc, j asc) of Delta_{i,j,k};
  (ii)  per-worker accumulation in the plan's W-op order, then a live-peer sum
        in ascending k_s (how the GPU path reduces: local fp32 accumulate,
        then the DP all-reduce over live peers);
  (iii) work conservation: the W ops of all workers partition all (i, j, k).
"""
from __future__ import annotations

import numpy as np

from . import layer as L
from . import planner as PL


def microbatch_pass(stages, cfg, x, r):
    """Forward through all N stages, MSE head, decoupled backward.
    Returns (loss, per-stage list of per-layer grad dicts)."""
    caches = []
    for layers in stages:
        x, c = L.stage_forward(layers, x, cfg)
        caches.append(c)
    loss, dy = L.loss_mse(x, r)
    grads = [None] * len(stages)
    for i in reversed(range(len(stages))):
        dy, bg, st = L.stage_backward_input(stages[i], caches[i], dy, cfg)
        grads[i] = L.merge_grads(bg, L.stage_backward_weight(st))
    return loss, grads


def contributions(stages, cfg, DP, m, inputs, targets):
    """Delta[(i, j, k)] = per-layer grad dicts of micro-batch (j, k) at stage i."""
    delta, losses = {}, {}
    for k in range(DP):
        for j in range(m):
            losses[(j, k)], g = microbatch_pass(stages, cfg, inputs[(k, j)], targets[(k, j)])
            for i in range(len(stages)):
                delta[(i, j, k)] = g[i]
    return delta, losses


def _zeros_like(gl):
    return [{n: np.zeros_like(a) for n, a in d.items()} for d in gl]


def _acc(acc, gl):
    for a, g in zip(acc, gl):
        for n in a:
            a[n] += g[n]


def canonical_sum(delta, i, DP, m):
    """Form (i): sum over k ascending, then j ascending."""
    acc = _zeros_like(delta[(i, 0, 0)])
    for k in range(DP):
        for j in range(m):
            _acc(acc, delta[(i, j, k)])
    return acc


def per_worker_sum(delta, plan, live, i):
    """Form (ii): each live worker accumulates its W ops in plan order (by
    start time), then the all-reduce sums live peers in ascending k_s."""
    DP = len(live[i])
    total = None
    for ks in range(DP):
        if not live[i][ks]:
            continue
        w_ops = sorted((o for o in plan.ops if o.stage == i and o.exec == ks and o.phase in (PL.W, PL.BC)
                        and o.it == 0), key=lambda o: o.start)
        acc = _zeros_like(delta[(i, 0, 0)])
        for o in w_ops:
            _acc(acc, delta[(i, o.mb, o.origin)])
        if total is None:
            total = acc
        else:
            _acc(total, acc)
    return total


def w_partition(plan, N, DP, m):
    """Form (iii): multiset of (i, j, k) covered by iteration-0 W ops."""
    seen = sorted((o.stage, o.mb, o.origin) for o in plan.ops if o.phase in (PL.W, PL.BC) and o.it == 0)
    return seen == sorted((i, j, k) for i in range(N) for j in range(m) for k in range(DP))
