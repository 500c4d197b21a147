"""AdamW step in fp64 — TEST INFRASTRUCTURE (see oracle/__init__.py).

PAPER.md §4.3 (line 583) names only "AdamW" and states that each stage steps
after its own all-reduce and local validation.  DESIGN.md reading R11 fixes the
hyper-parameters and form (Loshchilov & Hutter decoupled weight decay, bias
correction on, eps outside the square root, no global-norm clipping); reading
R8 fixes the gradient normalisation (mean over the DP*m micro-batches, applied
as ``grad_scale`` inside the step).  Step t >= 1, g <- grad_scale * g:
    m <- b1 m + (1 - b1) g
    v <- b2 v + (1 - b2) g^2
    mhat = m / (1 - b1^t),  vhat = v / (1 - b2^t)
    p <- p - lr wd p - lr mhat / (sqrt(vhat) + eps)
Weight decay applies to the 2-D weight matrices only.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class AdamCfg:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1


def adamw_step(p, m, v, g, step, cfg: AdamCfg, grad_scale=1.0, decay=True):
    """Returns (p, m, v) after one step; arrays are not modified in place."""
    g = grad_scale * g
    m = cfg.beta1 * m + (1.0 - cfg.beta1) * g
    v = cfg.beta2 * v + (1.0 - cfg.beta2) * g * g
    mhat = m / (1.0 - cfg.beta1 ** step)
    vhat = v / (1.0 - cfg.beta2 ** step)
    wd = cfg.weight_decay if decay else 0.0
    p = p - cfg.lr * wd * p - cfg.lr * mhat / (np.sqrt(vhat) + cfg.eps)
    return p, m, v


def adamw_step_layer(params, m, v, grads, step, cfg: AdamCfg, grad_scale=1.0):
    """Per-tensor dicts; decay only for 2-D tensors (weight matrices)."""
    newp, newm, newv = {}, {}, {}
    for name, p in params.items():
        newp[name], newm[name], newv[name] = adamw_step(
            p, m[name], v[name], grads[name], step, cfg, grad_scale, decay=(np.ndim(p) == 2))
    return newp, newm, newv


def nonfinite(grads) -> bool:
    """Local post-step validation flag (§4.3): any non-finite
    gradient element in this stage."""
    return any(not np.all(np.isfinite(g)) for g in grads.values())


def adamw_inverse(p1, m1, v1, g, step, cfg: AdamCfg, grad_scale=1.0, decay=True):
    """The arithmetic reversal of adamw_step (§4.3: AdamW rollbacks
    "do not entail additional memory costs because the operations involved are
    arithmetically reversible"), given the post-step state and the same gradient:
        m0 = (m1 - (1 - b1) g) / b1,   v0 = (v1 - (1 - b2) g^2) / b2,
        p0 = (p1 + lr mhat1 / (sqrt(vhat1) + eps)) / (1 - lr wd).
    Exact in real arithmetic; v0 is clamped at 0 against rounding (reading R31)."""
    g = grad_scale * g
    mhat = m1 / (1.0 - cfg.beta1 ** step)
    vhat = v1 / (1.0 - cfg.beta2 ** step)
    wd = cfg.weight_decay if decay else 0.0
    p0 = (p1 + cfg.lr * mhat / (np.sqrt(vhat) + cfg.eps)) / (1.0 - cfg.lr * wd)
    m0 = (m1 - (1.0 - cfg.beta1) * g) / cfg.beta1
    v0 = np.maximum((v1 - (1.0 - cfg.beta2) * g * g) / cfg.beta2, 0.0)
    return p0, m0, v0
