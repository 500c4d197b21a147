"""GPT model ends in fp64 numpy — token + position embedding (first stage) and final
LayerNorm + LM head + softmax cross-entropy (last stage) — TEST INFRASTRUCTURE (see
oracle/__init__.py).

PAPER.md §5.1 (line 607) trains "the Megatron implementation of GPT-3"; the ends are
not on the paper's method path (SURVEY.md §8(f) NEXT-3 adds them to make the stage
step GPT-complete).  Readings (R33): learned absolute position embeddings,
untied LM head W_out [V, h] (no bias), vocabulary padded to a multiple of 128
(50257 -> 50304, the padded classes are ordinary classes that no label names), loss =
mean over the T tokens of the micro-batch of  lse(logits_t) - logits_t[label_t].
Split like the layers (reading R9): B computes input gradients (and the final
LayerNorm's gamma / beta), W the weight products dW_out = dLogits^T Y and the embedding
scatter dE[v] = sum_{t: tok_t = v} dX_t, dP[p] = sum_{t: t mod s = p} dX_t.
"""
from __future__ import annotations

import numpy as np

from .layer import layernorm_bwd, layernorm_fwd, wgrad


def embed_fwd(E, P, tok, seq):
    """X[t] = E[tok[t]] + P[t mod seq]."""
    T = len(tok)
    return E[tok] + P[np.arange(T) % seq]


def embed_bwd(dX, tok, seq, V):
    """(dE, dP) with duplicates summed in token order."""
    T, h = dX.shape
    dE = np.zeros((V, h))
    dP = np.zeros((seq, h))
    for t in range(T):
        dE[tok[t]] += dX[t]
        dP[t % seq] += dX[t]
    return dE, dP


def head_forward(x, gf, bf, Wout, labels, eps):
    """Final LayerNorm, logits = Y W_out^T, mean cross-entropy.  Returns (loss, cache)."""
    y, xhat, rstd = layernorm_fwd(x, gf, bf, eps)
    logits = y @ Wout.T
    mx = logits.max(axis=1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(axis=1))
    T = len(labels)
    loss = float(np.mean(lse - logits[np.arange(T), labels]))
    return loss, dict(y=y, xhat=xhat, rstd=rstd, logits=logits, lse=lse, labels=labels, gf=gf, Wout=Wout)


def head_backward_input(c):
    """B of the head: dLogits = (softmax - onehot) / T, dY = dLogits W_out, then the
    final LayerNorm backward.  Returns (dx, {"gf": dgf, "bf": dbf}, wstash)."""
    T = len(c["labels"])
    p = np.exp(c["logits"] - c["lse"][:, None])
    dlog = p.copy()
    dlog[np.arange(T), c["labels"]] -= 1.0
    dlog /= T
    dy = dlog @ c["Wout"]
    dx, dg, db = layernorm_bwd(dy, c["xhat"], c["rstd"], c["gf"])
    return dx, {"gf": dg, "bf": db}, (c["y"], dlog)


def head_backward_weight(wstash):
    """W of the head: dW_out = dLogits^T Y."""
    y, dlog = wstash
    return {"Wout": wgrad(y, dlog)}
