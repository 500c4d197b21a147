"""One pre-LN GPT layer in fp64 numpy — forward, coupled backward, and the
decoupled split into B (input gradients) and W (weight gradients).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Plain definitions, no blocking,
no fusion.  Citations:
  * PAPER.md §3.2 (lines 250-255): "the backward pass calculates two distinct
    outputs: the gradients relative to the input (B_Input) and the gradients
    relative to parameters (weights) ... (B_Weight)".  W is "dependence-free"
    and deferrable.
  * PAPER.md §5.1 (line 607): "Megatron implementation of GPT-3" — the layer
    architecture itself is not spelled out; reading R1 fixes it:
    pre-LN, biased-variance LayerNorm (eps 1e-5), causal softmax attention,
    4h tanh-GeLU FFN, all linears with bias.
  * DESIGN.md reading R9: W = exactly the four dW products per layer; bias
    and LayerNorm gamma/beta gradients are produced by B.

Shapes: X [T, h] with T = micro_batch * seq, token t = b*seq + pos.
Weights are [out, in]; QKV rows are the [Q; K; V] blocks, head n uses rows
n*d..(n+1)*d of each block (so columns n*d..(n+1)*d of the QKV activation).
"""
from __future__ import annotations

import numpy as np

GELU_C = np.sqrt(2.0 / np.pi)
GELU_A = 0.044715


# ---------------------------------------------------------------- primitives
def layernorm_fwd(x, gamma, beta, eps):
    """y = xhat*gamma + beta, xhat = (x - mean) / sqrt(var + eps), biased var."""
    mu = x.mean(axis=1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = xc * rstd
    return xhat * gamma + beta, xhat, rstd


def layernorm_bwd(dy, xhat, rstd, gamma):
    """Returns (dx, dgamma, dbeta) for y = xhat*gamma + beta."""
    dgamma = (dy * xhat).sum(axis=0)
    dbeta = dy.sum(axis=0)
    g = dy * gamma
    dx = rstd * (g - g.mean(axis=1, keepdims=True) - xhat * (g * xhat).mean(axis=1, keepdims=True))
    return dx, dgamma, dbeta


def gelu(x):
    """tanh GeLU: 0.5 x (1 + tanh(c (x + 0.044715 x^3)))."""
    return 0.5 * x * (1.0 + np.tanh(GELU_C * (x + GELU_A * x ** 3)))


def gelu_grad(x):
    tau = np.tanh(GELU_C * (x + GELU_A * x ** 3))
    return 0.5 * (1.0 + tau) + 0.5 * x * (1.0 - tau * tau) * GELU_C * (1.0 + 3.0 * GELU_A * x * x)


def linear(x, w, b):
    """x [T, in], w [out, in], b [out] -> x w^T + b."""
    return x @ w.T + b


def wgrad(x, dy):
    """The single W product, dW = dY^T X ([out, in]).  Every weight gradient in
    the oracle goes through this one function so that coupled and decoupled
    runs perform the identical floating-point operation."""
    return dy.T @ x


def _heads(a, cfg, which):
    """View block `which` (0=Q,1=K,2=V) of QKV [T,3h] as [b, heads, s, d]."""
    h, d, s, b = cfg.hidden, cfg.head_dim, cfg.seq, cfg.micro_batch
    blk = a[:, which * h:(which + 1) * h]
    return blk.reshape(b, s, cfg.heads, d).transpose(0, 2, 1, 3)


def _merge(o, cfg):
    """[b, heads, s, d] -> [T, h]."""
    b, a, s, d = o.shape
    return o.transpose(0, 2, 1, 3).reshape(b * s, a * d)


def attention_fwd(qkv, cfg):
    """Causal softmax attention.  S = Q K^T / sqrt(d), S[t,u] = -inf for u > t,
    P = softmax_row(S), O = P V.  Returns (O [T,h], P [b,heads,s,s])."""
    q, k, v = (_heads(qkv, cfg, w) for w in range(3))
    d = cfg.head_dim
    s = q @ k.transpose(0, 1, 3, 2) / np.sqrt(d)
    mask = np.triu(np.ones((cfg.seq, cfg.seq), dtype=bool), 1)
    s = np.where(mask, -np.inf, s)
    s = s - s.max(axis=-1, keepdims=True)
    e = np.exp(s)
    p = e / e.sum(axis=-1, keepdims=True)
    o = p @ v
    return _merge(o, cfg), p


def attention_bwd(do, qkv, p, cfg):
    """dV = P^T dO; dP = dO V^T; dS = P (dP - rowsum(dP P)) / sqrt(d);
    dQ = dS K; dK = dS^T Q.  Returns dQKV [T, 3h] and the intermediates."""
    q, k, v = (_heads(qkv, cfg, w) for w in range(3))
    dO = do.reshape(cfg.micro_batch, cfg.seq, cfg.heads, cfg.head_dim).transpose(0, 2, 1, 3)
    dv = p.transpose(0, 1, 3, 2) @ dO
    dp = dO @ v.transpose(0, 1, 3, 2)
    ds = p * (dp - (dp * p).sum(axis=-1, keepdims=True)) / np.sqrt(cfg.head_dim)
    dq = ds @ k
    dk = ds.transpose(0, 1, 3, 2) @ q
    dqkv = np.concatenate([_merge(dq, cfg), _merge(dk, cfg), _merge(dv, cfg)], axis=1)
    return dqkv, {"dp": dp, "ds": ds}


# ---------------------------------------------------------------- forward
def layer_forward(P, x, cfg):
    """One layer, §5.1 GPT (reading R1).  Returns (Out, cache)."""
    y1, xhat1, rstd1 = layernorm_fwd(x, P["g1"], P["b1n"], cfg.ln_eps)
    qkv = linear(y1, P["wqkv"], P["bqkv"])
    o, p = attention_fwd(qkv, cfg)
    x2 = x + linear(o, P["wo"], P["bo"])
    y2, xhat2, rstd2 = layernorm_fwd(x2, P["g2"], P["b2n"], cfg.ln_eps)
    hpre = linear(y2, P["w1"], P["b1"])
    g = gelu(hpre)
    out = x2 + linear(g, P["w2"], P["b2"])
    cache = dict(x=x, y1=y1, xhat1=xhat1, rstd1=rstd1, qkv=qkv, p=p, o=o, x2=x2,
                 y2=y2, xhat2=xhat2, rstd2=rstd2, h=hpre, g=g)
    return out, cache


def stage_forward(layers, x, cfg):
    caches = []
    for P in layers:
        x, c = layer_forward(P, x, cfg)
        caches.append(c)
    return x, caches


# ---------------------------------------------------------------- backward
def layer_backward_input(P, c, dout, cfg):
    """B: input gradient of one layer plus the bias / LayerNorm parameter
    gradients (reading R9).  Also returns the W-stash (WeightGradStore,
    PAPER.md §4.3): the (X, dY) pairs of the four W products."""
    grads = {}
    grads["b2"] = dout.sum(axis=0)
    dg = dout @ P["w2"]
    dh = dg * gelu_grad(c["h"])
    grads["b1"] = dh.sum(axis=0)
    dy2 = dh @ P["w1"]
    dx2_ln, grads["g2"], grads["b2n"] = layernorm_bwd(dy2, c["xhat2"], c["rstd2"], P["g2"])
    dx2 = dout + dx2_ln
    grads["bo"] = dx2.sum(axis=0)
    do = dx2 @ P["wo"]
    dqkv, _ = attention_bwd(do, c["qkv"], c["p"], cfg)
    grads["bqkv"] = dqkv.sum(axis=0)
    dy1 = dqkv @ P["wqkv"]
    dx1_ln, grads["g1"], grads["b1n"] = layernorm_bwd(dy1, c["xhat1"], c["rstd1"], P["g1"])
    dx = dx2 + dx1_ln
    wstash = {"w2": (c["g"], dout), "w1": (c["y2"], dh), "wo": (c["o"], dx2), "wqkv": (c["y1"], dqkv)}
    return dx, grads, wstash


def layer_backward_weight(wstash):
    """W: exactly four products per layer, dW = dY^T X (§3.2)."""
    return {name: wgrad(xx, dy) for name, (xx, dy) in wstash.items()}


def layer_backward_coupled(P, c, dout, cfg):
    """Conventional backward: each W product right after its dY exists, in the
    order FC2, FC1, O, QKV.  Same formulas, same arrays, different timing."""
    grads = {}
    grads["b2"] = dout.sum(axis=0)
    grads["w2"] = wgrad(c["g"], dout)
    dg = dout @ P["w2"]
    dh = dg * gelu_grad(c["h"])
    grads["b1"] = dh.sum(axis=0)
    grads["w1"] = wgrad(c["y2"], dh)
    dy2 = dh @ P["w1"]
    dx2_ln, grads["g2"], grads["b2n"] = layernorm_bwd(dy2, c["xhat2"], c["rstd2"], P["g2"])
    dx2 = dout + dx2_ln
    grads["bo"] = dx2.sum(axis=0)
    grads["wo"] = wgrad(c["o"], dx2)
    do = dx2 @ P["wo"]
    dqkv, _ = attention_bwd(do, c["qkv"], c["p"], cfg)
    grads["bqkv"] = dqkv.sum(axis=0)
    grads["wqkv"] = wgrad(c["y1"], dqkv)
    dy1 = dqkv @ P["wqkv"]
    dx1_ln, grads["g1"], grads["b1n"] = layernorm_bwd(dy1, c["xhat1"], c["rstd1"], P["g1"])
    dx = dx2 + dx1_ln
    return dx, grads


def stage_backward_input(layers, caches, dout, cfg):
    """B over a stage (layers in reverse).  Returns dX, per-layer B grads and
    per-layer W-stashes."""
    bgrads, stashes = [None] * len(layers), [None] * len(layers)
    for l in reversed(range(len(layers))):
        dout, bgrads[l], stashes[l] = layer_backward_input(layers[l], caches[l], dout, cfg)
    return dout, bgrads, stashes


def stage_backward_weight(stashes):
    return [layer_backward_weight(s) for s in stashes]


def stage_backward_coupled(layers, caches, dout, cfg):
    grads = [None] * len(layers)
    for l in reversed(range(len(layers))):
        dout, grads[l] = layer_backward_coupled(layers[l], caches[l], dout, cfg)
    return dout, grads


def merge_grads(bgrads, wgrads):
    """Per-layer dict union of B grads and W grads."""
    return [dict(**b, **w) for b, w in zip(bgrads, wgrads)]


# ---------------------------------------------------------------- loss heads
def loss_inner(out, r):
    """Stage-level test loss l = <Out, R>, so dOut = R exactly."""
    return float((out * r).sum()), r.copy()


def loss_mse(out, r):
    """Pipeline loss head: l = 1/2 ||Out - R||^2 / (T h),
    dOut = (Out - R) / (T h)."""
    n = out.size
    diff = out - r
    return 0.5 * float((diff * diff).sum()) / n, diff / n
