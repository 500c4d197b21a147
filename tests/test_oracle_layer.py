"""Pins for oracle/layer.py against things other than itself:
torch fp64 library routines, torch.autograd, central finite differences,
closed-form special cases and algebraic identities."""
import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

import slipdata as sd
from oracle import layer as L

CFG = sd.C1_TINY
TINY2 = sd.ModelCfg(hidden=32, heads=2, ffn=128, seq=8, micro_batch=2, layers=2)


def relerr(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _torch_layer(P, x, cfg):
    """Library-routine forward (torch fp64): F.layer_norm, F.linear,
    F.scaled_dot_product_attention(is_causal=True), F.gelu(tanh)."""
    h, a, d = cfg.hidden, cfg.heads, cfg.head_dim
    y1 = Fn.layer_norm(x, (h,), P["g1"], P["b1n"], cfg.ln_eps)
    qkv = Fn.linear(y1, P["wqkv"], P["bqkv"])
    b, s = cfg.micro_batch, cfg.seq

    def heads(t):
        return t.reshape(b, s, a, d).transpose(1, 2)
    q, k, v = heads(qkv[:, :h]), heads(qkv[:, h:2 * h]), heads(qkv[:, 2 * h:])
    o = Fn.scaled_dot_product_attention(q, k, v, is_causal=True)
    o = o.transpose(1, 2).reshape(b * s, h)
    x2 = x + Fn.linear(o, P["wo"], P["bo"])
    y2 = Fn.layer_norm(x2, (h,), P["g2"], P["b2n"], cfg.ln_eps)
    g = Fn.gelu(Fn.linear(y2, P["w1"], P["b1"]), approximate="tanh")
    return x2 + Fn.linear(g, P["w2"], P["b2"])


def _setup(cfg, stage=0):
    P = sd.layer_params(cfg, stage, 0)
    x = sd.stage_input(cfg, 0, 0)
    r = sd.stage_target(cfg, 0, 0)
    return P, x, r


@pytest.mark.parametrize("cfg", [CFG, TINY2])
def test_forward_matches_torch_fp64(cfg):
    P, x, _ = _setup(cfg)
    out, _ = L.layer_forward(P, x, cfg)
    with torch.no_grad():
        ref = _torch_layer({k: torch.tensor(v) for k, v in P.items()}, torch.tensor(x), cfg).numpy()
    assert relerr(out, ref) <= 1e-12


@pytest.mark.parametrize("cfg", [CFG, TINY2])
def test_coupled_backward_matches_autograd(cfg):
    P, x, r = _setup(cfg)
    out, cache = L.layer_forward(P, x, cfg)
    _, dout = L.loss_inner(out, r)
    dx, grads = L.layer_backward_coupled(P, cache, dout, cfg)
    tp = {k: torch.tensor(v, requires_grad=True) for k, v in P.items()}
    tx = torch.tensor(x, requires_grad=True)
    loss = (_torch_layer(tp, tx, cfg) * torch.tensor(r)).sum()
    loss.backward()
    assert relerr(dx, tx.grad.numpy()) <= 1e-12
    for name in sd.PARAM_ORDER:
        assert relerr(grads[name], tp[name].grad.numpy()) <= 1e-12, name


def test_finite_differences_c1():
    """Central differences of l = <Out, R> on C1: random unit directions over
    all parameters and X, plus sampled coordinates per tensor (BJ: <= 1e-6)."""
    cfg = CFG
    P, x, r = _setup(cfg)
    out, cache = L.layer_forward(P, x, cfg)
    dx, grads = L.layer_backward_coupled(P, cache, r, cfg)
    names = list(sd.PARAM_ORDER) + ["X"]
    theta = dict(P, X=x)
    grad = dict(grads, X=dx)

    def loss(th):
        Pp = {k: th[k] for k in sd.PARAM_ORDER}
        o, _ = L.layer_forward(Pp, th["X"], cfg)
        return float((o * r).sum())

    rng = np.random.default_rng(7)
    tmax = max(np.max(np.abs(v)) for v in theta.values())
    delta = 1e-5 * max(1.0, tmax)
    worst = 0.0
    for _ in range(32):
        v = {k: rng.normal(size=theta[k].shape) for k in names}
        nrm = np.sqrt(sum((vv * vv).sum() for vv in v.values()))
        v = {k: vv / nrm for k, vv in v.items()}
        lp = loss({k: theta[k] + delta * v[k] for k in names})
        lm = loss({k: theta[k] - delta * v[k] for k in names})
        fd = (lp - lm) / (2 * delta)
        an = sum((grad[k] * v[k]).sum() for k in names)
        worst = max(worst, abs(fd - an) / abs(an))
    assert worst <= 1e-6, worst
    gmax = max(np.max(np.abs(g)) for g in grad.values())
    for k in names:
        flat = theta[k].reshape(-1)
        idx = rng.choice(flat.size, size=min(200, flat.size), replace=False)
        for ii in idx:
            th_p = dict(theta)
            th_m = dict(theta)
            a = flat.copy(); a[ii] += delta; th_p[k] = a.reshape(theta[k].shape)
            b = flat.copy(); b[ii] -= delta; th_m[k] = b.reshape(theta[k].shape)
            fd = (loss(th_p) - loss(th_m)) / (2 * delta)
            an = grad[k].reshape(-1)[ii]
            assert abs(fd - an) <= 1e-6 * max(abs(an), 1e-3 * gmax), (k, ii, fd, an)


@pytest.mark.parametrize("cfg", [CFG, TINY2])
def test_decoupled_equals_coupled_bitexact(cfg):
    """B + W == coupled backward, bit for bit in fp64 (BJ invariant)."""
    layers = sd.stage_params(cfg, 0, 2)
    x = sd.stage_input(cfg, 0, 1)
    r = sd.stage_target(cfg, 0, 1)
    out, caches = L.stage_forward(layers, x, cfg)
    dxc, gc = L.stage_backward_coupled(layers, caches, r, cfg)
    dxd, gb, st = L.stage_backward_input(layers, caches, r, cfg)
    gw = L.stage_backward_weight(st)
    gd = L.merge_grads(gb, gw)
    assert np.array_equal(dxc, dxd)
    for lc, ld in zip(gc, gd):
        assert set(lc) == set(ld) == set(sd.PARAM_ORDER)
        for n in sd.PARAM_ORDER:
            assert np.array_equal(lc[n], ld[n]), n


def test_wgrad_is_sum_of_outer_products():
    """dW = sum_t dY_t^T X_t, evaluated by an explicit loop (not matmul)."""
    rng = np.random.default_rng(3)
    x = rng.normal(size=(9, 5))
    dy = rng.normal(size=(9, 4))
    ref = np.zeros((4, 5))
    for t in range(9):
        for o in range(4):
            for i in range(5):
                ref[o, i] += dy[t, o] * x[t, i]
    assert relerr(L.wgrad(x, dy), ref) <= 1e-14


def test_layernorm_identities():
    rng = np.random.default_rng(4)
    x = rng.normal(size=(6, 16))
    gamma = 1 + 0.1 * rng.normal(size=16)
    beta = 0.1 * rng.normal(size=16)
    y, xhat, rstd = L.layernorm_fwd(x, gamma, beta, 1e-5)
    dy = rng.normal(size=(6, 16))
    dx, dgamma, dbeta = L.layernorm_bwd(dy, xhat, rstd, gamma)
    # LN is shift invariant: rows of dx are orthogonal to 1
    assert np.max(np.abs(dx.sum(axis=1))) < 1e-12
    # with eps = 0 it is also scale invariant: rows of dx orthogonal to x
    _, xh0, r0 = L.layernorm_fwd(x, gamma, beta, 0.0)
    dx0, _, _ = L.layernorm_bwd(dy, xh0, r0, gamma)
    assert np.max(np.abs((dx0 * x).sum(axis=1))) < 1e-12
    # constant row -> xhat = 0 -> output = beta
    y2, _, _ = L.layernorm_fwd(np.full((1, 16), 3.25), gamma, beta, 1e-5)
    assert np.allclose(y2[0], beta, atol=0, rtol=0)


def test_attention_identities():
    cfg = CFG
    P, x, r = _setup(cfg)
    out, cache = L.layer_forward(P, x, cfg)
    do = sd.rng(99).normal(size=(cfg.tokens, cfg.hidden))
    _, inter = L.attention_bwd(do, cache["qkv"], cache["p"], cfg)
    # softmax Jacobian: rows of dS sum to zero; causal mask -> P upper triangle exactly 0
    assert np.max(np.abs(inter["ds"].sum(axis=-1))) < 1e-13
    assert np.all(cache["p"][..., np.triu_indices(cfg.seq, 1)[0], np.triu_indices(cfg.seq, 1)[1]] == 0.0)
    assert np.allclose(cache["p"].sum(axis=-1), 1.0, rtol=0, atol=1e-14)


def test_special_cases():
    cfg = CFG
    P, x, _ = _setup(cfg)
    # Wo = W2 = 0  =>  Out = X + bo + b2
    Q = dict(P, wo=np.zeros_like(P["wo"]), w2=np.zeros_like(P["w2"]))
    out, _ = L.layer_forward(Q, x, cfg)
    assert relerr(out, x + P["bo"] + P["b2"]) <= 1e-15
    # seq = 1  =>  attention output O = V exactly
    c1 = sd.ModelCfg(hidden=64, heads=2, ffn=256, seq=1, micro_batch=3, layers=1)
    qkv = sd.rng(5).normal(size=(3, 192))
    o, p = L.attention_fwd(qkv, c1)
    assert np.array_equal(o, qkv[:, 128:])
    assert np.all(p == 1.0)


def test_gelu_grad_matches_torch():
    x = np.linspace(-6, 6, 1001)
    tx = torch.tensor(x, requires_grad=True)
    Fn.gelu(tx, approximate="tanh").sum().backward()
    assert relerr(L.gelu_grad(x), tx.grad.numpy()) <= 1e-14
    assert relerr(L.gelu(x), Fn.gelu(torch.tensor(x), approximate="tanh").numpy()) <= 1e-14


def test_mse_head_gradient():
    rng = np.random.default_rng(8)
    out = rng.normal(size=(4, 6))
    r = rng.normal(size=(4, 6))
    loss, d = L.loss_mse(out, r)
    t = torch.tensor(out, requires_grad=True)
    (0.5 * ((t - torch.tensor(r)) ** 2).mean()).backward()
    assert abs(loss - 0.5 * np.mean((out - r) ** 2)) < 1e-15
    assert relerr(d, t.grad.numpy()) <= 1e-15
