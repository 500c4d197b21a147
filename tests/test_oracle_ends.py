"""Pins of oracle/ends.py (GPT model ends, reading R33) against
PyTorch fp64 autograd (torch.nn.functional embedding / layer_norm / linear /
cross_entropy — library routines independent of the oracle), closed forms and brute force."""
import numpy as np
import torch
import torch.nn.functional as F

from oracle import ends as OE


def rng_case(V=96, h=32, seq=16, b=2, seed=3, scale=0.5):
    r = np.random.default_rng(seed)
    T = b * seq
    return dict(E=r.standard_normal((V, h)) * scale, P=r.standard_normal((seq, h)) * scale,
                tok=r.integers(0, V, T), labels=r.integers(0, V - 7, T), x=r.standard_normal((T, h)),
                gf=1.0 + 0.1 * r.standard_normal(h), bf=0.1 * r.standard_normal(h),
                W=r.standard_normal((V, h)) * 0.3, dX=r.standard_normal((T, h)), seq=seq, V=V)


def test_embedding_vs_torch_and_duplicates():
    c = rng_case()
    c["tok"][3] = c["tok"][5] = c["tok"][11]  # repeated tokens
    X = OE.embed_fwd(c["E"], c["P"], c["tok"], c["seq"])
    Et = torch.tensor(c["E"], requires_grad=True)
    Pt = torch.tensor(c["P"], requires_grad=True)
    tok = torch.tensor(c["tok"])
    Xt = F.embedding(tok, Et) + Pt[torch.arange(len(tok)) % c["seq"]]
    assert np.abs(X - Xt.detach().numpy()).max() == 0.0
    Xt.backward(torch.tensor(c["dX"]))
    dE, dP = OE.embed_bwd(c["dX"], c["tok"], c["seq"], c["V"])
    assert np.allclose(dE, Et.grad.numpy(), rtol=0, atol=1e-12)
    assert np.allclose(dP, Pt.grad.numpy(), rtol=0, atol=1e-12)
    # brute force for the repeated token: the three rows summed
    v = c["tok"][3]
    others = [t for t in range(len(c["tok"])) if c["tok"][t] == v]
    assert np.allclose(dE[v], sum(c["dX"][t] for t in others), atol=1e-12)
    assert np.count_nonzero(np.abs(dE).sum(1)) == len(set(c["tok"].tolist()))


def test_head_forward_backward_vs_torch():
    c = rng_case()
    loss, cache = OE.head_forward(c["x"], c["gf"], c["bf"], c["W"], c["labels"], 1e-5)
    dx, bg, ws = OE.head_backward_input(cache)
    wg = OE.head_backward_weight(ws)
    x = torch.tensor(c["x"], requires_grad=True)
    gf = torch.tensor(c["gf"], requires_grad=True)
    bf = torch.tensor(c["bf"], requires_grad=True)
    W = torch.tensor(c["W"], requires_grad=True)
    y = F.layer_norm(x, (x.shape[1],), gf, bf, 1e-5)
    lt = F.cross_entropy(F.linear(y, W), torch.tensor(c["labels"]))
    lt.backward()
    assert abs(loss - lt.item()) <= 1e-12 * max(1.0, abs(loss))
    assert np.allclose(dx, x.grad.numpy(), rtol=1e-10, atol=1e-13)
    assert np.allclose(bg["gf"], gf.grad.numpy(), rtol=1e-10, atol=1e-13)
    assert np.allclose(bg["bf"], bf.grad.numpy(), rtol=1e-10, atol=1e-13)
    assert np.allclose(wg["Wout"], W.grad.numpy(), rtol=1e-10, atol=1e-13)


def test_head_closed_forms():
    """W_out = 0: every logit 0, loss = ln V exactly, dLogits = (1/V - onehot)/T, so
    dY = 0 and dx = 0; rows of dLogits sum to zero for any weights."""
    c = rng_case()
    V, T = c["V"], len(c["labels"])
    loss, cache = OE.head_forward(c["x"], c["gf"], c["bf"], np.zeros_like(c["W"]), c["labels"], 1e-5)
    assert abs(loss - np.log(V)) < 1e-14
    dx, bg, (y, dlog) = OE.head_backward_input(cache)
    ref = np.full((T, V), 1.0 / V)
    ref[np.arange(T), c["labels"]] -= 1.0
    assert np.allclose(dlog, ref / T, atol=1e-16)
    assert np.abs(dx).max() == 0.0
    _, cache = OE.head_forward(c["x"], c["gf"], c["bf"], c["W"], c["labels"], 1e-5)
    _, _, (y, dlog) = OE.head_backward_input(cache)
    assert np.abs(dlog.sum(axis=1)).max() < 1e-15
