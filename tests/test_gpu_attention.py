"""Kernel-level parity of the fused causal attention (slip_attention) on the same bf16
inputs: O, the log2-domain LSE, and dQ / dK / dV against the fp64 oracle
(oracle/layer.py attention_fwd / attention_bwd) where it finishes in seconds, and against
a plain PyTorch fp32 reference of the same operation at the full GPT shapes — at sizes
that span several tiles, ragged tails (s % 128 != 0, s % 64 != 0), every supported head
dim, batch > 1.  Metric: the element-wise infinity-norm ratio of SURVEY §8(c.10)."""
import math

import numpy as np

import pytest
import torch

pytestmark = pytest.mark.gpu

GATE = 2e-2  # normwise, bf16 operands / fp32 accumulation (SURVEY §8(c) Gate A)


def rel(a, b):
    """||a - b||_inf / ||b||_inf (SURVEY §8(c.10) Gate A)."""
    a, b = a.double(), b.double()
    return ((a - b).abs().max() / b.abs().max()).item()


def oracle_reference(qkv, s, heads, batch, d, do):
    """fp64 oracle (oracle/layer.py) on the kernel's exact bf16 inputs."""
    import slipdata as sd
    from oracle import layer as OL
    cfg = sd.ModelCfg(hidden=heads * d, heads=heads, ffn=4 * heads * d, seq=s, micro_batch=batch, layers=1)
    q64 = qkv.double().cpu().numpy()
    o, p = OL.attention_fwd(q64, cfg)
    dqkv, _ = OL.attention_bwd(do.double().cpu().numpy(), q64, p, cfg)
    sc = np.einsum("bhsd,bhtd->bhst", *(OL._heads(q64, cfg, w) for w in range(2))) / np.sqrt(d)
    sc = np.where(np.triu(np.ones((s, s), dtype=bool), 1), -np.inf, sc)
    mx = sc.max(-1, keepdims=True)
    lse2 = (np.log(np.exp(sc - mx).sum(-1)) + mx[..., 0]) / np.log(2.0)
    dev = qkv.device
    return (torch.from_numpy(o).to(dev), torch.from_numpy(lse2.reshape(batch * heads, s)).to(dev),
            torch.from_numpy(dqkv).to(dev))


def reference(qkv, s, heads, batch, d, do):
    h = heads * d
    x = qkv.float().view(batch, s, 3, heads, d).permute(2, 0, 3, 1, 4)  # 3, b, H, s, d
    q, k, v = (t.clone().requires_grad_(True) for t in x)
    sc = (q @ k.transpose(-1, -2)) / math.sqrt(d)
    mask = torch.ones(s, s, dtype=torch.bool, device=qkv.device).tril()
    sc = sc.masked_fill(~mask, float("-inf"))
    lse2 = torch.logsumexp(sc, -1) / math.log(2.0)  # log2 domain
    p = torch.softmax(sc, -1)
    o = p @ v
    o.backward(do.float().view(batch, s, heads, d).permute(0, 2, 1, 3))
    o2 = o.permute(0, 2, 1, 3).reshape(batch * s, h)
    dqkv = torch.stack([q.grad, k.grad, v.grad]).permute(1, 3, 0, 2, 4).reshape(batch * s, 3 * h)
    return o2, lse2.reshape(batch * heads, s), dqkv


@pytest.mark.parametrize("s,heads,batch,d,scale", [
    (128, 2, 1, 128, 1.0), (256, 4, 1, 128, 1.0), (1024, 16, 1, 128, 1.0), (200, 3, 2, 128, 1.0),
    (300, 2, 1, 80, 1.0), (256, 2, 1, 80, 1.0), (384, 4, 2, 64, 1.0), (96, 2, 1, 32, 1.0),
    (2048, 16, 1, 128, 1.0), (2048, 32, 1, 80, 1.0),
    # large logits: the running max of the online softmax jumps by more than 2^8 (rescale path)
    (512, 2, 1, 128, 4.0), (1024, 4, 1, 128, 6.0), (300, 2, 1, 80, 5.0)])
def test_attention_fwd_bwd_vs_torch(s, heads, batch, d, scale):
    from paper_2405_14009_b200 import runtime as rt
    torch.manual_seed(s * 7 + heads + d)
    h = heads * d
    T = batch * s
    qkv = (torch.randn(T, 3 * h, device="cuda") * scale).to(torch.bfloat16)
    do = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    o = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(batch * heads, s, device="cuda")
    rt.attention(qkv, s, heads, batch, d, o, lse)
    dqkv = torch.empty(T, 3 * h, device="cuda", dtype=torch.bfloat16)
    dsum = torch.empty(batch * heads, s, device="cuda")
    rt.attention(qkv, s, heads, batch, d, dqkv, lse, o=o, d_o=do, dsum=dsum, backward=True)
    torch.cuda.synchronize()
    small = s * s * heads * batch <= (1 << 23)
    o_ref, lse_ref, dqkv_ref = (oracle_reference if small else reference)(qkv, s, heads, batch, d, do)
    bad = (~torch.isfinite(dqkv.float())).nonzero()
    assert torch.isfinite(o.float()).all() and bad.numel() == 0, (bad[:8].tolist(), bad[-8:].tolist())
    assert rel(o, o_ref) <= GATE
    assert (lse.double() - lse_ref.double()).abs().max().item() <= 1e-2
    for blk, name in enumerate(("dQ", "dK", "dV")):
        assert rel(dqkv[:, blk * h:(blk + 1) * h], dqkv_ref[:, blk * h:(blk + 1) * h]) <= GATE, name
    d_ref = (do.float() * o.float()).view(T, heads, d).sum(-1).view(batch, s, heads).permute(0, 2, 1)
    assert (dsum.view(batch, heads, s) - d_ref).abs().max().item() <= 1e-2 * d_ref.abs().max().item()
