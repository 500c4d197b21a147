"""Kernel-level parity of the fused causal attention (slip_attention) against a plain
PyTorch fp32 reference of the same operation on the same bf16 inputs: O, the log2-domain
LSE, and dQ / dK / dV — at sizes that span several tiles, ragged tails (s % 128 != 0,
s % 64 != 0), every supported head dim, batch > 1, and the full GPT-1.3B shape."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

GATE = 2e-2  # normwise, bf16 operands / fp32 accumulation (SURVEY §8(c) Gate A)


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


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
    o_ref, lse_ref, dqkv_ref = reference(qkv, s, heads, batch, d, do)
    bad = (~torch.isfinite(dqkv.float())).nonzero()
    assert torch.isfinite(o.float()).all() and bad.numel() == 0, (bad[:8].tolist(), bad[-8:].tolist())
    assert rel(o, o_ref) <= GATE
    assert (lse - lse_ref).abs().max().item() <= 1e-2
    for blk, name in enumerate(("dQ", "dK", "dV")):
        assert rel(dqkv[:, blk * h:(blk + 1) * h], dqkv_ref[:, blk * h:(blk + 1) * h]) <= GATE, name
    d_ref = (do.float() * o.float()).view(T, heads, d).sum(-1).view(batch, s, heads).permute(0, 2, 1)
    assert (dsum.view(batch, heads, s) - d_ref).abs().max().item() <= 1e-2 * d_ref.abs().max().item()
