import sys, os, math, torch
sys.path.insert(0, os.getcwd())
from paper_2405_14009_b200 import runtime as rt
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_gpu_attention import reference
for it in range(6):
    for (s, heads, batch, d) in [(300, 2, 1, 80), (200, 3, 2, 128), (256, 2, 1, 128)]:
        torch.manual_seed(it)
        h = heads * d; T = batch * s
        qkv = torch.randn(T, 3 * h, device="cuda").to(torch.bfloat16)
        do = torch.randn(T, h, device="cuda").to(torch.bfloat16)
        o = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(batch * heads, s, device="cuda")
        rt.attention(qkv, s, heads, batch, d, o, lse)
        dqkv = torch.zeros(T, 3 * h, device="cuda", dtype=torch.bfloat16)
        dsum = torch.empty(batch * heads, s, device="cuda")
        rt.attention(qkv, s, heads, batch, d, dqkv, lse, o=o, d_o=do, dsum=dsum, backward=True)
        torch.cuda.synchronize()
        o_ref, lse_ref, dref = reference(qkv, s, heads, batch, d, do)
        dq = dqkv[:, :h].float(); dqr = dref[:, :h]
        out = []
        for b in range(batch):
            for t in range(0, s, 64):
                rows = slice(b * s + t, b * s + min(s, t + 64))
                e = dq[rows] - dqr[rows]
                fin = torch.isfinite(e)
                out.append("%d:%d nan=%d err=%.3g" % (b, t, (~fin).sum().item(), (e[fin].norm() / dqr[rows].norm()).item()))
        print(it, s, d, " | ".join(out), flush=True)
