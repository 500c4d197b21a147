import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2405_14009_b200 import runtime as rt
for it in range(20):
    for (s, heads, batch, d) in [(200, 3, 2, 128), (300, 2, 1, 80)]:
        torch.manual_seed(it)
        h = heads * d; T = batch * s
        qkv = torch.randn(T, 3 * h, device="cuda").to(torch.bfloat16)
        do = torch.randn(T, h, device="cuda").to(torch.bfloat16)
        o = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(batch * heads, s, device="cuda")
        rt.attention(qkv, s, heads, batch, d, o, lse)
        dqkv = torch.empty(T, 3 * h, device="cuda", dtype=torch.bfloat16)
        dsum = torch.empty(batch * heads, s, device="cuda")
        rt.attention(qkv, s, heads, batch, d, dqkv, lse, o=o, d_o=do, dsum=dsum, backward=True)
        torch.cuda.synchronize()
        bad = (~torch.isfinite(dqkv.float())).nonzero()
        if bad.numel():
            print(it, s, "bad", bad.shape[0], "blocks", sorted(set((bad[:,1] // h).tolist())), "rows", sorted(set(bad[:,0].tolist()))[:10], "lse finite", torch.isfinite(lse).all().item(), flush=True)
