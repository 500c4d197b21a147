import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import slipdata as sd
from paper_2405_14009_b200 import runtime as rt
for cfg in [sd.ModelCfg(hidden=2048, heads=16, ffn=8192, seq=2048, micro_batch=1, layers=24),
            sd.ModelCfg(hidden=512, heads=4, ffn=2048, seq=1024, micro_batch=1, layers=24),
            sd.ModelCfg(hidden=512, heads=4, ffn=2048, seq=2048, micro_batch=1, layers=24),
            sd.ModelCfg(hidden=2048, heads=16, ffn=8192, seq=1024, micro_batch=1, layers=24)]:
    st = rt.Stage(cfg, 1, n_slots=1)
    rt.init_master_(st.master, cfg, 1, cfg.layers)
    rt.call("slip_weights_from_master", st.ctx, rt._stream())
    T, h = cfg.tokens, cfg.hidden
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(T, h, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(T, h, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    y = torch.empty_like(x); dx = torch.empty_like(x)
    st.forward(0, x, y); st.backward_input(0, dy, dx); torch.cuda.synchronize()
    bad = torch.isnan(dx.float()).any(1).nonzero().flatten().tolist()
    print(cfg.hidden, cfg.seq, "y nan", torch.isnan(y.float()).sum().item(), "dx nan rows", len(bad), bad[:20], bad[-5:] if bad else None, flush=True)
    st.close()
