"""Per-op timing of one GPT-shaped stage on one B200 (CUDA events), and a short
fixed launch sequence for ncu captures.

    python tools/kernel_bench.py [--cfg c2|c3|c5] [--layers 1] [--reps 10] [--once | --phases]

--once runs F, B, W exactly once each after one warm-up (for `ncu -k regex:... -s/-c`).
Prints one JSON line: ms per op and TFLOP/s of the W GEMMs (4 per layer)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import slipdata as sd  # noqa: E402
from paper_2405_14009_b200 import runtime as rt  # noqa: E402

CFGS = {"c2": sd.C2_1P3B, "c3": sd.C3_2P7B, "c5": sd.C5_6P7B}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c2")
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--phases", action="store_true",
                    help="F, B, W, AdamW once each between marker kernels, inside cudaProfilerStart/Stop "
                         "(ncu --profile-from-start off; summarise with tools/ncu_summary.py phases)")
    ap.add_argument("--no-sk", action="store_true", help="disable stream-K for the F / B linears")
    ap.add_argument("--sk", action="store_true", help="enable (hybrid) stream-K for the F / B linears")
    ap.add_argument("--profile", action="store_true",
                    help="per-kernel live durations (torch.profiler / CUPTI, warm caches) of --reps steps")
    a = ap.parse_args()
    cfg = CFGS[a.cfg]
    L = a.layers
    st = rt.Stage(cfg, L, n_slots=1)
    if a.no_sk:
        rt.call("slip_set_stream_k", st.ctx, 0)
    if a.sk:
        rt.call("slip_set_stream_k", st.ctx, 1)
    rt.init_master_(st.master, cfg, L, cfg.layers)
    rt.call("slip_weights_from_master", st.ctx, rt._stream())
    T, h, f = cfg.tokens, cfg.hidden, cfg.ffn
    x = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    dy = (torch.randn(T, h, device="cuda") * 1e-3).to(torch.bfloat16)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)

    def step():
        st.forward(0, x, y)
        st.backward_input(0, dy, dx)
        st.backward_weight(0)

    step()
    torch.cuda.synchronize()
    if a.once:
        step()
        torch.cuda.synchronize()
        return
    if a.phases:
        # F, B, W and one AdamW step once each, separated by one torch fill kernel per
        # boundary so tools/ncu_summary.py phases can attribute every launch to its phase.
        st.optimizer_step(1)
        marker = torch.zeros(1, device="cuda")
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        marker.fill_(1.0)
        st.forward(0, x, y)
        marker.fill_(2.0)
        st.backward_input(0, dy, dx)
        marker.fill_(3.0)
        st.backward_weight(0)
        marker.fill_(4.0)
        st.optimizer_step(2)
        marker.fill_(5.0)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    if a.profile:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(a.reps):
                step()
            torch.cuda.synchronize()
        ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
        seq = []  # kernels of the last step in launch order
        per = len(ev) // a.reps
        for e in ev[-per:]:
            seq.append((e.name, e.device_time if hasattr(e, "device_time") else e.cuda_time))
        tot = {}
        for e in ev:
            d = e.device_time if hasattr(e, "device_time") else e.cuda_time
            k = e.name.split("(")[0][:60]
            tot[k] = tot.get(k, 0.0) + d
        import re
        for name, d in seq:
            short = re.sub(r"^void |slip::|\(anonymous namespace\)::|<unnamed>::", "", name).split("(")[0]
            print(f"{d:9.1f} us  {short[:90]}")
        print("total per step (us):", round(sum(tot.values()) / a.reps, 1))
        return
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tf = tb = tw = 0.0
    for _ in range(a.reps):
        ev[0].record()
        st.forward(0, x, y)
        ev[1].record()
        st.backward_input(0, dy, dx)
        ev[2].record()
        st.backward_weight(0)
        ev[3].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
        tb += ev[1].elapsed_time(ev[2])
        tw += ev[2].elapsed_time(ev[3])
    n = a.reps
    wflop = 2.0 * T * (4 * h * h + 2 * f * h) * L
    s, d = cfg.seq, cfg.head_dim
    fflop = wflop + 2.0 * cfg.micro_batch * cfg.heads * s * s * d * 2 / 2 * L
    print(json.dumps({"cfg": a.cfg, "layers": L, "F_ms": tf / n, "B_ms": tb / n, "W_ms": tw / n,
                      "W_tflops": wflop / (tw / n / 1e3) / 1e12,
                      "F_tflops": fflop / (tf / n / 1e3) / 1e12,
                      "B_tflops": (wflop + 2 * fflop - 2 * wflop) / (tb / n / 1e3) / 1e12}))


if __name__ == "__main__":
    main()
