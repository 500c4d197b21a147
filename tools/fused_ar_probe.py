"""The fused DP = 2 all-reduce + AdamW kernel (slip_optimizer_step_peer, the compute half of
slip_comm_fuse_ar_adam; SURVEY §8(e) option (i)) in ONE process driving two GPUs, so that
ncu can wrap it (ncu may not wrap a multi-rank command on this pool):

    python tools/fused_ar_probe.py [--model 1.3b] [--layers 24] [--iters 10] [--both]
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
nvlrx__bytes.sum,nvltx__bytes.sum --devices 0 -k regex:adamw python tools/fused_ar_probe.py --iters 2

The stage (GPT shape, `layers` layers: its fp32 master / grad / m / v) lives on cuda:0, the
peer's fp32 gradient on cuda:1 with peer access enabled; each call reads g_own + g_peer
(4 B per parameter over NVLink) and streams the local state (30 B per parameter of HBM).
Prints one JSON line: the kernel time (CUDA events, cuda:0), the NVLink and HBM bytes per
call, and the roofline of a fused compute + collective kernel (B200_PROFILING.md: the
slower of the HBM time at the measured copy bandwidth and the NVLink time at the measured
770 GB/s peer copy)."""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NVLINK_GBPS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="1.3b")
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--both", action="store_true",
                    help="the DP = 2 situation: a stage on each GPU, each reading the other's gradient, concurrently")
    a = ap.parse_args()
    if torch.cuda.device_count() < 2:
        print(json.dumps({"skipped": "needs 2 GPUs"}))
        return
    from cuda.bindings import runtime as cudart
    import slipdata as sd
    from paper_2405_14009_b200 import runtime as rt
    from paper_2405_14009_b200._binding import slip_adam

    for d, o in ((0, 1), (1, 0)):
        torch.cuda.set_device(d)
        err = cudart.cudaDeviceEnablePeerAccess(o, 0)[0]
        if err not in (cudart.cudaError_t.cudaSuccess, cudart.cudaError_t.cudaErrorPeerAccessAlreadyEnabled):
            raise SystemExit(f"cudaDeviceEnablePeerAccess({d} -> {o}): {err}")
    cfg = {"1.3b": sd.C2_1P3B, "2.7b": sd.C3_2P7B, "6.7b": sd.C5_6P7B}[a.model]
    devs = (0, 1) if a.both else (0,)
    st, flag, strm = {}, {}, {}
    for d in devs:
        torch.cuda.set_device(d)
        st[d] = rt.Stage(cfg, a.layers, n_slots=1, device=f"cuda:{d}")
        n = st[d].master.numel()
        g = torch.Generator(device=f"cuda:{d}").manual_seed(1 + d)
        st[d].master.copy_(torch.randn(n, generator=g, device=f"cuda:{d}") * 0.02)
        st[d].grad.copy_(torch.randn(n, generator=g, device=f"cuda:{d}") * 1e-3)
        flag[d] = torch.zeros(1, dtype=torch.int32, device=f"cuda:{d}")
        strm[d] = torch.cuda.current_stream(d)
    if a.both:
        peer = {0: st[1].grad, 1: st[0].grad}
    else:
        peer = {0: torch.randn(n, generator=torch.Generator(device="cuda:1").manual_seed(2), device="cuda:1") * 1e-3}
    for d in (0, 1):
        torch.cuda.synchronize(d)
    adam = slip_adam(1e-4, 0.9, 0.95, 1e-8, 0.1)

    def step(d, k):
        torch.cuda.set_device(d)
        rt.call("slip_optimizer_step_peer", st[d].ctx, C.byref(adam), k, 1.0, C.c_void_p(flag[d].data_ptr()),
                C.c_void_p(peer[d].data_ptr()), rt._stream(strm[d]))

    for d in devs:
        step(d, 1)
    for d in (0, 1):
        torch.cuda.synchronize(d)
    ev = {}
    for d in devs:
        torch.cuda.set_device(d)
        ev[d] = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[d][0].record(strm[d])
    for k in range(a.iters):
        for d in devs:
            step(d, 2 + k)
    for d in devs:
        torch.cuda.set_device(d)
        ev[d][1].record(strm[d])
    for d in (0, 1):
        torch.cuda.synchronize(d)
    ms = max(ev[d][0].elapsed_time(ev[d][1]) for d in devs) / a.iters
    torch.cuda.set_device(0)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    nvl_bytes = 4.0 * n
    # read p, m, v, g (16 B), write p, m, v (12 B) + w bf16 (2 B); + the peer's 4 B reads of
    # this GPU's gradient when both directions run
    hbm_bytes = (34.0 if a.both else 30.0) * n
    t_nvl = nvl_bytes / (NVLINK_GBPS * 1e9) * 1e3
    t_hbm = hbm_bytes / (peaks["hbm_gbs"] * 1e9) * 1e3
    bound = max(t_nvl, t_hbm)
    print(json.dumps({
        "kernel": "adamw_kernel with g_peer (slip_optimizer_step_peer), 1 process, cuda:0 reading cuda:1",
        "both_directions": a.both, "model": a.model, "layers": a.layers, "params": n, "ms": ms,
        "nvlink_bytes_per_call": nvl_bytes, "hbm_bytes_per_call": hbm_bytes,
        "nvlink_GBps_achieved": nvl_bytes / ms / 1e6, "hbm_GBps_achieved": hbm_bytes / ms / 1e6,
        "roofline": {"bound": "nvlink" if t_nvl >= t_hbm else "hbm", "target_ms": bound,
                     "nvlink_ms_at_770": t_nvl, "hbm_ms_at_measured": t_hbm, "frac": bound / ms},
        "nonfinite": sum(int(f.item()) for f in flag.values())}))


if __name__ == "__main__":
    main()
