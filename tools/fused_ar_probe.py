"""The fused DP = 2 all-reduce + AdamW kernel (slip_optimizer_step_peer, the compute half of
slip_comm_fuse_ar_adam; SURVEY §8(e) option (i)) in ONE process driving two GPUs, so that
ncu can wrap it (ncu may not wrap a multi-rank command on this pool):

    python tools/fused_ar_probe.py [--model 1.3b] [--layers 24] [--iters 10]
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
    a = ap.parse_args()
    if torch.cuda.device_count() < 2:
        print(json.dumps({"skipped": "needs 2 GPUs"}))
        return
    from cuda.bindings import runtime as cudart
    import slipdata as sd
    from paper_2405_14009_b200 import runtime as rt
    from paper_2405_14009_b200._binding import slip_adam

    torch.cuda.set_device(0)
    err = cudart.cudaDeviceEnablePeerAccess(1, 0)[0]
    if err not in (cudart.cudaError_t.cudaSuccess, cudart.cudaError_t.cudaErrorPeerAccessAlreadyEnabled):
        raise SystemExit(f"cudaDeviceEnablePeerAccess: {err}")
    cfg = {"1.3b": sd.C2_1P3B, "2.7b": sd.C3_2P7B, "6.7b": sd.C5_6P7B}[a.model]
    st = rt.Stage(cfg, a.layers, n_slots=1)
    n = st.master.numel()
    g = torch.Generator(device="cuda:0").manual_seed(1)
    st.master.copy_(torch.randn(n, generator=g, device="cuda:0") * 0.02)
    st.grad.copy_(torch.randn(n, generator=g, device="cuda:0") * 1e-3)
    peer = (torch.randn(n, generator=torch.Generator(device="cuda:1").manual_seed(2), device="cuda:1") * 1e-3)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    adam = slip_adam(1e-4, 0.9, 0.95, 1e-8, 0.1)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    s = torch.cuda.current_stream(0)
    sp = rt._stream(s)

    def step(k):
        rt.call("slip_optimizer_step_peer", st.ctx, C.byref(adam), k, 1.0, C.c_void_p(flag.data_ptr()),
                C.c_void_p(peer.data_ptr()), sp)

    step(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for k in range(a.iters):
        step(2 + k)
    e1.record(s)
    torch.cuda.synchronize(0)
    ms = e0.elapsed_time(e1) / a.iters
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    nvl_bytes = 4.0 * n
    hbm_bytes = 30.0 * n  # read p, m, v, g (16 B), write p, m, v (12 B) + w bf16 (2 B)
    t_nvl = nvl_bytes / (NVLINK_GBPS * 1e9) * 1e3
    t_hbm = hbm_bytes / (peaks["hbm_gbs"] * 1e9) * 1e3
    bound = max(t_nvl, t_hbm)
    print(json.dumps({
        "kernel": "adamw_kernel with g_peer (slip_optimizer_step_peer), 1 process, cuda:0 reading cuda:1",
        "model": a.model, "layers": a.layers, "params": n, "ms": ms,
        "nvlink_bytes_per_call": nvl_bytes, "hbm_bytes_per_call": hbm_bytes,
        "nvlink_GBps_achieved": nvl_bytes / ms / 1e6, "hbm_GBps_achieved": hbm_bytes / ms / 1e6,
        "roofline": {"bound": "nvlink" if t_nvl >= t_hbm else "hbm", "target_ms": bound,
                     "nvlink_ms_at_770": t_nvl, "hbm_ms_at_measured": t_hbm, "frac": bound / ms},
        "nonfinite": int(flag.item())}))


if __name__ == "__main__":
    main()
