"""Context for the attention kernels' roofline: time PyTorch's own fused causal attention
(scaled_dot_product_attention; cuDNN / flash backends as PyTorch picks them on B200) on the
shape of one GPT layer's attention, forward and forward+backward, with CUDA events.

    python tools/attn_reference_timing.py [--heads 16] [--seq 2048] [--d 128]

Not on the product path: a library comparison point only."""
import argparse
import json

import torch
import torch.nn.functional as F


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    q, k, v = (torch.randn(1, a.heads, a.seq, a.d, device="cuda", dtype=torch.bfloat16, requires_grad=True)
               for _ in range(3))
    do = torch.randn(1, a.heads, a.seq, a.d, device="cuda", dtype=torch.bfloat16)
    out = {}
    for name, backends in (("default", None),
                           ("cudnn", [torch.nn.attention.SDPBackend.CUDNN_ATTENTION]),
                           ("flash", [torch.nn.attention.SDPBackend.FLASH_ATTENTION])):
        try:
            ctx = torch.nn.attention.sdpa_kernel(backends) if backends else torch.enable_grad()
            with ctx:
                for _ in range(3):
                    o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                    o.backward(do)
                torch.cuda.synchronize()
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                tf = tfb = 0.0
                for _ in range(a.reps):
                    e[0].record()
                    o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                    e[1].record()
                    o.backward(do)
                    e[2].record()
                    torch.cuda.synchronize()
                    tf += e[0].elapsed_time(e[1])
                    tfb += e[0].elapsed_time(e[2])
            flops_f = 4.0 * a.heads * a.seq * a.seq * a.d / 2
            out[name] = {"fwd_us": 1e3 * tf / a.reps, "fwd_bwd_us": 1e3 * tfb / a.reps,
                         "fwd_tflops": flops_f / (tf / a.reps / 1e3) / 1e12,
                         "fwd_bwd_tflops": 3.5 * flops_f / (tfb / a.reps / 1e3) / 1e12}
        except Exception as ex:  # backend unavailable for this shape
            out[name] = {"error": str(ex)[:200]}
    print(json.dumps({"shape": vars(a), **out}))


if __name__ == "__main__":
    main()
