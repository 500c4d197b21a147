"""Does a TMA store / reduce-add from a GEMM epilogue on cuda:0 reach memory on cuda:1
(peer access enabled)?  One process, two GPUs (diagnostic)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from cuda.bindings import runtime as cudart
    from paper_2405_14009_b200 import runtime as rt
    for d, o in ((0, 1), (1, 0)):
        torch.cuda.set_device(d)
        cudart.cudaDeviceEnablePeerAccess(o, 0)
    torch.cuda.set_device(0)
    M, N, K = 512, 512, 256
    g = torch.Generator(device="cuda:0").manual_seed(0)
    a = torch.randn(K, M, generator=g, device="cuda:0").to(torch.bfloat16)  # MN-major A: [K][M]
    b = torch.randn(K, N, generator=g, device="cuda:0").to(torch.bfloat16)
    ref = a.float().t() @ b.float()
    for mode, name in ((3, "store"), (4, "reduce-add")):
        c1 = torch.zeros(M, N, device="cuda:1")
        if mode == 4:
            c1.fill_(1.0)
        rt.gemm(a, b, c1, M, N, K, M, N, N, a_mn=True, b_mn=True, mode=mode, bn=256, accumulate=(mode == 4))
        torch.cuda.synchronize(0)
        got = c1.cpu() - (1.0 if mode == 4 else 0.0)
        err = ((got - ref.cpu()).abs().max() / ref.abs().max()).item()
        print(f"TMA {name} to peer memory: relerr {err:.3e}", flush=True)


if __name__ == "__main__":
    main()
