"""Out-of-bounds access checks without compute-sanitizer (the GPU pool disables it: runs
under it have left GPUs needing a reset).  Every buffer the library touches — bf16 weights,
fp32 master / grad / m / v, the stash arena, the workspace, the stage input / output and
the gradients in / out — is allocated inside a larger tensor whose guard bands (64 KB on
each side) hold a NaN bit pattern.  On ragged shapes (partial GEMM tiles, s % 128 != 0,
s % 64 != 0, b > 1, d = 80) a full F, B, merged W and AdamW step must

  * leave every guard band bit-identical (no write outside any buffer), and
  * produce finite results equal to the oracle (a read of a guard band would inject NaN),

and the GEMM family (every epilogue mode, pair and single-CTA tiles) likewise on operands
and outputs with NaN guards."""
import ctypes as C

import numpy as np
import pytest
import torch

import slipdata as sd
from oracle import layer as OL

pytestmark = pytest.mark.gpu

GUARD = 64 * 1024  # bytes on each side
PAT32 = 0x7FC17FC1  # an fp32 NaN whose two halves are bf16 NaNs


def _rt():
    from paper_2405_14009_b200 import runtime
    return runtime


class Guarded:
    """`nbytes` usable bytes at a 256-byte aligned offset inside a NaN-guarded allocation."""

    def __init__(self, nbytes, dtype):
        self.nbytes = int(nbytes)
        words = (GUARD * 2 + self.nbytes + 3) // 4 + 64
        self.raw = torch.full((words,), PAT32, dtype=torch.int32, device="cuda")
        self.off = GUARD // 4
        esz = torch.tensor([], dtype=dtype).element_size()
        n = self.nbytes // esz
        self.t = self.raw[self.off:self.off + (self.nbytes + 3) // 4].view(dtype)[:n]
        self.guard_lo = self.raw[:self.off].clone()
        end = self.off + (self.nbytes + 3) // 4
        self.end = end
        self.guard_hi = self.raw[end:].clone()

    def ptr(self):
        return C.c_void_p(self.t.data_ptr())

    def intact(self):
        return bool(torch.equal(self.raw[:self.off], self.guard_lo)) and bool(
            torch.equal(self.raw[self.end:], self.guard_hi))


def dev_bf16_into(buf, x):
    bits = torch.from_numpy(sd.to_bf16_bits(x).view(np.int16).copy()).view(torch.bfloat16)
    buf.t.copy_(bits.reshape(-1).cuda())


CFGS = {
    "d80_ragged": (sd.ModelCfg(hidden=640, heads=8, ffn=2560, seq=200, micro_batch=1, layers=2), 2),
    "d64_b2": (sd.ModelCfg(hidden=256, heads=4, ffn=1024, seq=136, micro_batch=2, layers=1), 1),
    "c1": (sd.C1_TINY, 1),
}


@pytest.mark.parametrize("name", list(CFGS))
def test_stage_step_stays_in_bounds(name):
    rt = _rt()
    from paper_2405_14009_b200._binding import slip_adam
    cfg, L = CFGS[name]
    model = rt.make_model(cfg)
    npar, sb, wb = C.c_int64(0), C.c_size_t(0), C.c_size_t(0)
    n_slots = 3
    rt.call("slip_param_count", C.byref(model), L, C.byref(npar))
    rt.call("slip_stash_bytes", C.byref(model), L, n_slots, C.byref(sb))
    rt.call("slip_workspace_bytes", C.byref(model), C.byref(wb))
    P = npar.value
    w = Guarded(2 * P, torch.bfloat16)
    bufs32 = {n: Guarded(4 * P, torch.float32) for n in ("master", "grad", "m", "v")}
    arena = Guarded(sb.value, torch.uint8)
    ws = Guarded(wb.value, torch.uint8)
    for n in ("grad", "m", "v"):
        bufs32[n].t.zero_()
    layers = sd.stage_params(cfg, 0, L, total_layers=max(L, 2))
    bufs32["master"].t.copy_(torch.from_numpy(sd.pack_stage(layers)).float())
    ctx = C.c_void_p()
    rt.call("slip_ctx_create", C.byref(ctx), C.byref(model), L, n_slots)
    rt.call("slip_stage_bind", ctx, w.ptr(), bufs32["master"].ptr(), bufs32["grad"].ptr(), bufs32["m"].ptr(),
            bufs32["v"].ptr(), P, arena.ptr(), sb.value, ws.ptr(), wb.value)
    s = rt._stream()
    rt.call("slip_weights_from_master", ctx, s)
    T, h = cfg.tokens, cfg.hidden
    io = {n: Guarded(2 * T * h, torch.bfloat16) for n in ("x0", "x1", "y", "r0", "r1", "dx")}
    dev_bf16_into(io["x0"], sd.stage_input(cfg, 0, 0))
    dev_bf16_into(io["x1"], sd.stage_input(cfg, 0, 1))
    dev_bf16_into(io["r0"], sd.stage_target(cfg, 0, 0))
    dev_bf16_into(io["r1"], sd.stage_target(cfg, 0, 1))
    for j, slot in enumerate((2, 0)):
        rt.call("slip_stage_forward", ctx, slot, io[f"x{j}"].ptr(), io["y"].ptr(), s)
        rt.call("slip_backward_input", ctx, slot, io[f"r{j}"].ptr(), io["dx"].ptr(), int(j > 0), s)
    arr = (C.c_int32 * 2)(2, 0)
    rt.call("slip_backward_weight_multi", ctx, C.cast(arr, C.c_void_p), 2, 0, s)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    a = slip_adam(1e-3, 0.9, 0.95, 1e-8, 0.1)
    rt.call("slip_optimizer_step", ctx, C.byref(a), 1, 0.5, C.c_void_p(flag.data_ptr()), s)
    torch.cuda.synchronize()
    lib = rt.lib()
    lib.slip_ctx_destroy(ctx)
    for n, g in [("w", w), ("arena", arena), ("ws", ws)] + list(bufs32.items()) + list(io.items()):
        assert g.intact(), f"write outside {n}"
    assert int(flag.item()) == 0
    assert torch.isfinite(bufs32["grad"].t).all() and torch.isfinite(bufs32["master"].t).all()
    # the summed gradient of the two micro-batches equals the oracle's (no guard NaN was read)
    ref = None
    for j in range(2):
        out, c = OL.stage_forward(layers, sd.stage_input(cfg, 0, j), cfg)
        _, g = OL.stage_backward_coupled(layers, c, sd.stage_target(cfg, 0, j), cfg)
        ref = g if ref is None else [{n: x[n] + y[n] for n in x} for x, y in zip(ref, g)]
    got = sd.unpack_stage(bufs32["grad"].t.cpu().numpy().astype(np.float64), cfg, L)
    for l in range(L):
        for n in sd.PARAM_ORDER:
            e = float(np.max(np.abs(got[l][n] - ref[l][n])) / np.max(np.abs(ref[l][n])))
            assert e <= 2e-2, (name, l, n, e)


GEMM_CASES = [
    # M, N, K, a_mn, b_mn, bn, mode
    (200, 72, 136, False, False, 256, 0),
    (130, 104, 200, False, True, 256, 0),
    (136, 200, 72, True, True, 256, 3),
    (136, 200, 72, True, True, 256, 4),
    (256, 80, 320, True, True, 80, 4),
    (96, 32, 64, True, True, 32, 3),
    (520, 776, 264, False, False, 256, 0),
]


@pytest.mark.parametrize("M,N,K,a_mn,b_mn,bn,mode", GEMM_CASES)
def test_gemm_stays_in_bounds(M, N, K, a_mn, b_mn, bn, mode):
    rt = _rt()
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = Guarded(2 * M * K, torch.bfloat16)
    B = Guarded(2 * N * K, torch.bfloat16)
    A.t.copy_(torch.randn(M * K, generator=g, device="cuda").to(torch.bfloat16))
    B.t.copy_(torch.randn(N * K, generator=g, device="cuda").to(torch.bfloat16))
    f32 = mode >= 3
    Cb = Guarded((4 if f32 else 2) * M * N, torch.float32 if f32 else torch.bfloat16)
    Cb.t.zero_()
    a2 = A.t.view(K, M) if a_mn else A.t.view(M, K)
    b2 = B.t.view(K, N) if b_mn else B.t.view(N, K)
    lda = M if a_mn else K
    ldb = N if b_mn else K
    rt.gemm(A.t, B.t, Cb.t, M, N, K, lda, ldb, N, a_mn=a_mn, b_mn=b_mn, mode=mode, bn=bn)
    if mode == 4:  # accumulate a second time on top
        rt.gemm(A.t, B.t, Cb.t, M, N, K, lda, ldb, N, a_mn=a_mn, b_mn=b_mn, mode=mode, bn=bn, accumulate=True)
    torch.cuda.synchronize()
    assert A.intact() and B.intact() and Cb.intact()
    Am = a2.t().float() if a_mn else a2.float()
    Bm = b2.float() if b_mn else b2.t().float()
    ref = Am @ Bm * (2.0 if mode == 4 else 1.0)
    got = Cb.t.float().view(M, N)
    assert torch.isfinite(got).all()
    assert ((got - ref).abs().max() / ref.abs().max()).item() <= 2e-2
