"""Kernel-level parity of the tcgen05 GEMM family (slip_gemm diagnostic entry)
against a plain fp32 PyTorch product of the same bf16 operands."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rt():
    from paper_2405_14009_b200 import runtime
    return runtime


def relerr(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-30)).item()


CASES = [
    # M, N, K, a_mn, b_mn, bn
    (128, 256, 64, False, False, 256),
    (256, 512, 1024, False, False, 256),
    (200, 72, 136, False, False, 256),
    (384, 256, 512, False, True, 256),
    (130, 104, 200, False, True, 256),
    (512, 768, 2048, True, True, 256),
    (136, 200, 72, True, True, 256),
    (256, 256, 128, False, False, 128),
    (256, 80, 256, False, True, 80),
    (256, 80, 320, True, True, 80),
    (64, 32, 32, False, True, 32),
    (96, 32, 64, True, True, 32),
    (1024, 1536, 2048, False, False, 128),
]


def _operands(M, N, K, a_mn, b_mn, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn((K, M) if a_mn else (M, K), generator=g, device="cuda").to(torch.bfloat16)
    b = torch.randn((K, N) if b_mn else (N, K), generator=g, device="cuda").to(torch.bfloat16)
    A = a.t() if a_mn else a
    B = b if b_mn else b.t()
    lda = M if a_mn else K
    ldb = N if b_mn else K
    return a, b, A, B, lda, ldb


@pytest.mark.parametrize("M,N,K,a_mn,b_mn,bn", CASES)
def test_gemm_bf16_out(M, N, K, a_mn, b_mn, bn):
    rt = _rt()
    a, b, A, B, lda, ldb = _operands(M, N, K, a_mn, b_mn)
    c = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    rt.gemm(a, b, c, M, N, K, lda, ldb, N, a_mn=a_mn, b_mn=b_mn, mode=0, bn=bn, alpha=0.5)
    torch.cuda.synchronize()
    ref = 0.5 * (A.float() @ B.float())
    assert relerr(c, ref) <= 1e-2


@pytest.mark.parametrize("M,N,K,a_mn,b_mn,bn", CASES)
def test_gemm_f32_store_and_accumulate(M, N, K, a_mn, b_mn, bn):
    rt = _rt()
    a, b, A, B, lda, ldb = _operands(M, N, K, a_mn, b_mn, seed=1)
    ref = A.float() @ B.float()
    c = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    rt.gemm(a, b, c, M, N, K, lda, ldb, N, a_mn=a_mn, b_mn=b_mn, mode=4, bn=bn, accumulate=False)
    torch.cuda.synchronize()
    assert relerr(c, ref) <= 1e-5
    base = torch.randn(M, N, device="cuda")
    c2 = base.clone()
    rt.gemm(a, b, c2, M, N, K, lda, ldb, N, a_mn=a_mn, b_mn=b_mn, mode=4, bn=bn, accumulate=True)
    torch.cuda.synchronize()
    assert relerr(c2, base + ref) <= 1e-5
