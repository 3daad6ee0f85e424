"""GPU parity of the library's tcgen05 GEMM (tt_gemm: CTA pairs, TMEM accumulators; the building block
of NEXT-f3's LM head) against a plain fp64 matmul of the same bf16 operands:
every operand major combination the LM head uses (H W^T, G W, G^T H) plus the fourth, ragged M / N /
K (tile tails zero-filled by TMA and masked in the epilogue), strided operands, bf16 and fp32
outputs and fp32 accumulation.  Tolerance: fp32 accumulation of K products of bf16 values -> the
result differs from the fp64 sum by rounding only (max-abs <= 1e-5 of sum |a||b| per element for
fp32 out; bf16 out adds its own rounding, 2^-8 relative)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2511_00413_b200 as P
    P.lib()
    return P


def _ref(a, b, a_mn, b_mn):
    A = a.double().T if a_mn else a.double()
    B = b.double() if b_mn else b.double().T
    return A @ B, A.abs() @ B.abs()


CASES = [
    # M, N, K, a_mn, b_mn
    (256, 256, 64, 0, 0),
    (512, 768, 320, 0, 0),
    (300, 200, 104, 0, 0),       # ragged everywhere, K not a multiple of 64
    (1000, 4096 + 72, 256, 0, 0),
    (384, 256, 1000, 0, 1),      # dH shape: G (K-major) . W_c (MN-major)
    (520, 136, 777, 1, 1),       # dW shape: G^T (MN-major) . H (MN-major)
    (264, 392, 192, 1, 0),
    (64, 64, 64, 0, 0),          # smaller than one pair tile
    (2048, 2048, 1024, 0, 0),    # many tiles per pair (persistent loop, both accumulator buffers)
]


@pytest.mark.parametrize("M,N,K,a_mn,b_mn", CASES)
def test_gemm_fp32_out(tt, M, N, K, a_mn, b_mn):
    import torch
    g = torch.Generator().manual_seed(M * 7 + N + K)
    a = torch.randn(*((K, M) if a_mn else (M, K)), generator=g).to(torch.bfloat16)
    b = torch.randn(*((K, N) if b_mn else (N, K)), generator=g).to(torch.bfloat16)
    d = tt.tt_gemm(a.cuda(), b.cuda(), a_mn=a_mn, b_mn=b_mn)
    torch.cuda.synchronize()
    ref, mag = _ref(a, b, a_mn, b_mn)
    err = (d.cpu().double() - ref).abs()
    assert bool((err <= 1e-5 * mag + 1e-6).all()), float((err / (mag + 1e-30)).max())


def test_gemm_bf16_out_strided_and_accumulate(tt):
    import torch
    g = torch.Generator().manual_seed(5)
    M, N, K = 700, 520, 448
    a_big = torch.randn(M, K + 64, generator=g).to(torch.bfloat16)
    a = a_big[:, 32:32 + K]                       # row stride K + 64, 64-byte offset
    b = torch.randn(N, K, generator=g).to(torch.bfloat16)
    ref, mag = _ref(a, b, 0, 0)
    out = torch.full((M, N + 8), 7.0, dtype=torch.bfloat16, device="cuda")
    d = tt.tt_gemm(a.cuda(), b.cuda(), out=out[:, :N])
    torch.cuda.synchronize()
    err = (d.cpu().double() - ref).abs()
    assert bool((err <= 2.0 ** -8 * ref.abs() + 1e-5 * mag + 1e-6).all())
    assert bool((out[:, N:] == 7.0).all())        # columns beyond N untouched
    acc = torch.ones(M, N, dtype=torch.float32, device="cuda")
    tt.tt_gemm(a.cuda(), b.cuda(), out=acc, accumulate=True)
    tt.tt_gemm(a.cuda(), b.cuda(), out=acc, accumulate=True)
    torch.cuda.synchronize()
    err = (acc.cpu().double() - (2 * ref + 1)).abs()
    assert bool((err <= 2e-5 * mag + 1e-5).all())


def test_gemm_rejects_bad_arguments(tt):
    import torch
    a = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        tt.tt_gemm(a, torch.zeros(64, 32, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(tt.TTError):
        tt.tt_gemm(a, a, out=torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda"), accumulate=True)
