"""tcgen05 GEMM engine vs a plain fp32 torch reference (same bf16-rounded
operands), every operand-major combination, tile width, split-K and epilogue
the model uses."""
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2006_11751_b200 as appo  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return appo.Context(0)


def operands(M, N, K, a_mn, b_mn, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    a_store = A.t().contiguous() if a_mn else A  # MN-major: [K][M]
    b_store = B.t().contiguous() if b_mn else B
    lda = M if a_mn else K
    ldb = N if b_mn else K
    return A, B, a_store, lda, b_store, ldb


def ref(A, B):
    return A.float() @ B.float().t()


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("bn", [64, 128, 192, 256])
def test_majors_and_tiles(ctx, a_mn, b_mn, bn):
    M, N, K = 296, 2 * bn + 64 if bn < 256 else 320, 384
    A, B, a, lda, b, ldb = operands(M, N, K, a_mn, b_mn)
    out = torch.zeros(M, N, device="cuda")
    ctx.gemm(M, N, K, a, lda, a_mn, b, ldb, b_mn, out, N, bn=bn)
    torch.cuda.synchronize()
    r = ref(A, B)
    assert (out - r).abs().max().item() <= 1e-3 * r.abs().max().item()


def test_bn32_kmajor(ctx):
    M, N, K = 1000, 32, 192
    A, B, a, lda, b, ldb = operands(M, N, K, False, False, 1)
    out = torch.zeros(M, N, device="cuda")
    ctx.gemm(M, N, K, a, lda, False, b, ldb, False, out, N, bn=32)
    torch.cuda.synchronize()
    r = ref(A, B)
    assert (out - r).abs().max().item() <= 1e-3 * r.abs().max().item()


@pytest.mark.parametrize("splits", [2, 7])
def test_split_k_and_small_m(ctx, splits):
    # weight-gradient shape: M = 32 (OOB-filled MN-major A), huge K
    M, N, K = 32, 192, 64 * 50
    A, B, a, lda, b, ldb = operands(M, N, K, True, True, 2)
    out = torch.zeros(M, N, device="cuda")
    ctx.gemm(M, N, K, a, lda, True, b, ldb, True, out, N, bn=192, splits=splits)
    torch.cuda.synchronize()
    r = ref(A, B)
    assert (out - r).abs().max().item() <= 1e-3 * r.abs().max().item()


def test_epilogues(ctx):
    M, N, K = 257, 128, 576
    A, B, a, lda, b, ldb = operands(M, N, K, False, False, 3)
    bias = torch.randn(N, device="cuda")
    r = ref(A, B)
    # scale + bias + ELU -> bf16
    out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    ctx.gemm(M, N, K, a, lda, False, b, ldb, False, out, N,
             flags=appo.EPI_BIAS | appo.EPI_ELU | appo.EPI_BF16, scale=0.5, bias=bias, bn=128)
    exp = torch.nn.functional.elu(r * 0.5 + bias)
    torch.cuda.synchronize()
    assert (out.float() - exp).abs().max().item() <= 1e-2 * exp.abs().max().item()
    # ELU' by aux
    aux = torch.nn.functional.elu(torch.randn(M, N, device="cuda")).bfloat16()
    out2 = torch.zeros(M, N, device="cuda")
    ctx.gemm(M, N, K, a, lda, False, b, ldb, False, out2, N, flags=appo.EPI_DELU, aux=aux,
             ld_aux=N, bn=128)
    a32 = aux.float()
    exp2 = r * torch.where(a32 > 0, torch.ones_like(a32), a32 + 1)
    torch.cuda.synchronize()
    assert (out2 - exp2).abs().max().item() <= 1e-3 * exp2.abs().max().item()
    # accumulate + transposed store
    out3 = torch.ones(N, M, device="cuda")
    ctx.gemm(M, N, K, a, lda, False, b, ldb, False, out3, M,
             flags=appo.EPI_ACCUM | appo.EPI_TRANS, bn=128)
    torch.cuda.synchronize()
    assert (out3 - (r.t() + 1)).abs().max().item() <= 1e-3 * r.abs().max().item()


def test_strided_rows(ctx):
    # the BPTT GEMM reads every T-th row of a [B][1536] buffer (lda = T*1536)
    T, n, K, N = 8, 64, 1536, 512
    big = torch.randn(n * T, K, device="cuda").bfloat16()
    W = torch.randn(K, N, device="cuda").bfloat16()  # [K][N] -> MN-major B
    t = 3
    a = big[t::T]
    out = torch.zeros(n, N, device="cuda")
    ctx.gemm(n, N, K, big[t:], T * K, False, W, N, True, out, N, bn=64, splits=4)
    torch.cuda.synchronize()
    r = a.float() @ W.float()
    assert (out - r).abs().max().item() <= 1e-3 * r.abs().max().item()


@pytest.mark.parametrize("bn,flags", [(64, 0), (128, appo.EPI_BIAS | appo.EPI_ELU | appo.EPI_BF16),
                                      (256, appo.EPI_BIAS)])
def test_many_tiles_per_cta(ctx, bn, flags):
    # production-size M (the inference FC / gate GEMMs run M = 16,384; conv GEMMs
    # millions of rows): every persistent CTA cycles its smem ring's mbarrier
    # phases and the double-buffered TMEM accumulator over dozens of tiles
    M, N, K = 148 * 128 * 6 + 77, bn * 2, 512
    A, B, a, lda, b, ldb = operands(M, N, K, False, False, 11)
    bias = torch.randn(N, device="cuda")
    dt = torch.bfloat16 if flags & appo.EPI_BF16 else torch.float32
    out = torch.zeros(M, N, device="cuda", dtype=dt)
    ctx.gemm(M, N, K, a, lda, False, b, ldb, False, out, N, flags=flags, bias=bias, bn=bn)
    torch.cuda.synchronize()
    r = ref(A, B)
    if flags & appo.EPI_BIAS:
        r = r + bias
    if flags & appo.EPI_ELU:
        r = torch.nn.functional.elu(r)
    tol = (1e-2 if dt == torch.bfloat16 else 1e-3) * r.abs().max().item()
    assert (out.float() - r).abs().max().item() <= tol
