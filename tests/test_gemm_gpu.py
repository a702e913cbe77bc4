"""GPU parity: int8 tcgen05 GEMM (raw accumulators bit-exact, exact fp64 epilogue bit-exact,
bf16 epilogue within tolerance), bf16 MN-major dW GEMM, exact sequential matmul, fp8 GEMM."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2304_13013_b200 import lowprec as L
from paper_2304_13013_b200 import _capi as A
from tests._util import bf16, dev, fp8_decode, host, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[A.SB_GEMM_1CTA, A.SB_GEMM_2CTA, A.SB_GEMM_WIDE, A.SB_GEMM_2CTA_MC],
                ids=["1cta", "2cta", "wide", "2cta_mc"])
def gemm_path(request):
    """Run the test on every tensor-core tiling (1-CTA 128x256, cta_group::2 256x256, the
    transposed cta_group::2 256x384 int8 / fp8 kernel, and the 256x256 kernel in clusters of two
    pairs sharing B by TMA multicast)."""
    h = A.handle()
    h.set_gemm_path(request.param)
    yield request.param
    h.set_gemm_path(A.SB_GEMM_AUTO)


def rand_q(rng, r, c):
    q = rng.integers(-127, 128, (r, c)).astype(np.int8)
    return q


def exact_raw(qa, qb):
    return qa.astype(np.float64) @ qb.astype(np.float64).T  # exact: |sum| < 2^53


def exact_dequant(raw, sa, sb):
    # float(double(acc) * sa_i * sb_j / 16129.0), linear.cpp:49
    return ((raw * sa.astype(np.float64)[:, None]) * sb.astype(np.float64)[None, :] / 16129.0).astype(np.float32)


GEMM_SHAPES = [(128, 256, 128), (200, 300, 160), (1, 1, 16), (130, 520, 1024), (512, 1024, 1280), (300, 1280, 5120),
               (7, 9, 5), (33, 17, 100)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_int8_raw_and_exact_dequant(M, N, K, gemm_path):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    qa, qb = rand_q(rng, M, K), rand_q(rng, N, K)
    sa = rng.uniform(0.1, 5, M).astype(np.float32)
    sb = np.array([rng.uniform(0.1, 5)], np.float32)
    A = L.QuantizedMatrix(dev(qa, torch.int8), dev(sa), L.ROW)
    B = L.QuantizedMatrix(dev(qb, torch.int8), dev(sb), L.TENSOR)
    raw = host(L.int8_matmul_dequant(A, B, out_dtype="raw"))
    want = exact_raw(qa, qb)
    assert np.array_equal(raw.astype(np.float64), want)
    y = host(L.int8_matmul_dequant(A, B, out_dtype=torch.float32, exact=True))
    assert np.array_equal(y, exact_dequant(want, sa, np.full(N, sb[0], np.float32)))
    yb = host(L.int8_matmul_dequant(A, B, out_dtype=torch.bfloat16, exact=False))
    assert rel_err(yb, exact_dequant(want, sa, np.full(N, sb[0], np.float32))) < 4e-3


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (77, 130, 48)])
def test_int8_dual_rowwise(M, N, K, gemm_path):
    rng = np.random.default_rng(3)
    qa, qb = rand_q(rng, M, K), rand_q(rng, N, K)
    sa = rng.uniform(0.1, 5, M).astype(np.float32)
    sb = rng.uniform(0.1, 5, N).astype(np.float32)
    A = L.QuantizedMatrix(dev(qa, torch.int8), dev(sa), L.ROW)
    B = L.QuantizedMatrix(dev(qb, torch.int8), dev(sb), L.ROW)
    y = host(L.matmul_dequant_dual_rowwise(A, B, exact=True))
    assert np.array_equal(y, exact_dequant(exact_raw(qa, qb), sa, sb))


def test_int8_pinned_and_int64():  # linear_test.cpp:62-72, :97-105
    qx = L.quantize_rowwise(dev([[1.0, 4.0]]))
    qw = L.quantize_tensorwise(dev([[2.0, 0.0], [0.0, 2.0]]))
    y = host(L.int8_matmul_dequant(qx, qw))
    assert y[0, 0] == np.float32(4064.0 * 4.0 * 2.0 / 16129.0) and y[0, 1] == 8.0
    for k in (1000, 140000):
        qx = L.quantize_rowwise(dev(np.ones((1, k), np.float32)))
        qw = L.quantize_tensorwise(dev(np.ones((1, k), np.float32)))
        assert host(L.int8_matmul_dequant(qx, qw))[0, 0] == np.float32(k)
        raw = host(L.int8_matmul_dequant(qx, qw, out_dtype="raw"))
        assert raw[0, 0] == 16129 * k


def test_int8_full_size_sampled_rows(gemm_path):
    """C2 fc1 forward shape: M=65792, N=5120, K=1280; sampled rows checked exactly."""
    M, N, K = 65792, 5120, 1280
    g = torch.Generator(device="cuda").manual_seed(0)
    qa = torch.randint(-127, 128, (M, K), device="cuda", dtype=torch.int8, generator=g)
    qb = torch.randint(-127, 128, (N, K), device="cuda", dtype=torch.int8, generator=g)
    sa = torch.rand(M, device="cuda", generator=g) + 0.5
    sb = torch.tensor([0.75], device="cuda")
    A = L.QuantizedMatrix(qa, sa, L.ROW)
    B = L.QuantizedMatrix(qb, sb, L.TENSOR)
    raw = L.int8_matmul_dequant(A, B, out_dtype="raw")
    rows = torch.tensor([0, 1, 127, 128, 4095, 33333, M - 129, M - 1], device="cuda")
    want = (qa[rows].double() @ qb.double().T)
    assert torch.equal(raw[rows].double(), want)
    y = L.int8_matmul_dequant(A, B, out_dtype=torch.bfloat16, exact=False)
    ref = (want * sa[rows].double()[:, None] * 0.75 / 16129.0)
    assert (y[rows].double() - ref).abs().max().item() <= (ref.abs() * 2 ** -8).max().item() + 1e-30


@pytest.mark.parametrize("T,m,n", [(64, 128, 256), (8192, 256, 512), (1000, 384, 264), (100, 24, 40), (65792, 128, 256)])
def test_wgrad_bf16_tensor_core(T, m, n, gemm_path):
    rng = np.random.default_rng(T)
    g = bf16(rng.standard_normal((T, m)).astype(np.float32))
    x = bf16(rng.standard_normal((T, n)).astype(np.float32))
    dw = host(L.wgrad(dev(g, torch.bfloat16), dev(x, torch.bfloat16), exact=False))
    want = g.astype(np.float64).T @ x.astype(np.float64)
    # fp32 accumulation in TMEM over T tokens (the reference's own sequential fp32 sum is
    # tolerance-equal too): 2e-4 relative at T = 65792
    tol = 2e-4 if T > 10000 else 2e-5
    assert rel_err(dw, want) < tol
    dw2 = L.wgrad(dev(g, torch.bfloat16), dev(x, torch.bfloat16), exact=False)
    L.wgrad(dev(g, torch.bfloat16), dev(x, torch.bfloat16), exact=False, out=dw2, accumulate=True)
    assert rel_err(host(dw2), 2 * want) < tol


@pytest.mark.parametrize("T,m,n", [(1024, 1280, 5120), (1024, 5120, 1280), (640, 1024, 6144), (200, 1280, 4992),
                                   (520, 4992, 1280)])
def test_wgrad_one_wave_wide_tiles(T, m, n):
    """The 256 x 384 one-wave dW kernel (tc_dw_wide.cuh), direct and transposed-store forms,
    incl. partial last tiles; against fp64, and equal to the split-K 256 x 256 path within fp32."""
    rng = np.random.default_rng(m + n + T)
    g = bf16(rng.standard_normal((T, m)).astype(np.float32))
    x = bf16(rng.standard_normal((T, n)).astype(np.float32))
    want = g.astype(np.float64).T @ x.astype(np.float64)
    dw = host(L.wgrad(dev(g, torch.bfloat16), dev(x, torch.bfloat16), exact=False))
    assert rel_err(dw, want) < 2e-5
    h = A.handle()
    h.set_gemm_path(A.SB_GEMM_1CTA)
    try:
        dw1 = host(L.wgrad(dev(g, torch.bfloat16), dev(x, torch.bfloat16), exact=False))
    finally:
        h.set_gemm_path(A.SB_GEMM_AUTO)
    assert rel_err(dw, dw1) < 2e-6


@pytest.mark.parametrize("T,m,n", [(37, 29, 53), (256, 64, 96)])
def test_wgrad_exact_bit_identical(T, m, n):
    rng = np.random.default_rng(5)
    g = rng.standard_normal((T, m)).astype(np.float32)
    x = rng.standard_normal((T, n)).astype(np.float32)
    dw = host(L.wgrad(dev(g), dev(x), exact=True))
    assert np.array_equal(dw, O.wgrad_f32(g, x))


@pytest.mark.parametrize("r,c,k", [(5, 7, 11), (64, 64, 64), (100, 33, 257)])
def test_matmul_exact_bit_identical(r, c, k):
    rng = np.random.default_rng(r)
    a = rng.standard_normal((r, k)).astype(np.float32)
    b = rng.standard_normal((c, k)).astype(np.float32)
    assert np.array_equal(host(L.matmul(dev(a), dev(b))), O.matmul_f32(a, b))


@pytest.mark.parametrize("fa,fb", [(L.E4M3, L.E4M3), (L.E5M2, L.E4M3)])
@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (130, 300, 160)])
def test_fp8_gemm(fa, fb, M, N, K, gemm_path):
    rng = np.random.default_rng(11)
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((N, K)).astype(np.float32)
    qa = L.quantize_fp8(dev(a), fa, L.ROW)
    qb = L.quantize_fp8(dev(b), fb, L.TENSOR)
    y = host(L.gemm_fp8(qa, qb))
    da = fp8_decode(host(qa.payload), fa).astype(np.float64) * host(qa.state)[:, None]
    db = fp8_decode(host(qb.payload), fb).astype(np.float64) * host(qb.state)[0]
    assert rel_err(y, da @ db.T) < 1e-5


def test_gemm_path_option_rejects_bad_values():
    h = A.handle()
    with pytest.raises(A.InvalidArgument, match="sb_set_gemm_path: bad path"):
        h.set_gemm_path(7)
    h.set_gemm_path(A.SB_GEMM_AUTO)


@pytest.mark.parametrize("M,N,K", [(70000, 40, 1000), (3, 70, 140001), (65, 129, 37)])
def test_int8_simt_fallback_large_m_and_int64(M, N, K):
    """Operands the TMA path cannot take (K % 16 != 0) run on the tiled dp4a SIMT kernel:
    exact integer products for any K (int64 tile sums past 133144, linear.cpp:62-65) and no
    65535-row grid limit (M = 70000 token rows)."""
    g = torch.Generator(device="cuda").manual_seed(M + K)
    qa = torch.randint(-127, 128, (M, K), device="cuda", dtype=torch.int8, generator=g)
    qb = torch.randint(-127, 128, (N, K), device="cuda", dtype=torch.int8, generator=g)
    sa = torch.rand(M, device="cuda", generator=g) + 0.5
    sb = torch.tensor([0.75], device="cuda")
    A_ = L.QuantizedMatrix(qa, sa, L.ROW)
    B_ = L.QuantizedMatrix(qb, sb, L.TENSOR)
    want = qa.double() @ qb.double().T
    y = L.int8_matmul_dequant(A_, B_, out_dtype=torch.float32, exact=True)
    t = (want * sa.double()[:, None]) * 0.75
    ref = (t / torch.full_like(t, 16129.0)).float()  # IEEE division (a Python-scalar divisor becomes a reciprocal)
    assert torch.equal(y, ref)
    if K <= 133144:
        raw = L.int8_matmul_dequant(A_, B_, out_dtype="raw")
        assert torch.equal(raw.double(), want)
