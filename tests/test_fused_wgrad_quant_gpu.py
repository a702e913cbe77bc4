"""GPU parity: the dW GEMM with G's row-wise quantize fused into its idle warps
(sb_wgrad_quantize_rowwise, tc_dw_wide.cuh QV) against the two standalone launches it replaces
(quantize_rowwise(G), linear.cpp:232 / quantize.cpp:131-133, and wgrad_full_precision(G, X),
linear.cpp:193-195, :245): payload and states bit for bit (and against the C oracle, which is
pinned to the reference), dW bit for bit (the same GEMM tiles), non-finite rows latched."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2304_13013_b200 import _capi as A
from paper_2304_13013_b200 import lowprec as L

pytestmark = pytest.mark.gpu

T_VIT = 256 * 257

# (T, m, n): G is T x m, X is T x n. The first three run the one-wave kernel with the quantize
# fused (m = 5120 / 1280 in registers, 3840 two-pass rows); the rest fall back to the separate
# quantizer (shapes the one-wave tiling does not take, or ragged rows).
SHAPES = [(T_VIT, 5120, 1280), (T_VIT, 1280, 5120), (20000, 3840, 1280), (8192, 4096, 1024), (1000, 1280, 640),
          (77, 40, 24)]


def _g(T, m, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    g = torch.randn(T, m, device="cuda", generator=gen)
    if T > 8:
        g[1] = 0  # all-zero row: state sentinel 1.0 (quantize.cpp:98-99)
        g[2] *= 1e-30  # tiny row: power-of-two prescale path
        g[3, ::5] *= 1e4  # outlier columns
        g[4] = torch.arange(m, device="cuda") % 255 - 127.0  # exact ties (x.5 quotients)
        g[5] *= 3e30  # huge row
    return g.to(torch.bfloat16)


@pytest.mark.parametrize("T,m,n", SHAPES)
def test_fused_matches_standalone(T, m, n):
    g = _g(T, m, 7 + m)
    x = torch.randn(T, n, device="cuda").to(torch.bfloat16)
    dw, qg = L.wgrad_quantize_rowwise(g, x)
    q_ref = L.quantize_rowwise(g)
    dw_ref = L.wgrad(g, x, exact=False)
    torch.cuda.synchronize()
    assert torch.equal(qg.payload, q_ref.payload), "payload differs from quantize_rowwise"
    assert torch.equal(qg.state, q_ref.state), "states differ from quantize_rowwise"
    assert torch.equal(dw, dw_ref), "dW differs from wgrad"
    if T <= 20000:
        # and against the pinned oracle on every row
        qo, so = O.quantize(g.float().cpu().numpy(), O.ROW)
        assert np.array_equal(qg.payload.cpu().numpy(), qo)
        assert np.array_equal(qg.state.cpu().numpy(), so)


def test_fused_empty_g_rejected_like_quantize_rowwise():
    g = torch.empty(0, 1280, device="cuda", dtype=torch.bfloat16)
    x = torch.empty(0, 640, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(A.InvalidArgument, match="quantize_rowwise: empty matrix"):
        L.wgrad_quantize_rowwise(g, x)
    with pytest.raises(A.InvalidArgument, match="quantize_rowwise: empty matrix"):
        L.quantize_rowwise(g)


def test_fused_full_c2_against_oracle():
    """C2 fc1's G (T = 65792 x 5120): every row's payload / state against the C oracle."""
    g = _g(T_VIT, 5120, 11)
    x = torch.randn(T_VIT, 1280, device="cuda").to(torch.bfloat16)
    _, qg = L.wgrad_quantize_rowwise(g, x)
    qo, so = O.quantize(g.float().cpu().numpy(), O.ROW)
    assert np.array_equal(qg.payload.cpu().numpy(), qo)
    assert np.array_equal(qg.state.cpu().numpy(), so)


@pytest.mark.parametrize("m,n", [(5120, 1280), (1280, 5120), (3840, 1280)])
def test_fused_nonfinite_latched(m, n):
    g = _g(T_VIT if m != 3840 else 20000, m, 3)
    g[17, 9] = float("nan")
    x = torch.randn(g.shape[0], n, device="cuda").to(torch.bfloat16)
    with pytest.raises(A.InvalidArgument, match="non-finite"):
        L.wgrad_quantize_rowwise(g, x)


def test_linear_backward_uses_fused_path():
    """sb_linear_backward (SwitchBack int8, bf16) issues the fused dW + G quantize: one launch
    fewer than quantize + dW + dX, and the same G payload, dX and dW as the standalone ops."""
    T, n, m = T_VIT, 1280, 5120
    gen = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(T, n, device="cuda", generator=gen).to(torch.bfloat16)
    w = (torch.randn(m, n, device="cuda", generator=gen) * n ** -0.5).to(torch.bfloat16)
    g = torch.randn(T, m, device="cuda", generator=gen).to(torch.bfloat16)
    mode = L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8)
    ctx = L.LinearContext()
    L.linear_forward(mode, x, w, ctx)
    h = A.handle()
    l0 = h.launches()
    dx, dw = L.linear_backward(mode, ctx, g)
    torch.cuda.synchronize()
    assert h.launches() - l0 == 2  # fused dW + G quantize, then the int8 dX GEMM
    dw_ref = L.wgrad(g, x, exact=False)
    qg = L.quantize_rowwise(g)
    qwt = L.quantize_tensorwise(w, with_transpose=True)[1]
    dx_ref = L.int8_matmul_dequant(qg, qwt, out_dtype=torch.bfloat16, exact=False)
    assert torch.equal(dw, dw_ref)
    assert torch.equal(dx, dx_ref)
