"""GPU parity: the MLP-block host entry sb_switchback_mlp_fwd_bwd_host (two chained SwitchBack
int8 linears, model.cpp:324-329 / 351-360, hidden activation kept on the device) against
(1) the reference itself (oracle/_ref, the unmodified lowprec::linear_forward / linear_backward
chained) in exact fp32 mode, and (2) the device-resident layer API in the bf16 performance path.
Token chunks are per-row independent, so Y and dX are bit-identical to the unchunked path;
dW sums the chunks in order."""
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2304_13013_b200 import _capi as A
from paper_2304_13013_b200 import lowprec as L
from tests._util import rel_err

pytestmark = pytest.mark.gpu


def _inputs(b, n, hd, m, seed, dtype):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(b, n, generator=g)
    w1 = torch.randn(hd, n, generator=g) / n ** 0.5
    w2 = torch.randn(m, hd, generator=g) / hd ** 0.5
    gg = torch.randn(b, m, generator=g)
    return [t.to(dtype).pin_memory() for t in (x, w1, w2, gg)]


@pytest.fixture
def chunk_env():
    old = os.environ.get("SB_HOST_CHUNK")
    yield lambda v: os.environ.__setitem__("SB_HOST_CHUNK", str(v))
    if old is None:
        os.environ.pop("SB_HOST_CHUNK", None)
    else:
        os.environ["SB_HOST_CHUNK"] = old


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("b,n,hd,m", [(300, 64, 96, 48), (1024, 128, 256, 128)])
def test_exact_one_chunk_bit_identical_to_reference(b, n, hd, m):
    """exact=1, fp32, one chunk: Y, dX, dW1, dW2 equal the reference's chained MLP bit for bit."""
    x, w1, w2, g = _inputs(b, n, hd, m, 1, torch.float32)
    y, dx, dw1, dw2 = L.switchback_mlp_fwd_bwd_host(x, w1, w2, g, exact=True)
    xn, w1n, w2n, gn = (t.numpy() for t in (x, w1, w2, g))
    ry, rdx = np.zeros((b, m), np.float32), np.zeros((b, n), np.float32)
    rd1, rd2 = np.zeros((hd, n), np.float32), np.zeros((m, hd), np.float32)
    P = lambda a: a.ctypes.data  # noqa: E731
    assert O.ref().ref_switchback_mlp_fwd_bwd_threaded(xn, w1n, w2n, gn, b, n, hd, m, 1, P(ry), P(rdx), P(rd1),
                                                       P(rd2)) == 0
    assert np.array_equal(y.numpy(), ry), "Y"
    assert np.array_equal(dx.numpy(), rdx), "dX"
    assert np.array_equal(dw1.numpy(), rd1), "dW1"
    assert np.array_equal(dw2.numpy(), rd2), "dW2"


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_exact_many_chunks_vs_reference(chunk_env):
    """exact=1 over 5 ragged chunks: Y / dX per row equal the reference; dW differs only by the
    chunked fp32 summation order."""
    b, n, hd, m = 1100, 64, 128, 64
    chunk_env(256)
    x, w1, w2, g = _inputs(b, n, hd, m, 2, torch.float32)
    y, dx, dw1, dw2 = L.switchback_mlp_fwd_bwd_host(x, w1, w2, g, exact=True)
    ry, rdx = np.zeros((b, m), np.float32), np.zeros((b, n), np.float32)
    rd1, rd2 = np.zeros((hd, n), np.float32), np.zeros((m, hd), np.float32)
    P = lambda a: a.ctypes.data  # noqa: E731
    assert O.ref().ref_switchback_mlp_fwd_bwd_threaded(*(t.numpy() for t in (x, w1, w2, g)), b, n, hd, m, 1, P(ry),
                                                       P(rdx), P(rd1), P(rd2)) == 0
    assert np.array_equal(y.numpy(), ry)
    assert np.array_equal(dx.numpy(), rdx)
    assert rel_err(dw1.numpy(), rd1) < 1e-6 and rel_err(dw2.numpy(), rd2) < 1e-6


def _device_mlp(x, w1, w2, g, gelu):
    """The same block on device tensors through the layer API (one launch sequence, no chunks)."""
    md = L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8)
    x, w1, w2, g = (t.cuda() for t in (x, w1, w2, g))
    c1, c2 = L.LinearContext(), L.LinearContext()
    pre = L.linear_forward(md, x, w1, c1)
    if gelu:
        act, aq = L.gelu_quantize_rowwise(pre)
        y = L.linear_forward(md, act, w2, c2, x_q=aq)
    else:
        y = L.linear_forward(md, pre, w2, c2)
    da, dw2 = L.linear_backward(md, c2, g)
    if gelu:
        g1, g1q = L.gelu_backward_quantize_rowwise(da, pre)
        dx, dw1 = L.linear_backward(md, c1, g1, g_q=g1q)
    else:
        dx, dw1 = L.linear_backward(md, c1, da)
    return y.cpu(), dx.cpu(), dw1.cpu(), dw2.cpu()


@pytest.mark.parametrize("gelu", [False, True])
@pytest.mark.parametrize("b,chunk", [(20000, None), (9000, 1024), (65792, None)])
def test_bf16_matches_device_path(gelu, b, chunk, chunk_env):
    """bf16 performance path at ViT-H widths (65792 = the C2 token count): Y and dX bit-identical to
    the device-resident layer API; dW1 / dW2 within the chunked fp32 summation tolerance."""
    n, hd, m = 1280, 5120, 1280
    if chunk:
        chunk_env(chunk)
    x, w1, w2, g = _inputs(b, n, hd, m, 3, torch.bfloat16)
    act = A.SB_ACT_GELU if gelu else A.SB_ACT_NONE
    y, dx, dw1, dw2 = L.switchback_mlp_fwd_bwd_host(x, w1, w2, g, activation=act)
    yd, dxd, dw1d, dw2d = _device_mlp(x, w1, w2, g, gelu)
    assert torch.equal(y, yd), "Y"
    assert torch.equal(dx, dxd), "dX"
    assert rel_err(dw1.numpy(), dw1d.numpy()) < 1e-4
    assert rel_err(dw2.numpy(), dw2d.numpy()) < 1e-4


def test_async_back_to_back_and_repeatable():
    """Two async calls alternate the device pools (the second call's uploads overlap the first's
    drain); both equal the synchronous call."""
    b, n, hd, m = 12000, 512, 1536, 512
    ins = [_inputs(b, n, hd, m, s, torch.bfloat16) for s in (4, 5)]
    outs = [L.switchback_mlp_fwd_bwd_host(*t, wait=False) for t in ins]
    L.host_pipeline_wait()
    for t, o in zip(ins, outs):
        ref = L.switchback_mlp_fwd_bwd_host(*t)
        for a, r in zip(o, ref):
            assert torch.equal(a, r)


def test_argument_errors():
    x, w1, w2, g = _inputs(64, 32, 48, 32, 6, torch.bfloat16)
    with pytest.raises(ValueError):
        L.switchback_mlp_fwd_bwd_host(x, w2, w1, g)
    with pytest.raises(A.SBError):  # GELU is the bf16 performance path only
        L.switchback_mlp_fwd_bwd_host(x.float().pin_memory(), w1.float().pin_memory(), w2.float().pin_memory(),
                                      g.float().pin_memory(), activation=A.SB_ACT_GELU, exact=True)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_unaligned_widths_take_the_fallback_kernels(dtype, chunk_env):
    """Widths that are not TMA-legal (n, hidden, m not multiples of 16) run the SIMT fallbacks inside
    the pipeline (several ragged chunks): Y / dX still equal the device-resident layer API."""
    b, n, hd, m = 3000, 100, 72, 40
    chunk_env(1024)
    x, w1, w2, g = _inputs(b, n, hd, m, 8, dtype)
    y, dx, dw1, dw2 = L.switchback_mlp_fwd_bwd_host(x, w1, w2, g)
    yd, dxd, dw1d, dw2d = _device_mlp(x, w1, w2, g, False)
    assert torch.equal(y, yd) and torch.equal(dx, dxd)
    assert rel_err(dw1.numpy(), dw1d.numpy()) < 1e-4 and rel_err(dw2.numpy(), dw2d.numpy()) < 1e-4


@pytest.mark.parametrize("taper,first,w2late", [("0", None, "1"), ("1", "512", "1"), ("2", "300", "0"), ("2", None, "1")])
def test_chunk_schedules_agree(taper, first, w2late, chunk_env):
    """Every chunk schedule of the pipeline (no taper, one short last chunk, chunks halving at the
    end, odd first-chunk sizes, W2 quantized up front or after the first chunk) gives Y / dX
    bit-identical to the device-resident layer API; dW differs only by the chunked fp32 sum order."""
    b, n, hd, m = 9000, 256, 512, 256
    chunk_env(2048)
    keys = ("SB_HOST_TAPER", "SB_HOST_FIRST", "SB_HOST_W2LATE")
    old = {k: os.environ.get(k) for k in keys}
    try:
        os.environ["SB_HOST_TAPER"] = taper
        os.environ["SB_HOST_W2LATE"] = w2late
        if first:
            os.environ["SB_HOST_FIRST"] = first
        else:
            os.environ.pop("SB_HOST_FIRST", None)
        x, w1, w2, g = _inputs(b, n, hd, m, 11, torch.bfloat16)
        for act in (A.SB_ACT_NONE, A.SB_ACT_GELU):
            y, dx, dw1, dw2 = L.switchback_mlp_fwd_bwd_host(x, w1, w2, g, activation=act)
            yd, dxd, dw1d, dw2d = _device_mlp(x, w1, w2, g, act == A.SB_ACT_GELU)
            assert torch.equal(y, yd) and torch.equal(dx, dxd)
            assert rel_err(dw1.numpy(), dw1d.numpy()) < 1e-4 and rel_err(dw2.numpy(), dw2d.numpy()) < 1e-4
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_async_into_alternating_out_buffers():
    """Back-to-back async calls writing into two alternating preallocated output sets (the
    pipelined use): every call's outputs equal the synchronous call's."""
    b, n, hd, m = 10000, 256, 768, 256
    x, w1, w2, g = _inputs(b, n, hd, m, 12, torch.bfloat16)
    ref = L.switchback_mlp_fwd_bwd_host(x, w1, w2, g)
    outs = [tuple(torch.empty_like(t).pin_memory() for t in ref) for _ in range(2)]
    for i in range(5):
        L.switchback_mlp_fwd_bwd_host(x, w1, w2, g, wait=False, out=outs[i % 2])
    L.host_pipeline_wait()
    for o in outs:
        for a, r in zip(o, ref):
            assert torch.equal(a, r)
    with pytest.raises(ValueError):
        L.switchback_mlp_fwd_bwd_host(x, w1, w2, g, out=(outs[0][0], outs[0][1], outs[0][3], outs[0][2]))  # dw1 / dw2 swapped
