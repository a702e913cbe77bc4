"""GPU: the PyTorch-facing SwitchBackLinear (autograd.Function over the C-ABI) equals the
explicit lowprec forward/backward, is tolerance-equal to an fp32 nn.Linear, takes any leading
shape, and is CUDA-graph capturable."""
import numpy as np
import pytest
import torch

from paper_2304_13013_b200 import _capi as A
from paper_2304_13013_b200 import lowprec as L
from paper_2304_13013_b200.nn import SwitchBackLinear

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a.detach() - b.detach()).norm() / b.detach().norm())


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_matches_lowprec_and_fp32_linear(dtype):
    torch.manual_seed(0)
    lin = SwitchBackLinear(256, 384, bias=False)
    x = torch.randn(4, 97, 256, device="cuda").to(dtype).requires_grad_(True)
    y = lin(x)
    g = torch.randn_like(y)
    y.backward(g)
    # the explicit lowprec path: identical outputs
    mode = L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8)
    ctx = L.LinearContext()
    y2 = L.linear_forward(mode, x.detach().reshape(-1, 256), lin.weight.detach().to(dtype), ctx)
    dx2, dw2 = L.linear_backward(mode, ctx, g.reshape(-1, 384))
    assert torch.equal(y.detach().reshape(-1, 384), y2)
    assert torch.equal(x.grad.reshape(-1, 256), dx2)
    assert torch.equal(lin.weight.grad, dw2)  # fp32 dW straight into the fp32 master weight
    # fp32 reference linear
    xr = x.detach().float().requires_grad_(True)
    wr = lin.weight.detach().float().requires_grad_(True)
    yr = torch.nn.functional.linear(xr, wr)
    yr.backward(g.float())
    assert rel(y.detach(), yr) < 2e-2
    assert rel(x.grad, xr.grad) < 2e-2
    assert rel(lin.weight.grad, wr.grad) < (1e-2 if dtype == torch.bfloat16 else 1e-5)


def test_bias_and_shapes():
    torch.manual_seed(2)
    lin = SwitchBackLinear(128, 64, bias=True)
    with torch.no_grad():
        lin.bias.copy_(torch.randn(64, device="cuda"))
    x = torch.randn(3, 5, 7, 128, device="cuda").bfloat16().requires_grad_(True)
    y = lin(x)
    assert y.shape == (3, 5, 7, 64) and y.dtype == torch.bfloat16
    g = torch.randn_like(y)
    y.backward(g)
    assert torch.allclose(lin.bias.grad, g.float().reshape(-1, 64).sum(0), rtol=1e-2, atol=1e-1)
    assert x.grad.shape == x.shape


def test_cuda_graph_capture_replays_identically():
    torch.manual_seed(1)
    l1, l2 = SwitchBackLinear(512, 2048), SwitchBackLinear(2048, 512)
    x = torch.randn(1024, 512, device="cuda").bfloat16()
    g = torch.randn(1024, 512, device="cuda").bfloat16()

    def step():
        xx = x.detach().requires_grad_(True)
        out = l2(torch.nn.functional.gelu(l1(xx)))
        out.backward(g)
        return out.detach().clone(), xx.grad.clone()

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            for p in (*l1.parameters(), *l2.parameters()):
                p.grad = None
            ref_y, ref_dx = step()
    torch.cuda.current_stream().wait_stream(s)
    for p in (*l1.parameters(), *l2.parameters()):
        p.grad = None
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out_y, out_dx = step()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out_y, ref_y) and torch.equal(out_dx, ref_dx)
    L.check_error()
