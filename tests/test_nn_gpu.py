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


@pytest.mark.parametrize("rows,cols", [(1000, 5120), (37, 1280), (8, 8), (7, 100)])
def test_gelu_quantize_fused_matches_composition(rows, cols):
    """act == gelu(pre) within one bf16 ulp of torch's, and its payload / states are exactly
    quantize_rowwise(act) (the fused kernel quantizes the values it stores)."""
    torch.manual_seed(rows + cols)
    pre = (torch.randn(rows, cols, device="cuda") * 2).bfloat16()
    pre[0, :3] = 0
    act, q = L.gelu_quantize_rowwise(pre)
    ref = torch.nn.functional.gelu(pre.float())
    assert ((act.float() - ref).abs() <= ref.abs() * 2 ** -7 + 1e-6).all()
    q2 = L.quantize_rowwise(act)
    assert torch.equal(q.payload, q2.payload) and torch.equal(q.state, q2.state)
    dact = torch.randn(rows, cols, device="cuda").bfloat16()
    g, gq = L.gelu_backward_quantize_rowwise(dact, pre)
    x = pre.float().requires_grad_(True)
    torch.nn.functional.gelu(x).backward(dact.float())
    assert ((g.float() - x.grad).abs() <= x.grad.abs() * 2 ** -7 + 1e-5).all()
    g2 = L.quantize_rowwise(g)
    assert torch.equal(gq.payload, g2.payload) and torch.equal(gq.state, g2.state)


def test_mlp_fused_module_matches_fp32():
    from paper_2304_13013_b200.nn import SwitchBackMLP

    torch.manual_seed(5)
    mlp = SwitchBackMLP(256, 1024)
    with torch.no_grad():
        mlp.fc1.bias.normal_()
        mlp.fc2.bias.normal_()
    x = torch.randn(3, 333, 256, device="cuda").bfloat16().requires_grad_(True)
    y = mlp(x)
    g = torch.randn_like(y)
    y.backward(g)
    xr = x.detach().float().requires_grad_(True)
    w1 = mlp.fc1.weight.detach().clone().requires_grad_(True)
    w2 = mlp.fc2.weight.detach().clone().requires_grad_(True)
    b1 = mlp.fc1.bias.detach().clone().requires_grad_(True)
    b2 = mlp.fc2.bias.detach().clone().requires_grad_(True)
    F = torch.nn.functional
    yr = F.linear(F.gelu(F.linear(xr, w1, b1)), w2, b2)
    yr.backward(g.float())
    assert rel(y, yr) < 2e-2
    assert rel(x.grad, xr.grad) < 3e-2
    for p, r in ((mlp.fc1.weight, w1), (mlp.fc2.weight, w2), (mlp.fc1.bias, b1), (mlp.fc2.bias, b2)):
        assert rel(p.grad, r.grad) < 2e-2


def test_gelu_table_equals_formula_for_every_bf16():
    """The fused kernels read GELU / GELU' from per-handle tables for |x| < 8; the (n x 1)
    shape takes the elementwise formula path. Every one of the 65536 bf16 inputs must give
    the same bits both ways (forward and backward)."""
    allx = torch.arange(65536, dtype=torch.int32, device="cuda").to(torch.int16).view(torch.bfloat16)
    a_vec, _ = L.gelu_quantize_rowwise(allx.view(8192, 8), check=False)
    a_sc, _ = L.gelu_quantize_rowwise(allx.view(65536, 1), check=False)
    assert torch.equal(a_vec.view(-1).view(torch.int16), a_sc.view(-1).view(torch.int16))
    dy = torch.randn(65536, device="cuda").bfloat16()
    g_vec, _ = L.gelu_backward_quantize_rowwise(dy.view(8192, 8), allx.view(8192, 8), check=False)
    g_sc, _ = L.gelu_backward_quantize_rowwise(dy.view(65536, 1), allx.view(65536, 1), check=False)
    assert torch.equal(g_vec.view(-1).view(torch.int16), g_sc.view(-1).view(torch.int16))
    with pytest.raises(L.InvalidArgument):  # the inf / NaN inputs latched the error word: consume it
        L.check_error()


@pytest.mark.parametrize("rows,cols", [(4000, 1280), (33, 256), (7, 2048)])
def test_layernorm_quantize_fused(rows, cols):
    """LayerNorm + row-wise quantize in one kernel: the output is torch's LayerNorm within bf16
    rounding, and the payload / states are exactly quantize_rowwise(out)."""
    torch.manual_seed(rows)
    x = (torch.randn(rows, cols, device="cuda") * 3 + 0.5).bfloat16()
    g = torch.randn(cols, device="cuda") * 0.5 + 1
    b = torch.randn(cols, device="cuda") * 0.1
    out, q, mean, rstd = L.layernorm_quantize_rowwise(x, g, b, 1e-5)
    ref = torch.nn.functional.layer_norm(x.float(), (cols,), g, b, 1e-5)
    assert ((out.float() - ref).abs() <= ref.abs() * 2 ** -7 + 2e-3).all()
    q2 = L.quantize_rowwise(out)
    assert torch.equal(q.payload, q2.payload) and torch.equal(q.state, q2.state)
    assert torch.allclose(mean, x.float().mean(1), rtol=1e-5, atol=1e-5)


def test_prenorm_modules_match_fp32():
    from paper_2304_13013_b200.nn import SwitchBackLinear, SwitchBackMLP

    torch.manual_seed(9)
    F = torch.nn.functional
    for mod in (SwitchBackLinear(256, 384, prenorm=True), SwitchBackMLP(256, 512, prenorm=True)):
        with torch.no_grad():
            mod.norm.weight.normal_(1.0, 0.2)
            mod.norm.bias.normal_(0.0, 0.1)
        x = torch.randn(2, 300, 256, device="cuda").bfloat16().requires_grad_(True)
        y = mod(x)
        g = torch.randn_like(y)
        y.backward(g)
        xr = x.detach().float().requires_grad_(True)
        params = {n: p.detach().clone().requires_grad_(True) for n, p in mod.named_parameters()}
        h = F.layer_norm(xr, (256,), params["norm.weight"], params["norm.bias"], mod.norm.eps)
        if isinstance(mod, SwitchBackLinear):
            yr = F.linear(h, params["weight"], params["bias"])
        else:
            yr = F.linear(F.gelu(F.linear(h, params["fc1.weight"], params["fc1.bias"])), params["fc2.weight"],
                          params["fc2.bias"])
        yr.backward(g.float())
        assert rel(y, yr) < 3e-2  # int8 noise of one or two quantized GEMMs on top of bf16 LN rounding
        assert rel(x.grad, xr.grad) < 3e-2
        for n, p in mod.named_parameters():
            assert rel(p.grad, params[n].grad) < 3e-2, n


@pytest.mark.parametrize("rows,cols", [(5000, 1280), (37, 256), (300, 1000)])
def test_layernorm_backward_kernel(rows, cols):
    """sb_layernorm_backward against torch's LayerNorm backward (fp32) with the same mean /
    rstd; dgamma / dbeta are fixed-order sums: bit-identical across runs."""
    torch.manual_seed(cols)
    x = (torch.randn(rows, cols, device="cuda") * 2 + 0.3).bfloat16()
    g = torch.randn(cols, device="cuda") * 0.3 + 1
    b = torch.randn(cols, device="cuda") * 0.1
    _, _, mean, rstd = L.layernorm_quantize_rowwise(x, g, b)
    dh = torch.randn(rows, cols, device="cuda").bfloat16()
    dx, dg, db = L.layernorm_backward(dh, x, mean, rstd, g)
    xr = x.float().requires_grad_(True)
    gr, br = g.clone().requires_grad_(True), b.clone().requires_grad_(True)
    torch.nn.functional.layer_norm(xr, (cols,), gr, br, 1e-5).backward(dh.float())
    assert rel(dx, xr.grad) < 1e-2
    assert rel(dg, gr.grad) < 1e-4 and rel(db, br.grad) < 1e-5
    dx2, dg2, db2 = L.layernorm_backward(dh, x, mean, rstd, g)
    assert torch.equal(dx, dx2) and torch.equal(dg, dg2) and torch.equal(db, db2)


def test_fused_producers_edge_rows():
    """Constant rows (zero variance: out = beta, all-equal payload), all-zero rows (state
    sentinel 1.0), and a non-finite row (latched, reported by check_error) through the fused
    LayerNorm and GELU quantizers."""
    cols = 1280
    x = torch.randn(6, cols, device="cuda").bfloat16()
    x[1] = 3.0
    x[2] = 0.0
    g = torch.ones(cols, device="cuda")
    b = torch.zeros(cols, device="cuda")
    out, q, mean, rstd = L.layernorm_quantize_rowwise(x, g, b)
    assert (out[1] == 0).all() and (out[2] == 0).all()
    assert float(q.state[1]) == 1.0 and float(q.state[2]) == 1.0  # zero rows: sentinel state
    assert float(mean[1]) == 3.0
    act, aq = L.gelu_quantize_rowwise(x)
    assert float(aq.state[2]) == 1.0 and (aq.payload[2] == 0).all()
    bad = x.clone()
    bad[4, 7] = float("nan")
    with pytest.raises(L.InvalidArgument):
        L.gelu_quantize_rowwise(bad)
    with pytest.raises(L.InvalidArgument):
        L.layernorm_quantize_rowwise(bad, g, b)


@pytest.mark.parametrize("variant,fmt", [("switchback_q", "int8"), ("switchback_m", "int8"), ("switchback", "fp8"),
                                         ("allquant", "int8")])
def test_linear_module_variants(variant, fmt):
    """SwitchBackLinear over the other reference variants / formats (prenorm fused where the
    variant quantizes X row-wise in int8, unfused otherwise) against an fp32 reference."""
    from paper_2304_13013_b200.nn import SwitchBackLinear

    torch.manual_seed(4)
    F = torch.nn.functional
    mod = SwitchBackLinear(256, 320, variant=variant, fmt=fmt, prenorm=True)
    x = torch.randn(600, 256, device="cuda").bfloat16().requires_grad_(True)
    y = mod(x)
    g = torch.randn_like(y)
    y.backward(g)
    xr = x.detach().float().requires_grad_(True)
    ps = {n: p.detach().clone().requires_grad_(True) for n, p in mod.named_parameters()}
    yr = F.linear(F.layer_norm(xr, (256,), ps["norm.weight"], ps["norm.bias"], mod.norm.eps), ps["weight"], ps["bias"])
    yr.backward(g.float())
    tol = 8e-2 if fmt == "fp8" else 3e-2
    assert rel(y, yr) < tol and rel(x.grad, xr.grad) < tol
    assert rel(mod.weight.grad, ps["weight"].grad) < tol


def test_residual_in_epilogue_modules():
    """SwitchBackLinear / SwitchBackMLP with residual=: the skip connection added in the GEMM
    epilogue, and its gradient passed straight through."""
    from paper_2304_13013_b200.nn import SwitchBackLinear, SwitchBackMLP

    torch.manual_seed(12)
    F = torch.nn.functional
    for mod in (SwitchBackLinear(256, 256), SwitchBackMLP(256, 512, prenorm=True)):
        x = torch.randn(500, 256, device="cuda").bfloat16().requires_grad_(True)
        r = torch.randn(500, 256, device="cuda").bfloat16().requires_grad_(True)
        y = mod(x, residual=r)
        y0 = mod(x) + r
        assert rel(y, y0) < 1e-2
        g = torch.randn_like(y)
        y.backward(g)
        assert torch.equal(r.grad, g)


@pytest.mark.parametrize("prenorm", [False, True])
def test_grouped_qkv_module_equals_three_linears(prenorm):
    """SwitchBackLinear(groups=3): q / k / v with three tensor-wise scales (model.cpp:303-305) as
    one GEMM. Forward: bit-identical to three separate SwitchBackLinear layers (same per-element
    arithmetic); dW / db: equal to the separate layers' to fp32 accumulation order; dX: the sum
    of the three layers' input gradients within bf16 rounding."""
    torch.manual_seed(3)
    T, D = 4096, 256
    grp = SwitchBackLinear(D, 3 * D, groups=3, prenorm=prenorm)
    sep = [SwitchBackLinear(D, D, prenorm=prenorm) for _ in range(3)]
    with torch.no_grad():
        for i, s in enumerate(sep):
            s.weight.copy_(grp.weight[i * D:(i + 1) * D])
            s.bias.copy_(torch.randn(D, device="cuda"))
            grp.bias[i * D:(i + 1) * D] = s.bias
            if prenorm:
                s.norm.load_state_dict(grp.norm.state_dict())
    x = torch.randn(T, D, device="cuda").bfloat16()
    gy = torch.randn(T, 3 * D, device="cuda").bfloat16()
    xg = x.clone().requires_grad_(True)
    yg = grp(xg)
    yg.backward(gy)
    xs = x.clone().requires_grad_(True)
    ys = torch.cat([s(xs) for s in sep], 1)
    ys.backward(gy)
    assert torch.equal(yg, ys)
    for i, s in enumerate(sep):
        assert rel(grp.weight.grad[i * D:(i + 1) * D], s.weight.grad) < 1e-5
        assert rel(grp.bias.grad[i * D:(i + 1) * D], s.bias.grad) < 1e-6
    assert rel(xg.grad.float(), xs.grad.float()) < 1e-2


@pytest.mark.parametrize("prenorm", [False, True])
def test_qkv_heads_matches_split_copies(prenorm):
    """SwitchBackLinear.qkv_heads (q / k / v as head views, gradients packed + quantized by one kernel)
    gives the same outputs and gradients, bit for bit, as the grouped linear followed by a
    torch split / transpose (whose backward copies the heads into the packed G)."""
    from paper_2304_13013_b200.nn import SwitchBackLinear

    B, S, D, H = 3, 37, 256, 4
    torch.manual_seed(4)
    lin = SwitchBackLinear(D, 3 * D, device="cuda", prenorm=prenorm, groups=3)
    with torch.no_grad():
        lin.bias.normal_()
    x0 = torch.randn(B, S, D, device="cuda").bfloat16()
    gq, gk, gv = (torch.randn(B, H, S, D // H, device="cuda").bfloat16() for _ in range(3))

    def run(fused):
        lin.zero_grad(set_to_none=True)
        x = x0.clone().requires_grad_(True)
        if fused:
            q, k, v = lin.qkv_heads(x, H)
        else:
            t = lin(x).view(B, S, 3, H, D // H)
            q, k, v = (t[:, :, i].transpose(1, 2) for i in range(3))
        ((q.float() * gq.float()).sum() + (k.float() * gk.float()).sum() + (v.float() * gv.float()).sum()).backward()
        return [q.detach().clone(), x.grad.clone()] + [p.grad.clone() for p in lin.parameters()]

    a, b = run(True), run(False)
    for u, w in zip(a, b):
        assert torch.equal(u, w)
