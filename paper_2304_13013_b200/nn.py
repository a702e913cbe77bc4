"""PyTorch-facing SwitchBack layer: an ``autograd.Function`` over the C-ABI linear forward /
backward (``sb_linear_forward`` / ``sb_linear_backward``, linear.cpp:113-278) and an
``nn.Linear``-shaped module. This is a CALLER of the drop-in path (SURVEY.md §8b "PyTorch
autograd.Function wrapper", §8f row 2 model-level caller), not part of the measured kernels.

* Weights are fp32 master parameters; each forward feeds a bf16 (or fp32) copy to the kernels
  and the weight gradient comes back in fp32 (the reference's dW precision, linear.cpp:245),
  so no gradient precision is lost to a bf16 round trip.
* No host synchronisation on the hot path (non-finite inputs still latch in the handle's
  device error word; ``lowprec.check_error()`` / ``sb_synchronize`` report them), so the layer
  is CUDA-graph capturable.
* Inputs of any leading shape (..., in_features) are flattened to token rows.
"""
from __future__ import annotations

import torch

from . import _capi as A
from . import lowprec as L

_VARIANTS = {"switchback": A.SB_SWITCHBACK, "switchback_m": A.SB_SWITCHBACK_M, "switchback_q": A.SB_SWITCHBACK_Q,
             "allquant": A.SB_ALLQUANT, "standard": A.SB_STANDARD}


class _SwitchBackLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x2d: torch.Tensor, weight: torch.Tensor, bias, mode: L.LinearMode, resid=None):
        w = weight.detach().to(x2d.dtype).contiguous()
        lctx = L.LinearContext()
        b = bias.detach().float() if bias is not None else None
        # bias (and the residual, if any) fused in the GEMM epilogue
        y = L.linear_forward(mode, x2d.contiguous(), w, lctx, check=False, bias=b,
                             residual=resid.detach() if resid is not None else None)
        ctx.lctx = lctx
        ctx.mode = mode
        ctx.has_bias = bias is not None
        ctx.keep_w = w  # the device context references it until the backward
        return y

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        g = g.contiguous()
        dx, dw = L.linear_backward(ctx.mode, ctx.lctx, g, check=False)
        db = L.column_sums(g) if ctx.has_bias and ctx.needs_input_grad[2] else None
        ctx.lctx = None
        ctx.keep_w = None
        return dx, dw, db, None, (g if ctx.needs_input_grad[4] else None)


class SwitchBackLinear(torch.nn.Module):
    """y = x W^T (+ b) with the int8 SwitchBack forward / input gradient and the 16-bit weight
    gradient (arXiv 2304.13013), on the B200 kernels of this package."""

    def __init__(self, in_features: int, out_features: int, bias: bool = True, variant: str = "switchback",
                 fmt: str = "int8", device=None, prenorm: bool = False, eps: float = 1e-5, groups: int = 1):
        super().__init__()
        self.in_features, self.out_features = in_features, out_features
        # groups > 1: out_features = groups projections of one shared input (q / k / v), each with
        # its own tensor-wise weight scale as separate linears would have (model.cpp:303-305),
        # computed as one GEMM (sb_gemm_i8_epilogue, per-column scales)
        if groups > 1 and (out_features % groups or variant != "switchback" or fmt != "int8"):
            raise ValueError("grouped SwitchBackLinear: int8 SwitchBack with out_features divisible by groups")
        self.groups = groups
        # prenorm: y = linear(LayerNorm(x)) with the norm fused into the input quantization
        self.norm = torch.nn.LayerNorm(in_features, eps=eps, device=device or "cuda") if prenorm else None
        self.mode = L.LinearMode(_VARIANTS[variant], A.SB_INT8 if fmt == "int8" else A.SB_FP8)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        # the reference's init (model.cpp:199-202): N(0, 1/n)
        self.weight = torch.nn.Parameter(torch.randn(out_features, in_features, device=dev) * in_features ** -0.5)
        self.bias = torch.nn.Parameter(torch.zeros(out_features, device=dev)) if bias else None

    def forward(self, x: torch.Tensor, residual: torch.Tensor | None = None) -> torch.Tensor:
        """y = x W^T + b (+ residual, added in the GEMM epilogue: the block's skip connection)."""
        shape = x.shape
        x2d = x.reshape(-1, self.in_features)
        r2d = residual.reshape(-1, self.out_features) if residual is not None else None
        # the fused LayerNorm + quantize kernel takes bf16 rows of <= 2048 columns, 8-aligned
        # (sb_layernorm_quantize_rowwise); anything else normalises unfused, then quantizes
        fusable = (self.mode.format == A.SB_INT8 and x.dtype == torch.bfloat16 and _ln_fusable(self.in_features)
                   and self.mode.variant in (A.SB_SWITCHBACK, A.SB_SWITCHBACK_M, A.SB_SWITCHBACK_Q))
        if self.groups > 1:
            n = self.norm
            ln_ok = n is not None and x.dtype == torch.bfloat16 and _ln_fusable(self.in_features)
            if n is not None and not ln_ok:
                x2d, n = n(x2d.float()).to(x2d.dtype), None
            y = _GroupedLinearFn.apply(x2d, n.weight if n is not None else None, n.bias if n is not None else None,
                                       n.eps if n is not None else 0.0, self.weight, self.bias, self.groups, r2d)
        elif self.norm is not None and fusable:
            y = _LNLinearFn.apply(x2d, self.norm.weight, self.norm.bias, self.norm.eps, self.weight, self.bias,
                                  self.mode, r2d)
        elif self.norm is not None:  # fp8 / tensor-wise X / wide rows: LayerNorm unfused, then the layer
            h = self.norm(x2d.float()).to(x2d.dtype)
            y = _SwitchBackLinearFn.apply(h, self.weight, self.bias, self.mode, r2d)
        else:
            y = _SwitchBackLinearFn.apply(x2d, self.weight, self.bias, self.mode, r2d)
        return y.reshape(*shape[:-1], self.out_features)

    def qkv_heads(self, x: torch.Tensor, heads: int):
        """The grouped q/k/v projection (groups = 3) for attention: x [B, S, in] -> q, k, v as
        [B, heads, S, Dh] views of the packed output; their gradients go straight into the fused
        pack + quantize kernel (_QKVHeadsFn)."""
        if self.groups != 3:
            raise ValueError("qkv_heads: a groups=3 SwitchBackLinear")
        B, S = x.shape[0], x.shape[1]
        x2d = x.reshape(-1, self.in_features)
        n = self.norm
        ln_ok = n is not None and x.dtype == torch.bfloat16 and _ln_fusable(self.in_features)
        if n is not None and not ln_ok:
            x2d, n = n(x2d.float()).to(x2d.dtype), None
        return _QKVHeadsFn.apply(x2d, n.weight if n is not None else None, n.bias if n is not None else None,
                                 n.eps if n is not None else 0.0, self.weight, self.bias, B, S, heads)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, bias={self.bias is not None}"
                + (f", groups={self.groups}" if self.groups > 1 else ""))


def _ln_fusable(cols: int) -> bool:
    return cols <= 2048 and cols % 8 == 0


def _ln_backward(dh, x2d, mean, rstd, ln_w, ln_b, needs):
    """LayerNorm backward with the forward's own mean / rstd: our bf16-in / bf16-out kernel
    (sb_layernorm_backward, fp32 math, deterministic column sums) for rows of <= 1280 columns,
    else torch's fp32 kernel."""
    if x2d.shape[1] <= 1280 and x2d.shape[1] % 8 == 0:
        dx, dg, db = L.layernorm_backward(dh, x2d, mean, rstd, ln_w.detach())
        return (dx if needs[0] else None), (dg if needs[1] else None), (db if needs[2] else None)
    dx, dg, db = torch.ops.aten.native_layer_norm_backward(
        dh.float(), x2d.float(), [x2d.shape[1]], mean.view(-1, 1), rstd.view(-1, 1), ln_w.detach().float(),
        ln_b.detach().float(), list(needs))
    return (dx.to(x2d.dtype) if dx is not None else None), dg, db


class _LNLinearFn(torch.autograd.Function):
    """y = SwitchBackLinear(LayerNorm(x)) with the normalisation fused into the row-wise
    quantization of the linear's input (sb_layernorm_quantize_rowwise + prequantized forward)."""

    @staticmethod
    def forward(ctx, x2d, ln_w, ln_b, eps: float, weight, bias, mode: L.LinearMode, resid=None):
        x2d = x2d.contiguous()
        h, hq, mean, rstd = L.layernorm_quantize_rowwise(x2d, ln_w.detach(), ln_b.detach(), eps, check=False)
        w = weight.detach().to(x2d.dtype).contiguous()
        lctx = L.LinearContext()
        y = L.linear_forward(mode, h, w, lctx, check=False, bias=bias.detach().float() if bias is not None else None,
                             x_q=hq, residual=resid.detach() if resid is not None else None)
        ctx.state = (x2d, mean, rstd, lctx, w)
        ctx.ln = (ln_w, ln_b)
        ctx.mode = mode
        ctx.has_bias = bias is not None
        return y

    @staticmethod
    def backward(ctx, g):
        x2d, mean, rstd, lctx, _ = ctx.state
        g = g.contiguous()
        dh, dw = L.linear_backward(ctx.mode, lctx, g, check=False)
        db = L.column_sums(g) if ctx.has_bias and ctx.needs_input_grad[5] else None
        dx, dg, dbeta = _ln_backward(dh, x2d, mean, rstd, *ctx.ln, ctx.needs_input_grad[:3])
        ctx.state = None
        return dx, dg, dbeta, None, dw, db, None, (g if ctx.needs_input_grad[7] else None)


def _grouped_forward(ctx, x2d, ln_w, ln_b, eps, weight, bias, groups, resid=None):
    x2d = x2d.contiguous()
    dt = x2d.dtype
    if ln_w is not None:
        h, hq, mean, rstd = L.layernorm_quantize_rowwise(x2d, ln_w.detach(), ln_b.detach(), eps, check=False)
        ln_state = (x2d, mean, rstd)
    else:
        h, hq, ln_state = x2d, L.quantize_rowwise(x2d, check=False), None
    m, n = weight.shape
    mg = m // groups
    w = weight.detach().to(dt).contiguous()
    wq = torch.empty((m, n), dtype=torch.int8, device=w.device)
    scale = torch.empty(m, dtype=torch.float32, device=w.device)
    wts = []
    for i in range(groups):
        q, qt = L.quantize_tensorwise(w[i * mg:(i + 1) * mg], check=False, with_transpose=True)
        wq[i * mg:(i + 1) * mg] = q.payload
        scale[i * mg:(i + 1) * mg] = q.state.expand(mg)
        wts.append(qt)
    y = L.int8_gemm_epilogue(hq, L.QuantizedMatrix(wq, scale, L.ROW), out_dtype=dt,
                             bias=bias.detach().float().contiguous() if bias is not None else None,
                             residual=resid.detach() if resid is not None else None)
    ctx.state = (h, wts, ln_state, groups)
    ctx.ln = (ln_w, ln_b)
    ctx.has_bias = bias is not None
    return y


def _grouped_backward(ctx, g, gqs=None):
    """dX = sum_i dequant(qrow(G_i) . W_i^T-payload) through the residual epilogue, one dW GEMM over
    the packed G; gqs: the groups' row-wise payloads when a producer already made them."""
    h, wts, ln_state, groups = ctx.state
    g = g.contiguous()
    mg = g.shape[1] // groups
    dx = None
    for i, wt in enumerate(wts):
        gq = gqs[i] if gqs is not None else L.quantize_rowwise(g[:, i * mg:(i + 1) * mg], check=False)  # own row scales
        dx = L.int8_gemm_epilogue(gq, wt, out_dtype=g.dtype, residual=dx)  # dX_0 + dX_1 + ... in order
    dw = L.wgrad(g, h, exact=False)
    db = L.column_sums(g) if ctx.has_bias and ctx.needs_input_grad[5] else None
    dg = dbeta = None
    if ln_state is not None:
        x2d, mean, rstd = ln_state
        dx, dg, dbeta = _ln_backward(dx, x2d, mean, rstd, *ctx.ln, ctx.needs_input_grad[:3])
    ctx.state = None
    return dx, dg, dbeta, dw, db


class _GroupedLinearFn(torch.autograd.Function):
    """`groups` SwitchBack int8 linears of one input, each with its own tensor-wise W scale
    (model.cpp:303-305): the input's row-wise quantization once (fused with the LayerNorm when
    prenorm), the groups' weights quantized into one packed payload, ONE GEMM with the
    per-column scale of each group (row x row dequant mode, + bias fused). Backward: each
    group's output gradient quantized row-wise on its own (a column slice, read in place), the
    groups' dX products summed through the GEMM's residual epilogue, one dW GEMM for all groups."""

    @staticmethod
    def forward(ctx, x2d, ln_w, ln_b, eps, weight, bias, groups, resid=None):
        return _grouped_forward(ctx, x2d, ln_w, ln_b, eps, weight, bias, groups, resid)

    @staticmethod
    def backward(ctx, g):
        dx, dg, dbeta, dw, db = _grouped_backward(ctx, g)
        return dx, dg, dbeta, None, dw, db, None, (g if ctx.needs_input_grad[7] else None)


class _QKVHeadsFn(torch.autograd.Function):
    """The grouped q/k/v projection handing attention its heads: forward returns q, k, v as
    [B, H, S, Dh] views of the packed output; backward receives the attention gradients in that
    head-major layout and turns them into the packed G plus the three projections' row-wise
    payloads in ONE kernel (sb_heads_pack_quantize) — the layout copy a caller would otherwise
    make, with the quantization riding on it — then runs the grouped backward."""

    @staticmethod
    def forward(ctx, x2d, ln_w, ln_b, eps, weight, bias, B, S, H):
        y = _grouped_forward(ctx, x2d, ln_w, ln_b, eps, weight, bias, 3)
        ctx.heads = (B, S, H)
        t = y.view(B, S, 3, H, y.shape[1] // (3 * H))
        return tuple(t[:, :, i].transpose(1, 2) for i in range(3))

    @staticmethod
    def backward(ctx, dq, dk, dv):
        g, gqs = L.heads_pack_quantize(dq, dk, dv, check=False)
        dx, dg, dbeta, dw, db = _grouped_backward(ctx, g, gqs)
        return dx, dg, dbeta, None, dw, db, None, None, None


class _SwitchBackMLPFn(torch.autograd.Function):
    """fc1 -> GELU -> fc2 with the producer fusions of SURVEY.md §8f row 1: GELU writes fc2's
    row-wise int8 input in the same pass (sb_gelu_quantize_rowwise), and GELU's backward
    writes fc1's quantized output gradient (sb_gelu_backward_quantize_rowwise), so neither
    activation is re-read just to be quantized."""

    @staticmethod
    def forward(ctx, x2d, ln_w, ln_b, eps, w1, b1, w2, b2, mode: L.LinearMode, resid=None):
        dt = x2d.dtype
        x2d = x2d.contiguous()
        w1b, w2b = w1.detach().to(dt).contiguous(), w2.detach().to(dt).contiguous()
        c1, c2 = L.LinearContext(), L.LinearContext()
        ln_state = None
        if ln_w is not None:  # pre-norm: LayerNorm fused with fc1's input quantization
            h, hq, mean, rstd = L.layernorm_quantize_rowwise(x2d, ln_w.detach(), ln_b.detach(), eps, check=False)
            ln_state = (x2d, mean, rstd)
        else:
            h, hq = x2d, None
        pre = L.linear_forward(mode, h, w1b, c1, check=False, bias=b1.detach().float() if b1 is not None else None,
                               x_q=hq)
        act, act_q = L.gelu_quantize_rowwise(pre, check=False)
        y = L.linear_forward(mode, act, w2b, c2, check=False, bias=b2.detach().float() if b2 is not None else None,
                             x_q=act_q, residual=resid.detach() if resid is not None else None)
        ctx.state = (c1, c2, pre, w1b, w2b, h, hq, ln_state)
        ctx.ln = (ln_w, ln_b)
        ctx.mode = mode
        ctx.bias = (b1 is not None, b2 is not None)
        return y

    @staticmethod
    def backward(ctx, gy):
        c1, c2, pre, _, _, _, _, ln_state = ctx.state
        gy = gy.contiguous()
        dact, dw2 = L.linear_backward(ctx.mode, c2, gy, check=False)
        g1, g1_q = L.gelu_backward_quantize_rowwise(dact, pre, check=False)
        dx, dw1 = L.linear_backward(ctx.mode, c1, g1, check=False, g_q=g1_q)
        db1 = L.column_sums(g1) if ctx.bias[0] and ctx.needs_input_grad[5] else None
        db2 = L.column_sums(gy) if ctx.bias[1] and ctx.needs_input_grad[7] else None
        dg = dbeta = None
        if ln_state is not None:
            x2d, mean, rstd = ln_state
            dx, dg, dbeta = _ln_backward(dx, x2d, mean, rstd, *ctx.ln, ctx.needs_input_grad[:3])
        ctx.state = None
        return dx, dg, dbeta, None, dw1, db1, dw2, db2, None, (gy if ctx.needs_input_grad[9] else None)


class SwitchBackMLP(torch.nn.Module):
    """Transformer MLP (fc1 -> GELU -> fc2) on SwitchBack linears with the activation fused into
    the quantization of its consumer (forward) and producer-gradient (backward). bf16 inputs."""

    def __init__(self, in_features: int, hidden_features: int, out_features: int | None = None, bias: bool = True,
                 variant: str = "switchback", device=None, prenorm: bool = False, eps: float = 1e-5):
        super().__init__()
        out_features = out_features or in_features
        # prenorm: LayerNorm fused into fc1's input quantization (sb_layernorm_quantize_rowwise)
        self.norm = torch.nn.LayerNorm(in_features, eps=eps, device=device or "cuda") if prenorm else None
        self.fc1 = SwitchBackLinear(in_features, hidden_features, bias=bias, variant=variant, device=device)
        self.fc2 = SwitchBackLinear(hidden_features, out_features, bias=bias, variant=variant, device=device)
        if variant not in ("switchback", "switchback_m", "switchback_q"):
            raise ValueError("SwitchBackMLP needs an int8 row-wise variant")

    def forward(self, x: torch.Tensor, residual: torch.Tensor | None = None) -> torch.Tensor:
        """fc2(gelu(fc1(norm(x)))) (+ residual, added in fc2's GEMM epilogue)."""
        if x.dtype != torch.bfloat16:
            raise TypeError("SwitchBackMLP runs in bf16")
        shape = x.shape
        n = self.norm
        x2d = x.reshape(-1, self.fc1.in_features)
        if n is not None and not _ln_fusable(self.fc1.in_features):
            x2d, n = n(x2d.float()).to(x.dtype), None  # rows the fused LayerNorm kernel cannot take
        r2d = residual.reshape(-1, self.fc2.out_features) if residual is not None else None
        y = _SwitchBackMLPFn.apply(x2d, n.weight if n is not None else None,
                                   n.bias if n is not None else None, n.eps if n is not None else 0.0,
                                   self.fc1.weight, self.fc1.bias, self.fc2.weight, self.fc2.bias, self.fc1.mode, r2d)
        return y.reshape(*shape[:-1], self.fc2.out_features)
