"""The reference's pre-norm transformer block (model.cpp:287-408) on the B200 kernels: the
model-level caller of the SwitchBack linears, with the reference's own
API shape (model.hpp: ModelConfig / BlockParams / BlockTape, transformer_block, and the block
backward that model_backward runs per block).

The block: x' = x + ls1 * attn(norm1(x)); out = x' + ls2 * mlp(norm2(x')), attention over all
rows as one sequence (model.hpp:13), q / k / v / out and mlp w1 / w2 through the linear mode.

Two numeric modes, picked by the input dtype:

* fp32 with ``linear_mode.exact`` — the reference's numerics: LayerNorm, softmax, GELU, the
  residual and layer-scale arithmetic in fp64 with fp32 stores exactly as model.cpp writes them;
  attention products on the reference-order sequential fp32 matmul (sb_matmul_f32); the linears
  bit-exact (fp64 dequant epilogue, sequential fp32 dW). Only the fp64 reductions inside
  LayerNorm / softmax run in a different summation order, so the block matches the reference to
  rounding (tests/test_block_gpu.py).
* bf16 — the performance path: LayerNorm fused with the row-wise quantization of the q/k/v and
  w1 inputs (sb_layernorm_quantize_rowwise), GELU with w2's (sb_gelu_quantize_rowwise) and
  GELU' with w1's output gradient (sb_gelu_backward_quantize_rowwise), the bf16 LayerNorm
  backward (sb_layernorm_backward), attention on torch SDPA.

q / k / v (model.cpp:303-305): three dim x dim projections with THREE tensor-wise scales. The
row-wise quantization of their shared input is computed once and the three weights are quantized
into one packed [3 dim x dim] payload, so the forward is ONE int8 GEMM whose per-output-column
scale is the scale of the projection the column belongs to (the row x row dequant mode,
linear.cpp:78-83): y = acc * s_x * s_W(p) / 16129 per column — the same value, bit for bit, as
the three separate linears. The backward keeps the reference's three row-wise quantizations of
dq / dk / dv (each projection's gradient has its own row scales) and three dX GEMMs summed in
the reference's order (model.cpp:392-397); the three weight gradients are one dW GEMM over the
packed [dq | dk | dv].
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch
import torch.nn.functional as F

from . import _capi as A
from . import lowprec as L

LN_EPS = 1e-5  # model.cpp:10
INV_SQRT2 = 0.70710678118654752440
INV_SQRT2PI = 0.39894228040143267794
PARAM_NAMES = ["norm1_gain", "norm1_bias", "wq", "wk", "wv", "wo", "ls1", "ls2", "norm2_gain", "norm2_bias", "w1",
               "w2"]


@dataclass
class BlockConfig:
    """The block fields of ModelConfig (model.hpp:15-31)."""
    dim: int = 64
    heads: int = 4
    mlp_ratio: float = 4.0
    layer_scale_enabled: bool = True
    linear_mode: L.LinearMode = field(default_factory=lambda: L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8))

    @property
    def mlp_hidden(self) -> int:
        return int(self.mlp_ratio * self.dim)

    def check(self) -> None:  # model.cpp:16-24
        if self.dim < 1 or self.heads < 1:
            raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "model config: dimensions must be >= 1")
        if self.dim % self.heads != 0:
            raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "model config: dim must be divisible by heads")
        if self.mlp_hidden < 1:
            raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "model config: mlp hidden width must be >= 1")


@dataclass
class BlockParams:
    """BlockParams (model.hpp:38-45) as device tensors: gains / biases / layer scales [dim]
    (fp32), weights [out x in] (fp32 or bf16, the block's compute dtype)."""
    norm1_gain: torch.Tensor
    norm1_bias: torch.Tensor
    wq: torch.Tensor
    wk: torch.Tensor
    wv: torch.Tensor
    wo: torch.Tensor
    ls1: torch.Tensor | None
    ls2: torch.Tensor | None
    norm2_gain: torch.Tensor
    norm2_bias: torch.Tensor
    w1: torch.Tensor
    w2: torch.Tensor


@dataclass
class _QKV:
    """The grouped q/k/v projection's forward state: the packed weight payload and each
    projection's transposed payload / scale (for the backward)."""
    x: torch.Tensor            # the shared input (ln1 output)
    wt: list                   # 3 x QuantizedMatrix: tensor-wise W_p^T payloads (the dX operands)


@dataclass
class BlockTape:
    """BlockTape (model.hpp:74-90): what the backward needs."""
    x_in: torch.Tensor | None = None
    ln1: tuple | None = None
    ln1_out: torch.Tensor | None = None
    qkv: object = None           # _QKV (grouped) or [LinearContext x 3]
    q: torch.Tensor | None = None
    k: torch.Tensor | None = None
    v: torch.Tensor | None = None
    attn: object = None          # exact: per-head attention weights; bf16: (q, k, v leaves, output)
    attn_concat: torch.Tensor | None = None
    o_ctx: L.LinearContext | None = None
    attn_out: torch.Tensor | None = None
    x_mid: torch.Tensor | None = None
    ln2: tuple | None = None
    ln2_out: torch.Tensor | None = None
    w1_ctx: L.LinearContext | None = None
    w2_ctx: L.LinearContext | None = None
    h_pre: torch.Tensor | None = None
    h: torch.Tensor | None = None
    mlp_out: torch.Tensor | None = None


def _exact(cfg: BlockConfig, x: torch.Tensor) -> bool:
    if x.dtype == torch.float32:
        if not cfg.linear_mode.exact:
            raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "transformer_block: fp32 input needs exact linears")
        return True
    if x.dtype != torch.bfloat16 or cfg.linear_mode.exact:
        raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "transformer_block: bf16 input needs the fast linears")
    return False


def _grouped(cfg: BlockConfig) -> bool:
    """Row-wise X and per-tensor (SwitchBack) or per-row (SwitchBackQ) W: the three projections
    share X's quantization and fold into one GEMM."""
    m = cfg.linear_mode
    return m.format == A.SB_INT8 and m.variant in (A.SB_SWITCHBACK, A.SB_SWITCHBACK_Q)


# ------------------------------------------------------- reference-order fp64 helpers (exact)
def _ln_forward_exact(x, gain, bias):
    """model.cpp:34-60: fp64 mean / var / inv_std, x_hat stored as float, y from the fp64 x_hat."""
    xd = x.double()
    mean = xd.mean(1, keepdim=True)
    var = ((xd - mean) ** 2).mean(1, keepdim=True)
    inv = 1.0 / torch.sqrt(var + LN_EPS)
    xh = (xd - mean) * inv
    y = (gain.double()[None, :] * xh + bias.double()[None, :]).float()
    return y, (xh.float(), inv)


def _ln_backward_exact(dy, gain, tape):
    """model.cpp:68-96."""
    x_hat, inv = tape
    dyd, xh = dy.double(), x_hat.double()
    dxh = dyd * gain.double()[None, :]
    m1 = dxh.mean(1, keepdim=True)
    m2 = (dxh * xh).mean(1, keepdim=True)
    dx = (inv * (dxh - m1 - xh * m2)).float()
    return dx, (dyd * xh).sum(0).float(), dyd.sum(0).float()


def _residual_add(x, branch, ls):  # model.cpp:133-142: float(double(x) + s * double(branch))
    s = ls.double()[None, :] if ls is not None else 1.0
    return (x.double() + s * branch.double()).float()


def _scale_cols(d, ls):  # model.cpp:144-151
    return d if ls is None else (d.double() * ls.double()[None, :]).float()


def _ls_grad(d, branch):  # model.cpp:153-161
    return (d.double() * branch.double()).sum(0).float()


def _gelu(x):  # model.cpp:127
    xd = x.double()
    return (0.5 * xd * (1.0 + torch.erf(xd * INV_SQRT2))).float()


def _gelu_grad(x):  # model.cpp:129-131
    xd = x.double()
    return 0.5 * (1.0 + torch.erf(xd * INV_SQRT2)) + xd * INV_SQRT2PI * torch.exp(-0.5 * xd * xd)


# ------------------------------------------------------------------------- the linears
def _linear(mode, x, w, ctx, **kw):
    return L.linear_forward(mode, x, w, ctx, check=False, **kw)


def _qkv_forward(cfg, p, h, hq, tape):
    """q, k, v = h Wq^T, h Wk^T, h Wv^T (model.cpp:303-305)."""
    mode = cfg.linear_mode
    if not _grouped(cfg):
        ctxs = [L.LinearContext() for _ in range(3)]
        outs = [_linear(mode, h, w, c) for w, c in zip((p.wq, p.wk, p.wv), ctxs)]
        tape.qkv = ctxs
        return outs
    d = cfg.dim
    hq = hq if hq is not None else L.quantize_rowwise(h, check=False)
    wp = torch.empty((3 * d, d), dtype=torch.int8, device=h.device)
    scale = torch.empty(3 * d, dtype=torch.float32, device=h.device)
    wts = []
    for i, w in enumerate((p.wq, p.wk, p.wv)):
        w = w.to(h.dtype).contiguous()
        if mode.variant == A.SB_SWITCHBACK_Q:  # row-wise W (linear.cpp:131-132): per-row scales
            q = L.quantize_rowwise(w, check=False)
            wp[i * d:(i + 1) * d] = q.payload
            scale[i * d:(i + 1) * d] = q.state
            wts.append(L.quantize_columnwise(w, check=False, transposed=True))  # linear.cpp:226-229
        else:  # tensor-wise W with its transpose from the same pass (quantize.cpp:143-159)
            q, qt = L.quantize_tensorwise(w, check=False, with_transpose=True)
            wp[i * d:(i + 1) * d] = q.payload
            scale[i * d:(i + 1) * d] = q.state.expand(d)
            wts.append(qt)
    # one GEMM, per-output-column scale = its projection's scale (row x row dequant mode)
    y = L.matmul_dequant_dual_rowwise(hq, L.QuantizedMatrix(wp, scale, L.ROW), out_dtype=h.dtype, exact=mode.exact)
    tape.qkv = _QKV(h, wts)
    return y[:, :d], y[:, d:2 * d], y[:, 2 * d:]


def _qkv_backward(cfg, p, tape, dq, dk, dv):
    """(d ln1_out, dWq, dWk, dWv) (model.cpp:392-397)."""
    mode = cfg.linear_mode
    if not _grouped(cfg):
        res = [L.linear_backward(mode, c, g, check=False) for c, g in zip(tape.qkv, (dq, dk, dv))]
        dx = (res[0][0].float() + res[1][0].float()) + res[2][0].float()  # add(add(q, k), v), fp32 rounding
        return dx.to(dq.dtype), res[0][1], res[1][1], res[2][1]
    st = tape.qkv
    d = cfg.dim
    dxs = []
    for g, wt in zip((dq, dk, dv), st.wt):
        gq = L.quantize_rowwise(g.contiguous(), check=False)  # each projection's own row scales
        if mode.variant == A.SB_SWITCHBACK_Q:
            dxs.append(L.matmul_dequant_dual_rowwise(gq, wt, out_dtype=torch.float32, exact=mode.exact))
        else:
            dxs.append(L.int8_matmul_dequant(gq, wt, out_dtype=torch.float32, exact=mode.exact))
    dx = (dxs[0] + dxs[1]) + dxs[2]
    # the three weight gradients in one GEMM over the packed [dq | dk | dv] (linear.cpp:245)
    dqkv = torch.cat((dq, dk, dv), 1)
    dw = L.wgrad(dqkv, st.x, exact=mode.exact)
    return dx.to(dq.dtype), dw[:d], dw[d:2 * d], dw[2 * d:]


# ---------------------------------------------------------------------------- forward
def transformer_block(cfg: BlockConfig, params: BlockParams, x: torch.Tensor, tape: BlockTape | None = None):
    """model.cpp:287-336. x: [tokens x dim] (fp32 exact or bf16). Returns the block output."""
    cfg.check()
    if x.dim() != 2 or x.shape[1] != cfg.dim:
        raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "transformer_block: input width != dim")
    exact = _exact(cfg, x)
    tp = tape if tape is not None else BlockTape()
    p = params
    T, d, H = x.shape[0], cfg.dim, cfg.heads
    dh = d // H
    scale = 1.0 / math.sqrt(dh)
    ls1 = p.ls1 if cfg.layer_scale_enabled else None
    ls2 = p.ls2 if cfg.layer_scale_enabled else None
    mode = cfg.linear_mode
    fused_ln = not exact and _grouped(cfg) and d <= 1280 and d % 8 == 0  # K11 / K12 row limits
    tp.x_in = x

    # norm1 -> q, k, v
    hq = None
    if exact:
        h, tp.ln1 = _ln_forward_exact(x, p.norm1_gain, p.norm1_bias)
    elif fused_ln:
        h, hq, mean, rstd = L.layernorm_quantize_rowwise(x, p.norm1_gain, p.norm1_bias, LN_EPS, check=False)
        tp.ln1 = (mean, rstd)
    else:
        h = F.layer_norm(x.float(), (d,), p.norm1_gain.float(), p.norm1_bias.float(), LN_EPS).to(x.dtype)
        tp.ln1 = None
    tp.ln1_out = h
    tp.q, tp.k, tp.v = _qkv_forward(cfg, p, h, hq, tp)

    # attention over all rows, per head (model.cpp:307-322)
    if exact:
        concat = torch.empty((T, d), dtype=torch.float32, device=x.device)
        weights = []
        for hd in range(H):
            c0, c1 = hd * dh, (hd + 1) * dh
            qh, kh, vh = (t[:, c0:c1].contiguous() for t in (tp.q, tp.k, tp.v))
            s = (L.matmul(qh, kh).double() * scale).float()
            sd = s.double()
            e = torch.exp(sd - sd.max(1, keepdim=True).values)
            a = (e / e.sum(1, keepdim=True)).float()  # softmax_rows, model.cpp:107-121
            concat[:, c0:c1] = L.matmul(a, vh.t().contiguous())
            weights.append(a)
        tp.attn = weights
    else:
        qkv = [t.reshape(T, H, dh).transpose(0, 1).unsqueeze(0).detach().requires_grad_(True)
               for t in (tp.q, tp.k, tp.v)]
        with torch.enable_grad():
            o = F.scaled_dot_product_attention(*qkv)
        concat = o.detach().squeeze(0).transpose(0, 1).reshape(T, d)
        tp.attn = (qkv, o)
    tp.attn_concat = concat

    tp.o_ctx = L.LinearContext()
    tp.attn_out = _linear(mode, concat.contiguous(), p.wo.to(x.dtype).contiguous(), tp.o_ctx)
    if exact:
        tp.x_mid = _residual_add(x, tp.attn_out, ls1)
    else:
        tp.x_mid = (x.float() + (ls1.float() if ls1 is not None else 1.0) * tp.attn_out.float()).to(x.dtype)

    # norm2 -> w1 -> gelu -> w2 (model.cpp:327-333)
    tp.w1_ctx, tp.w2_ctx = L.LinearContext(), L.LinearContext()
    w1, w2 = p.w1.to(x.dtype).contiguous(), p.w2.to(x.dtype).contiguous()
    if exact:
        h2, tp.ln2 = _ln_forward_exact(tp.x_mid, p.norm2_gain, p.norm2_bias)
        tp.ln2_out = h2
        tp.h_pre = _linear(mode, h2, w1, tp.w1_ctx)
        tp.h = _gelu(tp.h_pre)
        tp.mlp_out = _linear(mode, tp.h, w2, tp.w2_ctx)
    else:
        h2q = None
        if fused_ln:
            h2, h2q, mean2, rstd2 = L.layernorm_quantize_rowwise(tp.x_mid, p.norm2_gain, p.norm2_bias, LN_EPS,
                                                                 check=False)
            tp.ln2 = (mean2, rstd2)
        else:
            h2 = F.layer_norm(tp.x_mid.float(), (d,), p.norm2_gain.float(), p.norm2_bias.float(), LN_EPS).to(x.dtype)
            tp.ln2 = None
        tp.ln2_out = h2
        tp.h_pre = _linear(mode, h2, w1, tp.w1_ctx, **({"x_q": h2q} if h2q is not None else {}))
        if fused_ln:
            tp.h, hq2 = L.gelu_quantize_rowwise(tp.h_pre, check=False)
            tp.mlp_out = _linear(mode, tp.h, w2, tp.w2_ctx, x_q=hq2)
        else:
            tp.h = F.gelu(tp.h_pre.float()).to(x.dtype)
            tp.mlp_out = _linear(mode, tp.h, w2, tp.w2_ctx)
    if exact:
        return _residual_add(tp.x_mid, tp.mlp_out, ls2)
    return (tp.x_mid.float() + (ls2.float() if ls2 is not None else 1.0) * tp.mlp_out.float()).to(x.dtype)


# --------------------------------------------------------------------------- backward
def block_backward(cfg: BlockConfig, params: BlockParams, tape: BlockTape, d_out: torch.Tensor):
    """model.cpp:341-408. Returns (d_input, grads: BlockParams of fp32 gradients)."""
    p, tp = params, tape
    exact = _exact(cfg, d_out)
    d, H = cfg.dim, cfg.heads
    dh = d // H
    scale = 1.0 / math.sqrt(dh)
    T = d_out.shape[0]
    ls1 = p.ls1 if cfg.layer_scale_enabled else None
    ls2 = p.ls2 if cfg.layer_scale_enabled else None
    mode = cfg.linear_mode
    g = {}
    fused = not exact and tp.ln2 is not None

    # out = x_mid + ls2 * mlp_out
    g["ls2"] = _ls_grad(d_out, tp.mlp_out) if ls2 is not None else None
    if exact:
        d_mlp_out = _scale_cols(d_out, ls2)
    else:
        d_mlp_out = (d_out.float() * ls2.float()).to(d_out.dtype) if ls2 is not None else d_out
    d_h, g["w2"] = L.linear_backward(mode, tp.w2_ctx, d_mlp_out.contiguous(), check=False)
    if exact:
        d_hpre = (d_h.double() * _gelu_grad(tp.h_pre)).float()
        d_ln2, g["w1"] = L.linear_backward(mode, tp.w1_ctx, d_hpre, check=False)
        ln2_dx, g["norm2_gain"], g["norm2_bias"] = _ln_backward_exact(d_ln2, p.norm2_gain, tp.ln2)
        d_xmid = (d_out + ln2_dx)  # add_into: float(double(a) + double(b)) == fp32 add
    else:
        if fused:
            d_hpre, d_hpre_q = L.gelu_backward_quantize_rowwise(d_h, tp.h_pre, check=False)
            d_ln2, g["w1"] = L.linear_backward(mode, tp.w1_ctx, d_hpre, check=False, g_q=d_hpre_q)
            ln2_dx, g["norm2_gain"], g["norm2_bias"] = L.layernorm_backward(d_ln2, tp.x_mid, *tp.ln2, p.norm2_gain)
        else:
            hp = tp.h_pre.float().requires_grad_(True)
            with torch.enable_grad():
                (d_hpre,) = torch.autograd.grad(F.gelu(hp), hp, d_h.float())
            d_ln2, g["w1"] = L.linear_backward(mode, tp.w1_ctx, d_hpre.to(d_h.dtype), check=False)
            ln2_dx, g["norm2_gain"], g["norm2_bias"] = _ln_backward_torch(d_ln2, tp.x_mid, p.norm2_gain, p.norm2_bias)
        d_xmid = (d_out.float() + ln2_dx.float()).to(d_out.dtype)

    # x_mid = x_in + ls1 * attn_out
    g["ls1"] = _ls_grad(d_xmid, tp.attn_out) if ls1 is not None else None
    if exact:
        d_attn_out = _scale_cols(d_xmid, ls1)
    else:
        d_attn_out = (d_xmid.float() * ls1.float()).to(d_xmid.dtype) if ls1 is not None else d_xmid
    d_concat, g["wo"] = L.linear_backward(mode, tp.o_ctx, d_attn_out.contiguous(), check=False)

    # attention backward (model.cpp:373-389)
    if exact:
        dq = torch.empty((T, d), dtype=torch.float32, device=d_out.device)
        dk, dv = torch.empty_like(dq), torch.empty_like(dq)
        for hd in range(H):
            c0, c1 = hd * dh, (hd + 1) * dh
            qh, kh, vh, doh = (t[:, c0:c1].contiguous() for t in (tp.q, tp.k, tp.v, d_concat))
            a = tp.attn[hd]
            da = L.matmul(doh, vh)                               # dO . V^T
            dv[:, c0:c1] = L.matmul(a.t().contiguous(), doh.t().contiguous())  # A^T . dO
            ad, dad = a.double(), da.double()
            dot = (dad * ad).sum(1, keepdim=True)
            ds = (ad * (dad - dot) * scale).float()              # softmax_backward, model.cpp:124-132
            dq[:, c0:c1] = L.matmul(ds, kh.t().contiguous())     # dS . K
            dk[:, c0:c1] = L.matmul(ds.t().contiguous(), qh.t().contiguous())  # dS^T . Q
    else:
        qkv, o = tp.attn
        go = d_concat.reshape(T, H, dh).transpose(0, 1).unsqueeze(0)
        dqh, dkh, dvh = torch.autograd.grad(o, qkv, go)
        dq, dk, dv = (t.squeeze(0).transpose(0, 1).reshape(T, d) for t in (dqh, dkh, dvh))
    d_ln1, g["wq"], g["wk"], g["wv"] = _qkv_backward(cfg, p, tp, dq, dk, dv)

    if exact:
        ln1_dx, g["norm1_gain"], g["norm1_bias"] = _ln_backward_exact(d_ln1, p.norm1_gain, tp.ln1)
        d_x = d_xmid + ln1_dx
    else:
        if tp.ln1 is not None:
            ln1_dx, g["norm1_gain"], g["norm1_bias"] = L.layernorm_backward(d_ln1, tp.x_in, *tp.ln1, p.norm1_gain)
        else:
            ln1_dx, g["norm1_gain"], g["norm1_bias"] = _ln_backward_torch(d_ln1, tp.x_in, p.norm1_gain, p.norm1_bias)
        d_x = (d_xmid.float() + ln1_dx.float()).to(d_out.dtype)
    return d_x, BlockParams(**{k: g.get(k) for k in PARAM_NAMES})


def _ln_backward_torch(dy, x, gain, bias):
    xf = x.float().requires_grad_(True)
    gf, bf = gain.float().detach().requires_grad_(True), bias.float().detach().requires_grad_(True)
    with torch.enable_grad():
        y = F.layer_norm(xf, (x.shape[1],), gf, bf, LN_EPS)
        dx, dg, db = torch.autograd.grad(y, (xf, gf, bf), dy.float())
    return dx.to(x.dtype), dg, db
