"""Python face of the reference's ``lowprec`` operator API, on B200 device tensors.

Same names, argument meaning and error behaviour as the C++ reference
(proj/core/include/lowprec/{quantize,linear,optimizer}.hpp), so parity tests read
like the reference's own tests. Tensors are torch CUDA tensors (plumbing only:
device memory and the current stream); every operation is a call through the
C-ABI (include/switchback_b200.h) into hand-written sm_100a kernels.

Differences from the reference, by design:
  * the performance path keeps bf16 activations/weights (exact=False); exact=True
    reproduces the reference's fp32 numerics bit for bit (fp64 dequant epilogue,
    sequential fp32 weight gradient),
  * non-finite inputs are detected on the device; with ``check=True`` (default for the
    drop-in API) the call synchronizes and raises InvalidArgument("<op>: non-finite input").
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import _capi as A
from ._capi import InvalidArgument, SBError  # noqa: F401  (re-exported)

ROW, COLUMN, TENSOR = A.SB_AXIS_ROW, A.SB_AXIS_COLUMN, A.SB_AXIS_TENSOR
E4M3, E5M2 = A.SB_E4M3, A.SB_E5M2

_VARIANTS = ["Standard", "SwitchBack", "SwitchBackM", "SwitchBackQ", "AllQuant"]  # linear.cpp:8-25


def to_string(variant: int) -> str:
    return _VARIANTS[variant]


def parse_linear_variant(name: str) -> int:
    if name not in _VARIANTS:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, f"unknown linear variant: {name}")
    return _VARIANTS.index(name)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return A.SB_F32
    if t.dtype == torch.bfloat16:
        return A.SB_BF16
    raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, f"unsupported dtype {t.dtype}")


def _p(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None else 0)


def _need_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda:
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "switchback_b200: tensors must live on the B200")


def _check_nonfinite(h: A.Handle, check: bool) -> None:
    if check:
        h.synchronize()


def check_error(device: int | None = None) -> None:
    """Synchronise the handle's stream and raise InvalidArgument if any kernel since the last
    check saw a non-finite input (the deferred form of the per-call check, for async /
    CUDA-graph callers such as nn.SwitchBackLinear)."""
    try:
        A.handle(device).synchronize()
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "switchback: non-finite input") from None


@dataclass
class QuantizedMatrix:
    """quantize.hpp:48-65. payload int8 (or uint8 fp8 bytes) row-major; state per axis."""
    payload: torch.Tensor
    state: torch.Tensor
    axis: int
    fp8: bool = False
    fmt: int = E4M3

    @property
    def rows(self) -> int:
        return self.payload.shape[0]

    @property
    def cols(self) -> int:
        return self.payload.shape[1]


# ------------------------------------------------------------------ quantize
def quantize_rowwise(x: torch.Tensor, check: bool = True) -> QuantizedMatrix:
    """quantize.cpp:131-133."""
    _need_cuda(x)
    if x.dim() != 2 or x.stride(1) != 1 or x.stride(0) < x.shape[1]:
        x = x.contiguous()  # row-strided views (a column slice of a wider tensor) are read in place
    r, c = x.shape
    q = torch.empty((r, c), dtype=torch.int8, device=x.device)
    st = torch.empty(r, dtype=torch.float32, device=x.device)
    h = A.handle(x.device.index)
    A.check(h.lib.sb_quantize_rowwise(h.h, _p(x), _dt(x), r, c, x.stride(0), _p(q), c, _p(st)))
    try:
        _check_nonfinite(h, check)
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "quantize_rowwise: non-finite input") from None
    return QuantizedMatrix(q, st, ROW)


def gelu_quantize_rowwise(pre: torch.Tensor, check: bool = True) -> tuple[torch.Tensor, QuantizedMatrix]:
    """Producer fusion: act = gelu(pre) (bf16) and quantize_rowwise(act)
    from one read of pre."""
    _need_cuda(pre)
    pre = pre.contiguous()
    r, c = pre.shape
    act = torch.empty_like(pre)
    q = torch.empty((r, c), dtype=torch.int8, device=pre.device)
    st = torch.empty(r, dtype=torch.float32, device=pre.device)
    h = A.handle(pre.device.index)
    A.check(h.lib.sb_gelu_quantize_rowwise(h.h, _p(pre), _dt(pre), r, c, _p(act), _p(q), _p(st)))
    _check_nonfinite(h, check)
    return act, QuantizedMatrix(q, st, ROW)


def gelu_backward_quantize_rowwise(dact: torch.Tensor, pre: torch.Tensor,
                                   check: bool = True) -> tuple[torch.Tensor, QuantizedMatrix]:
    """g = dact * gelu'(pre) (bf16) and quantize_rowwise(g) from one read of dact and pre."""
    _need_cuda(dact, pre)
    dact, pre = dact.contiguous(), pre.contiguous()
    r, c = pre.shape
    g = torch.empty_like(pre)
    q = torch.empty((r, c), dtype=torch.int8, device=pre.device)
    st = torch.empty(r, dtype=torch.float32, device=pre.device)
    h = A.handle(pre.device.index)
    A.check(h.lib.sb_gelu_backward_quantize_rowwise(h.h, _p(dact), _p(pre), _dt(pre), r, c, _p(g), _p(q), _p(st)))
    _check_nonfinite(h, check)
    return g, QuantizedMatrix(q, st, ROW)


def heads_pack_quantize(dq: torch.Tensor, dk: torch.Tensor, dv: torch.Tensor, check: bool = True):
    """sb_heads_pack_quantize: attention gradients [B, H, S, Dh] (bf16, Dh contiguous) -> the
    packed q/k/v output gradient G [B*S, 3*H*Dh] and each projection's row-wise int8 payload /
    states (== quantize_rowwise(G[:, i*D:(i+1)*D])) from one pass. Returns (G, [QuantizedMatrix]*3)."""
    _need_cuda(dq, dk, dv)
    B, H, S, Dh = dq.shape
    ts = []
    for t in (dq, dk, dv):
        if t.shape != (B, H, S, Dh) or t.dtype != torch.bfloat16:
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "heads_pack_quantize: three bf16 [B, H, S, Dh] tensors")
        ts.append(t if t.stride(3) == 1 else t.contiguous())
    D = H * Dh
    dev = dq.device
    g = torch.empty((B * S, 3 * D), dtype=torch.bfloat16, device=dev)
    qs = [torch.empty((B * S, D), dtype=torch.int8, device=dev) for _ in range(3)]
    sts = [torch.empty(B * S, dtype=torch.float32, device=dev) for _ in range(3)]
    srcs = (C.c_void_p * 3)(*[t.data_ptr() for t in ts])
    strides = (C.c_int64 * 9)(*[v for t in ts for v in (t.stride(0), t.stride(1), t.stride(2))])
    qp = (C.c_void_p * 3)(*[q.data_ptr() for q in qs])
    sp = (C.c_void_p * 3)(*[x.data_ptr() for x in sts])
    h = A.handle(dev.index)
    A.check(h.lib.sb_heads_pack_quantize(h.h, srcs, strides, B, S, H, Dh, _p(g), qp, sp))
    _check_nonfinite(h, check)
    return g, [QuantizedMatrix(q, st, ROW) for q, st in zip(qs, sts)]


def layernorm_quantize_rowwise(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float = 1e-5,
                               check: bool = True):
    """Producer fusion: out = LayerNorm(x) (bf16, fp32 affine) and quantize_rowwise(out) from
    one read of x; returns (out, QuantizedMatrix, mean, rstd) (mean / rstd fp32 per row)."""
    _need_cuda(x, gamma, beta)
    x = x.contiguous()
    r, c = x.shape
    gamma, beta = gamma.float().contiguous(), beta.float().contiguous()
    out = torch.empty_like(x)
    q = torch.empty((r, c), dtype=torch.int8, device=x.device)
    st = torch.empty(r, dtype=torch.float32, device=x.device)
    mean = torch.empty(r, dtype=torch.float32, device=x.device)
    rstd = torch.empty(r, dtype=torch.float32, device=x.device)
    h = A.handle(x.device.index)
    A.check(h.lib.sb_layernorm_quantize_rowwise(h.h, _p(x), _dt(x), r, c, _p(gamma), _p(beta), C.c_float(eps),
                                                _p(out), _p(q), _p(st), _p(mean), _p(rstd)))
    _check_nonfinite(h, check)
    return out, QuantizedMatrix(q, st, ROW), mean, rstd


def column_sums(x: torch.Tensor) -> torch.Tensor:
    """fp32 column sums of a 2-D bf16 / fp32 matrix (row stride may exceed the width): the nn
    module's bias gradient, deterministic (sb_column_sums)."""
    _need_cuda(x)
    if x.dim() != 2 or x.stride(1) != 1 or x.stride(0) < x.shape[1]:
        x = x.reshape(-1, x.shape[-1]).contiguous()
    r, c = x.shape
    out = torch.empty(c, dtype=torch.float32, device=x.device)
    h = A.handle(x.device.index)
    A.check(h.lib.sb_column_sums(h.h, _p(x), _dt(x), r, c, x.stride(0), _p(out)))
    return out


def layernorm_backward(dh: torch.Tensor, x: torch.Tensor, mean: torch.Tensor, rstd: torch.Tensor,
                       gamma: torch.Tensor):
    """Backward of layernorm_quantize_rowwise's LayerNorm: (dx bf16, dgamma fp32, dbeta fp32),
    deterministic. Rows of up to 1280 columns."""
    _need_cuda(dh, x, mean, rstd, gamma)
    dh, x = dh.contiguous(), x.contiguous()
    r, c = x.shape
    h = A.handle(x.device.index)
    nbytes = C.c_size_t()
    A.check(h.lib.sb_layernorm_backward_workspace_size(h.h, c, C.byref(nbytes)))
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=x.device)
    dx = torch.empty_like(x)
    dg = torch.empty(c, dtype=torch.float32, device=x.device)
    db = torch.empty(c, dtype=torch.float32, device=x.device)
    A.check(h.lib.sb_layernorm_backward(h.h, _p(dh), _p(x), _dt(x), r, c, _p(mean), _p(rstd),
                                        _p(gamma.float().contiguous()), _p(dx), _p(dg), _p(db), _p(ws), ws.numel()))
    return dx, dg, db


def quantize_columnwise(x: torch.Tensor, check: bool = True, transposed: bool = False) -> QuantizedMatrix:
    """quantize.cpp:135-137. transposed=True returns quantize_rowwise(x^T) (linear.cpp:228-229)."""
    _need_cuda(x)
    x = x.contiguous()
    r, c = x.shape
    st = torch.empty(c, dtype=torch.float32, device=x.device)
    h = A.handle(x.device.index)
    if transposed:
        qt = torch.empty((c, r), dtype=torch.int8, device=x.device)
        A.check(h.lib.sb_quantize_columnwise(h.h, _p(x), _dt(x), r, c, c, _p(None), 0, _p(qt), r, _p(st)))
        out = QuantizedMatrix(qt, st, ROW)
    else:
        q = torch.empty((r, c), dtype=torch.int8, device=x.device)
        A.check(h.lib.sb_quantize_columnwise(h.h, _p(x), _dt(x), r, c, c, _p(q), c, _p(None), 0, _p(st)))
        out = QuantizedMatrix(q, st, COLUMN)
    try:
        _check_nonfinite(h, check)
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "quantize_columnwise: non-finite input") from None
    return out


def quantize_tensorwise(x: torch.Tensor, check: bool = True, with_transpose: bool = False):
    """quantize.cpp:139-141. with_transpose=True also returns the transposed payload
    from the same pass (quantize.cpp:143-159) -> (q, q_t)."""
    _need_cuda(x)
    x = x.contiguous()
    r, c = x.shape
    q = torch.empty((r, c), dtype=torch.int8, device=x.device)
    qt = torch.empty((c, r), dtype=torch.int8, device=x.device) if with_transpose else None
    st = torch.empty(1, dtype=torch.float32, device=x.device)
    h = A.handle(x.device.index)
    A.check(h.lib.sb_quantize_tensorwise(h.h, _p(x), _dt(x), r, c, c, _p(q), c, _p(qt), r, _p(st)))
    try:
        _check_nonfinite(h, check)
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "quantize_tensorwise: non-finite input") from None
    if with_transpose:
        return QuantizedMatrix(q, st, TENSOR), QuantizedMatrix(qt, st, TENSOR)
    return QuantizedMatrix(q, st, TENSOR)


def quantize_tensorwise_transpose(x: torch.Tensor, check: bool = True) -> QuantizedMatrix:
    """quantize.cpp:143-159: == quantize_tensorwise(x^T), written transposed in one pass."""
    _need_cuda(x)
    x = x.contiguous()
    r, c = x.shape
    qt = torch.empty((c, r), dtype=torch.int8, device=x.device)
    st = torch.empty(1, dtype=torch.float32, device=x.device)
    h = A.handle(x.device.index)
    A.check(h.lib.sb_quantize_tensorwise(h.h, _p(x), _dt(x), r, c, c, _p(None), 0, _p(qt), r, _p(st)))
    try:
        _check_nonfinite(h, check)
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "quantize_tensorwise_transpose: non-finite input") from None
    return QuantizedMatrix(qt, st, TENSOR)


def quantize_tensorwise_from_absmax(x: torch.Tensor, absmax_word: torch.Tensor, check: bool = True,
                                    with_transpose: bool = False):
    """quantize_tensorwise with the absmax already known (the word optimizer_step_ex writes with
    the bf16 shadow weight): one pass, payloads bit-identical to quantize_tensorwise(x)."""
    _need_cuda(x, absmax_word)
    x = x.contiguous()
    r, c = x.shape
    q = torch.empty((r, c), dtype=torch.int8, device=x.device)
    qt = torch.empty((c, r), dtype=torch.int8, device=x.device) if with_transpose else None
    st = torch.empty(1, dtype=torch.float32, device=x.device)
    h = A.handle(x.device.index)
    A.check(h.lib.sb_quantize_tensorwise_from_absmax(h.h, _p(x), _dt(x), r, c, c, _p(absmax_word), _p(q), c, _p(qt),
                                                      r, _p(st)))
    try:
        _check_nonfinite(h, check)
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "quantize_tensorwise: non-finite input") from None
    if with_transpose:
        return QuantizedMatrix(q, st, TENSOR), QuantizedMatrix(qt, st, TENSOR)
    return QuantizedMatrix(q, st, TENSOR)


def quantize_fp8(x: torch.Tensor, fmt: int, axis: int, check: bool = True) -> QuantizedMatrix:
    """quantize.cpp:161-176; payload stored as e4m3/e5m2 bytes (uint8)."""
    _need_cuda(x)
    x = x.contiguous()
    r, c = x.shape
    q = torch.empty((r, c), dtype=torch.uint8, device=x.device)
    st = torch.empty(r if axis == ROW else c if axis == COLUMN else 1, dtype=torch.float32, device=x.device)
    h = A.handle(x.device.index)
    A.check(h.lib.sb_quantize_fp8(h.h, _p(x), _dt(x), r, c, c, fmt, axis, _p(q), c, _p(st)))
    try:
        _check_nonfinite(h, check)
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "quantize_fp8: non-finite input") from None
    return QuantizedMatrix(q, st, axis, fp8=True, fmt=fmt)


def dequantize(q: QuantizedMatrix, dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """quantize.cpp:178-197."""
    want = q.rows if q.axis == ROW else q.cols if q.axis == COLUMN else 1
    if q.state.numel() != want:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "dequantize: state length does not match axis")
    y = torch.empty((q.rows, q.cols), dtype=dtype, device=q.payload.device)
    h = A.handle(q.payload.device.index)
    if q.fp8:
        A.check(h.lib.sb_dequantize_fp8(h.h, _p(q.payload), q.rows, q.cols, q.cols, q.fmt, _p(q.state), q.axis,
                                        _p(y), _dt(y), q.cols))
    else:
        A.check(h.lib.sb_dequantize(h.h, _p(q.payload), q.rows, q.cols, q.cols, _p(q.state), q.axis, _p(y), _dt(y),
                                    q.cols))
    return y


# -------------------------------------------------------------------- GEMMs
def _int8_product(qa: QuantizedMatrix, qb: QuantizedMatrix, mode: int, out_dtype, exact: bool) -> torch.Tensor:
    if qa.cols != qb.cols:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "int8 matmul: inner dimension mismatch")  # linear.cpp:55
    M, K, N = qa.rows, qa.cols, qb.rows
    dev = qa.payload.device
    h = A.handle(dev.index)
    if out_dtype == "raw":
        out = torch.empty((M, N), dtype=torch.int64 if K > 133144 else torch.int32, device=dev)
        odt = A.SB_I64 if K > 133144 else A.SB_I32
        A.check(h.lib.sb_gemm_i8(h.h, _p(qa.payload), _p(None), _p(qb.payload), _p(None), A.SB_SCALE_NONE, M, N, K,
                                 _p(out), odt, 0))
        return out
    out = torch.empty((M, N), dtype=out_dtype, device=dev)
    A.check(h.lib.sb_gemm_i8(h.h, _p(qa.payload), _p(qa.state), _p(qb.payload), _p(qb.state), mode, M, N, K, _p(out),
                             _dt(out), int(exact)))
    return out


def int8_matmul_dequant(qx: QuantizedMatrix, qw: QuantizedMatrix, out_dtype=torch.float32,
                        exact: bool = True) -> torch.Tensor:
    """linear.cpp:71-76: row-wise X against tensor-wise W, int32 accumulate, dequant epilogue.
    out_dtype='raw' returns the integer accumulators."""
    if qx.fp8 or qw.fp8:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "int8_matmul_dequant: fp8 operand")
    if qx.axis != ROW or qw.axis != TENSOR:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "int8_matmul_dequant: need row-wise X and tensor-wise W")
    return _int8_product(qx, qw, A.SB_SCALE_ROW_TENSOR, out_dtype, exact)


def matmul_dequant_dual_rowwise(qa: QuantizedMatrix, qb: QuantizedMatrix, out_dtype=torch.float32,
                                exact: bool = True) -> torch.Tensor:
    """linear.cpp:78-83."""
    if qa.fp8 or qb.fp8:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "matmul_dequant_dual_rowwise: fp8 operand")
    if qa.axis != ROW or qb.axis != ROW:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT,
                              "matmul_dequant_dual_rowwise: both operands must be row-wise")
    return _int8_product(qa, qb, A.SB_SCALE_ROW_ROW, out_dtype, exact)


def int8_gemm_epilogue(qa: QuantizedMatrix, qb: QuantizedMatrix, out_dtype=torch.bfloat16, bias=None, residual=None,
                       exact: bool = False) -> torch.Tensor:
    """sb_gemm_i8_epilogue: the row x tensor (qb tensor-wise) or row x row (qb row-wise: a
    per-output-column scale) int8 product with an fp32 bias and a residual of the output dtype
    added before the single output rounding."""
    if qa.cols != qb.cols:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "int8 matmul: inner dimension mismatch")
    M, K, N = qa.rows, qa.cols, qb.rows
    dev = qa.payload.device
    out = torch.empty((M, N), dtype=out_dtype, device=dev)
    mode = A.SB_SCALE_ROW_ROW if qb.axis == ROW else A.SB_SCALE_ROW_TENSOR
    ld = 0
    if residual is not None:
        if residual.dtype != out_dtype or residual.shape != (M, N) or residual.stride(1) != 1:
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "int8 matmul: residual must be M x N of the output dtype")
        ld = residual.stride(0)
    h = A.handle(dev.index)
    A.check(h.lib.sb_gemm_i8_epilogue(h.h, _p(qa.payload), _p(qa.state), _p(qb.payload), _p(qb.state), mode, M, N, K,
                                      _p(bias), _p(residual), ld, _p(out), _dt(out), int(exact)))
    return out


def matmul(a: torch.Tensor, b_transposed: torch.Tensor) -> torch.Tensor:
    """matrix.cpp:53-68: A . B^T, sequential fp32 reduction, bit-identical to the reference."""
    _need_cuda(a, b_transposed)
    if a.shape[1] != b_transposed.shape[1]:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "matmul: inner dimension mismatch")
    a = a.contiguous().float()
    b = b_transposed.contiguous().float()
    y = torch.empty((a.shape[0], b.shape[0]), dtype=torch.float32, device=a.device)
    h = A.handle(a.device.index)
    A.check(h.lib.sb_matmul_f32(h.h, _p(a), _p(b), a.shape[0], b.shape[0], a.shape[1], _p(y)))
    return y


def wgrad(g: torch.Tensor, x: torch.Tensor, exact: bool | None = None, out: torch.Tensor | None = None,
          accumulate: bool = False) -> torch.Tensor:
    """wgrad_full_precision, linear.cpp:193-195: G^T X (fp32 out)."""
    _need_cuda(g, x)
    b, m = g.shape
    n = x.shape[1]
    if exact is None:
        exact = g.dtype == torch.float32
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=g.device)
    h = A.handle(g.device.index)
    A.check(h.lib.sb_wgrad(h.h, _p(g), _p(x), _dt(g), b, m, n, _p(out), int(exact), int(accumulate)))
    return out


def wgrad_quantize_rowwise(g: torch.Tensor, x: torch.Tensor, check: bool = True) -> tuple[torch.Tensor, QuantizedMatrix]:
    """The backward's two uses of G in one launch: (wgrad_full_precision(G, X), quantize_rowwise(G))
    (linear.cpp:232, :245). dW as wgrad(exact=False); the payload / states equal
    quantize_rowwise(G) bit for bit."""
    _need_cuda(g, x)
    g, x = g.contiguous(), x.contiguous()
    b, m = g.shape
    n = x.shape[1]
    dw = torch.empty((m, n), dtype=torch.float32, device=g.device)
    q = torch.empty((b, m), dtype=torch.int8, device=g.device)
    st = torch.empty(b, dtype=torch.float32, device=g.device)
    h = A.handle(g.device.index)
    A.check(h.lib.sb_wgrad_quantize_rowwise(h.h, _p(g), _p(x), _dt(g), b, m, n, _p(dw), _p(q), m, _p(st)))
    try:
        _check_nonfinite(h, check)
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "quantize_rowwise: non-finite input") from None
    return dw, QuantizedMatrix(q, st, ROW)


def gemm_fp8(qa: QuantizedMatrix, qb: QuantizedMatrix, out_dtype=torch.float32) -> torch.Tensor:
    """fp8 SwitchBack product (linear.cpp:151-153): snapped operands, tensor-core accumulation."""
    M, K, N = qa.rows, qa.cols, qb.rows
    out = torch.empty((M, N), dtype=out_dtype, device=qa.payload.device)
    h = A.handle(qa.payload.device.index)
    A.check(h.lib.sb_gemm_fp8(h.h, _p(qa.payload), qa.fmt, _p(qa.state), qa.axis, _p(qb.payload), qb.fmt,
                              _p(qb.state), qb.axis, M, N, K, _p(out), _dt(out)))
    return out


# -------------------------------------------------------------------- layer
@dataclass
class LinearMode:
    """linear.hpp:30-35 (+ exact: reference-bit-exact numerics)."""
    variant: int = A.SB_STANDARD
    format: int = A.SB_INT8
    fp8_forward: int = E4M3
    fp8_gradient: int = E5M2
    exact: bool = False

    def c(self) -> A.LinearMode:
        return A.LinearMode(self.variant, self.format, self.fp8_forward, self.fp8_gradient, int(self.exact))

    def __eq__(self, o) -> bool:  # linear.cpp:27-32
        if self.variant != o.variant or self.format != o.format or self.exact != o.exact:
            return False
        return self.format == A.SB_INT8 or (self.fp8_forward == o.fp8_forward and self.fp8_gradient == o.fp8_gradient)


@dataclass
class LinearContext:
    """linear.hpp:39-48. Holds the device context plus the tensors it references."""
    mode: LinearMode | None = None
    raw: A.LinearCtx = field(default_factory=A.LinearCtx)
    keep: tuple = ()
    workspace: torch.Tensor | None = None


def _workspace(mode: LinearMode, b: int, n: int, m: int, device) -> torch.Tensor:
    nbytes = C.c_size_t()
    A.check(A.load().sb_linear_workspace_size(C.byref(mode.c()), b, n, m, C.byref(nbytes)))
    return torch.empty(nbytes.value, dtype=torch.uint8, device=device)


def workspace_views(ctx: LinearContext) -> dict:
    """The int8 operands a linear wrote into its workspace (sb_linear_workspace_layout), as
    QuantizedMatrix views: "x" (row-wise X), "w" (W; tensor-wise, or row-wise for SwitchBackQ),
    "w_t" (W^T payload, tensor-wise state) and "g" (row-wise G, valid after linear_backward
    unless G came prequantized). No copies: they alias ctx.workspace."""
    r = ctx.raw
    lay = A.LinearWsLayout()
    A.check(A.load().sb_linear_workspace_layout(C.byref(ctx.mode.c()), r.b, r.n, r.m, C.byref(lay)))
    ws = ctx.workspace

    def view(off, count, dtype, shape):
        es = torch.empty((), dtype=dtype).element_size()
        return ws[off:off + count * es].view(dtype).view(*shape)

    b, n, m = r.b, r.n, r.m
    w_rows = ctx.mode.variant == A.SB_SWITCHBACK_Q
    return {
        "x": QuantizedMatrix(view(lay.x_q, b * n, torch.int8, (b, n)), view(lay.x_state, b, torch.float32, (b,)), ROW),
        "w": QuantizedMatrix(view(lay.w_q, m * n, torch.int8, (m, n)),
                             view(lay.w_state, m if w_rows else 1, torch.float32, (m if w_rows else 1,)),
                             ROW if w_rows else TENSOR),
        "w_t": QuantizedMatrix(view(lay.w_q_t, n * m, torch.int8, (n, m)), view(lay.w_state, 1, torch.float32, (1,)),
                               TENSOR),
        "g": QuantizedMatrix(view(lay.g_q, b * m, torch.int8, (b, m)), view(lay.g_state, b, torch.float32, (b,)), ROW),
    }


def linear_forward(mode: LinearMode, x: torch.Tensor, w: torch.Tensor, ctx: LinearContext | None = None,
                   workspace: torch.Tensor | None = None, check: bool = True,
                   bias: torch.Tensor | None = None, x_q: QuantizedMatrix | None = None,
                   residual: torch.Tensor | None = None, w_absmax: torch.Tensor | None = None) -> torch.Tensor:
    """linear.cpp:113-164: Y = X W^T through the variant's quantized path. `bias` (fp32, m)
    is optional and fused into the GEMM epilogue (sb_linear_forward_bias). `x_q`: X already
    quantized row-wise by its producer (gelu_quantize_rowwise), skipping that pass."""
    _need_cuda(x, w)
    if x.dim() != 2 or w.dim() != 2 or x.numel() == 0 or w.numel() == 0:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: empty operand")
    if x.shape[1] != w.shape[1]:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: X is b x n but W is not m x n")
    if x.dtype != w.dtype:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: X and W dtypes differ")
    x, w = x.contiguous(), w.contiguous()
    b, n = x.shape
    m = w.shape[0]
    if workspace is None:
        workspace = _workspace(mode, b, n, m, x.device)
    y = torch.empty((b, m), dtype=x.dtype, device=x.device)
    h = A.handle(x.device.index)
    raw = A.LinearCtx()
    if w_absmax is not None:  # W's tensor-wise absmax word from optimizer_step_ex: sb_linear_forward_ex
        if w_absmax.dtype != torch.int32 or w_absmax.numel() != 1 or not w_absmax.is_cuda:
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: w_absmax must be one int32 device word")
        if bias is not None:
            if bias.dtype != torch.float32 or bias.shape != (m,) or not bias.is_cuda:
                raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: bias must be fp32 of shape (m,)")
            bias = bias.contiguous()
        if residual is not None:
            if residual.shape != (b, m) or residual.dtype != x.dtype or not residual.is_cuda:
                raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: residual must be b x m of X's dtype")
            residual = residual.contiguous()
        st = h.lib.sb_linear_forward_ex(h.h, C.byref(mode.c()), _p(x), _p(x_q.payload if x_q else None),
                                        _p(x_q.state if x_q else None), _p(w), _p(w_absmax), _p(bias), _p(residual),
                                        _dt(x), b, n, m, _p(y), C.byref(raw), _p(workspace), workspace.numel())
    elif residual is not None:
        if residual.shape != (b, m) or residual.dtype != x.dtype or not residual.is_cuda:
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: residual must be b x m of X's dtype")
        residual = residual.contiguous()
        if bias is not None:
            if bias.dtype != torch.float32 or bias.shape != (m,) or not bias.is_cuda:
                raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: bias must be fp32 of shape (m,)")
            bias = bias.contiguous()
        st = h.lib.sb_linear_forward_residual(h.h, C.byref(mode.c()), _p(x), _p(x_q.payload if x_q else None),
                                              _p(x_q.state if x_q else None), _p(w), _p(bias), _p(residual), _dt(x),
                                              b, n, m, _p(y), C.byref(raw), _p(workspace), workspace.numel())
    elif x_q is not None:
        bp = None
        if bias is not None:
            if bias.dtype != torch.float32 or bias.shape != (m,) or not bias.is_cuda:
                raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: bias must be fp32 of shape (m,)")
            bias = bias.contiguous()
            bp = bias
        st = h.lib.sb_linear_forward_prequant(h.h, C.byref(mode.c()), _p(x), _p(x_q.payload), _p(x_q.state), _p(w), _p(bp),
                                              _dt(x), b, n, m, _p(y), C.byref(raw), _p(workspace), workspace.numel())
    elif bias is None:
        st = h.lib.sb_linear_forward(h.h, C.byref(mode.c()), _p(x), _p(w), _dt(x), b, n, m, _p(y), C.byref(raw),
                                     _p(workspace), workspace.numel())
    else:
        if bias.dtype != torch.float32 or bias.shape != (m,) or not bias.is_cuda:
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_forward: bias must be fp32 of shape (m,)")
        bias = bias.contiguous()
        st = h.lib.sb_linear_forward_bias(h.h, C.byref(mode.c()), _p(x), _p(w), _p(bias), _dt(x), b, n, m, _p(y),
                                          C.byref(raw), _p(workspace), workspace.numel())
    A.check(st)
    try:
        _check_nonfinite(h, check)
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "linear_forward: non-finite input") from None
    if ctx is not None:
        ctx.mode = mode
        ctx.raw = raw
        ctx.keep = ((x, w) if mode.variant != A.SB_SWITCHBACK_M else ()) + ((x_q,) if x_q is not None else ())
        ctx.workspace = workspace
    return y


def linear_backward(mode: LinearMode, ctx: LinearContext, g: torch.Tensor, dw: torch.Tensor | None = None,
                    dw_accumulate: bool = False, check: bool = True,
                    g_q: QuantizedMatrix | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """linear.cpp:199-278 -> (x_grad [b x n], w_grad [m x n] fp32). `g_q`: G already quantized
    row-wise by its producer (gelu_backward_quantize_rowwise)."""
    if ctx.mode is None or not (mode == ctx.mode):
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT,
                              "linear_backward: context was produced by a different mode")
    r = ctx.raw
    if g.dim() != 2 or g.shape[0] != r.b or g.shape[1] != r.m:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "linear_backward: G must be b x m")
    _need_cuda(g)
    g = g.contiguous()
    dx = torch.empty((r.b, r.n), dtype=g.dtype, device=g.device)
    if dw is None:
        dw = torch.empty((r.m, r.n), dtype=torch.float32, device=g.device)
    h = A.handle(g.device.index)
    if g_q is not None:
        A.check(h.lib.sb_linear_backward_prequant(h.h, C.byref(mode.c()), C.byref(r), _p(g), _p(g_q.payload), _p(g_q.state),
                                                  _p(dx), _p(dw), int(dw_accumulate)))
    else:
        A.check(h.lib.sb_linear_backward(h.h, C.byref(mode.c()), C.byref(r), _p(g), _p(dx), _p(dw),
                                         int(dw_accumulate)))
    try:
        _check_nonfinite(h, check)
    except InvalidArgument:
        raise InvalidArgument(A.SB_ERR_NONFINITE, "linear_backward: non-finite input") from None
    return dx, dw


def switchback_fwd_bwd_host_many(layers, exact: bool = False):
    """switchback_fwd_bwd_host over several (x, w, g) host triples (e.g. the linears of one
    step), enqueued back to back with sb_switchback_fwd_bwd_host_async so each layer's uploads
    overlap the previous layer's drain; one wait at the end. Returns [(y, dx, dw), ...]."""
    h = A.handle()
    md = LinearMode(A.SB_SWITCHBACK, A.SB_INT8, exact=exact)
    outs = []
    for x, w, g in layers:
        b, n = x.shape
        m = w.shape[0]
        y = torch.empty((b, m), dtype=x.dtype, pin_memory=True)
        dx = torch.empty((b, n), dtype=x.dtype, pin_memory=True)
        dw = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
        A.check(h.lib.sb_switchback_fwd_bwd_host_async(h.h, C.byref(md.c()), _p(x), _p(w), _p(g), _dt(x), b, n, m,
                                                       _p(y), _p(dx), _p(dw)))
        outs.append((y, dx, dw))
    A.check(h.lib.sb_host_pipeline_wait(h.h))
    return outs


def switchback_fwd_bwd_host(x, w, g, exact: bool = False):
    """bench.cpp:75-81 over HOST tensors (pinned CPU torch tensors): returns (y, dx, dw) on the
    host. Copies + kernels pipelined over token chunks inside the C-ABI call."""
    b, n = x.shape
    m = w.shape[0]
    y = torch.empty((b, m), dtype=x.dtype, pin_memory=True)
    dx = torch.empty((b, n), dtype=x.dtype, pin_memory=True)
    dw = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
    h = A.handle()
    md = LinearMode(A.SB_SWITCHBACK, A.SB_INT8, exact=exact)
    A.check(h.lib.sb_switchback_fwd_bwd_host(h.h, C.byref(md.c()), _p(x), _p(w), _p(g), _dt(x), b, n, m, _p(y),
                                             _p(dx), _p(dw)))
    return y, dx, dw


def switchback_mlp_fwd_bwd_host(x, w1, w2, g, activation: int = A.SB_ACT_NONE, exact: bool = False,
                                wait: bool = True, out=None):
    """The MLP block of transformer_block / block_backward (model.cpp:324-329, 351-360) over
    HOST tensors: y = fc2(act(fc1(x))) and its backward for the block-output gradient g, the
    hidden activation kept on the device. x (b, n), w1 (hd, n), w2 (m, hd), g (b, m) pinned CPU
    tensors; returns (y, dx, dw1, dw2) on the host. wait=False enqueues only
    (sb_switchback_mlp_fwd_bwd_host_async; call host_pipeline_wait() before reading).
    out: optional preallocated pinned (y, dx, dw1, dw2) to write into (e.g. alternating sets
    for back-to-back async calls)."""
    b, n = x.shape
    hd, m = w1.shape[0], w2.shape[0]
    if w1.shape[1] != n or w2.shape[1] != hd or tuple(g.shape) != (b, m):
        raise ValueError("switchback_mlp_fwd_bwd: shape mismatch")
    if out is not None:
        y, dx, dw1, dw2 = out
        want = (((b, m), x.dtype), ((b, n), x.dtype), ((hd, n), torch.float32), ((m, hd), torch.float32))
        for t, (shape, dtype) in zip(out, want):
            if tuple(t.shape) != shape or t.dtype != dtype or not t.is_contiguous() or t.is_cuda:
                raise ValueError("switchback_mlp_fwd_bwd: out buffers must be contiguous host tensors "
                                 "(y, dx in x's dtype; dw1, dw2 fp32) of the output shapes")
    else:
        y = torch.empty((b, m), dtype=x.dtype, pin_memory=True)
        dx = torch.empty((b, n), dtype=x.dtype, pin_memory=True)
        dw1 = torch.empty((hd, n), dtype=torch.float32, pin_memory=True)
        dw2 = torch.empty((m, hd), dtype=torch.float32, pin_memory=True)
    h = A.handle()
    md = LinearMode(A.SB_SWITCHBACK, A.SB_INT8, exact=exact)
    fn = h.lib.sb_switchback_mlp_fwd_bwd_host if wait else h.lib.sb_switchback_mlp_fwd_bwd_host_async
    A.check(fn(h.h, C.byref(md.c()), activation, _p(x), _p(w1), _p(w2), _p(g), _dt(x), b, n, hd, m, _p(y), _p(dx),
               _p(dw1), _p(dw2)))
    return y, dx, dw1, dw2


def host_pipeline_wait():
    h = A.handle()
    A.check(h.lib.sb_host_pipeline_wait(h.h))


# ---------------------------------------------------------------- optimizer
@dataclass
class OptimizerHyperparams:
    """optimizer.hpp:21-33; lr_schedule is a Python callable t -> alpha_t."""
    lr_schedule: object = None
    beta1: float = 0.9
    beta2: float = 0.99
    beta2_warmup_lambda: float = 0.0
    eps: float = 1e-6
    weight_decay: float = 0.0
    clipping: int = A.SB_CLIP_NONE
    max_grad_norm: float = 1.0


@dataclass
class TensorRef:
    """optimizer.hpp:74-79 (fp32 device tensors, updated in place)."""
    name: str
    param: torch.Tensor
    grad: torch.Tensor
    v: torch.Tensor
    u: torch.Tensor


def optimizer_step(tensors: list[TensorRef], hp: OptimizerHyperparams, t: int,
                   workspace: torch.Tensor | None = None, infos: bool = True):
    """optimizer.cpp:102-172. Returns [(rms, eta)] per tensor (TensorStepInfo), or the
    device tensor of shape [n, 2] when infos=False (no host sync)."""
    if t < 1:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "optimizer_step: t must be >= 1")
    if hp.lr_schedule is None:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "optimizer_step: lr_schedule not set")
    for r in tensors:
        if r.param is None or r.grad is None or r.v is None or r.u is None:
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "optimizer_step: null tensor reference")
        if not (r.param.shape == r.grad.shape == r.v.shape == r.u.shape):
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, f"optimizer_step: shape mismatch for {r.name}")
        for a in (r.param, r.grad, r.v, r.u):
            if a.dtype != torch.float32 or not a.is_cuda or not a.is_contiguous():
                raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "optimizer_step: tensors must be contiguous fp32 CUDA")
    n = len(tensors)
    arr = (A.AdamwTensor * max(n, 1))()
    for i, r in enumerate(tensors):
        arr[i] = A.AdamwTensor(r.param.data_ptr(), r.grad.data_ptr(), r.v.data_ptr(), r.u.data_ptr(), r.param.numel())
    dev = tensors[0].param.device if n else torch.device("cuda")
    if workspace is None:
        nbytes = C.c_size_t()
        A.check(A.load().sb_stableadamw_workspace_size(arr, n, C.byref(nbytes)))
        workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    out = torch.empty((2, max(n, 1)), dtype=torch.float64, device=dev)
    hpc = A.AdamwHparams(float(hp.lr_schedule(t)), hp.beta1, hp.beta2, hp.beta2_warmup_lambda, hp.eps,
                         hp.weight_decay, hp.max_grad_norm, int(hp.clipping))
    h = A.handle(dev.index)
    A.check(h.lib.sb_stableadamw_step(h.h, arr, n, C.byref(hpc), t, _p(out[0]), _p(out[1]), _p(workspace),
                                      workspace.numel()))
    if not infos:
        return out
    o = out.cpu()
    return [(float(o[0, i]), float(o[1, i])) for i in range(n)]


def optimizer_step_sharded(shards: list[TensorRef], numel_total: list[int], hp: OptimizerHyperparams, t: int,
                           allreduce=None, shadows: list | None = None, workspace: torch.Tensor | None = None,
                           allreduce_max=None):
    """ZeRO-1 StableAdamW (sb_stableadamw_shard_phase1 / _phase2): `shards[i]` holds this rank's
    contiguous slice of tensor i (param / grad / v / u views of the same elements), numel_total[i]
    the whole tensor's size. Between the phases the per-tensor fp64 sums of g^2 / max(u, eps^2)
    are summed over ranks by `allreduce(sums)` (in place on the float64 device tensor: e.g. a
    torch.distributed all_reduce; None = one rank, or the library's own NCCL communicator via
    sb_stableadamw_step_sharded when `allreduce == "nccl"`). shadows[i] = (bf16 view of the shard,
    int32 word) or None, as optimizer_step_ex. Returns {rms, eta} float64 device tensors."""
    if t < 1:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "optimizer_step: t must be >= 1")
    n = len(shards)
    arr = (A.AdamwTensor * max(n, 1))()
    tot = (C.c_int64 * max(n, 1))(*numel_total)
    for i, r in enumerate(shards):
        if not (r.param.numel() == r.grad.numel() == r.v.numel() == r.u.numel()):
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, f"optimizer_step: shape mismatch for {r.name}")
        arr[i] = A.AdamwTensor(r.param.data_ptr(), r.grad.data_ptr(), r.v.data_ptr(), r.u.data_ptr(), r.param.numel())
    dev = shards[0].param.device if n else torch.device("cuda")
    if workspace is None:
        nbytes = C.c_size_t()
        A.check(A.load().sb_stableadamw_sharded_workspace_size(arr, n, C.byref(nbytes)))
        workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    sh = (C.c_void_p * max(n, 1))()
    wd = (C.c_void_p * max(n, 1))()
    for i in range(n):
        s_ = shadows[i] if shadows else None
        if s_ is not None:
            sh[i], wd[i] = s_[0].data_ptr(), s_[1].data_ptr()
    shp = sh if shadows else None
    wdp = wd if shadows else None
    hpc = A.AdamwHparams(float(hp.lr_schedule(t)), hp.beta1, hp.beta2, hp.beta2_warmup_lambda, hp.eps,
                         hp.weight_decay, hp.max_grad_norm, int(hp.clipping))
    out = {"rms": torch.empty(max(n, 1), dtype=torch.float64, device=dev),
           "eta": torch.empty(max(n, 1), dtype=torch.float64, device=dev)}
    h = A.handle(dev.index)
    if allreduce == "nccl":
        A.check(h.lib.sb_stableadamw_step_sharded(h.h, arr, tot, n, C.byref(hpc), t, shp, wdp, _p(out["rms"]),
                                                  _p(out["eta"]), _p(workspace), workspace.numel()))
        return {k: v[:n] for k, v in out.items()}
    sums = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    A.check(h.lib.sb_stableadamw_shard_phase1(h.h, arr, tot, n, C.byref(hpc), t, _p(sums), _p(workspace),
                                              workspace.numel()))
    if allreduce is not None:
        allreduce(sums)
    h.bind_stream(torch.cuda.current_stream(dev).cuda_stream)
    A.check(h.lib.sb_stableadamw_shard_phase2(h.h, arr, tot, n, C.byref(hpc), t, _p(sums), shp, wdp, _p(out["rms"]),
                                              _p(out["eta"]), _p(workspace), workspace.numel()))
    if shadows and allreduce_max is not None:
        for s_ in shadows:
            if s_ is not None:
                allreduce_max(s_[1])
    return {k: v[:n] for k, v in out.items()}


@dataclass
class LossScaler:
    """optimizer.hpp:45-48."""
    scale: float = 1.0
    per_tensor_skip: bool = True


def optimizer_step_ex(tensors: list[TensorRef], hp: OptimizerHyperparams, t: int, scaler: LossScaler | None = None,
                      shadows: list | None = None, workspace: torch.Tensor | None = None):
    """The trainer's update path (trainer.cpp:127-155) fused into the optimizer's passes
    (sb_stableadamw_step_ex): filter_nonfinite's unscaling and per-tensor skip, grad_absmax
    telemetry, the in-step clip over the applied tensors, and — for tensors given a
    shadow = (bf16 tensor of the param's shape, int32 word) — the next forward's bf16 weight
    and its tensor-wise absmax. Returns a dict of device tensors: rms, eta (float64 [n]),
    skipped (int32 [n]), grad_absmax (float32 [n]); no host synchronisation."""
    if t < 1:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "optimizer_step: t must be >= 1")
    if hp.lr_schedule is None:
        raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "optimizer_step: lr_schedule not set")
    scaler = scaler or LossScaler()
    n = len(tensors)
    arr = (A.AdamwTensor * max(n, 1))()
    for i, r in enumerate(tensors):
        if not (r.param.shape == r.grad.shape == r.v.shape == r.u.shape):
            raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, f"optimizer_step: shape mismatch for {r.name}")
        arr[i] = A.AdamwTensor(r.param.data_ptr(), r.grad.data_ptr(), r.v.data_ptr(), r.u.data_ptr(), r.param.numel())
    dev = tensors[0].param.device if n else torch.device("cuda")
    if workspace is None:
        nbytes = C.c_size_t()
        A.check(A.load().sb_stableadamw_workspace_size(arr, n, C.byref(nbytes)))
        workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    out = {"rms": torch.empty(max(n, 1), dtype=torch.float64, device=dev),
           "eta": torch.empty(max(n, 1), dtype=torch.float64, device=dev),
           "skipped": torch.empty(max(n, 1), dtype=torch.int32, device=dev),
           "grad_absmax": torch.empty(max(n, 1), dtype=torch.float32, device=dev)}
    sh = (C.c_void_p * max(n, 1))()
    wd = (C.c_void_p * max(n, 1))()
    for i in range(n):
        s_ = shadows[i] if shadows else None
        if s_ is not None:
            if s_[0].dtype != torch.bfloat16 or s_[0].numel() != tensors[i].param.numel() or s_[1].dtype != torch.int32:
                raise InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "optimizer_step: shadow must be (bf16 like param, int32 word)")
            sh[i], wd[i] = s_[0].data_ptr(), s_[1].data_ptr()
    ex = A.AdamwExtras(float(scaler.scale), int(scaler.per_tensor_skip), out["skipped"].data_ptr(),
                       out["grad_absmax"].data_ptr(), sh, wd)
    hpc = A.AdamwHparams(float(hp.lr_schedule(t)), hp.beta1, hp.beta2, hp.beta2_warmup_lambda, hp.eps,
                         hp.weight_decay, hp.max_grad_norm, int(hp.clipping))
    h = A.handle(dev.index)
    A.check(h.lib.sb_stableadamw_step_ex(h.h, arr, n, C.byref(hpc), t, C.byref(ex), _p(out["rms"]), _p(out["eta"]),
                                         _p(workspace), workspace.numel()))
    return {k: v[:n] for k, v in out.items()}
