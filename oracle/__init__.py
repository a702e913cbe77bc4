"""ctypes face of the parity checker — TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liboracle.so`` (our C restatement of the reference path,
oracle/oracle.c) and, when present, ``oracle/_ref/libref_lowprec.so`` (the
unmodified reference sources compiled by oracle/Makefile). Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline / reference arm may
import this package; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libref_lowprec.so")

ROW, COL, TENSOR, TENSOR_T = 0, 1, 2, 3
E4M3 = (4, 3, 7, 0)  # ebits, mbits, bias, reserved_top_exponent (quantize.hpp:30)
E5M2 = (5, 2, 15, 1)  # (quantize.hpp:31)

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_lib = None
_ref = None


def build():
    """Build liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_quantize_int8.argtypes = [_f32p, C.c_int64, C.c_int64, C.c_int, _i8p, _f32p]
        L.orc_quantize_tensorwise_transpose.argtypes = [_f32p, C.c_int64, C.c_int64, _i8p, _f32p]
        L.orc_dequantize_int8.argtypes = [_i8p, _f32p, C.c_int, C.c_int64, C.c_int64, _f32p]
        L.orc_fp8_value_set.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _f32p]
        L.orc_fp8_cast_scalar.argtypes = [C.c_float, _f32p, C.c_int]
        L.orc_fp8_cast_scalar.restype = C.c_float
        L.orc_quantize_fp8.argtypes = [_f32p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, _f32p, _f32p]
        L.orc_int8_gemm.argtypes = [_i8p, _f32p, C.c_int64, _i8p, _f32p, C.c_int64, C.c_int64, C.c_int64,
                                    C.c_int64, C.c_void_p, C.c_void_p]
        L.orc_matmul_f32.argtypes = [_f32p, _f32p, C.c_int64, C.c_int64, C.c_int64, _f32p]
        L.orc_wgrad_f32.argtypes = [_f32p, _f32p, C.c_int64, C.c_int64, C.c_int64, _f32p]
        L.orc_switchback_forward.argtypes = [_f32p, _f32p, C.c_int64, C.c_int64, C.c_int64, _f32p]
        L.orc_switchback_backward.argtypes = [_f32p, _f32p, _f32p, C.c_int64, C.c_int64, C.c_int64,
                                              _f32p, _f32p]
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_gaussian_matrix.argtypes = [C.c_int64, C.c_int64, C.c_float, C.c_float, C.c_uint64, _f32p]
        L.orc_uniform_int_stream.argtypes = [C.c_uint64, C.c_int64, C.c_int64, _i64p]
        L.orc_debias.argtypes = [C.c_double, C.c_int64]
        L.orc_debias.restype = C.c_double
        L.orc_beta2_warmup.argtypes = [C.c_int64, C.c_double]
        L.orc_beta2_warmup.restype = C.c_double
        L.orc_compute_rms.argtypes = [_f32p, _f32p, C.c_int64, C.c_double]
        L.orc_compute_rms.restype = C.c_double
        pp = C.POINTER(C.c_void_p)
        L.orc_stableadamw_step.argtypes = [C.c_int, pp, pp, pp, pp, _i64p, C.c_double, C.c_double,
                                           C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                           C.c_double, C.c_int64, _f64p, _f64p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The unmodified reference library (oracle/_ref). Raises if not built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            raise FileNotFoundError(f"{REF_PATH} not built (needs /root/reference; see oracle/Makefile)")
        L = C.CDLL(REF_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_gaussian_matrix.argtypes = [C.c_int64, C.c_int64, C.c_float, C.c_float, C.c_uint64, _f32p]
        L.ref_quantize_int8.argtypes = [_f32p, C.c_int64, C.c_int64, C.c_int, _i8p, _f32p]
        L.ref_quantize_fp8.argtypes = [_f32p, C.c_int64, C.c_int64, C.c_int, C.c_int, _f32p, _f32p]
        L.ref_fp8_value_set.argtypes = [C.c_int, _f32p]
        L.ref_dequantize_int8.argtypes = [_i8p, _f32p, C.c_int, C.c_int64, C.c_int64, _f32p]
        L.ref_int8_matmul.argtypes = [_f32p, _f32p, C.c_int64, C.c_int64, C.c_int64, C.c_int, _f32p]
        L.ref_matmul.argtypes = [_f32p, _f32p, C.c_int64, C.c_int64, C.c_int64, _f32p]
        L.ref_linear_fwd_bwd.argtypes = [C.c_int, C.c_int, _f32p, _f32p, C.c_void_p, C.c_int64, C.c_int64,
                                         C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_switchback_fwd_bwd_threaded.argtypes = [_f32p, _f32p, _f32p, C.c_int64, C.c_int64, C.c_int64,
                                                      C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_switchback_mlp_fwd_bwd_threaded.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_int64, C.c_int64,
                                                          C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                                          C.c_void_p, C.c_void_p]
        L.ref_block_fwd_bwd.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                        C.POINTER(C.c_void_p), _f32p, _f32p, _f32p, _f32p, C.POINTER(C.c_void_p)]
        pp = C.POINTER(C.c_void_p)
        L.ref_optimizer_step.argtypes = [C.c_int, pp, pp, pp, pp, _i64p, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_double, C.c_int, C.c_double, C.c_int64,
                                         _f64p, _f64p]
        _ref = L
    return _ref


class OracleError(ValueError):
    pass


_ERRS = {1: "empty matrix", 2: "non-finite input", 3: "invalid argument"}


def _chk(rc, op):
    if rc != 0:
        raise OracleError(f"{op}: {_ERRS.get(rc, rc)}")


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ------------------------------------------------------------------ oracle API
def derive_seed(seed, stream):
    return lib().orc_derive_seed(seed, stream)


def gaussian_matrix(rows, cols, mean, stdev, seed):
    out = np.empty((rows, cols), np.float32)
    _chk(lib().orc_gaussian_matrix(rows, cols, mean, stdev, seed, out), "gaussian_matrix")
    return out


def uniform_int_stream(seed, n, count):
    out = np.empty(count, np.int64)
    lib().orc_uniform_int_stream(seed, n, count, out)
    return out


def quantize(x, axis):
    """int8 quantize: axis ROW/COL/TENSOR/TENSOR_T -> (payload int8, state f32)."""
    x = _f32(x)
    r, c = x.shape
    if axis == TENSOR_T:
        q = np.empty((c, r), np.int8)
        st = np.empty(1, np.float32)
        _chk(lib().orc_quantize_tensorwise_transpose(x, r, c, q, st), "quantize_tensorwise_transpose")
        return q, st
    q = np.empty((r, c), np.int8)
    st = np.empty(r if axis == ROW else c if axis == COL else 1, np.float32)
    _chk(lib().orc_quantize_int8(x, r, c, axis, q, st), "quantize")
    return q, st


def dequantize(q, state, axis):
    q = np.ascontiguousarray(q, np.int8)
    r, c = q.shape
    y = np.empty((r, c), np.float32)
    lib().orc_dequantize_int8(q, _f32(state), axis, r, c, y)
    return y


def fp8_value_set(fmt=E4M3):
    out = np.empty(512, np.float32)
    n = lib().orc_fp8_value_set(*fmt, out)
    return out[:n].copy()


def quantize_fp8(x, fmt, axis):
    x = _f32(x)
    r, c = x.shape
    p = np.empty((r, c), np.float32)
    st = np.empty(r if axis == ROW else c if axis == COL else 1, np.float32)
    _chk(lib().orc_quantize_fp8(x, r, c, *fmt, axis, p, st), "quantize_fp8")
    return p, st


def int8_gemm(qa, sa, qb, sb, want_raw=True):
    """acc = qa @ qb.T (exact, int64); y = f32(double(acc)*sa_i*sb_j/16129).
    sa/sb: per-row states (len rows) or a single tensor state (len 1)."""
    qa = np.ascontiguousarray(qa, np.int8)
    qb = np.ascontiguousarray(qb, np.int8)
    sa, sb = _f32(sa), _f32(sb)
    r, k = qa.shape
    c = qb.shape[0]
    raw = np.empty((r, c), np.int64) if want_raw else None
    y = np.empty((r, c), np.float32)
    lib().orc_int8_gemm(qa, sa, 0 if sa.size == 1 and r != 1 else 1, qb, sb, 0 if sb.size == 1 and c != 1 else 1,
                        r, c, k, _ptr(raw), _ptr(y))
    return (raw, y) if want_raw else y


def matmul_f32(a, bt):
    a, bt = _f32(a), _f32(bt)
    y = np.empty((a.shape[0], bt.shape[0]), np.float32)
    lib().orc_matmul_f32(a, bt, a.shape[0], bt.shape[0], a.shape[1], y)
    return y


def wgrad_f32(g, x):
    g, x = _f32(g), _f32(x)
    b, m = g.shape
    n = x.shape[1]
    dw = np.empty((m, n), np.float32)
    lib().orc_wgrad_f32(g, x, b, m, n, dw)
    return dw


def switchback_forward(x, w):
    x, w = _f32(x), _f32(w)
    b, n = x.shape
    m = w.shape[0]
    y = np.empty((b, m), np.float32)
    _chk(lib().orc_switchback_forward(x, w, b, n, m, y), "linear_forward")
    return y


def switchback_backward(x, w, g):
    x, w, g = _f32(x), _f32(w), _f32(g)
    b, n = x.shape
    m = w.shape[0]
    dx = np.empty((b, n), np.float32)
    dw = np.empty((m, n), np.float32)
    _chk(lib().orc_switchback_backward(x, w, g, b, n, m, dx, dw), "linear_backward")
    return dx, dw


def compute_rms(g, u, eps):
    g, u = _f32(g).ravel(), _f32(u).ravel()
    return lib().orc_compute_rms(g, u, g.size, eps)


def _pp(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def stableadamw_step(thetas, grads, vs, us, t, alpha, beta1=0.9, beta2=0.99, beta2_warmup_lambda=0.0,
                     eps=1e-6, weight_decay=0.0, clipping=0, max_grad_norm=1.0, use_ref=False):
    """In-place StableAdamW step (optimizer.cpp:102-172) over float32 arrays.
    Returns (rms[], eta[])."""
    n = len(thetas)
    numel = np.array([a.size for a in thetas], np.int64)
    rms = np.empty(n, np.float64)
    eta = np.empty(n, np.float64)
    for a in (*thetas, *grads, *vs, *us):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    L = ref() if use_ref else lib()
    fn = L.ref_optimizer_step if use_ref else L.orc_stableadamw_step
    rc = fn(n, C.cast(_pp(thetas), C.POINTER(C.c_void_p)), C.cast(_pp(grads), C.POINTER(C.c_void_p)),
            C.cast(_pp(vs), C.POINTER(C.c_void_p)), C.cast(_pp(us), C.POINTER(C.c_void_p)), numel, alpha,
            beta1, beta2, beta2_warmup_lambda, eps, weight_decay, clipping, max_grad_norm, t, rms, eta)
    _chk(rc, "optimizer_step")
    return rms, eta


BLOCK_PARAMS = ["norm1.gain", "norm1.bias", "wq", "wk", "wv", "wo", "ls1", "ls2", "norm2.gain", "norm2.bias", "w1",
                "w2"]


def block_param_shapes(dim, hidden):
    return {"norm1.gain": (1, dim), "norm1.bias": (1, dim), "wq": (dim, dim), "wk": (dim, dim), "wv": (dim, dim),
            "wo": (dim, dim), "ls1": (1, dim), "ls2": (1, dim), "norm2.gain": (1, dim), "norm2.bias": (1, dim),
            "w1": (hidden, dim), "w2": (dim, hidden)}


def ref_block_fwd_bwd(variant, fmt, params, x, d_out, heads, mlp_ratio=4.0, layer_scale=True):
    """The reference's transformer_block + block_backward (model.cpp:287-408, run through
    model_forward / model_backward at depth 1 with identity embedding and head; oracle/_ref).
    params: dict name -> float32 array (BLOCK_PARAMS). Returns (y, dx, grads dict)."""
    x, d_out = _f32(x), _f32(d_out)
    tokens, dim = x.shape
    hidden = int(mlp_ratio * dim)
    shapes = block_param_shapes(dim, hidden)
    ps = [_f32(params[k]) if k in params else np.zeros(shapes[k], np.float32) for k in BLOCK_PARAMS]
    grads = {k: np.zeros(shapes[k], np.float32) for k in BLOCK_PARAMS}
    y = np.empty((tokens, dim), np.float32)
    dx = np.empty((tokens, dim), np.float32)
    pin = (C.c_void_p * 12)(*[a.ctypes.data for a in ps])
    pout = (C.c_void_p * 12)(*[grads[k].ctypes.data for k in BLOCK_PARAMS])
    rc = ref().ref_block_fwd_bwd(variant, fmt, tokens, dim, heads, mlp_ratio, int(layer_scale), pin, x, d_out, y, dx,
                                 pout)
    if rc != 0:
        raise OracleError(f"block: {ref().ref_last_error().decode()}")
    if not layer_scale:
        grads.pop("ls1")
        grads.pop("ls2")
    return y, dx, grads


def ref_linear(variant, fmt, x, w, g):
    """The reference's linear_forward + linear_backward (oracle/_ref): (y, dx, dw)."""
    x, w, g = _f32(x), _f32(w), _f32(g)
    b, n = x.shape
    m = w.shape[0]
    y = np.empty((b, m), np.float32)
    dx = np.empty((b, n), np.float32)
    dw = np.empty((m, n), np.float32)
    rc = ref().ref_linear_fwd_bwd(variant, fmt, x, w, _ptr(g), b, n, m, _ptr(y), _ptr(dx), _ptr(dw))
    if rc != 0:
        raise OracleError(f"linear: {ref().ref_last_error().decode()}")
    return y, dx, dw
