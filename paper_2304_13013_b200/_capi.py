"""ctypes binding of the C-ABI (include/switchback_b200.h).

The product path: every call below enqueues hand-written sm_100a kernels from
libswitchback_b200.so. If the library is missing or no B200 is visible the
calls raise — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SB_LIB_PATH") or os.path.join(PKG, "libswitchback_b200.so")  # override: A/B builds

# enums (switchback_b200.h)
SB_OK, SB_ERR_INVALID_ARGUMENT, SB_ERR_NONFINITE, SB_ERR_CUDA, SB_ERR_UNSUPPORTED = range(5)
SB_F32, SB_BF16, SB_I32, SB_I8, SB_U8, SB_I64 = range(6)
SB_AXIS_ROW, SB_AXIS_COLUMN, SB_AXIS_TENSOR = range(3)
SB_E4M3, SB_E5M2 = range(2)
SB_STANDARD, SB_SWITCHBACK, SB_SWITCHBACK_M, SB_SWITCHBACK_Q, SB_ALLQUANT = range(5)
SB_INT8, SB_FP8 = range(2)
SB_SCALE_ROW_TENSOR, SB_SCALE_ROW_ROW, SB_SCALE_NONE = range(3)
SB_CLIP_NONE, SB_CLIP_UPDATE, SB_CLIP_GRAD = range(3)
SB_GEMM_AUTO, SB_GEMM_1CTA, SB_GEMM_2CTA, SB_GEMM_WIDE, SB_GEMM_2CTA_MC = range(5)
SB_ACT_NONE, SB_ACT_GELU = range(2)

# every symbol include/switchback_b200.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "sb_abi_version", "sb_create", "sb_destroy", "sb_set_stream", "sb_synchronize", "sb_error_word",
    "sb_last_error", "sb_launch_count", "sb_quantize_rowwise", "sb_quantize_columnwise",
    "sb_quantize_tensorwise", "sb_dequantize", "sb_quantize_fp8", "sb_dequantize_fp8", "sb_gemm_i8",
    "sb_gemm_i8_epilogue", "sb_matmul_f32", "sb_wgrad", "sb_wgrad_quantize_rowwise", "sb_gemm_fp8", "sb_linear_workspace_size", "sb_linear_workspace_layout", "sb_linear_forward", "sb_linear_forward_bias",
    "sb_linear_forward_prequant", "sb_linear_backward_prequant", "sb_linear_forward_ex", "sb_quantize_tensorwise_from_absmax",
    "sb_stableadamw_step_ex", "sb_gelu_quantize_rowwise", "sb_linear_forward_residual",
    "sb_gelu_backward_quantize_rowwise", "sb_layernorm_quantize_rowwise", "sb_layernorm_backward_workspace_size",
    "sb_layernorm_backward",
    "sb_linear_backward", "sb_switchback_fwd_bwd_host", "sb_switchback_fwd_bwd_host_async",
    "sb_switchback_mlp_fwd_bwd_host", "sb_switchback_mlp_fwd_bwd_host_async",
    "sb_host_pipeline_wait", "sb_stableadamw_workspace_size", "sb_stableadamw_step",
    "sb_device_alloc", "sb_device_free", "sb_copy_to_device", "sb_copy_to_host", "sb_check_finite", "sb_fp8_cast",
    "sb_transpose_i8", "sb_column_sums", "sb_compute_rms", "sb_grad_clip_global_norm", "sb_filter_nonfinite", "sb_dequantize_values",
    "sb_set_gemm_path", "sb_dp_available", "sb_dp_unique_id", "sb_dp_init", "sb_dp_rank",
    "sb_dp_allreduce_grads_async", "sb_dp_wait", "sb_dp_allreduce_max_u32", "sb_dp_allreduce_sum_f64",
    "sb_dp_destroy", "sb_dp_symmetric_alloc", "sb_dp_symmetric_open", "sb_dp_symmetric_exchange",
    "sb_dp_symmetric_free", "sb_dp_owned_rows", "sb_wgrad_reduce_scatter", "sb_dp_barrier", "sb_dp_allgather_rows",
    "sb_dp_wgrad_allreduce_fused", "sb_stableadamw_sharded_workspace_size", "sb_stableadamw_shard_phase1",
    "sb_stableadamw_shard_phase2", "sb_stableadamw_step_sharded", "sb_dp_allreduce_max_words",
    "sb_heads_pack_quantize",
]


class SBError(RuntimeError):
    """A failing C-ABI call; .status is the sb_status code."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class InvalidArgument(SBError, ValueError):
    """Mirrors the reference's std::invalid_argument."""


class LinearMode(C.Structure):
    _fields_ = [("variant", C.c_int32), ("format", C.c_int32), ("fp8_forward", C.c_int32),
                ("fp8_gradient", C.c_int32), ("exact", C.c_int32)]


class LinearCtx(C.Structure):
    _fields_ = [("mode", LinearMode), ("b", C.c_int64), ("n", C.c_int64), ("m", C.c_int64), ("dt", C.c_int),
                ("x", C.c_void_p), ("w", C.c_void_p), ("w_q_t", C.c_void_p), ("w_state", C.c_void_p),
                ("x_q", C.c_void_p), ("x_state", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("valid", C.c_int32)]


class LinearWsLayout(C.Structure):
    _fields_ = [(f, C.c_size_t) for f in ("x_q", "x_state", "w_q", "w_q_t", "w_state", "g_q", "g_state", "total")]


class AdamwTensor(C.Structure):
    _fields_ = [("theta", C.c_void_p), ("grad", C.c_void_p), ("v", C.c_void_p), ("u", C.c_void_p),
                ("numel", C.c_int64)]


class AdamwExtras(C.Structure):
    _fields_ = [("loss_scale", C.c_double), ("per_tensor_skip", C.c_int32), ("skipped", C.c_void_p),
                ("grad_absmax", C.c_void_p), ("shadow_bf16", C.POINTER(C.c_void_p)),
                ("absmax_word", C.POINTER(C.c_void_p))]


class AdamwHparams(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("beta2_warmup_lambda", C.c_double), ("eps", C.c_double), ("weight_decay", C.c_double),
                ("max_grad_norm", C.c_double), ("clipping", C.c_int32)]


_lib = None
_lock = threading.Lock()


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load libswitchback_b200.so (building it in-tree first if it is absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if not build_if_missing:
                raise FileNotFoundError(f"{LIB_PATH} is not built (run python -m paper_2304_13013_b200.build)")
            from . import build as _b
            _b.build()
        L = C.CDLL(LIB_PATH)
        v, i64, i32, sz = C.c_void_p, C.c_int64, C.c_int, C.c_size_t
        sig = {
            "sb_abi_version": ([], C.c_int),
            "sb_create": ([i32, C.POINTER(v)], i32),
            "sb_destroy": ([v], i32),
            "sb_set_stream": ([v, v], i32),
            "sb_synchronize": ([v], i32),
            "sb_error_word": ([v], v),
            "sb_last_error": ([], C.c_char_p),
            "sb_launch_count": ([v], C.c_uint64),
            "sb_set_gemm_path": ([v, i32], i32),
            "sb_quantize_rowwise": ([v, v, i32, i64, i64, i64, v, i64, v], i32),
            "sb_quantize_columnwise": ([v, v, i32, i64, i64, i64, v, i64, v, i64, v], i32),
            "sb_quantize_tensorwise": ([v, v, i32, i64, i64, i64, v, i64, v, i64, v], i32),
            "sb_dequantize": ([v, v, i64, i64, i64, v, i32, v, i32, i64], i32),
            "sb_quantize_fp8": ([v, v, i32, i64, i64, i64, i32, i32, v, i64, v], i32),
            "sb_dequantize_fp8": ([v, v, i64, i64, i64, i32, v, i32, v, i32, i64], i32),
            "sb_gemm_i8": ([v, v, v, v, v, i32, i64, i64, i64, v, i32, i32], i32),
            "sb_gemm_i8_epilogue": ([v, v, v, v, v, i32, i64, i64, i64, v, v, i64, v, i32, i32], i32),
            "sb_matmul_f32": ([v, v, v, i64, i64, i64, v], i32),
            "sb_wgrad": ([v, v, v, i32, i64, i64, i64, v, i32, i32], i32),
            "sb_wgrad_quantize_rowwise": ([v, v, v, i32, i64, i64, i64, v, v, i64, v], i32),
            "sb_gemm_fp8": ([v, v, i32, v, i32, v, i32, v, i32, i64, i64, i64, v, i32], i32),
            "sb_linear_workspace_size": ([C.POINTER(LinearMode), i64, i64, i64, C.POINTER(sz)], i32),
            "sb_linear_workspace_layout": ([C.POINTER(LinearMode), i64, i64, i64, C.POINTER(LinearWsLayout)], i32),
            "sb_linear_forward": ([v, C.POINTER(LinearMode), v, v, i32, i64, i64, i64, v, C.POINTER(LinearCtx), v, sz],
                                  i32),
            "sb_linear_forward_bias": ([v, C.POINTER(LinearMode), v, v, v, i32, i64, i64, i64, v, C.POINTER(LinearCtx), v,
                                        sz], i32),
            "sb_linear_backward": ([v, C.POINTER(LinearMode), C.POINTER(LinearCtx), v, v, v, i32], i32),
            "sb_linear_forward_prequant": ([v, C.POINTER(LinearMode), v, v, v, v, v, i32, i64, i64, i64, v,
                                            C.POINTER(LinearCtx), v, sz], i32),
            "sb_linear_forward_ex": ([v, C.POINTER(LinearMode), v, v, v, v, v, v, v, i32, i64, i64, i64, v,
                                      C.POINTER(LinearCtx), v, sz], i32),
            "sb_quantize_tensorwise_from_absmax": ([v, v, i32, i64, i64, i64, v, v, i64, v, i64, v], i32),
            "sb_stableadamw_step_ex": ([v, C.POINTER(AdamwTensor), i32, C.POINTER(AdamwHparams), i64,
                                        C.POINTER(AdamwExtras), v, v, v, sz], i32),
            "sb_dp_available": ([C.POINTER(i32)], i32),
            "sb_dp_unique_id": ([v], i32),
            "sb_dp_init": ([v, v, i32, i32], i32),
            "sb_dp_rank": ([v, C.POINTER(i32), C.POINTER(i32)], i32),
            "sb_dp_allreduce_grads_async": ([v, C.POINTER(v), C.POINTER(i64), i32], i32),
            "sb_dp_wait": ([v], i32),
            "sb_dp_allreduce_max_u32": ([v, v, i64], i32),
            "sb_dp_allreduce_sum_f64": ([v, v, i64], i32),
            "sb_dp_destroy": ([v], i32),
            "sb_dp_symmetric_alloc": ([v, sz, C.POINTER(v), v], i32),
            "sb_dp_symmetric_open": ([v, v, i32, i32, v], i32),
            "sb_dp_symmetric_exchange": ([v, v, v], i32),
            "sb_dp_symmetric_free": ([v, v], i32),
            "sb_dp_owned_rows": ([i64, i32, i32, C.POINTER(i64), C.POINTER(i64)], i32),
            "sb_wgrad_reduce_scatter": ([v, v, v, i32, i64, i64, i64, v, v, i64, v], i32),
            "sb_dp_barrier": ([v], i32),
            "sb_heads_pack_quantize": ([v, v, v, i64, i64, i32, i32, v, v, v], i32),
            "sb_dp_allreduce_max_words": ([v, v, i32], i32),
            "sb_stableadamw_sharded_workspace_size": ([C.POINTER(AdamwTensor), i32, C.POINTER(sz)], i32),
            "sb_stableadamw_shard_phase1": ([v, C.POINTER(AdamwTensor), v, i32, C.POINTER(AdamwHparams), i64, v, v,
                                             sz], i32),
            "sb_stableadamw_shard_phase2": ([v, C.POINTER(AdamwTensor), v, i32, C.POINTER(AdamwHparams), i64, v, v, v,
                                             v, v, v, sz], i32),
            "sb_stableadamw_step_sharded": ([v, C.POINTER(AdamwTensor), v, i32, C.POINTER(AdamwHparams), i64, v, v, v,
                                             v, v, sz], i32),
            "sb_dp_allgather_rows": ([v, v, i64, i64], i32),
            "sb_dp_wgrad_allreduce_fused": ([v, v, v, i32, i64, i64, i64, v, v, i64, v], i32),
            "sb_linear_backward_prequant": ([v, C.POINTER(LinearMode), C.POINTER(LinearCtx), v, v, v, v, v, i32], i32),
            "sb_linear_forward_residual": ([v, C.POINTER(LinearMode), v, v, v, v, v, v, i32, i64, i64, i64, v,
                                            C.POINTER(LinearCtx), v, sz], i32),
            "sb_gelu_quantize_rowwise": ([v, v, i32, i64, i64, v, v, v], i32),
            "sb_gelu_backward_quantize_rowwise": ([v, v, v, i32, i64, i64, v, v, v], i32),
            "sb_layernorm_quantize_rowwise": ([v, v, i32, i64, i64, v, v, C.c_float, v, v, v, v, v], i32),
            "sb_layernorm_backward_workspace_size": ([v, i64, C.POINTER(sz)], i32),
            "sb_layernorm_backward": ([v, v, v, i32, i64, i64, v, v, v, v, v, v, v, sz], i32),
            "sb_switchback_fwd_bwd_host": ([v, C.POINTER(LinearMode), v, v, v, i32, i64, i64, i64, v, v, v], i32),
            "sb_switchback_fwd_bwd_host_async": ([v, C.POINTER(LinearMode), v, v, v, i32, i64, i64, i64, v, v, v], i32),
            "sb_switchback_mlp_fwd_bwd_host": ([v, C.POINTER(LinearMode), i32, v, v, v, v, i32, i64, i64, i64, i64,
                                                v, v, v, v], i32),
            "sb_switchback_mlp_fwd_bwd_host_async": ([v, C.POINTER(LinearMode), i32, v, v, v, v, i32, i64, i64, i64,
                                                      i64, v, v, v, v], i32),
            "sb_host_pipeline_wait": ([v], i32),
            "sb_stableadamw_workspace_size": ([C.POINTER(AdamwTensor), i32, C.POINTER(sz)], i32),
            "sb_stableadamw_step": ([v, C.POINTER(AdamwTensor), i32, C.POINTER(AdamwHparams), i64, v, v, v, sz],
                                    i32),
            "sb_device_alloc": ([v, sz, C.POINTER(v)], i32),
            "sb_device_free": ([v, v], i32),
            "sb_copy_to_device": ([v, v, v, sz], i32),
            "sb_copy_to_host": ([v, v, v, sz], i32),
            "sb_check_finite": ([v, v, i32, i64], i32),
            "sb_fp8_cast": ([v, v, i64, i32, v], i32),
            "sb_transpose_i8": ([v, v, i64, i64, v], i32),
            "sb_column_sums": ([v, v, i32, i64, i64, i64, v], i32),
            "sb_compute_rms": ([v, v, v, i64, C.c_double, v], i32),
            "sb_grad_clip_global_norm": ([v, C.POINTER(v), C.POINTER(i64), i32, C.c_double], i32),
            "sb_filter_nonfinite": ([v, C.POINTER(v), C.POINTER(v), C.POINTER(i64), i32, C.c_double, i32, v], i32),
            "sb_dequantize_values": ([v, v, i64, i64, v, i32, v], i32),
        }
        for name, (args, res) in sig.items():
            if os.environ.get("SB_LIB_PATH") and not hasattr(L, name):
                continue  # A/B runs against an older build: bind what it exports
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def check(status: int) -> None:
    if status == SB_OK:
        return
    msg = (load().sb_last_error() or b"").decode()
    if status == SB_ERR_INVALID_ARGUMENT or status == SB_ERR_NONFINITE:
        raise InvalidArgument(status, msg)
    raise SBError(status, msg)


class Handle:
    """One sb_handle per (device, stream). Follows torch's current stream on each call."""

    def __init__(self, device: int = 0):
        self.lib = load()
        self.device = device
        h = C.c_void_p()
        check(self.lib.sb_create(device, C.byref(h)))
        self.h = h

    def bind_stream(self, stream_ptr: int) -> None:
        check(self.lib.sb_set_stream(self.h, C.c_void_p(stream_ptr)))

    def synchronize(self) -> None:
        check(self.lib.sb_synchronize(self.h))

    def launches(self) -> int:
        return int(self.lib.sb_launch_count(self.h))

    def set_gemm_path(self, path: int) -> None:
        """SB_GEMM_AUTO / SB_GEMM_1CTA / SB_GEMM_2CTA (tiling only; results are identical)."""
        check(self.lib.sb_set_gemm_path(self.h, path))

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and self.h.value:
                self.lib.sb_destroy(self.h)
        except Exception:
            pass


_handles: dict[int, Handle] = {}


def handle(device: int | None = None) -> Handle:
    """The per-device handle bound to torch's current CUDA stream."""
    import torch

    if not torch.cuda.is_available():
        raise SBError(SB_ERR_CUDA, "switchback_b200: no CUDA device (the B200 path has no CPU fallback)")
    if device is None:
        device = torch.cuda.current_device()
    hd = _handles.get(device)
    if hd is None:
        hd = _handles[device] = Handle(device)
    hd.bind_stream(torch.cuda.current_stream(device).cuda_stream)
    return hd
