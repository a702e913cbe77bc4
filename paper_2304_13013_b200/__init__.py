"""B200-native SwitchBack (arXiv 2304.13013) — the lowprec hot path on sm_100a.

The drop-in boundary is the C-ABI in include/switchback_b200.h (libswitchback_b200.so);
``lowprec`` mirrors the reference's operator API on device tensors, ``dp`` shards the
token dimension across GPUs with one NCCL all-reduce of dW.
"""
from . import _capi  # noqa: F401

__all__ = ["lowprec", "dp", "build"]
