"""CPU: the C-ABI library loads and exports every entry point include/switchback_b200.h declares;
without a device the product path fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2304_13013_b200 import _capi as A

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "switchback_b200.h")


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?\s\**)?(sb_[a-z0-9_]+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    assert declared_symbols() == sorted(A.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = A.load()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.sb_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", A.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    L = A.load()
    h = C.c_void_p()
    st = L.sb_create(0, C.byref(h))
    assert st != A.SB_OK
    assert b"no CUDA device" in L.sb_last_error()
    with pytest.raises(A.SBError):
        A.handle(0)


def test_lowprec_shim_exports_reference_api():
    """liblowprec_b200.so serves the reference's lowprec:: signatures (INTEGRATION.md option A)."""
    import subprocess

    shim = os.path.join(os.path.dirname(A.LIB_PATH), "liblowprec_b200.so")
    if not os.path.exists(shim):
        pytest.skip("shim not built")
    syms = subprocess.run(["nm", "-DC", "--defined-only", shim], capture_output=True, text=True).stdout
    for name in ["lowprec::quantize_rowwise(lowprec::Matrix const&)", "lowprec::quantize_tensorwise_transpose(",
                 "lowprec::int8_matmul_dequant(", "lowprec::matmul_dequant_dual_rowwise(", "lowprec::linear_forward(",
                 "lowprec::linear_backward(", "lowprec::optimizer_step(", "lowprec::dequantize(",
                 "lowprec::quantize_fp8(", "lowprec::matmul("]:
        assert name in syms, name


def test_pytorch_modules_have_no_cpu_fallback():
    """The nn layer and the fused producer ops refuse CPU tensors instead of computing
    anything on the host (the product path is the CUDA library or nothing)."""
    import torch

    from paper_2304_13013_b200 import lowprec as Lp
    from paper_2304_13013_b200.nn import SwitchBackLinear

    mod = SwitchBackLinear(16, 8, device="cpu")
    with pytest.raises(Lp.InvalidArgument):
        mod(torch.randn(4, 16).bfloat16())
    x = torch.randn(4, 16).bfloat16()
    with pytest.raises(Lp.InvalidArgument):
        Lp.gelu_quantize_rowwise(x)
    with pytest.raises(Lp.InvalidArgument):
        Lp.layernorm_quantize_rowwise(x, torch.ones(16), torch.zeros(16))
    with pytest.raises(Lp.InvalidArgument):
        Lp.linear_forward(Lp.LinearMode(A.SB_SWITCHBACK, A.SB_INT8), x, torch.randn(8, 16).bfloat16())


def test_workspace_layout_offsets():
    """sb_linear_workspace_layout (no device needed): operands are 256-byte aligned, in the
    carve order, non-overlapping, and inside sb_linear_workspace_size."""
    L = A.load()
    mode = A.LinearMode(A.SB_SWITCHBACK, A.SB_INT8, 0, 1, 0)
    b, n, m = 1000, 384, 520
    lay = A.LinearWsLayout()
    assert L.sb_linear_workspace_layout(C.byref(mode), b, n, m, C.byref(lay)) == 0
    total = C.c_size_t()
    assert L.sb_linear_workspace_size(C.byref(mode), b, n, m, C.byref(total)) == 0
    assert lay.total == total.value
    spans = [(lay.x_q, b * n), (lay.x_state, 4 * b), (lay.w_q, m * n), (lay.w_q_t, m * n), (lay.w_state, 4 * m),
             (lay.g_q, b * m), (lay.g_state, 4 * b)]
    assert lay.x_q == 0
    for (o1, s1), (o2, _) in zip(spans, spans[1:]):
        assert o1 % 256 == 0 and o1 + s1 <= o2
    assert spans[-1][0] + spans[-1][1] <= lay.total
