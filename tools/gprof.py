"""One launch each of the C2 GEMMs (int8 fc1 fwd, int8 fc2 fwd, bf16 dW) for ncu captures."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_13013_b200 import _capi as A
h = A.handle(0)
T = 65792
P = lambda t: C.c_void_p(t.data_ptr())
for n, m in [(1280, 5120), (5120, 1280)]:
    xq = torch.randint(-127, 128, (T, n), device="cuda", dtype=torch.int8)
    wq = torch.randint(-127, 128, (m, n), device="cuda", dtype=torch.int8)
    sa = torch.rand(T, device="cuda")
    sb = torch.rand(1, device="cuda")
    y = torch.empty(T, m, device="cuda", dtype=torch.bfloat16)
    A.check(h.lib.sb_gemm_i8(h.h, P(xq), P(sa), P(wq), P(sb), A.SB_SCALE_ROW_TENSOR, T, m, n, P(y), A.SB_BF16, 0))
g = torch.randn(T, 1280, device="cuda").bfloat16()
x = torch.randn(T, 5120, device="cuda").bfloat16()
dw = torch.empty(1280, 5120, device="cuda")
A.check(h.lib.sb_wgrad(h.h, P(g), P(x), A.SB_BF16, T, 1280, 5120, P(dw), 0, 0))
torch.cuda.synchronize()
