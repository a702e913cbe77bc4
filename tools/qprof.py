"""One row-wise quantize launch per kernel variant at 65792 x COLS bf16 (for ncu)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_13013_b200 import _capi as A
h = A.handle(0)
rows, cols = 65792, int(os.environ.get("COLS", "5120"))
x = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
q = torch.empty(rows, cols, device="cuda", dtype=torch.int8)
s = torch.empty(rows, device="cuda")
for _ in range(2):
    A.check(h.lib.sb_quantize_rowwise(h.h, C.c_void_p(x.data_ptr()), A.SB_BF16, rows, cols, cols,
                                      C.c_void_p(q.data_ptr()), cols, C.c_void_p(s.data_ptr())))
torch.cuda.synchronize()
