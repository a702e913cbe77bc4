"""ncu driver: the fc1 / fc2 dW GEMMs of C2 with and without the fused row-wise quantize of G
(sb_wgrad vs sb_wgrad_quantize_rowwise), one launch each after a warm-up.

    ncu --set full -k regex:k_dw_wide -s 4 -c 4 -o gpurun_out/prof_dwq python tools/prof_dwq.py
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_13013_b200 import _capi as A  # noqa: E402

h = A.handle(0)
T = 65792
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for rep in range(2):  # first pass = warm-up (ncu -s skips it)
    for m, n in [(5120, 1280), (1280, 5120)]:
        g = torch.randn(T, m, device="cuda").bfloat16()
        x = torch.randn(T, n, device="cuda").bfloat16()
        dw = torch.empty(m, n, device="cuda")
        gq = torch.empty(T, m, device="cuda", dtype=torch.int8)
        gs = torch.empty(T, device="cuda")
        A.check(h.lib.sb_wgrad(h.h, P(g), P(x), A.SB_BF16, T, m, n, P(dw), 0, 0))
        A.check(h.lib.sb_wgrad_quantize_rowwise(h.h, P(g), P(x), A.SB_BF16, T, m, n, P(dw), P(gq), m, P(gs)))
        torch.cuda.synchronize()
