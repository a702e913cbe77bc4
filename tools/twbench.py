"""Tensor-wise quantize (both layouts, one launch) of the ViT-H weight shapes, CUDA-event timed.
    python tools/twbench.py"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_13013_b200 import _capi as A

h = A.handle(0)
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for m, n in ((5120, 1280), (1280, 5120), (3840, 1280), (1280, 1280)):
    w = (torch.randn(m, n, device="cuda") / n ** 0.5).bfloat16()
    q = torch.empty(m, n, device="cuda", dtype=torch.int8)
    qt = torch.empty(n, m, device="cuda", dtype=torch.int8)
    st = torch.empty(1, device="cuda")
    run = lambda: A.check(h.lib.sb_quantize_tensorwise(h.h, P(w), A.SB_BF16, m, n, n, P(q), n, P(qt), m, P(st)))  # noqa: E731
    for _ in range(5):
        run()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(20):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    print(f"tensorwise {m}x{n}: median {ts[len(ts) // 2]:.1f} us (min {ts[0]:.1f}); bound {4 * m * n / 6.55e6:.1f} us")
