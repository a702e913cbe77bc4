"""Time the row-wise quantizer (sb_quantize_rowwise) at the C2 shapes; prints GB/s vs HBM peak.
SB_QUANT_KERNEL=tma selects the smem-ring kernel instead of the register kernel."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_13013_b200 import _capi as A  # noqa: E402

h = A.handle(0)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6550.0
for rows, cols in [(65792, 5120), (65792, 1280), (8192, 4096), (65792, 3840)]:
    for dt, tdt in [(A.SB_BF16, torch.bfloat16), (A.SB_F32, torch.float32)]:
        x = torch.randn(rows, cols, device="cuda").to(tdt)
        q = torch.empty(rows, cols, device="cuda", dtype=torch.int8)
        s = torch.empty(rows, device="cuda")
        flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)

        def run():
            A.check(h.lib.sb_quantize_rowwise(h.h, C.c_void_p(x.data_ptr()), dt, rows, cols, cols,
                                              C.c_void_p(q.data_ptr()), cols, C.c_void_p(s.data_ptr())))
        for _ in range(3):
            run()
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); run(); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[len(ts) // 2] * 1e-3
        byts = rows * cols * (x.element_size() + 1) + 4 * rows
        print(f"{os.environ.get('SB_QUANT_KERNEL','reg'):4s} {rows}x{cols} {str(tdt):15s} {t*1e6:8.1f} us "
              f"{byts/t/1e9:7.0f} GB/s  {byts/t/1e9/peak*100:5.1f}% of {peak:.0f}")
