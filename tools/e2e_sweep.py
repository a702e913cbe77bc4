"""Host-buffer pipeline (sb_switchback_fwd_bwd_host) throughput at config 2 for the current
SB_HOST_CHUNK / SB_HOST_SLOTS environment.

    SB_HOST_CHUNK=2048 SB_HOST_SLOTS=4 python tools/e2e_sweep.py
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_13013_b200 import lowprec as L

T = 256 * 257
g = torch.Generator().manual_seed(7)
bufs = []
for n, m in ((1280, 5120), (5120, 1280)):
    bufs.append((torch.randn(T, n, generator=g).bfloat16().pin_memory(), (torch.randn(m, n, generator=g) / n ** 0.5).bfloat16().pin_memory(),
                 torch.randn(T, m, generator=g).bfloat16().pin_memory()))
for mode in ("sync", "async"):
    def once():
        if mode == "sync":
            for x, w, gg in bufs:
                L.switchback_fwd_bwd_host(x, w, gg)
        else:
            L.switchback_fwd_bwd_host_many(bufs)
    for _ in range(2):
        once()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(4):
        once()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 4
    print(f"{mode} chunk={os.environ.get('SB_HOST_CHUNK', 'def')} slots={os.environ.get('SB_HOST_SLOTS', 'def')}: "
          f"{dt * 1e3:.2f} ms/step {T / dt / 1e6:.3f} M tokens/s")

# the same bytes with no compute: per layer, X and G in on one stream, Y and dX out on another
# (device buffers preallocated), chunked like the pipeline -- the PCIe bound for this pattern
if os.environ.get("PURE", "1") == "1":
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    dev = []
    for x, w, gg in bufs:
        m = w.shape[0]
        n = x.shape[1]
        dev.append((torch.empty_like(x, device="cuda"), torch.empty_like(gg, device="cuda"),
                    torch.empty(T, m, dtype=x.dtype, device="cuda"), torch.empty(T, n, dtype=x.dtype, device="cuda"),
                    torch.empty(T, m, dtype=x.dtype, pin_memory=True), torch.empty(T, n, dtype=x.dtype, pin_memory=True)))
    def pure():
        for (x, w, gg), (xd, gd, yd, dxd, yh, dxh) in zip(bufs, dev):
            with torch.cuda.stream(s_in):
                xd.copy_(x, non_blocking=True)
                gd.copy_(gg, non_blocking=True)
            with torch.cuda.stream(s_out):
                yh.copy_(yd, non_blocking=True)
                dxh.copy_(dxd, non_blocking=True)
        torch.cuda.synchronize()
    pure()
    t0 = time.perf_counter()
    for _ in range(4):
        pure()
    dt = (time.perf_counter() - t0) / 4
    print(f"pure copies (same bytes, both directions concurrent): {dt * 1e3:.2f} ms/step {T / dt / 1e6:.3f} M tokens/s")
