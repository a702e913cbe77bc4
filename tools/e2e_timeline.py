"""Timeline of one MLP host-entry call (sb_switchback_mlp_fwd_bwd_host at the C2 shape) from
CUPTI (torch.profiler): busy time and span of H2D copies, D2H copies and kernels, so the call's
ms can be set against the PCIe floor. Not a bench number (profiled)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2304_13013_b200 import lowprec as L  # noqa: E402

T, n, hd, m = 65792, 1280, 5120, 1280
x = torch.randn(T, n).bfloat16().pin_memory()
w1 = (torch.randn(hd, n) / n ** 0.5).bfloat16().pin_memory()
w2 = (torch.randn(m, hd) / hd ** 0.5).bfloat16().pin_memory()
g = torch.randn(T, m).bfloat16().pin_memory()
for _ in range(3):
    L.switchback_mlp_fwd_bwd_host(x, w1, w2, g)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    L.switchback_mlp_fwd_bwd_host(x, w1, w2, g)
path = "gpurun_out/e2e_trace.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")]
cls = {}
for e in ev:
    nm = e["name"]
    k = "H2D" if "HtoD" in nm else "D2H" if "DtoH" in nm else "kernel" if e["cat"] == "kernel" else nm
    cls.setdefault(k, []).append((e["ts"], e["ts"] + e["dur"], e.get("args", {}).get("bytes", 0)))
t0 = min(a for v in cls.values() for a, _, _ in v)
t1 = max(b for v in cls.values() for _, b, _ in v)
print(f"call span {(t1 - t0) / 1e3:.2f} ms")
for k, v in cls.items():
    busy = sum(b - a for a, b, _ in v)
    by = sum(x for _, _, x in v)
    s = min(a for a, _, _ in v) - t0
    e = max(b for _, b, _ in v) - t0
    print(f"{k:7s} n={len(v):4d} busy {busy / 1e3:6.2f} ms  span {s / 1e3:6.2f} .. {e / 1e3:6.2f} ms  "
          f"{by / 1e6:8.1f} MB  {by / max(busy, 1) / 1e3:6.1f} GB/s while busy")
