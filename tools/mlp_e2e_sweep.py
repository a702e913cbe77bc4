"""Chunk sweep of the MLP host entry (sb_switchback_mlp_fwd_bwd_host) at the C2 shape:
ms per synchronous call for each setting. argv[1]: comma list of chunk:first:taper
(first 0 = the default quarter chunk; taper 0 = fixed chunks after the first)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_13013_b200 import lowprec as L  # noqa: E402

T, n, hd, m = 65792, 1280, 5120, 1280
x = torch.randn(T, n).bfloat16().pin_memory()
w1 = (torch.randn(hd, n) / n ** 0.5).bfloat16().pin_memory()
w2 = (torch.randn(m, hd) / hd ** 0.5).bfloat16().pin_memory()
g = torch.randn(T, m).bfloat16().pin_memory()
spec = sys.argv[1] if len(sys.argv) > 1 else "8192:0:1,8192:0:0,8192:1024:1,16384:0:1,6144:0:1"
for _rep in range(2):
    for item in spec.split(","):
        chunk, first, taper = (int(v) for v in item.split(":"))
        os.environ["SB_HOST_CHUNK"] = str(chunk)
        os.environ["SB_HOST_TAPER"] = str(taper)
        if first:
            os.environ["SB_HOST_FIRST"] = str(first)
        else:
            os.environ.pop("SB_HOST_FIRST", None)
        for _ in range(2):
            L.switchback_mlp_fwd_bwd_host(x, w1, w2, g)
        t0 = time.perf_counter()
        for _ in range(5):
            L.switchback_mlp_fwd_bwd_host(x, w1, w2, g)
        ms = (time.perf_counter() - t0) / 5 * 1e3
        print(f"chunk {chunk:6d} first {first or chunk // 4:6d} taper {taper}: {ms:7.2f} ms/step "
              f"{T / ms * 1e3 / 1e6:6.2f} M tokens/s", flush=True)
