"""Per-kernel HBM rate of the bandwidth-bound kernels at the ViT-H shapes (CUDA events over 20
back-to-back launches each, inputs larger than L2): algorithmic bytes / time against the measured
HBM peak. Not the bench; the A/B tool for these kernels."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_13013_b200 import _capi as A  # noqa: E402
from paper_2304_13013_b200 import lowprec as L  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = 6457.7
p = os.path.join(ROOT, "MEASURED_PEAKS.json")
if os.path.exists(p):
    peak = json.load(open(p))["hbm_gbs"]
T = 256 * 257


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1000.0


rows = []


def report(name, us, nbytes):
    gbs = nbytes / us / 1e3
    rows.append((name, us, gbs, gbs / peak))
    print(f"{name:44s} {us:8.1f} us {gbs:7.0f} GB/s  {gbs / peak:5.1%} of HBM", flush=True)


x5 = torch.randn(T, 5120, device="cuda").bfloat16()
x1 = torch.randn(T, 1280, device="cuda").bfloat16()
report("quantize_rowwise bf16 65792x5120", timeit(lambda: L.quantize_rowwise(x5, check=False)), T * 5120 * 3 + 4 * T)
report("quantize_rowwise bf16 65792x1280", timeit(lambda: L.quantize_rowwise(x1, check=False)), T * 1280 * 3 + 4 * T)
for fmt, nm in ((A.SB_E4M3, "e4m3"), (A.SB_E5M2, "e5m2")):
    report(f"quantize_fp8 rows {nm} 65792x5120", timeit(lambda: L.quantize_fp8(x5, fmt, A.SB_AXIS_ROW, check=False)),
           T * 5120 * 3 + 4 * T)
g = torch.randn(1280, device="cuda")
b = torch.randn(1280, device="cuda")
report("layernorm_quantize_rowwise 65792x1280", timeit(lambda: L.layernorm_quantize_rowwise(x1, g, b, check=False)),
       T * 1280 * 5 + 12 * T)
_, _, mean, rstd = L.layernorm_quantize_rowwise(x1, g, b, check=False)
dh = torch.randn(T, 1280, device="cuda").bfloat16()
report("layernorm_backward 65792x1280", timeit(lambda: L.layernorm_backward(dh, x1, mean, rstd, g)), T * 1280 * 6 + 8 * T)
pre = torch.randn(T, 5120, device="cuda").bfloat16()
report("gelu_quantize_rowwise 65792x5120", timeit(lambda: L.gelu_quantize_rowwise(pre, check=False)), T * 5120 * 5 + 4 * T)
report("gelu_backward_quantize 65792x5120",
       timeit(lambda: L.gelu_backward_quantize_rowwise(x5, pre, check=False)), T * 5120 * 7 + 4 * T)
report("column_sums (bias grad) 65792x5120", timeit(lambda: L.column_sums(x5)), T * 5120 * 2)
report("column_sums (bias grad) 65792x1280", timeit(lambda: L.column_sums(x1)), T * 1280 * 2)
report("torch .sum(0) fp32 65792x5120 (yardstick)", timeit(lambda: x5.sum(0, dtype=torch.float32)), T * 5120 * 2)
w = torch.randn(5120, 1280, device="cuda").bfloat16()
report("quantize_tensorwise (+T) 5120x1280", timeit(lambda: L.quantize_tensorwise(w, check=False, with_transpose=True)),
       5120 * 1280 * 4 + 4)
