"""int8 GEMM with and without the residual epilogue (OUT_BF16_RESID) at the ViT-H block shapes:
    python tools/resid_gemm.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2304_13013_b200 import lowprec as L

T = 256 * 257


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000


for K, N in ((1280, 1280), (5120, 1280)):
    x = torch.randn(T, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    r = torch.randn(T, N, device="cuda").bfloat16()
    qa = L.quantize_rowwise(x, check=False)
    qb = L.quantize_tensorwise(w, check=False)
    t0 = timeit(lambda: L.int8_gemm_epilogue(qa, qb))
    t1 = timeit(lambda: L.int8_gemm_epilogue(qa, qb, residual=r))
    t2 = timeit(lambda: L.int8_gemm_epilogue(qa, qb) + r)
    y1 = L.int8_gemm_epilogue(qa, qb, residual=r)
    y0 = L.int8_gemm_epilogue(qa, qb).float() + r.float()
    err = ((y1.float() - y0).abs().max() / y0.abs().max()).item()
    print(f"M={T} N={N} K={K}: plain {t0:6.1f} us  +residual epilogue {t1:6.1f} us  plain + torch add {t2:6.1f} us"
          f"  (max |diff| / max |y| vs the fp32 sum {err:.1e})")
