"""Practical dense int8 tensor-core peak on this B200: cuBLASLt int8 GEMM (torch._int_mm, int32
out) at large square shapes, CUDA-event timed -- the library yardstick for our int8 GEMM's %.
    python tools/int8_peak.py"""
import torch

for n in (8192, 12288, 16384):
    a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        torch._int_mm(a, b)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"int8 {n}^3: {ms * 1e3:.0f} us -> {2 * n ** 3 / ms / 1e9:.0f} TOPS")
