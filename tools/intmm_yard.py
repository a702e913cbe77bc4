"""cuBLASLt int8 GEMM yardstick (torch._int_mm, int32 output) at the C2 int8 shapes."""
import torch
T = 65792
for (K, N) in [(1280, 5120), (5120, 1280)]:
    a = torch.randint(-127, 128, (T, K), device="cuda", dtype=torch.int8)
    b = torch.randint(-127, 128, (N, K), device="cuda", dtype=torch.int8).t()  # column-major K x N
    for _ in range(3):
        c = torch._int_mm(a, b)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); torch._int_mm(a, b); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    t = sorted(ts)[5] / 1e3
    print(f"_int_mm M={T} N={N} K={K}: {t*1e6:.1f} us  {2*T*N*K/t/1e12:.0f} TOPS (int32 out {T*N*4/1e6:.0f} MB)")
