# print cluster occupancy facts for the 2-CTA GEMM (debug helper)
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_13013_b200 import lowprec as L
p = torch.cuda.get_device_properties(0)
print("sms", p.multi_processor_count)
a = torch.randint(-127, 127, (4096, 1024), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 127, (4096, 1024), dtype=torch.int8, device="cuda")
A = L.QuantizedMatrix(a, torch.ones(4096, device="cuda"), L.ROW)
B = L.QuantizedMatrix(b, torch.ones(1, device="cuda"), L.TENSOR)
for _ in range(3):
    L.int8_matmul_dequant(A, B, out_dtype=torch.bfloat16, exact=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    L.int8_matmul_dequant(A, B, out_dtype=torch.bfloat16, exact=False)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print("4096^2 x 1024 int8: %.1f us  %.0f TOPS" % (ms * 1e3, 2 * 4096 * 4096 * 1024 / ms / 1e9))
