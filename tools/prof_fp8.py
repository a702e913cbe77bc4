"""Row-wise fp8 quantize (e4m3, then e5m2) at 65792 x 5120 bf16, two launches each (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_13013_b200 import _capi as A  # noqa: E402
from paper_2304_13013_b200 import lowprec as L  # noqa: E402

x = torch.randn(65792, 5120, device="cuda").bfloat16()
for fmt in (A.SB_E4M3, A.SB_E5M2):
    for _ in range(2):
        L.quantize_fp8(x, fmt, A.SB_AXIS_ROW, check=False)
torch.cuda.synchronize()
