"""K10 (fused GELU / GELU' + row-wise quantize) at the ViT-H MLP shape, for ncu:
    ncu --set full -k regex:act_quantize python tools/prof_k10.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2304_13013_b200 import lowprec as L

T, H = 256 * 257, 5120
pre = torch.randn(T, H, device="cuda").bfloat16()
dact = torch.randn(T, H, device="cuda").bfloat16()
for _ in range(2):
    L.gelu_quantize_rowwise(pre, check=False)
    L.gelu_backward_quantize_rowwise(dact, pre, check=False)
torch.cuda.synchronize()
