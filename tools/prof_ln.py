"""K11 (LayerNorm + quantize) and K12 (LayerNorm backward) at the ViT-H shape, for ncu:
    ncu --set full -k regex:ln_ python tools/prof_ln.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2304_13013_b200 import lowprec as L

T, D = 256 * 257, 1280
x = torch.randn(T, D, device="cuda").bfloat16()
dh = torch.randn(T, D, device="cuda").bfloat16()
g = torch.ones(D, device="cuda")
b = torch.zeros(D, device="cuda")
for _ in range(2):
    _, _, mean, rstd = L.layernorm_quantize_rowwise(x, g, b, check=False)
    L.layernorm_backward(dh, x, mean, rstd, g)
torch.cuda.synchronize()
