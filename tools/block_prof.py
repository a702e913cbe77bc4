"""One eager fwd+bwd of the ViT-H block (bench.py --config vit_block) per arm, for an ncu
launch list:  ARM=switchback|bf16 ncu --metrics gpu__time_duration.sum --csv python tools/block_prof.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

from paper_2304_13013_b200.nn import SwitchBackLinear, SwitchBackMLP

dev = torch.device("cuda", 0)
B, S, D, H = 256, 257, 1280, 16
arm = os.environ.get("ARM", "switchback")  # switchback | fused (prenorm SwitchBackLinear / SwitchBackMLP) | bf16
mk = (lambda i, o: SwitchBackLinear(i, o, device=dev)) if arm != "bf16" else (lambda i, o: torch.nn.Linear(i, o, device=dev))
mlp = SwitchBackMLP(D, 4 * D, device=dev, prenorm=True) if arm == "fused" else None
qkv_ln = SwitchBackLinear(D, 3 * D, device=dev, prenorm=True) if arm == "fused" else None
ln1, ln2 = torch.nn.LayerNorm(D, device=dev), torch.nn.LayerNorm(D, device=dev)
qkv, out, fc1, fc2 = mk(D, 3 * D), mk(D, D), mk(D, 4 * D), mk(4 * D, D)
x = torch.randn(B, S, D, device=dev).bfloat16().requires_grad_(True)
gy = torch.randn(B, S, D, device=dev).bfloat16()
for it in range(2):
    torch.cuda.nvtx.range_push(f"step{it}")
    with torch.autocast("cuda", dtype=torch.bfloat16, enabled=arm == "bf16"):
        qkv_out = qkv_ln(x) if qkv_ln is not None else qkv(ln1(x.float()).to(torch.bfloat16))
        q, k, v = qkv_out.view(B, S, 3, H, D // H).permute(2, 0, 3, 1, 4).unbind(0)
        a = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(B, S, D)
        x2 = x + out(a)
        y = x2 + (mlp(x2) if mlp is not None else fc2(F.gelu(fc1(ln2(x2.float()).to(torch.bfloat16)))))
    y.backward(gy)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
