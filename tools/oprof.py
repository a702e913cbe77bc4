"""One StableAdamW step over 4 ViT-H tensors (for ncu)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_13013_b200 import _capi as A, lowprec as L
sizes = [3840 * 1280, 1280 * 1280, 5120 * 1280, 1280 * 5120]
refs = [L.TensorRef(f"t{i}", torch.randn(s, device="cuda"), torch.randn(s, device="cuda") * 1e-3,
                    torch.zeros(s, device="cuda"), torch.zeros(s, device="cuda")) for i, s in enumerate(sizes)]
hp = L.OptimizerHyperparams(lr_schedule=lambda t: 1e-3, weight_decay=0.2, clipping=A.SB_CLIP_UPDATE)
for t in range(1, 4):
    L.optimizer_step(refs, hp, t, infos=False)
torch.cuda.synchronize()
