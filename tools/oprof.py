"""StableAdamW steps over NBLK ViT-H blocks (4 tensors each) — for ncu and quick timing.

    NBLK=8 SB_ADAMW_KERNEL=ring|reg python tools/oprof.py
"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_13013_b200 import _capi as A, lowprec as L
nblk = int(os.environ.get("NBLK", "1"))
sizes = [3840 * 1280, 1280 * 1280, 5120 * 1280, 1280 * 5120] * nblk
refs = [L.TensorRef(f"t{i}", torch.randn(s, device="cuda"), torch.randn(s, device="cuda") * 1e-3,
                    torch.zeros(s, device="cuda"), torch.zeros(s, device="cuda")) for i, s in enumerate(sizes)]
hp = L.OptimizerHyperparams(lr_schedule=lambda t: 1e-3, weight_decay=0.2, clipping=A.SB_CLIP_UPDATE)
steps = int(os.environ.get("STEPS", "3"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for t in range(1, steps + 1):
    if t == steps:
        e0.record()
    L.optimizer_step(refs, hp, t, infos=False)
e1.record()
torch.cuda.synchronize()
n = sum(sizes)
ms = e0.elapsed_time(e1)
print(f"oprof nblk={nblk} params={n} last step {ms:.3f} ms -> {n * 28 / ms / 1e6:.0f} GB/s algorithmic")
