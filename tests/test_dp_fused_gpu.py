"""GPU: the fused dW GEMM + reduce-scatter over peer memory (sb_wgrad_reduce_scatter, SURVEY.md
§8e stage 2) on one B200.

* one rank: the epilogue's TMA reduce-adds into the zeroed symmetric buffer give exactly the
  plain dW (0 + x == x), at both MLP weight shapes (direct and transposed one-wave kernel),
  with and without G's fused row-wise quantize;
* two processes sharing the GPU (CUDA IPC between processes works on one device; NCCL refuses
  two ranks on one GPU, so the handles and barriers travel over gloo): each process computes its
  token shard's G_r^T X_r and reduce-adds every 32-row block into the owner's copy, mapped from
  the other process; each owner's rows equal the full-batch dW within fp32 summation tolerance
  (1e-4 relative, as every dW check: two 16384-token partial sums against one 32768-token chain)."""
import os
import subprocess
import sys

import pytest
import torch

from paper_2304_13013_b200 import _capi as A
from paper_2304_13013_b200 import dp
from paper_2304_13013_b200 import lowprec as L

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("m,n", [(1280, 5120), (5120, 1280)])
@pytest.mark.parametrize("fuse_q", [False, True])
def test_one_rank_equals_plain_wgrad(m, n, fuse_q):
    T = 16384
    torch.manual_seed(m + n)
    g = torch.randn(T, m, device="cuda").bfloat16()
    x = torch.randn(T, n, device="cuda").bfloat16()
    h = A.handle(0)
    buf = dp.SymmetricBuffer(h, 4 * m * n + 4096)
    try:
        dw = buf.view((m, n), 4096)
        dw.zero_()
        gq = torch.empty(T, m, dtype=torch.int8, device="cuda") if fuse_q else None
        gs = torch.empty(T, dtype=torch.float32, device="cuda") if fuse_q else None
        dp.wgrad_reduce_scatter(h, g, x, dw, gq, gs)
        ref = L.wgrad(g, x)
        torch.cuda.synchronize()
        assert torch.equal(dw, ref)
        if fuse_q:
            q = L.quantize_rowwise(g)
            assert torch.equal(gq, q.payload) and torch.equal(gs, q.state)
        # the whole fused exchange without a communicator is the same GEMM into the zeroed buffer
        dw.fill_(7.0)
        A.check(h.lib.sb_dp_wgrad_allreduce_fused(h.h, L._p(g), L._p(x), A.SB_BF16, T, m, n, L._p(dw), None, m, None))
        torch.cuda.synchronize()
        assert torch.equal(dw, ref)
    finally:
        buf.close()


def test_reduce_scatter_rejects_foreign_buffer():
    h = A.handle(0)
    g = torch.randn(256, 64, device="cuda").bfloat16()
    dw = torch.zeros(64, 64, device="cuda")
    with pytest.raises(A.InvalidArgument, match="symmetric"):
        dp.wgrad_reduce_scatter(h, g, g, dw)


_TWO = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
from paper_2304_13013_b200 import _capi as A, dp, lowprec as L
rank, world = int(sys.argv[2]), 2
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[3], rank=rank, world_size=world)
torch.cuda.set_device(0)
T, m, n = 32768, int(sys.argv[4]), int(sys.argv[5])
gen = torch.Generator(device="cuda").manual_seed(11)
G = torch.randn(T, m, device="cuda", generator=gen).bfloat16()
X = torch.randn(T, n, device="cuda", generator=gen).bfloat16()
r0, r1 = T * rank // world, T * (rank + 1) // world
h = A.handle(0)
buf = dp.SymmetricBuffer(h, 4 * m * n, rank, world)
dw = buf.view((m, n))
dw.zero_()
torch.cuda.synchronize()
dist.barrier()                                   # every copy zeroed before any rank adds
dp.wgrad_reduce_scatter(h, G[r0:r1], X[r0:r1], dw)
torch.cuda.synchronize()
dist.barrier()                                   # every rank's reduce-adds landed
o0, o1 = dp.owned_rows(m, rank, world)
full = L.wgrad(G, X)
torch.cuda.synchronize()
rel = ((dw[o0:o1] - full[o0:o1]).norm() / full[o0:o1].norm()).item()
others = torch.cat([dw[:o0], dw[o1:]]).abs().max().item() if o1 - o0 < m else 0.0
dist.barrier()
buf.close()
print(f"rank {rank} rows {o0}:{o1} rel {rel:.3e} others {others}", flush=True)
sys.exit(0 if rel < 1e-4 and o1 > o0 and others == 0.0 else 1)
"""


@pytest.mark.parametrize("m,n", [(1280, 5120), (5120, 1280)])
def test_two_processes_one_gpu_reduce_scatter(tmp_path, m, n):
    script = tmp_path / "two.py"
    script.write_text(_TWO)
    port = str(29500 + (os.getpid() + m) % 1000)
    procs = [subprocess.Popen([sys.executable, str(script), ROOT, str(r), port, str(m), str(n)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        outs.append((p.returncode, out))
    for rc, out in outs:
        assert rc == 0, out[-3000:]


@pytest.mark.parametrize("m,n", [(1280, 1280), (3840, 1280)])
def test_fused_allreduce_every_layer_shape(m, n):
    """sb_dp_wgrad_allreduce_fused serves every ViT-H dW shape: the out-projection (1280 x 1280) is
    not a one-wave shape and takes the local GEMM + all-reduce form, qkv (3840 x 1280) the fused
    reduce-scatter epilogue; both equal the plain dW (one rank), G's payload equal to
    quantize_rowwise(G)."""
    T = 16384
    torch.manual_seed(m)
    g = torch.randn(T, m, device="cuda").bfloat16()
    x = torch.randn(T, n, device="cuda").bfloat16()
    h = A.handle(0)
    buf = dp.SymmetricBuffer(h, 4 * m * n)
    try:
        dw = buf.view((m, n))
        gq = torch.empty(T, m, dtype=torch.int8, device="cuda")
        gs = torch.empty(T, dtype=torch.float32, device="cuda")
        A.check(h.lib.sb_dp_wgrad_allreduce_fused(h.h, L._p(g), L._p(x), A.SB_BF16, T, m, n, L._p(dw), L._p(gq), m,
                                                  L._p(gs)))
        ref = L.wgrad(g, x)
        q = L.quantize_rowwise(g)
        torch.cuda.synchronize()
        assert torch.equal(dw, ref)
        assert torch.equal(gq, q.payload) and torch.equal(gs, q.state)
    finally:
        buf.close()
