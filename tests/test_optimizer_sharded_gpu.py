"""GPU: ZeRO-1 StableAdamW (sb_stableadamw_shard_phase1 / _phase2 / _step_sharded).

* one rank, each tensor whole: identical to the fused step (same fixed-order sums), bit for bit;
* a tensor split into world shards on ONE process (the shards' sums added on the host side as
  an all-reduce would): v, u bitwise the unsharded step's; RMS within 1e-12; theta bitwise where
  eta does not depend on the summation order (RMS <= 1 under update clipping, and no clipping);
* two processes sharing the GPU (gloo all-reduce of the fp64 sums), each updating its row shard
  of every ViT-H weight shape: the concatenated shards equal the one-process full step."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2304_13013_b200 import _capi as A
from paper_2304_13013_b200 import lowprec as L

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [(3840, 1280), (1280, 1280), (5120, 1280), (1280, 5120), (7, 13)]


def state(seed, shapes=SHAPES, gscale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    out = []
    for r, c in shapes:
        n = r * c
        out.append([torch.randn(n, device="cuda", generator=g), torch.randn(n, device="cuda", generator=g) * gscale,
                    torch.randn(n, device="cuda", generator=g) * 1e-3, torch.rand(n, device="cuda", generator=g) * 1e-4])
    return out


def refs(st, sl=None):
    return [L.TensorRef(f"t{i}", *(a if sl is None else a[sl[i]] for a in s)) for i, s in enumerate(st)]


@pytest.mark.parametrize("clipping", [A.SB_CLIP_NONE, A.SB_CLIP_UPDATE])
def test_one_rank_equals_fused_step(clipping):
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 1e-3, weight_decay=0.2, clipping=clipping)
    a, b = state(1), state(1)
    for t in (1, 2, 3):
        info = L.optimizer_step(refs(a), hp, t, infos=False)
        out = L.optimizer_step_sharded(refs(b), [s[0].numel() for s in b], hp, t)
        torch.cuda.synchronize()
        assert torch.equal(out["rms"], info[0]) and torch.equal(out["eta"], info[1])
        for x, y in zip(a, b):
            for u, w in zip(x, y):
                assert torch.equal(u, w)


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("gscale", [1e-4, 1.0])  # RMS <= 1 (eta = alpha) and RMS > 1 (eta = alpha / RMS)
def test_shards_on_one_process(world, gscale):
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 1e-3, weight_decay=0.2, clipping=A.SB_CLIP_UPDATE)
    full, sh = state(2, gscale=gscale), state(2, gscale=gscale)
    info = L.optimizer_step(refs(full), hp, 1, infos=False)
    tot = [s[0].numel() for s in sh]
    sums = []
    parts = []
    for r in range(world):
        sl = [slice(n * r // world, n * (r + 1) // world) for n in tot]
        parts.append(sl)
        h = A.handle(0)
        nb = C_size(refs(sh, sl))
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        arr = adamw_arr(refs(sh, sl))
        s_ = torch.empty(len(sh), dtype=torch.float64, device="cuda")
        hpc = A.AdamwHparams(1e-3, hp.beta1, hp.beta2, 0.0, hp.eps, hp.weight_decay, 1.0, int(hp.clipping))
        A.check(h.lib.sb_stableadamw_shard_phase1(h.h, arr, int64s(tot), len(sh), C.byref(hpc), 1, L._p(s_),
                                                  L._p(ws), ws.numel()))
        sums.append(s_)
    total = torch.stack(sums).sum(0)
    rms = torch.sqrt(total / torch.tensor(tot, dtype=torch.float64, device="cuda"))
    assert torch.allclose(rms, info[0], rtol=1e-12, atol=0)
    for r in range(world):
        h = A.handle(0)
        arr = adamw_arr(refs(sh, parts[r]))
        nb = C_size(refs(sh, parts[r]))
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        out = torch.empty(2, len(sh), dtype=torch.float64, device="cuda")
        hpc = A.AdamwHparams(1e-3, hp.beta1, hp.beta2, 0.0, hp.eps, hp.weight_decay, 1.0, int(hp.clipping))
        A.check(h.lib.sb_stableadamw_shard_phase2(h.h, arr, int64s(tot), len(sh), C.byref(hpc), 1, L._p(total), None,
                                                  None, L._p(out[0]), L._p(out[1]), L._p(ws), ws.numel()))
        assert torch.allclose(out[1], info[1], rtol=1e-12, atol=0)
    torch.cuda.synchronize()
    for x, y in zip(full, sh):
        assert torch.equal(x[2], y[2]) and torch.equal(x[3], y[3])  # v, u: no reduction feeds them
        if gscale < 1:  # RMS <= 1: eta = alpha exactly, theta bitwise
            assert torch.equal(x[0], y[0])
        else:
            assert torch.allclose(x[0], y[0], rtol=1e-6, atol=1e-9)


import ctypes as C  # noqa: E402


def adamw_arr(rs):
    arr = (A.AdamwTensor * len(rs))()
    for i, r in enumerate(rs):
        arr[i] = A.AdamwTensor(r.param.data_ptr(), r.grad.data_ptr(), r.v.data_ptr(), r.u.data_ptr(), r.param.numel())
    return arr


def int64s(v):
    return (C.c_int64 * len(v))(*v)


def C_size(rs):
    nb = C.c_size_t()
    A.check(A.load().sb_stableadamw_sharded_workspace_size(adamw_arr(rs), len(rs), C.byref(nb)))
    return nb.value


def test_shadow_rows_and_errors():
    """Phase 2 writes the shard's bf16 shadow rows and the tensor-wise absmax word; kGradClip is refused."""
    st = state(3, shapes=[(512, 256)])
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 1e-3, clipping=A.SB_CLIP_UPDATE)
    shadow = torch.empty(512 * 256, dtype=torch.bfloat16, device="cuda")
    word = torch.zeros(1, dtype=torch.int32, device="cuda")
    L.optimizer_step_sharded(refs(st), [512 * 256], hp, 1, shadows=[(shadow, word)])
    torch.cuda.synchronize()
    assert torch.equal(shadow, st[0][0].bfloat16())
    assert int(word.item()) == int(st[0][0].bfloat16().float().abs().max().view(torch.int32).item())
    with pytest.raises(A.SBError, match="grad_clip"):
        L.optimizer_step_sharded(refs(st), [512 * 256], L.OptimizerHyperparams(lr_schedule=lambda t: 1e-3,
                                                                               clipping=A.SB_CLIP_GRAD), 1)


_TWO = r"""
import sys, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
from paper_2304_13013_b200 import _capi as A, dp, lowprec as L
rank, world = int(sys.argv[2]), 2
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[3], rank=rank, world_size=world)
torch.cuda.set_device(0)
shapes = [(3840, 1280), (1280, 1280), (5120, 1280), (1280, 5120)]
hp = L.OptimizerHyperparams(lr_schedule=lambda t: 1e-3, weight_decay=0.2, clipping=A.SB_CLIP_UPDATE)
def make():
    g = torch.Generator(device="cuda").manual_seed(5)
    return [[torch.randn(r * c, device="cuda", generator=g), torch.randn(r * c, device="cuda", generator=g),
             torch.randn(r * c, device="cuda", generator=g) * 1e-3, torch.rand(r * c, device="cuda", generator=g) * 1e-4]
            for r, c in shapes]
full, mine = make(), make()
rows = [dp.owned_rows(r, rank, world) for r, _ in shapes]   # this rank's dW rows (the fused reduce-scatter's)
sl = [slice(r0 * c, r1 * c) for (r0, r1), (_, c) in zip(rows, shapes)]
def ar(t):
    h = t.cpu(); dist.all_reduce(h); t.copy_(h)
for step in (1, 2):
    info = L.optimizer_step([L.TensorRef(str(i), *s) for i, s in enumerate(full)], hp, step, infos=False)
    out = L.optimizer_step_sharded([L.TensorRef(str(i), *(a[sl[i]] for a in s)) for i, s in enumerate(mine)],
                                   [r * c for r, c in shapes], hp, step, allreduce=ar)
torch.cuda.synchronize()
ok = torch.allclose(out["rms"], info[0], rtol=1e-12, atol=0)
for i, (f, m) in enumerate(zip(full, mine)):
    ok &= torch.equal(f[2][sl[i]], m[2][sl[i]]) and torch.equal(f[3][sl[i]], m[3][sl[i]])
    ok &= torch.allclose(f[0][sl[i]], m[0][sl[i]], rtol=1e-6, atol=1e-9)
print(f"rank {rank} ok {ok} rms {out['rms'].tolist()}", flush=True)
sys.exit(0 if ok else 1)
"""


def test_two_processes_one_gpu(tmp_path):
    script = tmp_path / "zero1.py"
    script.write_text(_TWO)
    port = str(29700 + os.getpid() % 200)
    procs = [subprocess.Popen([sys.executable, str(script), ROOT, str(r), port], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        assert p.returncode == 0, out[-3000:]
