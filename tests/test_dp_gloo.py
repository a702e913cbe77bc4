"""CPU, world_size 2 over gloo: the data-parallel decomposition of the SwitchBack path
(paper_2304_13013_b200/dp.py). Each rank runs the oracle's SwitchBack
forward/backward (oracle/ = the CPU checker; the GPU ranks run the CUDA path) on its token
shard; the only collective is the dW sum all-reduce. Checks: the row shards of Y and dX are
bit-identical to the unsharded result (per-token-row independence of row-wise quantization
and of the fwd / dX GEMMs), dW matches within fp32 tolerance (the all-reduce changes the
summation order), and the max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(T, n, m):
    rng = np.random.default_rng(7)
    x = rng.standard_normal((T, n)).astype(np.float32)
    w = (rng.standard_normal((m, n)) / np.sqrt(n)).astype(np.float32)
    g = rng.standard_normal((T, m)).astype(np.float32)
    x[3] = 0.0  # an all-zero token row (state sentinel) lands on rank 0
    return x, w, g


def _worker(rank, world, port, T, n, m, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle as O
    from paper_2304_13013_b200 import dp

    r, w_, _ = dp.init_from_env(backend="gloo")
    assert (r, w_) == (rank, world) and dist.get_backend() == "gloo"
    x, w, g = _inputs(T, n, m)
    r0, r1 = dp.shard_rows(T, rank, world)
    y = O.switchback_forward(x[r0:r1], w)
    dx, dw = O.switchback_backward(x[r0:r1], w, g[r0:r1])
    dw_t = torch.from_numpy(dw)
    ar = dp.GradAllReduce()
    ar.launch(dw_t)
    ar.wait()
    t = dp.max_over_ranks(float(rank + 1))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), y=y, dx=dx, dw=dw_t.numpy(), r0=r0, r1=r1, t=t)
    dist.destroy_process_group()


@pytest.mark.parametrize("T", [64, 37])  # even and ragged token counts
def test_token_sharded_switchback_world2(tmp_path, T):
    import oracle as O
    from paper_2304_13013_b200 import dp

    n, m, world = 48, 80, 2
    mp.spawn(_worker, args=(world, _free_port(), T, n, m, str(tmp_path)), nprocs=world, join=True)
    x, w, g = _inputs(T, n, m)
    y_ref = O.switchback_forward(x, w)
    dx_ref, dw_ref = O.switchback_backward(x, w, g)
    seen = 0
    for rank in range(world):
        d = np.load(tmp_path / f"rank{rank}.npz")
        r0, r1 = int(d["r0"]), int(d["r1"])
        assert (r0, r1) == dp.shard_rows(T, rank, world)
        assert np.array_equal(d["y"], y_ref[r0:r1])      # bit-identical row shards
        assert np.array_equal(d["dx"], dx_ref[r0:r1])
        rel = np.linalg.norm(d["dw"].astype(np.float64) - dw_ref) / np.linalg.norm(dw_ref)
        assert rel < 1e-6                                 # all-reduced dW == unsharded dW (fp32 order)
        assert float(d["t"]) == float(world)              # max over ranks
        seen += r1 - r0
    assert seen == T


def test_shard_rows_cover_exactly():
    from paper_2304_13013_b200 import dp

    for total in (0, 1, 7, 65792):
        for world in (1, 2, 3, 8):
            spans = [dp.shard_rows(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
