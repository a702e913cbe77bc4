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


def _allquant_worker(rank, world, port, T, n, m, out_dir):
    """AllQuant int8 dW under token sharding, as csrc/dp.cu runs it: per-feature absmax maxed
    over ranks, column-wise quantization of the local rows, the local raw integer product,
    summed over ranks as int64, one dequantization (linear.cpp:239-241, :49)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle as O
    from paper_2304_13013_b200 import dp

    dp.init_from_env(backend="gloo")
    x, _, g = _inputs(T, n, m)
    r0, r1 = dp.shard_rows(T, rank, world)
    gl, xl = g[r0:r1], x[r0:r1]
    sg = torch.from_numpy(np.abs(gl).max(0, initial=0.0))   # absmax per feature, this rank's tokens
    sx = torch.from_numpy(np.abs(xl).max(0, initial=0.0))
    dist.all_reduce(sg, op=dist.ReduceOp.MAX)                # sb_dp_allreduce_max_u32
    dist.all_reduce(sx, op=dist.ReduceOp.MAX)
    sg = np.where(sg.numpy() == 0, 1.0, sg.numpy()).astype(np.float32)  # zero-slice sentinel
    sx = np.where(sx.numpy() == 0, 1.0, sx.numpy()).astype(np.float32)
    # lround(127 x / s): half away from zero (quantize.cpp:17-20)
    qg = (np.sign(gl) * np.floor(np.abs(127.0 * gl.astype(np.float64) / sg) + 0.5)).astype(np.int8).T.copy()
    qx = (np.sign(xl) * np.floor(np.abs(127.0 * xl.astype(np.float64) / sx) + 0.5)).astype(np.int8).T.copy()
    raw = torch.from_numpy(qg.astype(np.int64) @ qx.astype(np.int64).T)  # local int product [m x n]
    dist.all_reduce(raw, op=dist.ReduceOp.SUM)               # the int64 sum over ranks
    dw = ((raw.numpy().astype(np.float64) * sg.astype(np.float64)[:, None]) * sx.astype(np.float64)[None, :]
          / 16129.0).astype(np.float32)
    np.savez(os.path.join(out_dir, f"aq{rank}.npz"), dw=dw)
    dist.destroy_process_group()


def test_allquant_token_sharded_dw_is_bit_exact(tmp_path):
    """The data-parallel AllQuant dW (max-reduced feature scales, int64-summed accumulators) is
    bit-identical to the single-process reference (oracle/_ref when built, else the oracle)."""
    import oracle as O

    T, n, m, world = 50, 24, 40, 2
    mp.spawn(_allquant_worker, args=(world, _free_port(), T, n, m, str(tmp_path)), nprocs=world, join=True)
    x, w, g = _inputs(T, n, m)
    qgt, sgt = O.quantize(np.ascontiguousarray(g.T), O.ROW)
    qxt, sxt = O.quantize(np.ascontiguousarray(x.T), O.ROW)
    want = O.int8_gemm(qgt, sgt, qxt, sxt, want_raw=False)   # matmul_dequant_dual_rowwise, K = T
    if O.ref_available():
        _, _, dw_ref = O.ref_linear(4, 0, x, w, g)            # AllQuant int8 through the reference
        assert np.array_equal(want, dw_ref)
    for rank in range(world):
        assert np.array_equal(np.load(tmp_path / f"aq{rank}.npz")["dw"], want)


def test_lpt_partition_balances_c5():
    """C5 (BASELINE configs[4]): 51 ViT-H blocks x 4 weight tensors over 2 / 4 / 8 ranks, whole
    tensors per rank: max / mean <= 1.02 (round-robin by index: 1.17 / 1.33 / 1.36)."""
    from paper_2304_13013_b200 import dp

    sizes = [3840 * 1280, 1280 * 1280, 5120 * 1280, 1280 * 5120] * 51
    for world in (1, 2, 4, 8):
        parts = dp.lpt_partition(sizes, world)
        assert sorted(i for p in parts for i in p) == list(range(len(sizes)))
        loads = [sum(sizes[i] for i in p) for p in parts]
        assert max(loads) / (sum(loads) / world) <= 1.02


def test_owned_rows_partition_matches_library():
    """The fused reduce-scatter's row ownership (dp.owned_rows == sb_dp_owned_rows): contiguous,
    32-row aligned, covering every row once, balanced to one 32-row block."""
    import ctypes as C

    from paper_2304_13013_b200 import _capi as A
    from paper_2304_13013_b200 import dp

    lib = A.load(build_if_missing=False)
    for rows in (1, 31, 32, 100, 1280, 3840, 5120, 5121):
        for world in (1, 2, 3, 4, 8):
            prev = 0
            sizes = []
            for r in range(world):
                r0, r1 = dp.owned_rows(rows, r, world)
                a, b = C.c_int64(), C.c_int64()
                assert lib.sb_dp_owned_rows(rows, r, world, C.byref(a), C.byref(b)) == 0
                assert (a.value, b.value) == (r0, r1)
                assert r0 == prev and (r0 % 32 == 0 or r0 == rows)
                prev = r1
                sizes.append(-(-(r1 - r0) // 32))
            assert prev == rows
            assert max(sizes) - min(sizes) <= 1
