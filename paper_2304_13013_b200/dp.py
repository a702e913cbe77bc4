"""Data parallelism for the SwitchBack path: the token dimension is sharded across ranks
(one process per GPU); the only collective is the sum all-reduce of dW.

Why this is exact where it can be: row-wise quantization of X and G and
the forward / input-gradient GEMMs are per-token-row independent, and the tensor-wise W
scale comes from the replicated W, so each rank's Y and dX rows are bit-identical to the
single-GPU result. dW = sum_r G_r^T X_r is the one exchange step (NCCL all-reduce over
NVLink; gloo in the CPU tests); its summation order differs from the single-GPU GEMM,
so dW matches within fp32 tolerance.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def init_from_env(backend: str | None = None) -> tuple[int, int, int]:
    """(rank, world, local_rank) from torchrun's env; initializes the default group when
    WORLD_SIZE > 1. Backend: nccl when CUDA is available, else gloo."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Test hooks for exercising the multi-rank path on a one-GPU box: SB_DP_SHARE_GPU=1 maps
    # every rank to cuda:0, SB_DP_BACKEND=gloo replaces NCCL (which refuses two ranks on one GPU).
    if os.environ.get("SB_DP_SHARE_GPU") == "1":
        local = 0
    backend = backend or os.environ.get("SB_DP_BACKEND") or None
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def shard_rows(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous token-row shard [r0, r1) of `total` rows for `rank` (sizes differ by <= 1)."""
    r0 = total * rank // world
    r1 = total * (rank + 1) // world
    return r0, r1


class GradAllReduce:
    """Asynchronous sum all-reduce of weight gradients, issued as each layer's backward
    finishes so the transfer of layer L overlaps the backward of layer L-1."""

    def __init__(self, group=None):
        self.group = group
        self.pending: list = []

    def launch(self, dw: torch.Tensor) -> None:
        if not dist.is_initialized() or dist.get_world_size(self.group) == 1:
            return
        self.pending.append(dist.all_reduce(dw, op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def wait(self) -> None:
        for w in self.pending:
            w.wait()
        self.pending.clear()


def max_over_ranks(value: float, device=None) -> float:
    """Timing rule: the job's step time is the max over ranks."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
