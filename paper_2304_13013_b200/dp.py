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


class NcclComm:
    """The library's own NCCL communicator on a handle (sb_dp_init, csrc/dp.cu): rank 0 draws the
    128-byte id (sb_dp_unique_id) and torch.distributed broadcasts it — the out-of-band step of
    NCCL's setup; after that every exchange of the SwitchBack step (dW sum, AllQuant's absmax
    max, a sharded optimizer's RMS sums) goes through the C-ABI, with no torch collective."""

    def __init__(self, handle, rank: int, world: int, group=None):
        import ctypes as C

        from . import _capi as A

        self.h, self.rank, self.world = handle, rank, world
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            A.check(handle.lib.sb_dp_unique_id(uid))
        if world > 1:
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0, group=group)
            uid = (C.c_uint8 * 128)(*t.cpu().tolist())
        A.check(handle.lib.sb_dp_init(handle.h, uid, rank, world))

    def close(self) -> None:
        from . import _capi as A

        A.check(self.h.lib.sb_dp_destroy(self.h.h))


class GradAllReduce:
    """Asynchronous sum all-reduce of weight gradients, issued as each layer's backward
    finishes so the transfer of layer L overlaps the backward of layer L-1. With a NcclComm the
    library does it (sb_dp_allreduce_grads_async on its communication stream, joined by
    sb_dp_wait); otherwise torch.distributed (gloo in the CPU tests)."""

    def __init__(self, group=None, comm: NcclComm | None = None):
        self.group = group
        self.comm = comm
        self.pending: list = []

    def launch(self, dw: torch.Tensor) -> None:
        if self.comm is not None:
            if self.comm.world == 1:
                return
            import ctypes as C

            from . import _capi as A

            h = self.comm.h
            h.bind_stream(torch.cuda.current_stream(dw.device).cuda_stream)
            bufs = (C.c_void_p * 1)(dw.data_ptr())
            numel = (C.c_int64 * 1)(dw.numel())
            A.check(h.lib.sb_dp_allreduce_grads_async(h.h, bufs, numel, 1))
            self.pending.append(None)
            return
        if not dist.is_initialized() or dist.get_world_size(self.group) == 1:
            return
        self.pending.append(dist.all_reduce(dw, op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def wait(self) -> None:
        if self.comm is not None:
            from . import _capi as A

            if self.pending:
                A.check(self.comm.h.lib.sb_dp_wait(self.comm.h.h))
            self.pending.clear()
            return
        for w in self.pending:
            w.wait()
        self.pending.clear()


def lpt_partition(sizes: list[int], world: int) -> list[list[int]]:
    """Whole tensors to ranks, balanced by size (longest processing time first: largest tensor
    to the least-loaded rank, ties to the lower rank; deterministic). For the C5 set (51 ViT-H
    blocks x {3840x1280, 1280x1280, 5120x1280, 1280x5120}) max / mean load is <= 1.02 at 2, 4
    and 8 ranks, where round-robin by index gives 1.33-1.36."""
    loads = [0] * world
    parts: list[list[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(sizes)), key=lambda k: (-sizes[k], k)):
        r = min(range(world), key=lambda j: (loads[j], j))
        parts[r].append(i)
        loads[r] += sizes[i]
    for p in parts:
        p.sort()
    return parts


def max_over_ranks(value: float, device=None) -> float:
    """Timing rule: the job's step time is the max over ranks."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def owned_rows(rows: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r0, r1) of a `rows`-row dW owned by `rank` in the fused reduce-scatter (mirror of
    sb_dp_owned_rows, csrc/dp.cu): 32-row blocks, block rb -> rank rb * world // nblocks."""
    nb = (rows + 31) // 32

    def first(r):
        return (r * nb + world - 1) // world

    return min(rows, 32 * first(rank)), min(rows, 32 * first(rank + 1))


class _CudaView:
    """__cuda_array_interface__ over a raw device pointer (zero-copy torch view)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class SymmetricBuffer:
    """A device buffer allocated on every rank and mapped into every rank's process
    (sb_dp_symmetric_alloc + CUDA IPC), the target of the fused dW GEMM + reduce-scatter
    (sb_wgrad_reduce_scatter). The 64-byte IPC handles travel over the library's NCCL
    communicator (`comm`) or, without one, over torch.distributed (`all_gather_object`: gloo in
    the one-GPU multi-process tests)."""

    def __init__(self, handle, nbytes: int, rank: int = 0, world: int = 1, comm: NcclComm | None = None,
                 group=None):
        import ctypes as C

        from . import _capi as A

        self.h, self.rank, self.world = handle, rank, world
        ptr, ih = C.c_void_p(), (C.c_uint8 * 64)()
        A.check(handle.lib.sb_dp_symmetric_alloc(handle.h, nbytes, C.byref(ptr), ih))
        self.ptr, self.nbytes = ptr.value, nbytes
        if comm is not None:
            A.check(handle.lib.sb_dp_symmetric_exchange(handle.h, ptr, ih))
        else:
            mine = bytes(ih)
            if world > 1:
                allh: list = [None] * world
                dist.all_gather_object(allh, mine, group=group)
            else:
                allh = [mine]
            blob = (C.c_uint8 * (64 * world)).from_buffer_copy(b"".join(allh))
            A.check(handle.lib.sb_dp_symmetric_open(handle.h, ptr, rank, world, blob))

    def view(self, shape, offset_bytes: int = 0) -> torch.Tensor:
        """fp32 torch tensor over [offset, offset + prod(shape) * 4) of this rank's copy."""
        n = 1
        for s in shape:
            n *= s
        if offset_bytes < 0 or offset_bytes + 4 * n > self.nbytes or offset_bytes % 16:
            raise ValueError("view outside the symmetric buffer (or not 16-byte aligned)")
        return torch.as_tensor(_CudaView(self.ptr + offset_bytes, shape, "<f4"), device="cuda")

    def close(self) -> None:
        import ctypes as C

        from . import _capi as A

        if self.ptr:
            A.check(self.h.lib.sb_dp_symmetric_free(self.h.h, C.c_void_p(self.ptr)))
            self.ptr = 0


def wgrad_reduce_scatter(handle, g: torch.Tensor, x: torch.Tensor, dw: torch.Tensor, g_q=None, g_state=None) -> None:
    """dW GEMM whose epilogue reduce-adds each 32-row block into its owner rank's copy of the
    symmetric buffer behind `dw` (sb_wgrad_reduce_scatter). Every rank's dw must be zeroed and
    that ordered before this call on every rank."""
    import ctypes as C

    from . import _capi as A

    b, m = g.shape
    n = x.shape[1]
    handle.bind_stream(torch.cuda.current_stream(g.device).cuda_stream)
    A.check(handle.lib.sb_wgrad_reduce_scatter(
        handle.h, C.c_void_p(g.data_ptr()), C.c_void_p(x.data_ptr()), A.SB_BF16, b, m, n, C.c_void_p(dw.data_ptr()),
        C.c_void_p(g_q.data_ptr() if g_q is not None else None), m,
        C.c_void_p(g_state.data_ptr() if g_state is not None else None)))
