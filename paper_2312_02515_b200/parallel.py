"""Adapter-parallel multi-GPU plumbing.

The BatchFusion path shards by job: every rank owns a disjoint set of LoRA jobs
(their adapters, optimizer state and token rows) and a replica of the frozen
base weights.  The only collective is the one-off broadcast of W0 from rank 0
(NCCL over NVLink on B200; gloo in the CPU tests); the steady state exchanges
nothing — per-job losses stay with the rank that owns the job.  Timing takes
the max over ranks.
"""
from __future__ import annotations

import ctypes
import heapq

import torch
import torch.distributed as dist


def partition_jobs(expected_tokens, world: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of jobs to ranks by expected
    effective tokens per step.  Deterministic: ties go to the lower job index
    and the lower rank.  Returns, per rank, its job indices in ascending order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(expected_tokens)), key=lambda j: (-float(expected_tokens[j]), j))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    parts = [[] for _ in range(world)]
    for j in order:
        load, r = heapq.heappop(heap)
        parts[r].append(j)
        heapq.heappush(heap, (load + float(expected_tokens[j]), r))
    return [sorted(p) for p in parts]


def comm_rendezvous_id(group=None, rank: int | None = None, world: int | None = None) -> bytes:
    """The NCCL unique id for a native communicator: made by group rank 0
    (mlora_comm_unique_id — host only, no GPU needed) and shipped to the other
    ranks over the torch.distributed group; every rank returns the same bytes."""
    from . import _native as N
    L = N.lib()
    rank = dist.get_rank(group) if rank is None else rank
    world = dist.get_world_size(group) if world is None else world
    buf = (ctypes.c_uint8 * L.mlora_comm_id_bytes())()
    if rank == 0:
        N.check(L.mlora_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    if world == 1:
        return bytes(buf)
    box = [bytes(buf) if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return box[0]


class NativeComm:
    """The C ABI's NCCL communicator (include/mlora.h `mlora_comm_*`), bound to
    one context's GPU.  The 128-byte NCCL id travels from rank 0 to the others
    over the already-initialised torch.distributed group (any backend — gloo is
    enough); after that, the collectives run in libmlora.so, not in torch."""

    def __init__(self, ctx, group=None, rank: int | None = None, world: int | None = None):
        from . import _native as N
        self._N = N
        L = N.lib()
        rank = dist.get_rank(group) if rank is None else rank
        world = dist.get_world_size(group) if world is None else world
        buf = (ctypes.c_uint8 * L.mlora_comm_id_bytes()).from_buffer_copy(comm_rendezvous_id(group, rank, world))
        handle = ctypes.c_void_p()
        N.check(L.mlora_comm_create(ctx.handle, ctypes.cast(buf, ctypes.c_void_p), world, rank,
                                    ctypes.byref(handle)), ctx.handle)
        self.ctx, self.handle, self.rank, self.world = ctx, handle, rank, world

    def broadcast(self, tensors, root: int = 0, stream=None) -> None:
        """All buffers in one NCCL group (mlora_broadcast_base), in place."""
        N = self._N
        n = len(tensors)
        ptrs = (N.vp * n)(*[t.data_ptr() for t in tensors])
        sizes = (N.i64 * n)(*[t.numel() * t.element_size() for t in tensors])
        s = torch.cuda.current_stream(tensors[0].device).cuda_stream if stream is None and n else stream
        N.check(N.lib().mlora_broadcast_base(self.handle, n, ptrs, sizes, root, s), self.ctx.handle)

    def sum_(self, t: torch.Tensor, stream=None) -> torch.Tensor:
        """In-place fp32 sum over ranks (mlora_comm_sum_f32)."""
        if t.dtype != torch.float32 or not t.is_contiguous():
            raise TypeError("sum_ needs a contiguous float32 tensor")
        s = torch.cuda.current_stream(t.device).cuda_stream if stream is None else stream
        self._N.check(self._N.lib().mlora_comm_sum_f32(self.handle, t.data_ptr(), t.numel(), s), self.ctx.handle)
        return t

    def close(self) -> None:
        if self.handle:
            self._N.lib().mlora_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def broadcast_base_weights(weights: dict, src: int = 0, group=None, comm: NativeComm | None = None) -> None:
    """Replicate the frozen base weights from `src` to every rank, in place, in
    sorted-name order (all ranks agree on order).  With `comm` (the native
    communicator) every tensor goes in ONE NCCL group through libmlora.so;
    otherwise one torch.distributed broadcast per tensor (gloo on CPU)."""
    if comm is not None:
        comm.broadcast([weights[name] for name in sorted(weights)], root=src)
        return
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    for name in sorted(weights):
        dist.broadcast(weights[name], src=src, group=group)


def max_over_ranks(value: float, device=None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
