"""Adapter-parallel multi-GPU plumbing.

The BatchFusion path shards by job: every rank owns a disjoint set of LoRA jobs
(their adapters, optimizer state and token rows) and a replica of the frozen
base weights.  The only collective is the one-off broadcast of W0 from rank 0
(NCCL over NVLink on B200; gloo in the CPU tests); the steady state exchanges
nothing — per-job losses stay with the rank that owns the job.  Timing takes
the max over ranks.
"""
from __future__ import annotations

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


def broadcast_base_weights(weights: dict, src: int = 0, group=None) -> None:
    """Replicate the frozen base weights from `src` to every rank, in place,
    one broadcast per tensor in sorted-name order (all ranks agree on order)."""
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
