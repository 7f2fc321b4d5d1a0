"""The measured memory model — owned by the product.

PAPER Eq. 6: the memory of one job's fused training step is
M(B_t, L_n) = beta0 + beta1 * B_t * L_n + beta2 * B_t * L_n^2.  The reference
fits it from warm-up samples (fit_memory_model, /root/reference/proj/src/
memory_model.cpp:76-152), plans the warm-up probes (warmup_plan :241-259),
packs jobs under a budget (max_packing :200-239) and admits jobs per
scheduling step (greedy_admit, scheduler.cpp:61-72).  Here:

  * the probes are LIVE: each (B_t, L_n) of the warm-up plan runs the real
    fused step (FusedLoraLayer, one job, B_t * L_n rows) and its footprint is
    read with cudaMemGetInfo through the C ABI (mlora_mem_info) — adapters,
    optimizer state, activations, the context's workspace; the replicated
    frozen W0 is shared by every job and excluded, as in the reference's
    per-job estimate;
  * the fit, the prediction, the packer and the warm-up plan are the façade's
    C++ (include/fusim/memory_model.hpp, the same code a C++ fusim user links);
  * executor.FusedExecutor admits jobs per iteration under a budget with it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _native as N
from . import packer as P


@dataclass
class MemoryModel:
    """fusim::MemoryModel (memory_model.hpp): GB = b0 + b1 Bt Ln + b2 Bt Ln^2."""
    beta0: float = 0.0
    beta1: float = 0.0
    beta2: float = 0.0
    rmse: float = 0.0
    sample_count: int = 0

    def predict(self, batch_size: int, seq_len: int) -> float:
        """predict_memory (memory_model.cpp:154-157)."""
        u = float(batch_size) * seq_len
        return self.beta0 + u * (self.beta1 + self.beta2 * seq_len)

    def predict_clamped(self, batch_size: int, seq_len: int, floor_gb: float) -> float:
        """predict_memory_clamped (memory_model.cpp:159-167)."""
        return max(self.predict(batch_size, seq_len), floor_gb)


def fit_memory_model(samples, nonnegative: bool = False) -> MemoryModel:
    """samples: [(batch_size, seq_len, mem_gb)] -> MemoryModel (FitError as the reference)."""
    n = len(samples)
    bs = (C.c_int32 * max(n, 1))(*[int(s[0]) for s in samples])
    sl = (C.c_int32 * max(n, 1))(*[int(s[1]) for s in samples])
    mem = (C.c_double * max(n, 1))(*[float(s[2]) for s in samples])
    out = (C.c_double * 4)()
    P._chk(P.lib().fusim_c_fit_memory_model(n, bs, sl, mem, 1 if nonnegative else 0, out))
    return MemoryModel(out[0], out[1], out[2], out[3], n)


def max_packing(item_gb, budget_gb: float, greedy: bool = False) -> list[int]:
    """fusim::max_packing: a feasible subset of maximum total (ascending indices)."""
    n = len(item_gb)
    items = (C.c_double * max(n, 1))(*[float(x) for x in item_gb])
    out = (C.c_int32 * max(n, 1))()
    cnt = C.c_int32()
    P._chk(P.lib().fusim_c_max_packing(n, items, float(budget_gb), 1 if greedy else 0, out, C.byref(cnt)))
    return [int(out[i]) for i in range(cnt.value)]


def warmup_plan(batch_sizes, seq_lens) -> tuple[list[tuple[int, int]], bool]:
    """fusim::warmup_plan: (probes, sufficient)."""
    nb, nl = len(batch_sizes), len(seq_lens)
    b = (C.c_int32 * max(nb, 1))(*[int(x) for x in batch_sizes])
    s = (C.c_int32 * max(nl, 1))(*[int(x) for x in seq_lens])
    out = (C.c_int32 * max(2 * nb * nl, 2))()
    cnt, suff = C.c_int32(), C.c_int32()
    P._chk(P.lib().fusim_c_warmup_plan(nb, b, nl, s, out, C.byref(cnt), C.byref(suff)))
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(cnt.value)], bool(suff.value)


def device_free_bytes(ctx) -> int:
    free, total = C.c_size_t(), C.c_size_t()
    N.check(N.lib().mlora_mem_info(ctx.handle, C.byref(free), C.byref(total)), ctx.handle)
    return int(free.value)


def measure_step_gb(device, shapes, ranks, rows: int, W0: dict, seed: int = 0) -> float:
    """Device memory of one fused training step (cudaMemGetInfo before / after):
    a fresh context (its workspace counts), a FusedLoraLayer holding `ranks`
    jobs' adapters + AdamW state and activations for `rows` fused rows, one full
    step run, everything freed afterwards.  W0 (shared, replicated) is passed in
    and not counted, nor is the step's input x (the fused batch: host data in
    flight, double-buffered by the trainer).  The layer is one arena allocation,
    so the reading is its bytes to the driver's 2 MB page."""
    from . import fused as F
    from .layer import FusedLoraLayer
    import gc
    dev = torch.device(device)
    torch.cuda.synchronize(dev)
    gc.collect()  # a previous probe's layer must really be gone before the baseline
    torch.cuda.empty_cache()
    probe = F.Context(dev)
    free0 = device_free_bytes(probe)
    ctx = F.Context(dev)
    J = len(ranks)
    layer = FusedLoraLayer(ctx, shapes, ranks, [2.0] * J, [1e-4] * J, rows=rows, seed=seed, W0=W0)
    per = rows // J
    layer.set_layout([min(rows, j * per) if j < J else rows for j in range(J + 1)])
    x = F.fill_uniform(torch.empty(rows, shapes[0][2], dtype=torch.bfloat16, device=dev), seed + 1)
    layer.step(x)
    torch.cuda.synchronize(dev)
    del x
    torch.cuda.empty_cache()  # the init temporaries (per-job fp32 adapters before packing) are gone
    used = free0 - device_free_bytes(probe)
    layer.close()
    del layer
    ctx.close()
    torch.cuda.synchronize(dev)
    gc.collect()
    torch.cuda.empty_cache()
    probe.close()
    return used / 2 ** 30


def probe_samples(device, shapes, rank: int, batch_sizes, seq_lens, W0: dict) -> list[tuple[int, int, float]]:
    """The warm-up phase: every probe of warmup_plan(batch_sizes, seq_lens) runs
    one real fused step for one job of `rank` on B_t * L_n rows; returns the
    reference's MemSample rows (batch_size, seq_len, mem_gb)."""
    probes, _ = warmup_plan(batch_sizes, seq_lens)
    # one discarded probe first: the process's one-off device costs (lazily loaded
    # kernel modules, the stream-ordered pool) land there, not in a job's sample
    measure_step_gb(device, shapes, [rank], probes[0][0] * probes[0][1], W0)
    return [(bt, ln, measure_step_gb(device, shapes, [rank], bt * ln, W0)) for bt, ln in probes]


def greedy_admit(order, est: dict, budget_gb: float, max_concurrent: int) -> tuple[list, float]:
    """scheduler.cpp:61-72: walk `order`, admit while fewer than max_concurrent
    are in and the running estimate stays within the budget."""
    chosen, total = [], 0.0
    for j in order:
        if len(chosen) >= max_concurrent:
            break
        if total + est[j] <= budget_gb:
            chosen.append(j)
            total += est[j]
    return chosen, total


@dataclass
class QueuedJob:
    """What admission sees of a live job (JobState as schedule() reads it)."""
    id: str
    priority: int
    submit_time: float
    next_batch: list          # item lengths of its next candidate batch (next_candidate_batch)
    memory_gb: float          # its estimate (estimate_job_memory)


def admit(queue: list[QueuedJob], strategy: str, budget_gb: float, max_concurrent: int,
          admission: str = "greedy") -> list[int]:
    """schedule() for M1 / M2 / M3 (scheduler.cpp:74-130) -> indices into `queue`
    in admission order.  fifo: arrival order (submit, id); priority: urgency
    (priority desc, submit, id); minpad: the jobs that fit the budget alone,
    select_minpad(max_concurrent) (the façade's C++).  Then greedy_admit.
    admission="pack" first keeps the ordered list's max_packing subset (the
    M4 pack_admission step, :153-164)."""
    est = {i: q.memory_gb for i, q in enumerate(queue)}
    if strategy == "fifo":
        order = sorted(range(len(queue)), key=lambda i: (queue[i].submit_time, queue[i].id))
    elif strategy == "priority":
        order = sorted(range(len(queue)), key=lambda i: (-queue[i].priority, queue[i].submit_time, queue[i].id))
    elif strategy == "minpad":
        fits = [i for i in range(len(queue)) if est[i] <= budget_gb]
        if not fits:
            return []
        cands = [P.Candidate(i, queue[i].next_batch, queue[i].priority, queue[i].submit_time, id=queue[i].id)
                 for i in fits]
        order = [cands[c].job for c in P.select(cands, max_concurrent, "minpad").chosen]
    else:
        raise ValueError(f"unknown strategy {strategy!r}")
    if admission == "pack":
        keep = max_packing([est[i] for i in order], budget_gb)
        order = [order[k] for k in keep]
    elif admission != "greedy":
        raise ValueError("admission must be 'greedy' or 'pack'")
    return greedy_admit(order, est, budget_gb, max_concurrent)[0]
