"""A real executor behind the reference simulator's fused iteration.

The reference's discrete-event engine charges every fused iteration an
analytic time (`duration = base + per_token·ξ + per_launch·launches`,
/root/reference/proj/src/sim.cpp:177-179).  This executor runs the same
iteration for real on the B200:

  peek each running job's next batch      (JobState::next_candidate_batch, workload.cpp:50-60)
  choose the jobs to fuse                 (fifo / priority / MinPad, batch_select.cpp:56-128 — the
                                           façade's C++ via packer.select)
  lay the rows out, account ξ, ξ_p, δ      (fuse / fused_shape, lora.cpp:72-158)
  one fused fwd + bwd + per-job AdamW     (FusedLoraLayer.step — the sm_100a kernels)
  commit the consumed items               (JobState::commit_batch, workload.cpp:62-66)

and emits the reference's `iteration_done{ξ, ξ_p, jobs_in_batch}` event
(sim.cpp:185-191) with the MEASURED device time and the per-job losses (what
the reference's detect_stop consumes, progress.cpp:90-124).  Metrics follow
compute_metrics (sim.cpp:258-265): δ = Σξ_p / Σξ, T_tot = Σξ / makespan,
T_e = (1 − δ)·T_tot.

Memory-budget admission (`memory_budget_gb`): each live job's footprint is
estimated by the measured memory model (memory.MemoryModel — live cudaMemGetInfo
probes of the real step fitted to PAPER Eq. 6; predict_memory_clamped at the
job's batch size and longest item, as estimate_job_memory, scheduler.cpp:36-42)
or, without a model, by JobConfig.memory_gb.  Admission then follows the
reference's schedule() (scheduler.cpp:74-130): fifo / priority order the live
jobs by arrival / urgency and admit greedily (greedy_admit :61-72: up to
max_concurrent, running estimate within the budget); minpad keeps the jobs that
fit alone, runs select_minpad and admits its choice greedily.  admission="pack"
first reduces the ordered list to its max_packing subset (the M4 pack_admission
path, :153-164).  An iteration whose admission is empty ends the run with
`Trace.truncated = "budget_exhausted"` (sim.cpp:140-147).

Early stopping (`early_stopping=True`) applies the reference's rule,
detect_stop (progress.cpp:90-124, restated below), to the REAL per-job losses
(and to accuracies from an optional `accuracy_fn`).  It is checked where the
reference's stream_stop checks it (sim.cpp:85-101): a job stops once its event's
iteration is <= the iterations it has done.  The job then leaves the candidate
set, and a `job_stopped` record is appended to `Trace.stops` (the reference's
scheduler.on_stop_event).  A job stopped for a non-finite loss is also
quarantined (FusedLoraLayer.quarantine): its bf16 operand copies are zeroed, so
its NaN adapter cannot reach the shared rank k-blocks of other jobs' tiles.
Pipelined, a step's losses are read while the next step is already queued, so a
stop seen in step t's losses takes effect from step t+2.  With
`pipelined=False` it takes effect from step t+1, as in the reference.

With `checkpoint_dir`, each job's adapter and AdamW state is saved
(FusedLoraLayer.save_job: reference layout, atomic write) when the job
completes or is stopped.

Two step backends.  Default: one transformer layer's LoRA'd projections
(FusedLoraLayer) on synthetic hidden states, loss L_j = 1/2 sum ||Y||^2.  Every
job's dataset items live in HBM (bf16 [len, k], seeded per item, so an epoch
revisits the same data) and each step's fused batch is built on the device by
mlora_fuse_rows — the reference's fuse (lora.cpp:114-158), bit-exact — in the
packed or the padded layout.  With
`model=DecoderConfig`: the whole decoder (model.MultiLoraDecoder) on each job's
token sequences, so the per-job losses detect_stop consumes are the real
padding-masked cross-entropy (K4).  A job's dataset items are then token
sequences (JobConfig.tokens, or deterministic synthetic tokens per item when
absent), so an epoch revisits the same items and the CE falls as the adapters
learn.

Row order: the kernels need each job's rows contiguous and in adapter order, so
the fused rows are placed in job-index order; the selection (urgency) order is
kept as the routing order reported in the event.  The linear layer is
row-independent, so this changes no result.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from . import fused as F
from . import packer as P
from .layer import FusedLoraLayer


def detect_stop(losses, accuracies=(), patience: int = 3):
    """fusim::detect_stop (progress.cpp:90-124): the first non-finite loss stops
    the job at that (1-based) iteration; `patience` consecutive accuracy values
    not above the best so far stop it at the last of them; the earlier event
    wins and a tie goes to the NaN stop.  Returns None or (iteration, cause)."""
    nan_ev = None
    for i, v in enumerate(losses):
        if not math.isfinite(v):
            nan_ev = (i + 1, "nan_loss")
            break
    dec_ev = None
    if len(accuracies) > 0 and patience >= 1:
        best, streak = accuracies[0], 0
        for i in range(1, len(accuracies)):
            if accuracies[i] <= best:
                streak += 1
                if streak == patience:
                    dec_ev = (i + 1, "accuracy_decline")
                    break
            else:
                best, streak = accuracies[i], 0
    if nan_ev and dec_ev:
        return nan_ev if nan_ev[0] <= dec_ev[0] else dec_ev
    return nan_ev or dec_ev


@dataclass
class JobConfig:
    id: str
    lengths: list                  # dataset item token counts
    batch_size: int = 4
    rank: int = 16
    lr: float = 1e-4
    scale: float = 2.0
    priority: int = 1
    submit_time: float = 0.0
    iterations: int = 10           # true_iterations
    tokens: list | None = None     # decoder backend: token ids of each dataset item (len == lengths[i])
    memory_gb: float = 0.0         # static footprint used without a memory model (JobSpec::memory_gb)


@dataclass
class _JobState:
    cfg: JobConfig
    cursor: int = 0
    done: int = 0
    losses: list = field(default_factory=list)      # one per completed iteration
    accuracies: list = field(default_factory=list)
    stopped: str | None = None                      # stop cause once early-stopped
    saved: bool = False                             # adapter checkpoint written

    @property
    def finished(self) -> bool:
        return self.stopped is not None or self.done >= self.cfg.iterations

    def peek_items(self) -> range:
        n = len(self.cfg.lengths)
        pos = self.cursor % n
        return range(pos, pos + min(self.cfg.batch_size, n - pos))

    def peek(self) -> list:
        return [self.cfg.lengths[i] for i in self.peek_items()]

    def commit(self, n_items: int) -> None:
        self.cursor += n_items
        if self.cursor >= len(self.cfg.lengths):
            self.cursor = 0


@dataclass
class Trace:
    events: list = field(default_factory=list)
    stops: list = field(default_factory=list)       # job_stopped records (early stopping)
    checkpoints: list = field(default_factory=list)  # {job, path, iterations, cause} per saved adapter
    busy_time: float = 0.0
    truncated: str | None = None                    # "budget_exhausted" when admission came back empty

    def metrics(self) -> dict:
        xi = sum(e["total_tokens"] for e in self.events)
        xi_p = sum(e["padding_tokens"] for e in self.events)
        eff = sum(e["effective_tokens"] for e in self.events)
        delta = xi_p / xi if xi else 0.0
        t_tot = xi / self.busy_time if self.busy_time else 0.0
        return {"iterations": len(self.events), "delta": delta, "T_tot": t_tot, "T_e": (1.0 - delta) * t_tot,
                "effective_tokens": eff, "effective_tokens_per_s": eff / self.busy_time if self.busy_time else 0.0,
                "busy_time_s": self.busy_time}


class FusedExecutor:
    """Runs fused multi-LoRA training iterations of several jobs on one GPU."""

    def __init__(self, ctx: F.Context, shapes, jobs: list[JobConfig], max_concurrent: int,
                 strategy: str = "minpad", padded: bool = False, seed: int = 0, W0: dict | None = None,
                 pipelined: bool = True, early_stopping: bool = False, patience: int = 3,
                 accuracy_fn=None, checkpoint_dir: str | None = None, model=None,
                 memory_budget_gb: float | None = None, memory_model=None, memory_floor_gb: float = 0.1,
                 admission: str = "greedy"):
        if admission not in ("greedy", "pack"):
            raise ValueError("admission must be 'greedy' or 'pack'")
        self.memory_budget_gb = memory_budget_gb
        self.memory_model = memory_model
        self.memory_floor_gb = memory_floor_gb
        self.admission = admission
        self.ctx = ctx
        self.checkpoint_dir = checkpoint_dir  # a job's adapter is saved when it completes or stops
        self.early_stopping = early_stopping
        self.patience = patience
        self.accuracy_fn = accuracy_fn  # (job_id, iteration, loss) -> accuracy or None
        self.shapes = shapes
        self.jobs = [_JobState(j) for j in jobs]
        self.M = max_concurrent
        self.strategy = strategy
        self.padded = padded
        self.pipelined = pipelined
        max_len = max(max(j.lengths) for j in jobs)
        max_bs = max(j.batch_size for j in jobs)
        capacity = max_concurrent * max_bs * max_len
        self.model = model
        if model is None:
            self.layer = FusedLoraLayer(ctx, shapes, [j.rank for j in jobs], [j.scale for j in jobs],
                                        [j.lr for j in jobs], rows=capacity, seed=seed, W0=W0)
            self.k_in = shapes[0][2]
            # each job's dataset, resident in HBM: item `it` of job i is the counter-based
            # fill with seed mix_seed(seed, 3, i, it) (the C++ executor builds the same bytes)
            self.data = [[F.fill_uniform(torch.empty(n, self.k_in, dtype=torch.bfloat16, device=ctx.device),
                                         F.mix_seed(seed, 3, i, it), -1.0, 1.0)
                          for it, n in enumerate(j.lengths)] for i, j in enumerate(jobs)]
            self._x = torch.empty(capacity, self.k_in, dtype=torch.bfloat16, device=ctx.device)
            self._mask = torch.empty(capacity, dtype=torch.uint8, device=ctx.device)
        else:
            from .model import MultiLoraDecoder
            for j in jobs:
                if j.tokens is not None and [len(t) for t in j.tokens] != list(j.lengths):
                    raise ValueError(f"job {j.id}: token sequences do not match its lengths")
            self.layer = MultiLoraDecoder(ctx, model, [j.rank for j in jobs], [j.scale for j in jobs],
                                          [j.lr for j in jobs], capacity=capacity, seed=seed)
        self.trace = Trace()
        self.clock = 0.0
        self._pending = None  # the enqueued step whose time/losses have not been collected yet
        self._loss_host = [torch.empty(len(jobs), dtype=torch.float32).pin_memory() for _ in range(2)]
        self._slot = 0

    def _item_tokens(self, i: int, item: int) -> list:
        """Token ids of job i's dataset item (given, or synthetic and fixed per item)."""
        cfg = self.jobs[i].cfg
        if cfg.tokens is not None:
            return list(cfg.tokens[item])
        g = torch.Generator().manual_seed(1_000_003 * (i + 1) + item)
        return torch.randint(0, self.model.vocab, (cfg.lengths[item],), generator=g).tolist()

    def active(self) -> list[int]:
        return [i for i, js in enumerate(self.jobs) if not js.finished]

    def job_memory_gb(self, i: int) -> float:
        """estimate_job_memory (scheduler.cpp:36-42): the fitted model at the job's
        batch size and longest item, clamped to the floor; else its static size."""
        cfg = self.jobs[i].cfg
        if self.memory_model is not None:
            return self.memory_model.predict_clamped(cfg.batch_size, max(cfg.lengths), self.memory_floor_gb)
        return float(cfg.memory_gb)

    def _admit(self, live: list[int]) -> tuple[list[int], dict]:
        """schedule() (scheduler.cpp:74-130) under the memory budget -> admitted job
        indices in admission order, and their estimates (memory.admit)."""
        from . import memory as MM
        est = {i: self.job_memory_gb(i) for i in live}
        queue = [MM.QueuedJob(self.jobs[i].cfg.id, self.jobs[i].cfg.priority, self.jobs[i].cfg.submit_time,
                              self.jobs[i].peek(), est[i]) for i in live]
        picked = MM.admit(queue, self.strategy, float(self.memory_budget_gb), self.M, self.admission)
        return [live[q] for q in picked], est

    def _collect(self) -> dict | None:
        """Finish the pending step: wait for its end event, read its device time and
        its per-job losses (copied D2H into pinned memory when it was enqueued)."""
        if self._pending is None:
            return None
        pend, self._pending = self._pending, None
        pend["e1"].synchronize()
        duration = pend["e0"].elapsed_time(pend["e1"]) / 1e3
        losses = pend["loss"].tolist()
        self.clock += duration
        self.trace.busy_time += duration
        ev = {"type": "iteration_done", "time": self.clock, "duration_s": duration, **pend["meta"],
              "losses": {self.jobs[i].cfg.id: losses[i] for i in pend["chosen"]}}
        self.trace.events.append(ev)
        for i in pend["chosen"]:
            js = self.jobs[i]
            js.losses.append(losses[i])
            if self.accuracy_fn is not None:
                acc = self.accuracy_fn(js.cfg.id, len(js.losses), losses[i])
                if acc is not None:
                    js.accuracies.append(float(acc))
            if self.early_stopping and js.stopped is None:
                stop = detect_stop(js.losses, js.accuracies, self.patience)
                if stop is not None and stop[0] <= len(js.losses):
                    js.stopped = stop[1]
                    if stop[1] == "nan_loss":
                        self.layer.quarantine(i)  # a non-finite adapter must not reach other jobs' tiles
                    self.trace.stops.append({"type": "job_stopped", "time": self.clock, "job": js.cfg.id,
                                             "iteration": stop[0], "cause": stop[1],
                                             "iterations_done": js.done})
            if self.checkpoint_dir is not None and js.finished and not js.saved:
                self._checkpoint(i, js.stopped or "completed")
        return ev

    def _checkpoint(self, i: int, cause: str) -> None:
        """Save job i's adapter + AdamW state (reference layout, atomic write).
        The host copy waits for the work already queued on the stream."""
        import os
        js = self.jobs[i]
        path = os.path.join(self.checkpoint_dir, f"{js.cfg.id}.pt")
        self.layer.save_job(path, i)
        js.saved = True
        self.trace.checkpoints.append({"job": js.cfg.id, "path": path, "iterations": js.done, "cause": cause})

    def step(self) -> dict | None:
        """Select, pack and enqueue the next fused iteration.  Pipelined (default):
        returns the PREVIOUS iteration's event, so the host packing of step t+1
        overlaps the device executing step t; `flush()` collects the last one."""
        live = self.active()
        if not live or self.trace.truncated:
            return self._collect()
        mem_meta = {}
        if self.memory_budget_gb is None:
            cands = [P.Candidate(i, self.jobs[i].peek(), self.jobs[i].cfg.priority, self.jobs[i].cfg.submit_time,
                                 id=self.jobs[i].cfg.id) for i in live]
            sel = P.select(cands, self.M, self.strategy)
            chosen = [cands[c].job for c in sel.chosen]      # job indices, urgency (routing) order
        else:
            chosen, est = self._admit(live)                  # admission order
            if not chosen:
                self.trace.truncated = "budget_exhausted"
                return self._collect()
            mem_meta = {"estimated_memory_gb": sum(est[i] for i in chosen),
                        "per_job_memory_gb": {self.jobs[i].cfg.id: est[i] for i in chosen}}
        batches = {i: self.jobs[i].peek() for i in chosen}
        in_batch = sorted(chosen)                            # row order: job-index order
        lay = P.layout([batches[i] for i in in_batch], padded=self.padded)
        seg, r = [0], 0
        for j in range(len(self.jobs)):
            if j in batches:
                r = lay.seg[in_batch.index(j) + 1]
            seg.append(r)
        active = [j in batches for j in range(len(self.jobs))]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()  # the measured iteration includes building the fused batch on the device
        if self.model is None:
            self.layer.set_layout(seg)                       # stream-ordered plan update, no host sync
            seqs = [self.data[j][it] for j in in_batch for it in self.jobs[j].peek_items()]
            x, _, offs = F.fuse_rows(self.ctx, seqs, padded=self.padded, out=self._x[:lay.rows],
                                     mask=self._mask[:lay.rows])  # device fuse: pad rows zero as in fuse()
            if offs[:-1] != [r0 for rows in lay.seq_rows for r0, _ in rows]:
                raise RuntimeError("device fuse layout disagrees with the packer's layout")
        else:
            from .model import pack_tokens
            seqs = [[self._item_tokens(j, it) for it in self.jobs[j].peek_items()] if j in batches else []
                    for j in range(len(self.jobs))]
            tb = pack_tokens(seqs, padded=self.padded)
            if tb.seg != seg:
                raise RuntimeError("token layout disagrees with the packer's layout")
            self.layer.set_batch(tb)                         # stream-ordered uploads, no host sync
        slot = self._loss_host[self._slot]
        self._slot ^= 1
        if self.model is None:
            loss = self.layer.step(x, active=active)
        else:
            loss = self.layer.forward()
            self.layer.backward()
            self.layer.optimizer_step(active=active)
        slot.copy_(loss, non_blocking=True)                  # D2H of this step's per-job losses
        e1.record()
        prev = self._collect()                               # step t-1 (normally finished already)
        for i in chosen:
            self.jobs[i].commit(len(batches[i]))
            self.jobs[i].done += 1
        self._pending = {"e0": e0, "e1": e1, "loss": slot, "chosen": chosen,
                         "meta": {"total_tokens": lay.total_tokens, "padding_tokens": lay.padding_tokens,
                                  "effective_tokens": lay.effective_tokens, "rows": lay.rows,
                                  "jobs_in_batch": len(chosen), "routing": [self.jobs[i].cfg.id for i in chosen],
                                  **mem_meta}}
        if not self.pipelined:
            return self._collect()
        return prev

    def flush(self) -> dict | None:
        return self._collect()

    def run(self, max_iterations: int | None = None) -> Trace:
        n = 0
        while (max_iterations is None or n < max_iterations) and self.active() and not self.trace.truncated:
            self.step()
            n += 1
        self.flush()
        return self.trace
