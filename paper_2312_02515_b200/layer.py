"""One fused multi-LoRA training step over the LoRA'd projections of a transformer layer.

This is the executor that slots in at the reference simulator's fused-iteration
hook (/root/reference/proj/src/sim.cpp:163-191): given the fused batch's
segment layout (which rows belong to which job, from the MinPad packer) it runs
every projection's forward, the per-job loss, every backward and one per-job-lr
AdamW update — all on device, all through the C ABI, with no per-job launches.

Step semantics (stated in DESIGN.md §Measurement): the layer's hidden state x
feeds q, k, v, gate, up; o consumes v's output and down consumes up's output
(attention / SiLU-gating are outside the hot path).  The per-job loss is
L_j = 1/2 sum_p ||Y_p[rows of j]||^2, so dL/dY_p = Y_p (every projection's
backward is exact for this loss with its input detached).  FLOPs per effective
token per projection: 4dk + 6 r (d + k).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as N
from . import fused as F

# (name, d_out, k_in, input source)
LLAMA7B = [("q", 4096, 4096, "x"), ("k", 4096, 4096, "x"), ("v", 4096, 4096, "x"), ("o", 4096, 4096, "v"),
           ("gate", 11008, 4096, "x"), ("up", 11008, 4096, "x"), ("down", 4096, 11008, "up")]
LLAMA13B = [("q", 5120, 5120, "x"), ("k", 5120, 5120, "x"), ("v", 5120, 5120, "x"), ("o", 5120, 5120, "v"),
            ("gate", 13824, 5120, "x"), ("up", 13824, 5120, "x"), ("down", 5120, 13824, "up")]
# ChatGLM2-6B: multi-query attention -> fused qkv 4096 -> 4096 + 2*2*128 = 4608; h->4h is the fused
# gate/up (2 x 13696 = 27392); 4h->h 13696 -> 4096.
CHATGLM2_6B = [("qkv", 4608, 4096, "x"), ("dense", 4096, 4096, "x"), ("h_to_4h", 27392, 4096, "x"),
               ("4h_to_h", 4096, 13696, "h_to_4h_half")]
TINY = [("q", 256, 256, "x"), ("k", 256, 256, "x"), ("v", 256, 256, "x"), ("o", 256, 256, "v"),
        ("gate", 688, 256, "x"), ("up", 688, 256, "x"), ("down", 256, 688, "up")]

SHAPES = {"llama7b": LLAMA7B, "llama13b": LLAMA13B, "chatglm2_6b": CHATGLM2_6B, "tiny": TINY}


def flops_per_token(shapes, rank: int) -> int:
    """Algorithmic fwd+bwd FLOPs per effective token for one job of rank r (frozen W0)."""
    return sum(4 * d * k + 6 * rank * (d + k) for _, d, k, _ in shapes)


class AdapterJobsMixin:
    """Per-job adapter management shared by FusedLoraLayer and the decoder
    (model.MultiLoraDecoder): quarantine and checkpoint / resume.  Needs
    `ctx, plan, ranks, scales, lrs, step_count` and `named_projections()` ->
    [(key, projection with d, k, A, B: fused.AdamState)]."""

    def quarantine(self, job: int) -> None:
        """Zero job `job`'s bf16 operand copies (its rows of every A_cat, its
        columns of every B_cat, on every projection), stream-ordered.  The
        fused kernels rely on structural zeros: the other jobs' rows of H_cat / G_cat are exactly 0
        and multiply this job's adapter inside a shared 64-column rank k-block.
        0 * NaN is NaN, so a diverged adapter could poison its neighbours.  The
        executor calls this when early stopping retires a job with a
        non-finite loss.  Its fp32 masters and moments are kept for inspection."""
        r0, r1 = self.plan.rank_offsets[job], self.plan.rank_offsets[job + 1]
        for _, p in self.named_projections():
            p.A.p_bf16[r0:r1].zero_()
            p.B.p_bf16[:, r0:r1].zero_()

    # ------------------------------------------------------------ checkpoint / resume
    CKPT_FORMAT = "mlora-adapter-v1"

    def job_state(self, job: int) -> dict:
        """Job `job`'s adapter and AdamW state in the reference's layout
        (AdapterWeights, lora.hpp:34-41: A_j r x k, B_j d x r, fp32), copied to
        host after everything already queued on the current stream."""
        r0, r = self.plan.rank_offsets[job], self.ranks[job]
        proj = {}
        for key, p in self.named_projections():
            proj[key] = {"d": p.d, "k": p.k,
                         "A": p.A.p[r0:r0 + r].cpu(), "mA": p.A.m[r0:r0 + r].cpu(), "vA": p.A.v[r0:r0 + r].cpu(),
                         "B": p.B.p[:, r0:r0 + r].cpu(), "mB": p.B.m[:, r0:r0 + r].cpu(),
                         "vB": p.B.v[:, r0:r0 + r].cpu()}
        return {"format": self.CKPT_FORMAT, "rank": r, "scale": self.scales[job], "lr": self.lrs[job],
                "step": self.step_count[job], "proj": proj}

    def save_job(self, path: str, job: int) -> None:
        """Atomically write job `job`'s state (temp file + fsync + rename, as the
        reference writes its outputs: io.cpp:404-414 atomic_write)."""
        import os
        state = self.job_state(job)
        d = os.path.dirname(os.path.abspath(path))
        os.makedirs(d, exist_ok=True)
        tmp = path + ".tmp"
        with open(tmp, "wb") as f:
            torch.save(state, f)
            f.flush()
            os.fsync(f.fileno())
        os.replace(tmp, path)

    def load_job(self, path_or_state, job: int) -> None:
        """Resume job `job` from a saved state: fp32 masters, AdamW moments and
        step count go into the job's cat-layout slices, the bf16 operand copies
        are refreshed.  UsageError on a foreign file or a rank / scale mismatch
        (as AdapterWeights::validate, lora.cpp:62-70); ShapeError on projection
        dims."""
        from . import errors as E
        st = torch.load(path_or_state, map_location="cpu") if isinstance(path_or_state, str) else path_or_state
        if not isinstance(st, dict) or st.get("format") != self.CKPT_FORMAT:
            raise E.UsageError("not an mlora adapter checkpoint")
        if st["rank"] != self.ranks[job]:
            raise E.UsageError(f"checkpoint rank {st['rank']} != slot rank {self.ranks[job]}")
        if float(st["scale"]) != float(self.scales[job]):  # s_j lives in the plan's device tables
            raise E.UsageError(f"checkpoint scale {st['scale']} != slot scale {self.scales[job]}")
        named = self.named_projections()
        names = {key for key, _ in named}
        if set(st["proj"]) != names:
            raise E.ShapeError(f"checkpoint projections {sorted(st['proj'])} != layer {sorted(names)}")
        r0, r = self.plan.rank_offsets[job], self.ranks[job]
        for key, p in named:
            q = st["proj"][key]
            if (q["d"], q["k"]) != (p.d, p.k) or tuple(q["A"].shape) != (r, p.k) or tuple(q["B"].shape) != (p.d, r):
                raise E.ShapeError(f"projection {key}: checkpoint shape does not match the layer")
        dev = self.ctx.device
        for key, p in named:
            q = st["proj"][key]
            p.A.p[r0:r0 + r] = q["A"].to(dev)
            p.A.m[r0:r0 + r] = q["mA"].to(dev)
            p.A.v[r0:r0 + r] = q["vA"].to(dev)
            p.A.p_bf16[r0:r0 + r] = p.A.p[r0:r0 + r].to(torch.bfloat16)
            p.B.p[:, r0:r0 + r] = q["B"].to(dev)
            p.B.m[:, r0:r0 + r] = q["mB"].to(dev)
            p.B.v[:, r0:r0 + r] = q["vB"].to(dev)
            p.B.p_bf16[:, r0:r0 + r] = p.B.p[:, r0:r0 + r].to(torch.bfloat16)
        self.lrs[job] = float(st["lr"])
        self.step_count[job] = int(st["step"])


@dataclass
class Projection:
    name: str
    d: int
    k: int
    src: str
    W0: torch.Tensor                   # bf16 [d, k] frozen base weight (replicated)
    A: F.AdamState                     # A_cat fp32 master [R_pad, k] (+ bf16 copy)
    B: F.AdamState                     # B_cat fp32 master [d, R_pad] (+ bf16 copy)
    dA: torch.Tensor                   # fp32 [R_pad, k]
    dB: torch.Tensor                   # fp32 [d, R_pad]
    Y: torch.Tensor                    # bf16 [rows, d]
    H: torch.Tensor                    # bf16 [rows, R_pad]
    G: torch.Tensor                    # bf16 [rows, R_pad]
    dX: torch.Tensor                   # bf16 [rows, k]
    row_sq: torch.Tensor               # fp32 [ceil(d/256), rows] fused-loss row partials


class FusedLoraLayer(AdapterJobsMixin):
    """All adapters of J jobs on one layer's projections, cat layout, on one GPU."""

    def __init__(self, ctx: F.Context, shapes, ranks, scales, lrs, rows: int, seed: int = 0,
                 W0: dict | None = None, lora_init: str = "random"):
        self.ctx = ctx
        self.shapes = shapes
        self.ranks = list(ranks)
        self.scales = list(scales)
        self.lrs = list(lrs)
        self.J = len(ranks)
        self.rows = rows
        self.step_count = [0] * self.J
        dev = ctx.device
        # plan with a placeholder layout; set_layout() installs the real one
        self.plan = F.Plan(ctx, [0] * self.J + [rows], ranks, scales)
        R = self.plan.rank_padded
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.proj: list[Projection] = []
        for name, d, k, src in shapes:
            if W0 is not None and name in W0:
                w = W0[name]
            else:
                w = ((torch.rand(d, k, generator=g) * 2 - 1) / k ** 0.5).to(torch.bfloat16).to(dev)
            As, Bs = [], []
            for r in ranks:
                As.append(((torch.rand(r, k, generator=g) * 2 - 1) / k ** 0.5).to(dev))
                if lora_init == "zero_b":   # standard LoRA init: B = 0
                    Bs.append(torch.zeros(d, r, device=dev))
                else:
                    Bs.append(((torch.rand(d, r, generator=g) * 2 - 1) / r ** 0.5).to(dev))
            A32, B32, A16, B16 = F.pack_adapters(ctx, self.plan, d, k, As, Bs)
            self.proj.append(Projection(
                name, d, k, src, w, F.AdamState.of(A32, A16, 0), F.AdamState.of(B32, B16, 1),
                torch.zeros(R, k, device=dev), torch.zeros(d, R, device=dev),
                torch.empty(rows, d, dtype=torch.bfloat16, device=dev),
                torch.empty(rows, R, dtype=torch.bfloat16, device=dev),
                torch.empty(rows, R, dtype=torch.bfloat16, device=dev),
                torch.empty(rows, k, dtype=torch.bfloat16, device=dev),
                torch.empty(N.lib().mlora_rowsq_blocks(d), rows, dtype=torch.float32, device=dev)))
        self.loss = torch.zeros(self.J, dtype=torch.float32, device=dev)
        self._rowsq_d = (N.i32 * len(self.proj))(*[p.d for p in self.proj])

    def set_layout(self, seg_offsets) -> None:
        """Install the segment layout of the next fused batch: job j owns rows
        seg[j]:seg[j+1] (empty for jobs not in this batch); total rows <= capacity."""
        rows = int(seg_offsets[-1])
        if rows < 1 or rows > self.rows:
            raise ValueError(f"layout rows {rows} outside [1, capacity {self.rows}]")
        self.plan.update(seg_offsets)  # stream-ordered, no host sync
        self.cur_rows = rows

    def named_projections(self):
        return [(p.name, p) for p in self.proj]

    def _views(self, p: Projection, rows: int):
        nblk = p.row_sq.shape[0]
        return (p.Y[:rows], p.H[:rows], p.G[:rows], p.dX[:rows],
                p.row_sq.view(-1)[: nblk * rows].view(nblk, rows))

    def _input(self, src: str, x: torch.Tensor, rows: int) -> torch.Tensor:
        if src == "x":
            return x
        if src == "h_to_4h_half":
            p = next(q for q in self.proj if q.name == "h_to_4h")
            # first half of the fused gate/up output (stand-in for the gated act.)
            return p.Y[:rows, : p.d // 2].contiguous()
        return next(q for q in self.proj if q.name == src).Y[:rows]

    def forward_backward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """Grouped schedule: every HBM-bound op is issued once for all projections
        whose inputs are ready (mlora_down_group / mlora_grad_group), the tensor-
        bound base GEMMs once per projection.  LLaMA layer: 2 forward down-group
        launches, 7 base GEMMs, loss, non-finite guard, 1 backward down-group, 7 dX GEMMs,
        1 grad group."""
        ctx, plan = self.ctx, self.plan
        L, s = N.lib(), F._stream_handle(stream)
        rows = getattr(self, "cur_rows", self.rows)
        views = [self._views(p, rows) for p in self.proj]
        inputs: dict[int, torch.Tensor] = {}
        done: set[str] = set()
        # ---- forward, in dependency waves
        while len(done) < len(self.proj):
            source = lambda src: None if src == "x" else ("h_to_4h" if src == "h_to_4h_half" else src)
            wave = [i for i, p in enumerate(self.proj)
                    if p.name not in done and (source(p.src) is None or source(p.src) in done)]
            if not wave:
                raise RuntimeError("projection inputs form a cycle")
            for i in wave:
                inputs[i] = self._input(self.proj[i].src, x, rows)
            n = len(wave)
            N.check(L.mlora_down_group(ctx.handle, plan.handle, n, 0,
                                       (N.i32 * n)(*[self.proj[i].k for i in wave]),
                                       (N.vp * n)(*[inputs[i].data_ptr() for i in wave]),
                                       (N.vp * n)(*[self.proj[i].A.p_bf16.data_ptr() for i in wave]),
                                       (N.vp * n)(*[views[i][1].data_ptr() for i in wave]), s), ctx.handle)
            for i in wave:
                p = self.proj[i]
                Y, H, _, _, rsq = views[i]
                N.check(L.mlora_base_fwd(ctx.handle, plan.handle, p.d, p.k, inputs[i].data_ptr(), p.W0.data_ptr(),
                                         H.data_ptr(), p.B.p_bf16.data_ptr(), Y.data_ptr(), rsq.data_ptr(), s),
                        ctx.handle)
                done.add(p.name)
        # ---- per-job loss from the row sums the forward GEMM epilogues produced (no re-read of Y)
        n = len(self.proj)
        ptrs = (N.vp * n)(*[v[4].data_ptr() for v in views])
        N.check(L.mlora_loss_from_rowsq(ctx.handle, plan.handle, ptrs, self._rowsq_d, n, self.loss.data_ptr(), s),
                ctx.handle)
        # ---- a job whose loss is not finite contributes a zero gradient: its rows of
        # every tensor the backward reads — dY (= Y here), the saved H and every
        # projection input X — are zeroed.  No inf/NaN then meets the structural
        # zeros of other jobs' columns (dB = dY^T H, dA = G^T X), and the job's own
        # gradient is exactly 0, so its adapter stays finite and cannot leak into
        # its neighbours' forward tiles either.  (The caller's x rows of that job
        # are zeroed in place.)
        guard = {}
        for i, v in enumerate(views):
            guard[v[0].data_ptr()] = self.proj[i].d
            guard[v[1].data_ptr()] = self.plan.rank_padded
            guard[inputs[i].data_ptr()] = inputs[i].shape[1]
        ng = len(guard)
        N.check(L.mlora_zero_nonfinite_rows(ctx.handle, plan.handle, self.loss.data_ptr(),
                                            (N.vp * ng)(*guard.keys()), (N.i32 * ng)(*guard.values()), ng, s),
                ctx.handle)
        # ---- backward: dL/dY_p = Y_p for every projection
        N.check(L.mlora_down_group(ctx.handle, plan.handle, n, 1, (N.i32 * n)(*[p.d for p in self.proj]),
                                   (N.vp * n)(*[v[0].data_ptr() for v in views]),
                                   (N.vp * n)(*[p.B.p_bf16.data_ptr() for p in self.proj]),
                                   (N.vp * n)(*[v[2].data_ptr() for v in views]), s), ctx.handle)
        for i in reversed(range(n)):
            p = self.proj[i]
            Y, _, G, dX, _ = views[i]
            N.check(L.mlora_base_dx(ctx.handle, plan.handle, p.d, p.k, Y.data_ptr(), p.W0.data_ptr(), G.data_ptr(),
                                    p.A.p_bf16.data_ptr(), dX.data_ptr(), s), ctx.handle)
        N.check(L.mlora_grad_group(ctx.handle, plan.handle, n, (N.i32 * n)(*[p.d for p in self.proj]),
                                   (N.i32 * n)(*[p.k for p in self.proj]),
                                   (N.vp * n)(*[inputs[i].data_ptr() for i in range(n)]),
                                   (N.vp * n)(*[v[0].data_ptr() for v in views]),
                                   (N.vp * n)(*[v[1].data_ptr() for v in views]),
                                   (N.vp * n)(*[v[2].data_ptr() for v in views]),
                                   (N.vp * n)(*[p.dA.data_ptr() for p in self.proj]),
                                   (N.vp * n)(*[p.dB.data_ptr() for p in self.proj]), s), ctx.handle)
        return self.loss

    def optimizer_step(self, active=None, stream=None) -> None:
        """AdamW on every adapter; jobs not in `active` (bool per job) keep p, m, v
        untouched this step (their rows were absent from the fused batch)."""
        active = [True] * self.J if active is None else list(active)
        self.step_count = [s + (1 if a else 0) for s, a in zip(self.step_count, active)]
        steps = [s if a else 0 for s, a in zip(self.step_count, active)]
        states, grads = [], []
        for p in self.proj:
            states += [p.A, p.B]
            grads += [p.dA, p.dB]
        # loss_gate: a job whose loss this step is not finite keeps p, m, v and its
        # step count untouched on the device (its gradient was zeroed by the guard,
        # but stale momentum must not move its adapter either)
        F.adam_step(self.ctx, self.plan, states, grads, self.lrs, steps, stream=stream, loss_gate=self.loss)

    def step(self, x: torch.Tensor, active=None, stream=None) -> torch.Tensor:
        """One fused training iteration over the installed layout; returns the
        per-job loss (device fp32 [J]).  Note: when a job's loss is not finite
        the non-finite guard zeroes that job's rows of every tensor the backward
        reads, including the caller's `x` (in place) — the rows are already
        poisoned for this step and a zero row is what keeps the other jobs'
        fused reductions exact."""
        loss = self.forward_backward(x, stream)
        self.optimizer_step(active, stream)
        return loss
