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

import ctypes as C
from dataclasses import dataclass

import torch

from . import _native as N
from . import errors as E
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


class _DeviceBlock:
    """One cudaMalloc'd block owned through the C ABI (mlora_malloc / mlora_free),
    exposed to torch by the CUDA array interface (no copy).  Outside torch's
    caching allocator, so the layer's footprint on the device is exactly its bytes."""

    def __init__(self, ctx, nbytes: int):
        self.ctx = ctx
        p = N.vp()
        N.check(N.lib().mlora_malloc(ctx.handle, max(int(nbytes), 1), C.byref(p)), ctx.handle)
        self.ptr, self.nbytes = p.value, int(nbytes)
        self.__cuda_array_interface__ = {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False),
                                         "version": 3, "strides": None}

    def free(self) -> None:
        if self.ptr:
            N.lib().mlora_free(self.ctx.handle, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class _Arena:
    """Tensors carved from one device allocation (256-byte aligned views)."""
    ALIGN = 256

    def __init__(self, ctx, nbytes: int):
        self.block = _DeviceBlock(ctx, nbytes)
        self.buf = torch.as_tensor(self.block, device=ctx.device)
        assert self.buf.data_ptr() == self.block.ptr and self.buf.numel() == nbytes
        self.off = 0

    @staticmethod
    def size(shape, itemsize: int) -> int:
        n = itemsize
        for s in shape:
            n *= s
        return (n + _Arena.ALIGN - 1) // _Arena.ALIGN * _Arena.ALIGN

    def take(self, shape, dtype, zero: bool = False) -> torch.Tensor:
        itemsize = torch.empty((), dtype=dtype).element_size()
        n = self.size(shape, itemsize)
        if self.off + n > self.buf.numel():
            raise MemoryError("layer arena exhausted (size computation out of date)")
        count = 1
        for s in shape:
            count *= s
        t = self.buf[self.off:self.off + count * itemsize].view(dtype).view(*shape)
        self.off += n
        if zero:
            t.zero_()
        return t


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
    """All adapters of J jobs on one layer's projections, cat layout, on one GPU.

    The step itself is native: the tensors are described once to
    mlora_layer_create (include/mlora.h) and every iteration is ONE C-ABI call,
    mlora_layer_step (forward waves, loss, guard, backward, AdamW).  Synthetic
    weights come from the device's counter-based fill (fused.fill_uniform with
    fused.mix_seed per tensor), so the C++ façade's executor
    (fusim::b200::FusedIterationExecutor) builds the bit-identical layer."""

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
        names = [name for name, _, _, _ in shapes]
        # every per-layer tensor (adapters, moments, gradients, activations, the
        # loss) is carved from ONE device allocation: no allocator fragmentation,
        # and the layer's footprint is exactly its bytes (what the memory model's
        # cudaMemGetInfo probes measure, memory.py)
        arena = _Arena(ctx, self._arena_bytes(shapes, names, self.J, R, rows))
        self._arena = arena
        self.proj: list[Projection] = []
        for pi, (name, d, k, src) in enumerate(shapes):
            if W0 is not None and name in W0:
                w = W0[name]
            else:
                w = F.fill_uniform(torch.empty(d, k, dtype=torch.bfloat16, device=dev), F.mix_seed(seed, 0, pi),
                                   -k ** -0.5, k ** -0.5)
            As, Bs = [], []
            for j, r in enumerate(ranks):
                As.append(F.fill_uniform(torch.empty(r, k, device=dev), F.mix_seed(seed, 1, pi, j), -k ** -0.5,
                                         k ** -0.5))
                if lora_init == "zero_b":   # standard LoRA init: B = 0
                    Bs.append(torch.zeros(d, r, device=dev))
                else:
                    Bs.append(F.fill_uniform(torch.empty(d, r, device=dev), F.mix_seed(seed, 2, pi, j), -r ** -0.5,
                                             r ** -0.5))
            f32, b16 = torch.float32, torch.bfloat16
            A32, B32, A16, B16 = F.pack_adapters(ctx, self.plan, d, k, As, Bs,
                                                 out=(arena.take((R, k), f32), arena.take((d, R), f32),
                                                      arena.take((R, k), b16), arena.take((d, R), b16)))
            del As, Bs
            sA = F.AdamState(A32, arena.take((R, k), f32, zero=True), arena.take((R, k), f32, zero=True), A16, 0)
            sB = F.AdamState(B32, arena.take((d, R), f32, zero=True), arena.take((d, R), f32, zero=True), B16, 1)
            self.proj.append(Projection(
                name, d, k, src, w, sA, sB, arena.take((R, k), f32, zero=True), arena.take((d, R), f32, zero=True),
                arena.take((rows, d), b16), arena.take((rows, R), b16), arena.take((rows, R), b16),
                arena.take((rows, k), b16), arena.take((N.lib().mlora_rowsq_blocks(d), rows), f32)))
        self.loss = arena.take((self.J,), torch.float32, zero=True)
        # ---- the native layer: one descriptor per projection (pointers into the tensors above)
        self._scratch = {}
        desc = (N.LayerProjC * len(self.proj))()
        for i, p in enumerate(self.proj):
            if p.src == "x":
                src, col0 = -1, 0
            else:
                base = "h_to_4h" if p.src == "h_to_4h_half" else p.src
                src, col0 = names.index(base), 0
            scratch = None
            if src >= 0 and self.proj[src].d != p.k:  # column slice of a wider source (ChatGLM2 4h_to_h)
                scratch = self._scratch[p.name] = arena.take((rows, p.k), torch.bfloat16)
            desc[i] = N.LayerProjC(p.d, p.k, src, col0, p.W0.data_ptr(), p.A.p.data_ptr(), p.B.p.data_ptr(),
                                   p.A.m.data_ptr(), p.A.v.data_ptr(), p.B.m.data_ptr(), p.B.v.data_ptr(),
                                   p.A.p_bf16.data_ptr(), p.B.p_bf16.data_ptr(), p.dA.data_ptr(), p.dB.data_ptr(),
                                   p.Y.data_ptr(), p.H.data_ptr(), p.G.data_ptr(), p.dX.data_ptr(),
                                   p.row_sq.data_ptr(), None if scratch is None else scratch.data_ptr())
        h = N.vp()
        N.check(N.lib().mlora_layer_create(ctx.handle, self.plan.handle, len(self.proj), desc, rows, C.byref(h)),
                ctx.handle)
        self._layer = h
        self._hp = N.AdamHparamsC(0.9, 0.999, 1e-8, 0.0)

    @staticmethod
    def _arena_bytes(shapes, names, J: int, R: int, rows: int) -> int:
        total = _Arena.size((J,), 4)  # the per-job loss
        for name, d, k, src in shapes:
            total += 4 * _Arena.size((R, k), 4) + _Arena.size((R, k), 2)      # A_cat: p, m, v, grad; bf16 copy
            total += 4 * _Arena.size((d, R), 4) + _Arena.size((d, R), 2)      # B_cat: the same
            total += _Arena.size((rows, d), 2) + 2 * _Arena.size((rows, R), 2) + _Arena.size((rows, k), 2)
            total += _Arena.size((N.lib().mlora_rowsq_blocks(d), rows), 4)
            if src != "x":
                base = "h_to_4h" if src == "h_to_4h_half" else src
                if shapes[names.index(base)][1] != k:
                    total += _Arena.size((rows, k), 2)
        return total

    def close(self) -> None:
        if getattr(self, "_layer", None):
            N.lib().mlora_layer_destroy(self._layer)
            self._layer = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

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

    def input_of(self, p: Projection, x: torch.Tensor) -> torch.Tensor:
        """The tensor projection p read in the last step (x, or its source's Y / slice)."""
        rows = getattr(self, "cur_rows", self.rows)
        if p.src == "x":
            return x[:rows]
        if p.name in self._scratch:
            return self._scratch[p.name][:rows]
        return next(q for q in self.proj if q.name == p.src).Y[:rows]

    def _check_x(self, x: torch.Tensor) -> None:
        rows = getattr(self, "cur_rows", self.rows)
        k0 = next((p.k for p in self.proj if p.src == "x"), None)
        if not (x.is_cuda and x.dtype == torch.bfloat16 and x.is_contiguous() and x.dim() == 2
                and x.shape[0] >= rows and x.shape[1] == k0):
            raise E.ShapeError(f"x must be a contiguous bf16 CUDA tensor of >= {rows} x {k0}")

    def forward_backward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """Forward (dependency waves: shared-input and grouped down-projections,
        base GEMMs with fused row sums), per-job loss, non-finite guard, backward
        (G group, dX GEMMs, grouped dA / dB): mlora_layer_forward_backward."""
        self._check_x(x)
        N.check(N.lib().mlora_layer_forward_backward(self._layer, x.data_ptr(), self.loss.data_ptr(),
                                                     F._stream_handle(stream)), self.ctx.handle)
        return self.loss

    def _steps(self, active):
        active = [True] * self.J if active is None else list(active)
        self.step_count = [s + (1 if a else 0) for s, a in zip(self.step_count, active)]
        return [s if a else 0 for s, a in zip(self.step_count, active)]

    def optimizer_step(self, active=None, stream=None) -> None:
        """AdamW on every adapter; jobs not in `active` (bool per job) keep p, m, v
        untouched this step (their rows were absent from the fused batch).
        loss_gate: a job whose loss this step is not finite keeps p, m, v
        untouched on the device (its gradient was zeroed by the guard, but
        stale momentum must not move its adapter either)."""
        steps = self._steps(active)
        states, grads = [], []
        for p in self.proj:
            states += [p.A, p.B]
            grads += [p.dA, p.dB]
        F.adam_step(self.ctx, self.plan, states, grads, self.lrs, steps, stream=stream, loss_gate=self.loss)

    def step(self, x: torch.Tensor, active=None, stream=None) -> torch.Tensor:
        """One fused training iteration over the installed layout, ONE native call
        (mlora_layer_step); returns the per-job loss (device fp32 [J]).  Note: when
        a job's loss is not finite the non-finite guard zeroes that job's rows of
        every tensor the backward reads, including the caller's `x` (in place) —
        the rows are already poisoned for this step and a zero row is what keeps
        the other jobs' fused reductions exact."""
        self._check_x(x)
        steps = self._steps(active)
        lr_c = (N.f32 * self.J)(*[float(v) for v in self.lrs])
        st_c = (N.i32 * self.J)(*steps)
        N.check(N.lib().mlora_layer_step(self._layer, x.data_ptr(), lr_c, st_c, C.byref(self._hp),
                                         self.loss.data_ptr(), F._stream_handle(stream)), self.ctx.handle)
        return self.loss
