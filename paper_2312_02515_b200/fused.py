"""Device executor for the BatchFusion multi-LoRA linear layer (host side, Python).

Thin, allocation-aware wrappers over the C ABI (include/mlora.h).  Torch is
used only for device memory and streams; every FLOP runs in the sm_100a
kernels of libmlora.so.

    ctx  = Context(device)                       # mlora_ctx: TMA-descriptor cache, workspace
    plan = Plan(ctx, seg_offsets, ranks, scales) # segment layout of one fused batch
    Y, H = linear_fwd(ctx, plan, X, W0, A_cat, B_cat)
    dX, dA_cat, dB_cat = linear_bwd(ctx, plan, dY, X, H, W0, A_cat, B_cat)

Reference correspondence: ``linear_fwd`` replaces fusim::fused_forward
(/root/reference/proj/src/lora.cpp:160-182) on packed rows; the backward has
no reference function and is pinned by composing the reference primitives
(SURVEY.md §8c).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _native as N
from . import errors


def _stream_handle(stream: torch.cuda.Stream | None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _require_cuda(t: torch.Tensor, name: str, dtype: torch.dtype, shape: tuple | None = None) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise errors.UsageError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise errors.UsageError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise errors.UsageError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise errors.ShapeError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


class Context:
    """mlora_ctx for one device (one per GPU / thread)."""

    def __init__(self, device: int | torch.device = 0):
        dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.device = dev
        L = N.lib()
        h = N.vp()
        N.check(L.mlora_ctx_create(dev.index or 0, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    @property
    def num_sms(self) -> int:
        return N.lib().mlora_ctx_num_sms(self._h)

    @property
    def launches(self) -> int:
        return N.lib().mlora_ctx_launch_count(self._h)

    KERNEL_KINDS = {0: "base_fwd", 1: "base_dx", 2: "down", 3: "grad", 4: "aux", 5: "adam"}

    def set_profiling(self, enable: bool) -> None:
        N.check(N.lib().mlora_ctx_set_profiling(self._h, 1 if enable else 0), self._h)

    def profile(self, reset: bool = False) -> dict:
        """{kind: (launches, total device ms)} of the live per-kernel timing."""
        out = {}
        names = list(self.KERNEL_KINDS.items())
        for i, (kind, name) in enumerate(names):
            cnt, ms = N.i64(), C.c_double()
            last = i == len(names) - 1
            N.check(N.lib().mlora_ctx_profile_read(self._h, kind, C.byref(cnt), C.byref(ms),
                                                   1 if (reset and last) else 0), self._h)
            out[name] = (cnt.value, ms.value)
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().mlora_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """Segment layout of one fused batch (mlora_plan).

    seg_offsets: J+1 non-decreasing row offsets (job j owns rows seg[j]:seg[j+1]),
    ranks: J adapter ranks, scales: J LoRA scales (alpha / r); s_j = 1 is the
    reference's (unscaled) arithmetic.
    """

    def __init__(self, ctx: Context, seg_offsets, ranks, scales=None, stream=None):
        J = len(ranks)
        if len(seg_offsets) != J + 1:
            raise errors.UsageError("seg_offsets must have len(ranks)+1 entries")
        self.ctx = ctx
        self.num_jobs = J
        self.seg = [int(x) for x in seg_offsets]
        self.ranks = [int(r) for r in ranks]
        self.scales = [1.0] * J if scales is None else [float(s) for s in scales]
        seg_c = (N.i64 * (J + 1))(*self.seg)
        rank_c = (N.i32 * J)(*self.ranks)
        scale_c = (N.f32 * J)(*self.scales)
        h = N.vp()
        with torch.cuda.device(ctx.device):
            N.check(N.lib().mlora_plan_create(ctx.handle, J, seg_c, rank_c, scale_c,
                                              _stream_handle(stream), C.byref(h)), ctx.handle)
        self._h = h
        self.rows = int(N.lib().mlora_plan_rows(h))
        self.rank_padded = int(N.lib().mlora_plan_rank_padded(h))
        roff = (N.i32 * (J + 1))()
        N.check(N.lib().mlora_plan_rank_offsets(h, roff))
        self.rank_offsets = list(roff)

    @property
    def handle(self):
        return self._h

    def update(self, seg_offsets, stream=None) -> None:
        """Next fused batch's segment layout (same jobs/ranks/scales): stream-ordered,
        no host sync, no allocation in steady state (mlora_plan_update)."""
        if len(seg_offsets) != self.num_jobs + 1:
            raise errors.UsageError("seg_offsets must have num_jobs+1 entries")
        seg = [int(x) for x in seg_offsets]
        with torch.cuda.device(self.ctx.device):
            N.check(N.lib().mlora_plan_update(self._h, (N.i64 * len(seg))(*seg), _stream_handle(stream)),
                    self.ctx.handle)
        self.seg = seg
        self.rows = int(N.lib().mlora_plan_rows(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().mlora_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def linear_fwd(ctx: Context, plan: Plan, X: torch.Tensor, W0: torch.Tensor, A_cat: torch.Tensor,
               B_cat: torch.Tensor, Y: torch.Tensor | None = None, H: torch.Tensor | None = None,
               row_sq: torch.Tensor | None = None, stream=None):
    """Y = X W0^T + s_j (X_j A_j^T) B_j^T on packed rows; returns (Y, H).
    row_sq (optional, fp32 [mlora_rowsq_blocks(d), rows]) receives the fused
    per-row sums of squares of Y from the GEMM epilogue."""
    d, k = W0.shape
    M, R = plan.rows, plan.rank_padded
    _require_cuda(X, "X", torch.bfloat16, (M, k))
    _require_cuda(W0, "W0", torch.bfloat16)
    _require_cuda(A_cat, "A_cat", torch.bfloat16, (R, k))
    _require_cuda(B_cat, "B_cat", torch.bfloat16, (d, R))
    if Y is None:
        Y = torch.empty((M, d), dtype=torch.bfloat16, device=X.device)
    if H is None:
        H = torch.empty((M, R), dtype=torch.bfloat16, device=X.device)
    _require_cuda(Y, "Y", torch.bfloat16, (M, d))
    _require_cuda(H, "H", torch.bfloat16, (M, R))
    if row_sq is not None:
        _require_cuda(row_sq, "row_sq", torch.float32, (N.lib().mlora_rowsq_blocks(d), M))
    N.check(N.lib().mlora_linear_fwd_ex(ctx.handle, plan.handle, d, k, N.ptr(X), N.ptr(W0), N.ptr(A_cat),
                                        N.ptr(B_cat), N.ptr(Y), N.ptr(H), N.ptr(row_sq), _stream_handle(stream)),
            ctx.handle)
    return Y, H


def linear_bwd(ctx: Context, plan: Plan, dY: torch.Tensor, X: torch.Tensor, H: torch.Tensor,
               W0: torch.Tensor, A_cat: torch.Tensor, B_cat: torch.Tensor, need_dX: bool = True,
               dX: torch.Tensor | None = None, dA_cat: torch.Tensor | None = None,
               dB_cat: torch.Tensor | None = None, G: torch.Tensor | None = None, stream=None):
    """Returns (dX | None, dA_cat fp32 [R_pad, k], dB_cat fp32 [d, R_pad])."""
    d, k = W0.shape
    M, R = plan.rows, plan.rank_padded
    _require_cuda(dY, "dY", torch.bfloat16, (M, d))
    _require_cuda(X, "X", torch.bfloat16, (M, k))
    _require_cuda(H, "H", torch.bfloat16, (M, R))
    dev = X.device
    if G is None:
        G = torch.empty((M, R), dtype=torch.bfloat16, device=dev)
    if need_dX and dX is None:
        dX = torch.empty((M, k), dtype=torch.bfloat16, device=dev)
    if dA_cat is None:
        dA_cat = torch.empty((R, k), dtype=torch.float32, device=dev)
    if dB_cat is None:
        dB_cat = torch.empty((d, R), dtype=torch.float32, device=dev)
    N.check(N.lib().mlora_linear_bwd(ctx.handle, plan.handle, d, k, N.ptr(dY), N.ptr(X), N.ptr(H), N.ptr(W0),
                                     N.ptr(A_cat), N.ptr(B_cat), N.ptr(G), N.ptr(dX if need_dX else None),
                                     N.ptr(dA_cat), N.ptr(dB_cat), _stream_handle(stream)), ctx.handle)
    return (dX if need_dX else None), dA_cat, dB_cat


def pack_adapters(ctx: Context, plan: Plan, d: int, k: int, As, Bs, stream=None, out=None):
    """Per-job fp32 device adapters (A_j r_j x k, B_j d x r_j) -> cat layout.
    Returns (A_cat_f32, B_cat_f32, A_cat_bf16, B_cat_bf16), written into `out`
    (the same 4-tuple of tensors) when given."""
    J = plan.num_jobs
    if len(As) != J or len(Bs) != J:
        raise errors.RoutingError("need one adapter per job")
    R = plan.rank_padded
    dev = ctx.device
    if out is not None:
        A32, B32, A16, B16 = out
        for t, name, dt, shp in ((A32, "A_cat_f32", torch.float32, (R, k)), (B32, "B_cat_f32", torch.float32, (d, R)),
                                 (A16, "A_cat_bf16", torch.bfloat16, (R, k)),
                                 (B16, "B_cat_bf16", torch.bfloat16, (d, R))):
            _require_cuda(t, name, dt, shp)
    else:
        A32 = torch.empty((R, k), dtype=torch.float32, device=dev)
        B32 = torch.empty((d, R), dtype=torch.float32, device=dev)
        A16 = torch.empty((R, k), dtype=torch.bfloat16, device=dev)
        B16 = torch.empty((d, R), dtype=torch.bfloat16, device=dev)
    for j in range(J):
        _require_cuda(As[j], f"A[{j}]", torch.float32, (plan.ranks[j], k))
        _require_cuda(Bs[j], f"B[{j}]", torch.float32, (d, plan.ranks[j]))
    ap = (N.vp * J)(*[a.data_ptr() for a in As])
    bp = (N.vp * J)(*[b.data_ptr() for b in Bs])
    N.check(N.lib().mlora_pack_adapters(ctx.handle, plan.handle, d, k, ap, bp, N.ptr(A32), N.ptr(B32),
                                        N.ptr(A16), N.ptr(B16), _stream_handle(stream)), ctx.handle)
    return A32, B32, A16, B16


@dataclass
class AdamState:
    p: torch.Tensor        # fp32 master (cat layout)
    m: torch.Tensor
    v: torch.Tensor
    p_bf16: torch.Tensor   # operand copy used by the GEMMs
    layout: int            # 0: rows by job (A_cat), 1: cols by job (B_cat)

    @staticmethod
    def of(p32: torch.Tensor, p16: torch.Tensor, layout: int) -> "AdamState":
        return AdamState(p32, torch.zeros_like(p32), torch.zeros_like(p32), p16, layout)


def adam_step(ctx: Context, plan: Plan, states, grads, lr, step, beta1=0.9, beta2=0.999, eps=1e-8,
              weight_decay=0.0, stream=None, loss_gate: torch.Tensor | None = None) -> None:
    """One fused AdamW launch over every adapter tensor (per-job lr and step).
    loss_gate (device fp32 [J]): jobs whose loss is not finite are skipped."""
    J = plan.num_jobs
    groups = (N.AdamGroupC * len(states))()
    for i, (st, g) in enumerate(zip(states, grads)):
        groups[i] = N.AdamGroupC(st.p.data_ptr(), g.data_ptr(), st.m.data_ptr(), st.v.data_ptr(),
                                 st.p_bf16.data_ptr() if st.p_bf16 is not None else None,
                                 st.p.shape[0], st.p.shape[1], st.layout, 0)
    lr_c = (N.f32 * J)(*[float(x) for x in lr])
    step_c = (N.i32 * J)(*[int(x) for x in step])
    N.check(N.lib().mlora_adam_step_ex(ctx.handle, plan.handle, groups, len(states), lr_c, step_c, beta1, beta2,
                                       eps, weight_decay, N.ptr(loss_gate), _stream_handle(stream)), ctx.handle)


def fuse_rows(ctx: Context, seqs, padded: bool = False, out: torch.Tensor | None = None,
              mask: torch.Tensor | None = None, stream=None):
    """Device fuse (mlora_fuse_rows; fusim::fuse, lora.cpp:114-158): copy each
    sequence's bf16 rows (device tensors [len_i, dim], FusedBatch order) into one
    fused matrix, packed or in the reference's padded layout (slot = max len,
    zero tail).  Returns (X [rows, dim], mask uint8 [rows], row offsets [S+1])."""
    S = len(seqs)
    if S == 0:
        raise errors.UsageError("fuse: no sequences")
    dim = seqs[0].shape[1]
    lens = [int(t.shape[0]) for t in seqs]
    rows = S * max(lens) if padded else sum(lens)
    dev = ctx.device
    for i, t in enumerate(seqs):
        if t.dtype != torch.bfloat16 or not t.is_cuda or t.dim() != 2 or t.shape[1] != dim or t.stride(1) != 1:
            raise errors.ShapeError(f"sequence {i}: needs a bf16 CUDA [len, {dim}] tensor with unit column stride")
    if out is None:
        out = torch.empty(rows, dim, dtype=torch.bfloat16, device=dev)
    if mask is None:
        mask = torch.empty(rows, dtype=torch.uint8, device=dev)
    offs = (N.i64 * (S + 1))()
    N.check(N.lib().mlora_fuse_rows(ctx.handle, S, (N.vp * S)(*[t.data_ptr() for t in seqs]),
                                    (N.i64 * S)(*[t.stride(0) for t in seqs]), (N.i32 * S)(*lens), dim,
                                    1 if padded else 0, out.data_ptr(), mask.data_ptr(), offs,
                                    _stream_handle(stream)), ctx.handle)
    return out, mask, list(offs)


_MASK64 = (1 << 64) - 1


def mix_seed(*parts: int) -> int:
    """64-bit FNV-1a over the parts: the per-tensor seed of the synthetic
    weights / data (the C++ façade's fusim::b200::mix_seed is the same), so a
    Python and a C++ host initialise bit-identical tensors."""
    h = 0xCBF29CE484222325
    for v in parts:
        h = ((h ^ (int(v) & _MASK64)) * 0x100000001B3) & _MASK64
    return h


def fill_uniform(t: torch.Tensor, seed: int, lo: float = -1.0, hi: float = 1.0, stream=None) -> torch.Tensor:
    """In place: t[i] = lo + (hi - lo) * u(seed, i) on the device (mlora_fill_uniform:
    counter-based, independent of launch shape and host language).  fp32 or bf16."""
    if not t.is_cuda or not t.is_contiguous() or t.dtype not in (torch.float32, torch.bfloat16):
        raise errors.UsageError("fill_uniform needs a contiguous fp32 / bf16 CUDA tensor")
    with torch.cuda.device(t.device):
        N.check(N.lib().mlora_fill_uniform(t.data_ptr(), t.numel(), 0 if t.dtype == torch.float32 else 1,
                                           int(seed) & _MASK64, float(lo), float(hi), _stream_handle(stream)))
    return t
