"""Python wrappers of the small model kernels (K4 masked CE, K5 RMSNorm / RoPE)
in libmlora.so (include/mlora.h).  Torch provides memory and streams only."""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from . import errors


def _s(stream):
    return (stream or torch.cuda.current_stream()).cuda_stream


def masked_ce(logits: torch.Tensor, labels: torch.Tensor, seg_offsets, mask: torch.Tensor | None = None,
              need_grad: bool = True, stream=None):
    """Per-job mean cross-entropy over the real rows of a fused batch.
    logits bf16 [rows, V]; labels int32 [rows]; mask uint8 [rows] (None: all real).
    Returns (loss fp32 [J], dlogits bf16 [rows, V] | None)."""
    rows, V = logits.shape
    if logits.dtype != torch.bfloat16 or labels.dtype != torch.int32:
        raise errors.UsageError("logits must be bf16 and labels int32")
    dev = logits.device
    J = len(seg_offsets) - 1
    seg = torch.tensor(list(seg_offsets), dtype=torch.int32, device=dev)
    row_loss = torch.empty(rows, dtype=torch.float32, device=dev)
    loss = torch.empty(J, dtype=torch.float32, device=dev)
    inv = torch.empty(J, dtype=torch.float32, device=dev)
    dl = torch.empty_like(logits) if need_grad else None
    N.check(N.lib().mlora_masked_ce(J, seg.data_ptr(), rows, V, logits.data_ptr(), labels.data_ptr(),
                                    None if mask is None else mask.data_ptr(), row_loss.data_ptr(), loss.data_ptr(),
                                    inv.data_ptr(), None if dl is None else dl.data_ptr(), _s(stream)))
    return loss, dl


def rmsnorm_fwd(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-6, stream=None):
    rows, h = x.shape
    y = torch.empty_like(x)
    rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    N.check(N.lib().mlora_rmsnorm_fwd(rows, h, x.data_ptr(), w.data_ptr(), eps, y.data_ptr(), rstd.data_ptr(),
                                      _s(stream)))
    return y, rstd


def rmsnorm_bwd(dy: torch.Tensor, x: torch.Tensor, w: torch.Tensor, rstd: torch.Tensor, rows_per_block: int = 64,
                stream=None):
    rows, h = x.shape
    dx = torch.empty_like(x)
    dw = torch.empty(h, dtype=torch.float32, device=x.device)
    nblk = -(-rows // rows_per_block)
    ws = torch.empty(nblk * h, dtype=torch.float32, device=x.device)
    N.check(N.lib().mlora_rmsnorm_bwd(rows, h, dy.data_ptr(), x.data_ptr(), w.data_ptr(), rstd.data_ptr(),
                                      dx.data_ptr(), dw.data_ptr(), ws.data_ptr(), rows_per_block, _s(stream)))
    return dx, dw


def rope(x: torch.Tensor, pos: torch.Tensor, base: float = 10000.0, inverse: bool = False, stream=None):
    rows, heads, hd = x.shape
    y = torch.empty_like(x)
    N.check(N.lib().mlora_rope(rows, heads, hd, x.data_ptr(), y.data_ptr(), pos.data_ptr(), base,
                               1 if inverse else 0, _s(stream)))
    return y


# ---------------------------------------------------------------- decoder-layer kernels (mlora_decoder.cu)
def _bf16(t: torch.Tensor, name: str) -> None:
    if t.dtype != torch.bfloat16 or not t.is_cuda:
        raise errors.UsageError(f"{name} must be a bf16 CUDA tensor")
    if t.stride(-1) != 1:
        raise errors.UsageError(f"{name} must have unit column stride")


def embed(tokens: torch.Tensor, E: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """x[t] = E[tokens[t]] (frozen bf16 table [V, h])."""
    V, h = E.shape
    out = torch.empty(tokens.shape[0], h, dtype=torch.bfloat16, device=E.device) if out is None else out
    N.check(N.lib().mlora_embed(tokens.shape[0], h, V, tokens.data_ptr(), E.data_ptr(), out.data_ptr(), _s(stream)))
    return out


def add_rmsnorm(x: torch.Tensor, delta: torch.Tensor | None, w: torch.Tensor, eps: float = 1e-6,
                x_out: torch.Tensor | None = None, y: torch.Tensor | None = None, rstd: torch.Tensor | None = None,
                stream=None):
    """(x_out = bf16(x + delta) | None, y = RMSNorm(x_out or x) * w, rstd)."""
    rows, h = x.shape
    if delta is not None and x_out is None:
        x_out = torch.empty_like(x)
    y = torch.empty_like(x) if y is None else y
    rstd = torch.empty(rows, dtype=torch.float32, device=x.device) if rstd is None else rstd
    N.check(N.lib().mlora_add_rmsnorm(rows, h, x.data_ptr(), None if delta is None else delta.data_ptr(),
                                      w.data_ptr(), eps, None if x_out is None else x_out.data_ptr(), y.data_ptr(),
                                      rstd.data_ptr(), _s(stream)))
    return x_out, y, rstd


def rmsnorm_bwd_sum(dys, dres: torch.Tensor | None, x: torch.Tensor, w: torch.Tensor, rstd: torch.Tensor,
                    out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """dx = dres + RMSNorm'(x)^T (w * sum(dys)) for a frozen norm weight."""
    rows, h = x.shape
    out = torch.empty_like(x) if out is None else out
    n = len(dys)
    N.check(N.lib().mlora_rmsnorm_bwd_sum(rows, h, n, (N.vp * n)(*[d.data_ptr() for d in dys]),
                                          None if dres is None else dres.data_ptr(), x.data_ptr(), w.data_ptr(),
                                          rstd.data_ptr(), out.data_ptr(), _s(stream)))
    return out


def swiglu_fwd(gate: torch.Tensor, up: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """silu(gate) * up; gate / up may be column slices (row stride = stride(0))."""
    rows, f = gate.shape
    out = torch.empty(rows, f, dtype=torch.bfloat16, device=gate.device) if out is None else out
    N.check(N.lib().mlora_swiglu_fwd(rows, f, gate.data_ptr(), gate.stride(0), up.data_ptr(), up.stride(0),
                                     out.data_ptr(), _s(stream)))
    return out


def swiglu_bwd(gate: torch.Tensor, up: torch.Tensor, dout: torch.Tensor, dgate: torch.Tensor, dup: torch.Tensor,
               stream=None) -> None:
    rows, f = gate.shape
    N.check(N.lib().mlora_swiglu_bwd(rows, f, gate.data_ptr(), gate.stride(0), up.data_ptr(), up.stride(0),
                                     dout.data_ptr(), dgate.data_ptr(), dgate.stride(0), dup.data_ptr(),
                                     dup.stride(0), _s(stream)))


class AttnLayout:
    """Sequence layout of a fused batch for mlora_attn_*: sequence s owns rows
    seq_offsets[s]:seq_offsets[s+1], its first seq_lens[s] rows are real."""

    def __init__(self, seq_offsets, seq_lens=None, device=None):
        off = [int(x) for x in seq_offsets]
        if len(off) < 2 or off[0] != 0 or any(b < a for a, b in zip(off, off[1:])):
            raise errors.UsageError("seq_offsets must start at 0 and be non-decreasing")
        lens = [b - a for a, b in zip(off, off[1:])] if seq_lens is None else [int(x) for x in seq_lens]
        if len(lens) != len(off) - 1 or any(not 0 <= n <= b - a for n, a, b in zip(lens, off, off[1:])):
            raise errors.UsageError("seq_lens must fit their slots")
        self.offsets, self.lens = off, lens
        self.rows = off[-1]
        self.max_len = max(1, max(b - a for a, b in zip(off, off[1:])))
        # pinned staging + async copies: stream-ordered, the host never waits for the device
        self.d_off = torch.tensor(off, dtype=torch.int32).pin_memory().to(device, non_blocking=True)
        self.d_len = torch.tensor(lens, dtype=torch.int32).pin_memory().to(device, non_blocking=True)

    def desc(self, heads: int, kv_heads: int, head_dim: int, rope_base: float = 10000.0,
             scale: float | None = None, prerotated: bool = False) -> "N.AttnDescC":
        return N.AttnDescC(self.d_off.data_ptr(), self.d_len.data_ptr(), self.rows, len(self.lens), self.max_len,
                           heads, kv_heads, head_dim, float(rope_base),
                           float(head_dim ** -0.5 if scale is None else scale), 1 if prerotated else 0)


def attn_rope(layout: AttnLayout, x: torch.Tensor, n_heads: int, head_dim: int, rope_base: float = 10000.0,
              out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """RoPE of n_heads heads of every row (position within its sequence); x may be a column slice."""
    out = torch.empty(x.shape[0], n_heads * head_dim, dtype=torch.bfloat16, device=x.device) if out is None else out
    d = layout.desc(n_heads, n_heads, head_dim, rope_base)
    N.check(N.lib().mlora_attn_rope(C.byref(d), x.data_ptr(), x.stride(0), n_heads, out.data_ptr(), out.stride(0),
                                    _s(stream)))
    return out


def attn_fwd(layout: AttnLayout, q, k, v, heads: int, kv_heads: int, head_dim: int, rope_base: float = 10000.0,
             out: torch.Tensor | None = None, lse: torch.Tensor | None = None, prerotated: bool = False,
             stream=None):
    """Causal attention (RoPE fused unless q/k come prerotated by attn_rope) over
    the fused rows; q/k/v may be column slices."""
    rows = layout.rows
    out = torch.empty(rows, heads * head_dim, dtype=torch.bfloat16, device=q.device) if out is None else out
    lse = torch.empty(heads, rows, dtype=torch.float32, device=q.device) if lse is None else lse
    d = layout.desc(heads, kv_heads, head_dim, rope_base, prerotated=prerotated)
    N.check(N.lib().mlora_attn_fwd(C.byref(d), q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0), v.data_ptr(),
                                   v.stride(0), out.data_ptr(), out.stride(0), lse.data_ptr(), _s(stream)))
    return out, lse


def attn_bwd(layout: AttnLayout, q, k, v, o, dout, lse, dq, dk, dv, heads: int, kv_heads: int, head_dim: int,
             rope_base: float = 10000.0, dsum: torch.Tensor | None = None, prerotated: bool = False,
             stream=None) -> None:
    """dq / dk are with respect to the unrotated q / k in both modes."""
    rows = layout.rows
    dsum = torch.empty(heads, rows, dtype=torch.float32, device=q.device) if dsum is None else dsum
    d = layout.desc(heads, kv_heads, head_dim, rope_base, prerotated=prerotated)
    N.check(N.lib().mlora_attn_bwd(C.byref(d), q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0), v.data_ptr(),
                                   v.stride(0), o.data_ptr(), o.stride(0), dout.data_ptr(), dout.stride(0),
                                   lse.data_ptr(), dsum.data_ptr(), dq.data_ptr(), dq.stride(0), dk.data_ptr(),
                                   dk.stride(0), dv.data_ptr(), dv.stride(0), _s(stream)))
