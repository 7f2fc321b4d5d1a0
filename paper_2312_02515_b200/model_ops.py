"""Python wrappers of the small model kernels (K4 masked CE, K5 RMSNorm / RoPE)
in libmlora.so (include/mlora.h).  Torch provides memory and streams only."""
from __future__ import annotations

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
