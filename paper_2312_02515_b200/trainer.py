"""Public training API over host batches: the call a user makes.

`PipelinedTrainer.run(batches)` takes fused batches that live in pinned host
memory, uploads each one (H2D on a dedicated copy stream, double-buffered so
batch i+1 streams in while step i computes), runs the fused multi-LoRA step
(FusedLoraLayer.step: every projection's fwd + loss + bwd + per-job AdamW) and
copies each step's per-job losses back to pinned host memory (D2H on the
compute stream).  Every byte of every step's input and result crosses PCIe
inside the loop; only the overlap is new.
"""
from __future__ import annotations

import torch

from .layer import FusedLoraLayer


class PipelinedTrainer:
    def __init__(self, layer: FusedLoraLayer, rows: int, k_in: int):
        dev = layer.ctx.device
        self.layer = layer
        self.buf = [torch.empty(rows, k_in, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.ready = [torch.cuda.Event() for _ in range(2)]      # upload of buf[i] finished
        self.free = [torch.cuda.Event() for _ in range(2)]       # step reading buf[i] finished
        for e in self.free:
            e.record(torch.cuda.current_stream(dev))

    def _upload(self, slot: int, host: torch.Tensor) -> None:
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(self.free[slot])
            self.buf[slot].copy_(host, non_blocking=True)
            self.ready[slot].record(self.copy_stream)

    def run(self, host_batches, losses_host: torch.Tensor) -> torch.Tensor:
        """host_batches: sequence of pinned bf16 [rows, k_in] tensors.
        losses_host: pinned fp32 [len(host_batches), J] receiving every step's losses."""
        n = len(host_batches)
        compute = torch.cuda.current_stream(self.layer.ctx.device)
        if n == 0:
            return losses_host
        self.copy_stream.wait_stream(compute)  # uploads start inside the caller's timed region
        self._upload(0, host_batches[0])
        for i in range(n):
            slot = i & 1
            if i + 1 < n:
                self._upload(slot ^ 1, host_batches[i + 1])
            compute.wait_event(self.ready[slot])
            loss = self.layer.step(self.buf[slot])
            self.free[slot].record(compute)
            losses_host[i].copy_(loss, non_blocking=True)
        return losses_host
