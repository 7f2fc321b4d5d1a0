"""§8f row 3 — measured memory samples for the reference's Eq. 6 memory model.

For a warm-up probe grid of (batch size B_t, sequence length L_n) — the
reference's warmup_plan cross product (memory_model.cpp:241-259) — run one
fused LoRA training step of a LLaMA-7B layer (7 projections, one job, r=16) on
the B200 and record the peak device memory.  Output: the reference's memory
sample CSV (`batch_size,seq_len,mem_gb`, proj/docs/schema.md:73-81), i.e. the
input of `fusim fit-mem` / fit_memory_model, plus a least-squares fit of
M = b0 + b1·B_t·L_n + b2·B_t·L_n² (Eq. 6) for reference.
"""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2312_02515_b200 import fused as F
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer


def main(out_csv):
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    g = torch.Generator(device="cpu").manual_seed(1)
    W0 = {n: ((torch.rand(d, k, generator=g) * 2 - 1) / k ** 0.5).to(torch.bfloat16).to(dev) for n, d, k, _ in LLAMA7B}
    torch.cuda.synchronize()
    rows_out = []
    for bs in (1, 2, 4, 8):
        for L in (128, 256, 512, 1024):
            torch.cuda.empty_cache()
            torch.cuda.reset_peak_memory_stats(dev)
            base = torch.cuda.memory_allocated(dev)
            layer = FusedLoraLayer(ctx, LLAMA7B, [16], [2.0], [1e-4], rows=bs * L, seed=2, W0=W0)
            layer.set_layout([0, bs * L])
            x = (torch.rand(bs * L, 4096, device=dev) * 2 - 1).to(torch.bfloat16)
            layer.step(x)
            torch.cuda.synchronize()
            peak = torch.cuda.max_memory_allocated(dev) - base
            # the frozen base weights are shared by every job; the per-job footprint
            # the scheduler budgets is adapters + optimizer state + activations
            rows_out.append((bs, L, peak / 2 ** 30))
            del layer, x
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["batch_size", "seq_len", "mem_gb"])
        for bs, L, m in rows_out:
            w.writerow([bs, L, f"{m:.6f}"])
    t = np.array([bs * L for bs, L, _ in rows_out], np.float64)
    Ln = np.array([L for _, L, _ in rows_out], np.float64)
    M = np.array([m for _, _, m in rows_out])
    A = np.stack([np.ones_like(t), t, t * Ln], 1)  # Eq. 6: (1, Bt*Ln, Bt*Ln^2)
    beta, *_ = np.linalg.lstsq(A, M, rcond=None)
    rmse = float(np.sqrt(np.mean((A @ beta - M) ** 2)))
    print(f"samples={len(rows_out)} beta0={beta[0]:.6g} GB beta1={beta[1]:.6g} GB/token beta2={beta[2]:.6g} "
          f"rmse={rmse:.3g} GB  (per LLaMA-7B layer, one r16 job, W0 excluded)")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/memory_samples.csv")
