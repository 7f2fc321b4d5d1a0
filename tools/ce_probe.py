"""Time the padding-masked cross-entropy (count + row pass + per-job mean) at C4 shape:
12 288 rows x V = 65 024 bf16 logits, 6 jobs, every row real.

    python tools/ce_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_02515_b200 import model_ops as M  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    rows, V = 12288, 65024
    logits = (torch.randn(rows, V, device=dev) * 3).to(torch.bfloat16)
    labels = torch.randint(0, V, (rows,), device=dev, dtype=torch.int32)
    mask = torch.ones(rows, dtype=torch.uint8, device=dev)
    seg = [0, 2048, 4096, 6144, 8192, 10240, 12288]
    for _ in range(2):
        M.masked_ce(logits, labels, seg, mask)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        M.masked_ce(logits, labels, seg, mask)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"masked_ce {ms:.3f} ms ({4 * rows * V / ms / 1e6:.0f} GB/s of 2V read + 2V written per row)")


if __name__ == "__main__":
    main()
