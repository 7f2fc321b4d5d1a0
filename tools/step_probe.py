"""Time and energy of the C2 layer step on one B200, for A/B runs of a build or
environment change (one process per variant):
  rested  — single steps after a 0.25 s rest (the power limiter relaxed): median ms;
  burst   — 20 back-to-back steps from a rested GPU (the bench's headline regime);
  sustained — 200 back-to-back steps: ms/step and mJ/step (NVML total-energy counter).

    python tools/step_probe.py [label]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_02515_b200 import fused as F
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer


def main(label="run"):
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    layer = FusedLoraLayer(ctx, LLAMA7B, [16] * 4, [2.0] * 4, [1e-4, 2e-4, 5e-5, 3e-4], rows=8192, seed=1)
    layer.set_layout([0, 2048, 4096, 6144, 8192])
    x = F.fill_uniform(torch.empty(8192, 4096, dtype=torch.bfloat16, device=dev), 5)
    for _ in range(5):
        layer.step(x)
    torch.cuda.synchronize()

    def region(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            layer.step(x)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / n

    rested = []
    for _ in range(12):
        time.sleep(0.25)
        rested.append(region(1))
    time.sleep(1.5)
    burst = region(20)
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    time.sleep(1.5)
    j0 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
    sus = region(200)
    j1 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
    print(json.dumps({"label": label, "rested_ms": round(sorted(rested)[6], 4), "burst_ms": round(burst, 4),
                      "sustained_ms": round(sus, 4), "sustained_mJ_per_step": round((j1 - j0) / 200, 1),
                      "sm_mhz_after": nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)}))


if __name__ == "__main__":
    main(*sys.argv[1:])
