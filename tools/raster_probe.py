"""Time and energy per C2 layer step for the base-GEMM raster (MLORA_RASTER,
read once per process): under the 1 kW cap, joules per step decide speed.

    MLORA_RASTER=8 python tools/raster_probe.py [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv  # noqa: E402
import torch  # noqa: E402

from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    ctx = F.Context(0)
    rows = 8192
    layer = FusedLoraLayer(ctx, LLAMA7B, [16] * 4, [2.0] * 4, [1e-4, 2e-4, 5e-5, 3e-4], rows, seed=1)
    layer.set_layout([j * 2048 for j in range(5)])
    x = (torch.rand(rows, 4096, generator=torch.Generator().manual_seed(2)) * 2 - 1).to(torch.bfloat16).cuda()
    for _ in range(20):
        layer.step(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    j0 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
    e0.record()
    for _ in range(steps):
        layer.step(x)
    e1.record()
    torch.cuda.synchronize()
    j1 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
    ms = e0.elapsed_time(e1) / steps
    print(json.dumps({"raster": os.environ.get("MLORA_RASTER", "default"), "ms_per_step": round(ms, 4),
                      "mJ_per_step": round((j1 - j0) / steps, 1), "W": round((j1 - j0) / (ms * steps), 1),
                      "clock": nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)}))


if __name__ == "__main__":
    main()
