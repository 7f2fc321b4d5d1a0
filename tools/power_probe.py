"""Base-GEMM throughput with SM clock and board power sampled (NVML) — decides
whether the CTA-pair kernel is power-bound (throughput ~ watts / energy-per-op)
or operand-bandwidth-bound.  Run once per MLORA_BASE_KERNEL variant (the variant
is latched per process)."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv
import torch

from paper_2312_02515_b200 import _native as N
from paper_2312_02515_b200 import fused as F

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)


def measured(fn, n):
    clk, pw, stop = [], [], threading.Event()

    def sample():
        while not stop.is_set():
            clk.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            pw.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)
            time.sleep(0.002)
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    th = threading.Thread(target=sample)
    th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    return s.elapsed_time(e) / n, statistics.median(clk), statistics.median(pw)


dev = torch.device("cuda", 0)
ctx = F.Context(dev)
M, J = 8192, 4
plan = F.Plan(ctx, [j * M // J for j in range(J + 1)], [16] * J, [2.0] * J)
R = plan.rank_padded
variant = os.environ.get("MLORA_BASE_KERNEL", "pair")
for d, k in ((4096, 4096), (11008, 4096)):
    X = torch.randn(M, k, device=dev).to(torch.bfloat16)
    W = (torch.randn(d, k, device=dev) / k ** 0.5).to(torch.bfloat16)
    H = torch.randn(M, R, device=dev).to(torch.bfloat16)
    B = torch.randn(d, R, device=dev).to(torch.bfloat16)
    Y = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    fn = lambda: N.lib().mlora_base_fwd(ctx.handle, plan.handle, d, k, X.data_ptr(), W.data_ptr(), H.data_ptr(),
                                        B.data_ptr(), Y.data_ptr(), None, s)
    fl = 2.0 * M * d * k
    for rep in range(2):
        ms, mhz, watts = measured(fn, 1000)
        tf = fl / ms / 1e9
        print(f"{variant:5s} {d:5d}x{k:5d}: {ms * 1e3:7.1f} us  {tf:7.1f} TF/s  SM {mhz:.0f} MHz  "
              f"{watts:.0f} W  {tf / watts:.3f} TF/s/W  {tf / mhz * 1e3:.1f} GF/s/MHz")
