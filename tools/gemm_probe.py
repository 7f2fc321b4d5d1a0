"""Sustained throughput of the CTA-pair base GEMM vs cuBLAS (torch.matmul) on the
LLaMA-7B projection shapes, 200 back-to-back launches each, with the SM clock
sampled (NVML) during each loop."""
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


def clocked(fn, n):
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            time.sleep(0.002)
    for _ in range(10):
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
    return s.elapsed_time(e) / n, statistics.median(samples) if samples else None


dev = torch.device("cuda", 0)
ctx = F.Context(dev)
M, J = 8192, 4
plan = F.Plan(ctx, [j * M // J for j in range(J + 1)], [16] * J, [2.0] * J)
R = plan.rank_padded
for d, k in ((4096, 4096), (11008, 4096), (4096, 11008)):
    X = torch.randn(M, k, device=dev).to(torch.bfloat16)
    W = (torch.randn(d, k, device=dev) / k ** 0.5).to(torch.bfloat16)
    H = torch.randn(M, R, device=dev).to(torch.bfloat16)
    B = torch.randn(d, R, device=dev).to(torch.bfloat16)
    Y = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    ours = lambda: N.lib().mlora_base_fwd(ctx.handle, plan.handle, d, k, X.data_ptr(), W.data_ptr(), H.data_ptr(),
                                          B.data_ptr(), Y.data_ptr(), None, s)
    cub = lambda: torch.matmul(X, W.t(), out=Y)
    fl = 2.0 * M * d * k
    for name, fn in (("mlora pair", ours), ("cuBLAS", cub), ("mlora pair", ours), ("cuBLAS", cub)):
        ms, mhz = clocked(fn, 200)
        print(f"{d:5d}x{k:5d} {name:10s}: {ms * 1e3:7.1f} us  {fl / ms / 1e9:7.1f} TF/s  median SM {mhz} MHz")
