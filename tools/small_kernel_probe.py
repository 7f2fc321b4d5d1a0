"""Time the HBM-bound kernels (down-projection H/G, dA/dB grads) vs rows: the
slope is the achieved streaming bandwidth, the intercept the fixed per-launch cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_02515_b200 import fused as F

dev = torch.device("cuda", 0)
ctx = F.Context(dev)
d = k = int(os.environ.get("DK", "4096"))
J, r = 4, 16
for M in (2048, 4096, 8192, 16384, 32768):
    seg = [j * (M // J) for j in range(J + 1)]
    plan = F.Plan(ctx, seg, [r] * J, [2.0] * J)
    R = plan.rank_padded
    X = torch.randn(M, k, device=dev).to(torch.bfloat16)
    W = (torch.randn(d, k, device=dev) / k ** 0.5).to(torch.bfloat16)
    A = (torch.randn(R, k, device=dev) / k ** 0.5).to(torch.bfloat16)
    B = (torch.randn(d, R, device=dev) / 4).to(torch.bfloat16)
    dY = torch.randn(M, d, device=dev).to(torch.bfloat16)
    Y, H = F.linear_fwd(ctx, plan, X, W, A, B)
    outs = F.linear_bwd(ctx, plan, dY, X, H, W, A, B)
    torch.cuda.synchronize()
    ctx.profile(reset=True)
    ctx.set_profiling(True)
    n = 20
    for _ in range(n):
        F.linear_fwd(ctx, plan, X, W, A, B, Y, H)
        F.linear_bwd(ctx, plan, dY, X, H, W, A, B, True, *outs[:3])
    ctx.set_profiling(False)
    p = ctx.profile(reset=True)
    mb = M * k * 2 / 1e6
    down_us = 1e3 * p["down"][1] / p["down"][0]
    grad_us = 1e3 * p["grad"][1] / p["grad"][0]
    aux_us = 1e3 * p["aux"][1] / max(p["aux"][0], 1)
    print(f"M={M:6d} X={mb:7.1f} MB | down {down_us:7.1f} us ({mb / down_us / 1e3:5.2f} TB/s) | "
          f"grad {grad_us:7.1f} us ({mb / grad_us / 1e3:5.2f} TB/s) | split-reduce {aux_us:5.1f} us "
          f"| base fwd {1e3 * p['base_fwd'][1] / p['base_fwd'][0]:7.1f} us")
