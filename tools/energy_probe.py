"""Where do the joules of a C2 layer step go?  Each launch type of the step is run
back to back for ~1.5 s (the 1 kW cap engaged, as in the sustained bench pass) and the
NVML total-energy counter read around the loop: average board power, time and energy
per launch, and energy per algorithmic FLOP / byte.  The step's own joules come from
the same counter over 200 steps.

    python tools/energy_probe.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv  # noqa: E402

from paper_2312_02515_b200 import _native as N  # noqa: E402
from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer  # noqa: E402

import ctypes  # noqa: E402
FP = ctypes.POINTER(ctypes.c_float)


def main():
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    rows = 8192
    layer = FusedLoraLayer(ctx, LLAMA7B, [16] * 4, [2.0] * 4, [1e-4, 2e-4, 5e-5, 3e-4], rows=rows, seed=1)
    layer.set_layout([0, 2048, 4096, 6144, 8192])
    x = F.fill_uniform(torch.empty(rows, 4096, dtype=torch.bfloat16, device=dev), 5)
    for _ in range(3):
        layer.step(x)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream().cuda_stream
    P = {p.name: p for p in layer.proj}
    L = N.lib()
    plan = layer.plan.handle
    R = layer.plan.rank_padded

    def inp(p):
        return x if p.src == "x" else P[p.src].Y

    def base_fwd(name):
        p = P[name]
        return lambda: N.check(L.mlora_base_fwd(ctx.handle, plan, p.d, p.k, inp(p).data_ptr(), p.W0.data_ptr(),
                                                p.H.data_ptr(), p.B.p_bf16.data_ptr(), p.Y.data_ptr(), None, s), ctx.handle)

    def base_dx(name):
        p = P[name]
        return lambda: N.check(L.mlora_base_dx(ctx.handle, plan, p.d, p.k, p.Y.data_ptr(), p.W0.data_ptr(),
                                               p.G.data_ptr(), p.A.p_bf16.data_ptr(), p.dX.data_ptr(), s), ctx.handle)

    projs = list(P.values())
    n = len(projs)

    def g_group():
        N.check(L.mlora_down_group(ctx.handle, plan, n, 1, (N.i32 * n)(*[p.d for p in projs]),
                                   (N.vp * n)(*[p.Y.data_ptr() for p in projs]),
                                   (N.vp * n)(*[p.B.p_bf16.data_ptr() for p in projs]),
                                   (N.vp * n)(*[p.G.data_ptr() for p in projs]), s), ctx.handle)

    xs = [p for p in projs if p.src == "x"]

    def down_multi():
        m = len(xs)
        N.check(L.mlora_down_group(ctx.handle, plan, m, 0, (N.i32 * m)(*[4096] * m), (N.vp * m)(*[x.data_ptr()] * m),
                                   (N.vp * m)(*[p.A.p_bf16.data_ptr() for p in xs]),
                                   (N.vp * m)(*[p.H.data_ptr() for p in xs]), s), ctx.handle)

    def grads():
        N.check(L.mlora_grad_group(ctx.handle, plan, n, (N.i32 * n)(*[p.d for p in projs]),
                                   (N.i32 * n)(*[p.k for p in projs]), (N.vp * n)(*[inp(p).data_ptr() for p in projs]),
                                   (N.vp * n)(*[p.Y.data_ptr() for p in projs]),
                                   (N.vp * n)(*[p.H.data_ptr() for p in projs]),
                                   (N.vp * n)(*[p.G.data_ptr() for p in projs]),
                                   (N.vp * n)(*[p.dA.data_ptr() for p in projs]), (N.vp * n)(*[p.dB.data_ptr() for p in projs]),
                                   s), ctx.handle)

    def C_f(t):
        import ctypes
        return ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_float))

    def step():
        layer.step(x)

    fl = lambda d, k: 2 * rows * d * k
    cases = [
        ("layer step (C2)", step, 8192 * 816996352, None),
        ("base fwd 4096x4096 (q)", base_fwd("q"), fl(4096, 4096), None),
        ("base fwd 11008x4096 (gate)", base_fwd("gate"), fl(11008, 4096), None),
        ("base fwd 4096x11008 (down)", base_fwd("down"), fl(4096, 11008), None),
        ("base dX 4096x4096 (q)", base_dx("q"), fl(4096, 4096), None),
        ("base dX 11008->4096 (gate)", base_dx("gate"), fl(11008, 4096), None),
        ("G group (7 projections)", g_group, None, sum(rows * p.d * 2 for p in projs)),
        ("shared-input down (5 projections)", down_multi, None, rows * 4096 * 2),
        ("dA + dB groups (+ reduce)", grads, None, sum(rows * (p.d + p.k) * 2 for p in projs)),
    ]
    if os.environ.get("ENERGY_AB"):  # interleaved A/B of the forward and dX GEMM on one shape
        cases = [c for c in cases if c[0] in ("base fwd 4096x4096 (q)", "base dX 4096x4096 (q)")] * 4
    for name, fn, flops, byts in cases:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        time.sleep(1.5)
        # size the loop to ~1.5 s
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        e1.synchronize()
        per = e0.elapsed_time(e1) / 5
        iters = max(10, int(1500.0 / per))
        j0 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        e1.synchronize()
        j1 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
        ms = e0.elapsed_time(e1) / iters
        mj = (j1 - j0) / iters
        rec = {"case": name, "ms": round(ms, 4), "mJ": round(mj, 2), "W": round(mj / ms, 1),
               "sm_mhz": nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)}
        if flops:
            rec["pJ_per_flop"] = round(mj * 1e9 / flops, 4)
            rec["TFLOPs"] = round(flops / ms / 1e9, 1)
        if byts:
            rec["pJ_per_byte"] = round(mj * 1e9 / byts, 2)
            rec["GBs"] = round(byts / ms / 1e6, 1)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
