"""Rested (full-clock) timing of the C2 base GEMMs: per projection vs one grouped
launch per wave, for forward wave 1 (q, k, v, gate, up <- x), forward wave 2
(o, down) and the 7 dX.  Each measurement is one call bracketed by CUDA events
after a 0.2 s rest; median of 9.

    python tools/base_group_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_02515_b200 import _native as N
from paper_2312_02515_b200 import fused as F
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer


def timed(fn, reps=9):
    ts = []
    for _ in range(reps):
        time.sleep(0.2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    layer = FusedLoraLayer(ctx, LLAMA7B, [16] * 4, [2.0] * 4, [1e-4] * 4, rows=8192, seed=1)
    layer.set_layout([0, 2048, 4096, 6144, 8192])
    x = F.fill_uniform(torch.empty(8192, 4096, dtype=torch.bfloat16, device=dev), 5)
    layer.step(x)
    torch.cuda.synchronize()
    L, s = N.lib(), torch.cuda.current_stream().cuda_stream
    P = {p.name: p for p in layer.proj}
    inp = lambda p: x if p.src == "x" else P[p.src].Y

    def fwd_single(names):
        for n in names:
            p = P[n]
            N.check(L.mlora_base_fwd(ctx.handle, layer.plan.handle, p.d, p.k, inp(p).data_ptr(), p.W0.data_ptr(),
                                     p.H.data_ptr(), p.B.p_bf16.data_ptr(), p.Y.data_ptr(), p.row_sq.data_ptr(), s),
                    ctx.handle)

    def fwd_group(names):
        ps = [P[n] for n in names]
        k = len(ps)
        arr = lambda f: (N.vp * k)(*[f(p) for p in ps])
        N.check(L.mlora_base_fwd_group(ctx.handle, layer.plan.handle, k, (N.i32 * k)(*[p.d for p in ps]),
                                       (N.i32 * k)(*[p.k for p in ps]), arr(lambda p: inp(p).data_ptr()),
                                       arr(lambda p: p.W0.data_ptr()), arr(lambda p: p.H.data_ptr()),
                                       arr(lambda p: p.B.p_bf16.data_ptr()), arr(lambda p: p.Y.data_ptr()),
                                       arr(lambda p: p.row_sq.data_ptr()), s), ctx.handle)

    def dx_single(names):
        for n in names:
            p = P[n]
            N.check(L.mlora_base_dx(ctx.handle, layer.plan.handle, p.d, p.k, p.Y.data_ptr(), p.W0.data_ptr(),
                                    p.G.data_ptr(), p.A.p_bf16.data_ptr(), p.dX.data_ptr(), s), ctx.handle)

    def dx_group(names):
        ps = [P[n] for n in names]
        k = len(ps)
        arr = lambda f: (N.vp * k)(*[f(p) for p in ps])
        N.check(L.mlora_base_dx_group(ctx.handle, layer.plan.handle, k, (N.i32 * k)(*[p.d for p in ps]),
                                      (N.i32 * k)(*[p.k for p in ps]), arr(lambda p: p.Y.data_ptr()),
                                      arr(lambda p: p.W0.data_ptr()), arr(lambda p: p.G.data_ptr()),
                                      arr(lambda p: p.A.p_bf16.data_ptr()), arr(lambda p: p.dX.data_ptr()), s),
                  ctx.handle)

    if "--ncu" in sys.argv:  # one call of each dX variant, for an ncu capture
        dx_single(["up", "gate"])
        dx_group(["up", "gate"])
        torch.cuda.synchronize()
        return
    cases = {
        "fwd qkv": ["q", "k", "v"], "fwd gate,up": ["gate", "up"], "fwd wave1": ["q", "k", "v", "gate", "up"],
        "fwd o,down": ["o", "down"], "fwd down": ["down"], "fwd q": ["q"],
    }
    out = {}
    for name, names in cases.items():
        out[name] = {"single": round(timed(lambda: fwd_single(names)), 4),
                     "group": round(timed(lambda: fwd_group(names)), 4)}
    dcases = {"dx all7": ["down", "up", "gate", "o", "v", "k", "q"], "dx qkvo": ["o", "v", "k", "q"],
              "dx gate,up": ["up", "gate"], "dx heavy-first": ["up", "gate", "down", "o", "v", "k", "q"]}
    for name, names in dcases.items():
        out[name] = {"single": round(timed(lambda: dx_single(names)), 4),
                     "group": round(timed(lambda: dx_group(names)), 4)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
