"""A/B on one box: the C2 layer step with the base GEMMs grouped per wave (the
product, mlora_layer_step) vs one base-GEMM launch per projection (the same
kernels through mlora_base_fwd / mlora_base_dx).  Alternating blocks of steps
cancel clock drift under the power cap.

    python tools/group_ab.py [steps_per_block] [blocks]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_02515_b200 import _native as N
from paper_2312_02515_b200 import fused as F
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer


def ungrouped_step(layer, x):
    ctx, plan, L = layer.ctx, layer.plan, N.lib()
    s = torch.cuda.current_stream().cuda_stream
    rows = layer.cur_rows
    P = layer.proj
    ins = {p.name: (x if p.src == "x" else next(q for q in P if q.name == p.src).Y[:rows]) for p in P}
    waves = [[p for p in P if p.src == "x"], [p for p in P if p.src != "x"]]
    for wave in waves:
        n = len(wave)
        N.check(L.mlora_down_group(ctx.handle, plan.handle, n, 0, (N.i32 * n)(*[p.k for p in wave]),
                                   (N.vp * n)(*[ins[p.name].data_ptr() for p in wave]),
                                   (N.vp * n)(*[p.A.p_bf16.data_ptr() for p in wave]),
                                   (N.vp * n)(*[p.H.data_ptr() for p in wave]), s), ctx.handle)
        for p in wave:
            N.check(L.mlora_base_fwd(ctx.handle, plan.handle, p.d, p.k, ins[p.name].data_ptr(), p.W0.data_ptr(),
                                     p.H.data_ptr(), p.B.p_bf16.data_ptr(), p.Y.data_ptr(), p.row_sq.data_ptr(), s),
                    ctx.handle)
    n = len(P)
    N.check(L.mlora_loss_from_rowsq(ctx.handle, plan.handle, (N.vp * n)(*[p.row_sq.data_ptr() for p in P]),
                                    (N.i32 * n)(*[p.d for p in P]), n, layer.loss.data_ptr(), s), ctx.handle)
    N.check(L.mlora_down_group(ctx.handle, plan.handle, n, 1, (N.i32 * n)(*[p.d for p in P]),
                               (N.vp * n)(*[p.Y.data_ptr() for p in P]), (N.vp * n)(*[p.B.p_bf16.data_ptr() for p in P]),
                               (N.vp * n)(*[p.G.data_ptr() for p in P]), s), ctx.handle)
    for p in reversed(P):
        N.check(L.mlora_base_dx(ctx.handle, plan.handle, p.d, p.k, p.Y.data_ptr(), p.W0.data_ptr(), p.G.data_ptr(),
                                p.A.p_bf16.data_ptr(), p.dX.data_ptr(), s), ctx.handle)
    N.check(L.mlora_grad_group(ctx.handle, plan.handle, n, (N.i32 * n)(*[p.d for p in P]),
                               (N.i32 * n)(*[p.k for p in P]), (N.vp * n)(*[ins[p.name].data_ptr() for p in P]),
                               (N.vp * n)(*[p.Y.data_ptr() for p in P]), (N.vp * n)(*[p.H.data_ptr() for p in P]),
                               (N.vp * n)(*[p.G.data_ptr() for p in P]), (N.vp * n)(*[p.dA.data_ptr() for p in P]),
                               (N.vp * n)(*[p.dB.data_ptr() for p in P]), s), ctx.handle)
    layer.optimizer_step()


def main(steps=30, blocks=6):
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    layer = FusedLoraLayer(ctx, LLAMA7B, [16] * 4, [2.0] * 4, [1e-4, 2e-4, 5e-5, 3e-4], rows=8192, seed=1)
    layer.set_layout([0, 2048, 4096, 6144, 8192])
    x = F.fill_uniform(torch.empty(8192, 4096, dtype=torch.bfloat16, device=dev), 5)
    arms = {"grouped": lambda: layer.step(x), "per_projection": lambda: ungrouped_step(layer, x)}
    for f in arms.values():
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    res = {k: [] for k in arms}
    for b in range(blocks):
        for name in (list(arms) if b % 2 == 0 else list(reversed(list(arms)))):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                arms[name]()
            e1.record()
            e1.synchronize()
            res[name].append(e0.elapsed_time(e1) / steps)
    out = {k: {"ms_per_step": [round(v, 4) for v in vs], "mean": round(sum(vs) / len(vs), 4)}
           for k, vs in res.items()}
    # rested single steps (the power limiter relaxes between them): kernel efficiency at
    # the full clock, the regime of a short burst
    import time
    rested = {k: [] for k in arms}
    for r in range(12):
        for name in (list(arms) if r % 2 == 0 else list(reversed(list(arms)))):
            time.sleep(0.25)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            arms[name]()
            e1.record()
            e1.synchronize()
            rested[name].append(e0.elapsed_time(e1))
    for k, vs in rested.items():
        vs = sorted(vs)
        out[k]["rested_median_ms"] = round(vs[len(vs) // 2], 4)
        out[k]["rested_min_ms"] = round(vs[0], 4)
    # energy per step under sustained load (NVML total-energy counter, mJ)
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(0)
        for name in arms:
            torch.cuda.synchronize()
            j0 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
            for _ in range(200):
                arms[name]()
            torch.cuda.synchronize()
            out[name]["mJ_per_step"] = round((nv.nvmlDeviceGetTotalEnergyConsumption(h) - j0) / 200, 2)
    except Exception as e:
        out["energy_error"] = str(e)
    print(json.dumps(out))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
