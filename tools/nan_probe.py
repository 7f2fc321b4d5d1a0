"""Where does a diverged job's inf/NaN first reach another job?  Replays the
executor's early-stopping scenario on a fixed layout and, after every step,
reports per job which tensors hold non-finite values in that job's rows
(Y, H, G, dX, inputs) or columns (dA, dB, A, B masters and bf16 copies)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_02515_b200 import fused as F
from paper_2312_02515_b200.layer import TINY, FusedLoraLayer

ctx = F.Context(0)
J = 4
lrs = [1e-3, 1e30, 1e-3, 1e-3]
layer = FusedLoraLayer(ctx, TINY, [8] * J, [2.0] * J, lrs, rows=4 * 72, seed=11)
seg = [0, 72, 144, 216, 288]
layer.set_layout(seg)
r = layer.plan.rank_offsets
g = torch.Generator(device="cpu").manual_seed(3)


def bad(t):
    return not bool(torch.isfinite(t.float()).all())


for step in range(1, 6):
    x = ((torch.rand(288, TINY[0][2], generator=g) * 2 - 1).to(torch.bfloat16)).cuda()
    loss = layer.forward_backward(x).clone()
    torch.cuda.synchronize()
    report = {}
    for j in range(J):
        rows = slice(seg[j], seg[j + 1])
        cols = slice(r[j], r[j + 1])
        hits = []
        for p in layer.proj:
            for nm, t in (("Y", p.Y[rows]), ("H", p.H[rows]), ("G", p.G[rows]), ("dX", p.dX[rows]),
                          ("dA", p.dA[cols]), ("dB", p.dB[:, cols])):
                if bad(t):
                    hits.append(f"{p.name}.{nm}")
        report[j] = hits
    print(f"step {step} loss {loss.tolist()}")
    for j in range(J):
        print(f"   job{j}: {report[j][:12]}{' ...' if len(report[j]) > 12 else ''}")
    layer.optimizer_step()
    torch.cuda.synchronize()
    for j in range(J):
        cols = slice(r[j], r[j + 1])
        pb = [p.name for p in layer.proj if bad(p.A.p[cols]) or bad(p.B.p[:, cols]) or bad(p.A.p_bf16[cols])
              or bad(p.B.p_bf16[:, cols])]
        if pb:
            print(f"   after adam job{j} params non-finite in {pb}")
