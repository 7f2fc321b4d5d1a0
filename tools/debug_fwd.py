"""Quick numerical probe of the device path vs the fp64 oracle (prints errors)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2312_02515_b200 import fused as F
from oracle import mlora_oracle as O


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def case(M_seg, ranks, scales, d, k, seed=0):
    g = torch.Generator().manual_seed(seed)
    seg = [0]
    for m in M_seg: seg.append(seg[-1] + m)
    M = seg[-1]
    X = (torch.rand(M, k, generator=g) * 2 - 1)
    W0 = (torch.rand(d, k, generator=g) * 2 - 1) / k ** 0.5
    As = [(torch.rand(r, k, generator=g) * 2 - 1) / k ** 0.5 for r in ranks]
    Bs = [(torch.rand(d, r, generator=g) * 2 - 1) / max(r, 1) ** 0.5 for r in ranks]
    dY = (torch.rand(M, d, generator=g) * 2 - 1)
    bf = lambda t: t.to(torch.bfloat16)
    f64 = lambda t: bf(t).double().numpy()
    ctx = F.Context(0)
    plan = F.Plan(ctx, seg, ranks, scales)
    dev = torch.device("cuda", 0)
    A32, B32, A16, B16 = F.pack_adapters(ctx, plan, d, k, [bf(a).float().to(dev) for a in As], [bf(b).float().to(dev) for b in Bs])
    Xd, Wd, dYd = bf(X).to(dev), bf(W0).to(dev), bf(dY).to(dev)
    Y, H = F.linear_fwd(ctx, plan, Xd, Wd, A16, B16)
    dX, dA, dB = F.linear_bwd(ctx, plan, dYd, Xd, H, Wd, A16, B16)
    torch.cuda.synchronize()
    Yref = O.segmented_forward(f64(X), f64(W0), [f64(a) for a in As], [f64(b) for b in Bs], scales, seg)
    dXr, dAr, dBr = O.segmented_backward(f64(dY), f64(X), f64(W0), [f64(a) for a in As], [f64(b) for b in Bs], scales, seg)
    Yg = Y.float().cpu().numpy()
    print(f"case M={M} d={d} k={k} ranks={ranks} seg={seg}")
    print("  Y  rel", rel(Yg, Yref), " base-only rel", rel(Yg, f64(X) @ f64(W0).T))
    ro = plan.rank_offsets
    # H check
    Hg = H.float().cpu().numpy()
    for j in range(len(ranks)):
        a, b = seg[j], seg[j+1]
        Href = scales[j] * f64(X)[a:b] @ f64(As[j]).T
        print(f"  H[{j}] rel", rel(Hg[a:b, ro[j]:ro[j]+ranks[j]], Href), "offblock max", float(np.abs(np.delete(Hg[a:b], np.s_[ro[j]:ro[j]+ranks[j]], axis=1)).max()) if Hg.shape[1] > ranks[j] else 0)
    print("  dX rel", rel(dX.float().cpu().numpy(), dXr))
    dAg = dA.cpu().numpy(); dBg = dB.cpu().numpy()
    for j in range(len(ranks)):
        print(f"  dA[{j}] rel", rel(dAg[ro[j]:ro[j]+ranks[j]], dAr[j]), f" dB[{j}] rel", rel(dBg[:, ro[j]:ro[j]+ranks[j]], dBr[j]))
    # timing of the big shape
    return ctx


if __name__ == "__main__":
    case([128], [16], [1.0], 256, 128)
    case([256, 128], [16, 16], [1.0, 2.0], 512, 256)
    case([37, 163, 133], [8, 16, 32], [1.0, 0.5, 2.0], 384, 328)
    case([2048] * 4, [16] * 4, [2.0] * 4, 4096, 4096)
    case([1000, 3000, 500, 2692], [8, 16, 32, 64], [1.0] * 4, 4096, 11008)


def bench(M=8192, d=4096, k=4096, J=4, r=16, iters=20):
    dev = torch.device("cuda", 0)
    seg = [i * (M // J) for i in range(J + 1)]
    ctx = F.Context(0)
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
    def t(fn):
        for _ in range(3): fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(iters): fn()
        e.record(); torch.cuda.synchronize()
        return s.elapsed_time(e) / iters
    tf = t(lambda: F.linear_fwd(ctx, plan, X, W, A, B, Y, H))
    tb = t(lambda: F.linear_bwd(ctx, plan, dY, X, H, W, A, B, True, *outs[:3]))
    tt = t(lambda: torch.matmul(X, W.t()))
    fl = 2 * M * d * k
    print(f"bench M={M} d={d} k={k}: fwd {tf*1e3:.1f} us ({fl/tf/1e9:.0f} TF/s base-equiv), bwd {tb*1e3:.1f} us ({2*fl/tb/1e9:.0f} TF/s), torch.matmul {tt*1e3:.1f} us ({fl/tt/1e9:.0f} TF/s)")


if __name__ == "__main__" and os.environ.get("BENCH", "1") == "1":
    bench()
    bench(d=11008, k=4096)
    bench(d=4096, k=11008)
