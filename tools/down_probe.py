"""Time the forward rank-r down-projection launches at C2 shapes (x 8192 x 4096,
4 jobs x r16) with CUDA events: the shared-input kernel (NB projections reading
one x) and the grouped kernel (the same NB problems, one each).

    python tools/down_probe.py [iters]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_02515_b200 import _native as N  # noqa: E402
from paper_2312_02515_b200 import fused as F  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    M, nb = 8192, 5
    K = int(os.environ.get("PROBE_K", "4096"))
    seg = [0, 2048, 4096, 6144, 8192]
    plan = F.Plan(ctx, seg, [16] * 4, [2.0] * 4)
    R = plan.rank_padded
    X = F.fill_uniform(torch.empty(M, K, dtype=torch.bfloat16, device=dev), 1)
    A = [F.fill_uniform(torch.empty(R, K, dtype=torch.bfloat16, device=dev), 2 + i, -0.02, 0.02) for i in range(nb)]
    H = [torch.empty(M, R, dtype=torch.bfloat16, device=dev) for _ in range(nb)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()

    def call(idx):
        m = len(idx)
        N.check(N.lib().mlora_down_group(ctx.handle, plan.handle, m, 0, (N.i32 * m)(*[K] * m),
                                         (N.vp * m)(*[X.data_ptr()] * m), (N.vp * m)(*[A[i].data_ptr() for i in idx]),
                                         (N.vp * m)(*[H[i].data_ptr() for i in idx]), s.cuda_stream), ctx.handle)

    for name, fn in (("shared-input NB=5", lambda: call(list(range(nb)))),
                     ("grouped, 1 problem (x once)", lambda: call([0]))):
        for _ in range(5):
            fn()
        ts = []
        for _ in range(iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        med = ts[len(ts) // 2]
        byt = M * K * 2 + M * R * 2 * (nb if "NB" in name else 1)
        print(f"{name:32s} median {med:7.1f} us  min {ts[0]:7.1f} us  {byt / med / 1e3:7.0f} GB/s (x + H)")


if __name__ == "__main__":
    main()
