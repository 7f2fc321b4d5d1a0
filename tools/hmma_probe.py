"""Cost of computing the rank-r intermediate H = X A^T INSIDE the forward base GEMM
(the north star's "keep X_i A_i on chip" alternative): the CTA-pair kernel issues,
per main k-step, one extra UMMA 256 x 16n next to the 256 x 256 one (MLORA_EXP_HMMA=n,
an experiment build flag: the extra product lands in the output tile, so results are
wrong; only the time is of interest).  Variants are interleaved in bursts so the
power-capped clock drifts equally over all of them.

    python tools/hmma_probe.py [rounds] [burst]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_02515_b200 import _native as N  # noqa: E402
from paper_2312_02515_b200 import fused as F  # noqa: E402


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    burst = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    M, J = 8192, 4
    plan = F.Plan(ctx, [j * M // J for j in range(J + 1)], [16] * J, [2.0] * J)
    R = plan.rank_padded
    s = torch.cuda.current_stream()
    for d, k in ((4096, 4096), (11008, 4096), (4096, 11008)):
        X = F.fill_uniform(torch.empty(M, k, dtype=torch.bfloat16, device=dev), 1)
        W0 = F.fill_uniform(torch.empty(d, k, dtype=torch.bfloat16, device=dev), 2, -k ** -0.5, k ** -0.5)
        H = F.fill_uniform(torch.empty(M, R, dtype=torch.bfloat16, device=dev), 3)
        B = F.fill_uniform(torch.empty(d, R, dtype=torch.bfloat16, device=dev), 4, -0.1, 0.1)
        Y = torch.empty(M, d, dtype=torch.bfloat16, device=dev)

        def launch():
            N.check(N.lib().mlora_base_fwd(ctx.handle, plan.handle, d, k, X.data_ptr(), W0.data_ptr(), H.data_ptr(),
                                           B.data_ptr(), Y.data_ptr(), None, s.cuda_stream), ctx.handle)
        times = {0: [], 1: [], 2: []}
        for _ in range(3):
            launch()
        for _ in range(rounds):
            for v in times:
                os.environ["MLORA_EXP_HMMA"] = str(v)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(burst):
                    launch()
                e1.record(s)
                e1.synchronize()
                times[v].append(e0.elapsed_time(e1) * 1e3 / burst)
        base = statistics.median(times[0])
        print(f"d={d} k={k}: " + "  ".join(
            f"extra N={16 * v}: {statistics.median(t):7.1f} us ({100 * (statistics.median(t) / base - 1):+.1f}%)"
            for v, t in times.items()), flush=True)


if __name__ == "__main__":
    main()
