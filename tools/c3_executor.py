"""BASELINE C3 through the executor: LLaMA-13B-shaped layer, 8 jobs with ranks
{8,16,32,64}x2 and per-job NormalTruncated sequence lengths, max_concurrent=4.

Compares selection strategies (FIFO vs MinPad, batch_select.cpp) and row
layouts (the reference's padded FusedBatch vs packed real tokens): reports the
reference accounting (δ = Σξ_p/Σξ, T_tot, T_e = (1-δ)·T_tot, sim.cpp:258-265)
with MEASURED step times, and effective tokens/s.  Prints one JSON line per run.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_02515_b200 import executor as X
from paper_2312_02515_b200 import fused as F
from paper_2312_02515_b200 import packer as P
from paper_2312_02515_b200.layer import LLAMA13B


def jobs(iterations):
    ranks = [8, 16, 32, 64] * 2
    means = [64, 128, 256, 512, 1024, 96, 192, 384]
    lrs = [1e-4, 2e-4, 5e-5, 3e-4] * 2
    out = []
    for j in range(8):
        lens = P.sample_lengths("normal", 64, seed=3000 + j, min_len=32, max_len=1024, mean=means[j], stddev=96.0)
        out.append(X.JobConfig(id=f"job{j}", lengths=lens, batch_size=4, rank=ranks[j], lr=lrs[j], scale=2.0,
                               priority=1 + j % 3, submit_time=float(j), iterations=iterations))
    return out


def main():
    iters = int(os.environ.get("C3_ITERS", "6"))
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    g = torch.Generator(device="cpu").manual_seed(1234)
    W0 = {name: ((torch.rand(d, k, generator=g) * 2 - 1) / k ** 0.5).to(torch.bfloat16).to(dev)
          for name, d, k, _ in LLAMA13B}
    for strategy in ("fifo", "minpad"):
        for padded in (True, False):
            ex = X.FusedExecutor(ctx, LLAMA13B, jobs(iters), max_concurrent=4, strategy=strategy, padded=padded,
                                 seed=5, W0=W0)
            ex.step()  # warm-up iteration (kernel attributes, tensor maps)
            ex.flush()
            ex.trace = X.Trace()
            trace = ex.run()
            m = trace.metrics()
            print(json.dumps({"config": "C3 llama13b-layer 8 jobs r{8,16,32,64}x2, M=4", "strategy": strategy,
                              "layout": "padded" if padded else "packed", **{k: round(v, 4) if isinstance(v, float)
                                                                               else v for k, v in m.items()}}))
            del ex
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
