"""C2 layer step (LLaMA-7B layer, 8192 tokens, r16) with the same tokens split
over J = 1 .. 64 fused jobs: step time, effective tokens/s and launches per step.
BatchFusion's claim is that fusing more jobs costs (almost) nothing: one launch
set per layer step whatever J is (the per-job scheme needs 4 launches per job
and projection, count_launches, lora.cpp:184-189).  Same timing as bench.py
(CUDA events over the steps, inputs resident).

    python tools/jobs_scaling_probe.py [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer, flops_per_token  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    ctx = F.Context(0)
    rows = 8192
    g = torch.Generator(device="cpu").manual_seed(1234)
    W0 = {n: ((torch.rand(d, k, generator=g) * 2 - 1) / k ** 0.5).to(torch.bfloat16).cuda() for n, d, k, _ in LLAMA7B}
    x = (torch.rand(rows, 4096, generator=g) * 2 - 1).to(torch.bfloat16).cuda()
    for J in (1, 4, 8, 16, 32, 64):
        layer = FusedLoraLayer(ctx, LLAMA7B, [16] * J, [2.0] * J, [1e-4] * J, rows, seed=J, W0=W0)
        layer.set_layout([j * rows // J for j in range(J + 1)])
        for _ in range(5):
            layer.step(x)
        torch.cuda.synchronize()
        l0 = ctx.launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            layer.step(x)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        print(json.dumps({"jobs": J, "rank": 16, "R_pad": layer.plan.rank_padded, "ms_per_step": round(ms, 3),
                          "tokens_per_s": round(rows / ms * 1e3), "tflops": round(rows * flops_per_token(LLAMA7B, 16)
                                                                               / ms / 1e9, 1),
                          "launches_per_step": (ctx.launches - l0) / steps,
                          "per_job_scheme_launches_per_step": 7 * 4 * J * 2}), flush=True)
        del layer
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
