"""Soak test: long runs of the C2 layer step and of a small decoder fine-tune.

* C2: 3000 steps, twice from the same seeds: every step's per-job losses must be
  finite and the two runs bitwise identical (deterministic kernels, no atomics);
  reports the step-time drift under the power cap.
* Decoder: TINY_LLAMA fine-tuning 4 jobs on fixed token batches for 400 steps:
  every job's CE must fall monotonically on average (first / last 20-step means).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200 import model as MD  # noqa: E402
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer  # noqa: E402


def c2_run(ctx, steps):
    layer = FusedLoraLayer(ctx, LLAMA7B, [16] * 4, [2.0] * 4, [1e-4, 2e-4, 5e-5, 3e-4], 8192, seed=3)
    layer.set_layout([j * 2048 for j in range(5)])
    x = (torch.rand(8192, 4096, generator=torch.Generator().manual_seed(4)) * 2 - 1).to(torch.bfloat16).cuda()
    losses = torch.empty(steps, 4, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    for i in range(steps):
        if i == 100:
            ev[1].record()
        if i == steps - 100:
            ev[2].record()
        losses[i] = layer.step(x)
    ev[3].record()
    torch.cuda.synchronize()
    return losses.cpu(), ev[0].elapsed_time(ev[1]) / 100, ev[2].elapsed_time(ev[3]) / 100


def main():
    ctx = F.Context(0)
    steps = int(os.environ.get("SOAK_STEPS", "3000"))
    a, t_first, t_last = c2_run(ctx, steps)
    b, _, _ = c2_run(ctx, steps)
    out = {"c2_steps": steps, "all_finite": bool(torch.isfinite(a).all()), "bitwise_identical_runs": bool(torch.equal(a, b)),
           "ms_per_step_first100": round(t_first, 3), "ms_per_step_last100": round(t_last, 3),
           "loss_first": a[0].tolist(), "loss_last": a[-1].tolist()}
    g = torch.Generator().manual_seed(7)
    seqs = [[torch.randint(0, 96, (64,), generator=g).tolist() for _ in range(4)] for _ in range(4)]
    batch = MD.pack_tokens(seqs)
    m = MD.MultiLoraDecoder(ctx, MD.TINY_LLAMA, [8, 8, 16, 16], [2.0] * 4, [1e-3, 2e-3, 5e-4, 3e-3], capacity=batch.rows,
                            seed=7, lora_init="zero_b")
    m.set_batch(batch)
    ce = torch.stack([m.step().clone() for _ in range(400)]).cpu()
    out["decoder_ce_first20"] = [round(v, 4) for v in ce[:20].mean(0).tolist()]
    out["decoder_ce_last20"] = [round(v, 4) for v in ce[-20:].mean(0).tolist()]
    out["decoder_all_finite"] = bool(torch.isfinite(ce).all())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
