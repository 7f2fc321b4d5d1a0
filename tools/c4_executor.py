"""BASELINE C4 end to end through the executor: the ChatGLM2-6B-shaped decoder
(multi-query attention, h 4096, V 65024; C4_LAYERS of its 28 layers) fine-tuning
6 LoRA jobs with per-job NormalTruncated sequence lengths, max_concurrent=4,
padding-masked cross-entropy as every job's loss (what detect_stop consumes).
C4_CFG=c3 runs BASELINE C3 at model level instead: the LLaMA-13B-shaped decoder
with 8 jobs of ranks {8, 16, 32, 64} x 2 (C4_LAYERS of its 40 layers).

Compares FIFO vs MinPad selection and the reference's padded FusedBatch layout
vs packed real tokens, with the reference accounting (δ, T_tot, T_e,
sim.cpp:258-265) on MEASURED step times, and each job's first / last CE.
One JSON line per run.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_02515_b200 import executor as X  # noqa: E402
from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200 import model as MD  # noqa: E402
from paper_2312_02515_b200 import packer as P  # noqa: E402


C3 = os.environ.get("C4_CFG") == "c3"


def jobs(iterations):
    if C3:
        means, ranks = [64, 128, 256, 512, 96, 192, 384, 448], [8, 16, 32, 64] * 2
        lrs = [1e-4, 2e-4, 5e-5, 3e-4] * 2
    else:
        means, ranks = [64, 128, 256, 384, 96, 192], [16] * 6
        lrs = [1e-4, 2e-4, 5e-5, 3e-4, 1e-4, 2e-4]
    out = []
    for j in range(len(means)):
        lens = P.sample_lengths("normal", 32, seed=4000 + j, min_len=16, max_len=512, mean=means[j], stddev=64.0)
        out.append(X.JobConfig(id=f"job{j}", lengths=lens, batch_size=4, rank=ranks[j], lr=lrs[j], scale=2.0,
                               priority=1 + j % 3, submit_time=float(j), iterations=iterations))
    return out


def main():
    iters = int(os.environ.get("C4_ITERS", "8"))
    layers = int(os.environ.get("C4_LAYERS", "8" if C3 else "28"))
    cfg = (MD.LLAMA_13B if C3 else MD.CHATGLM2_6B).with_layers(layers)
    name = (f"C3 llama-13b decoder ({layers} of 40 layers) 8 jobs r{{8,16,32,64}}x2, M=4" if C3 else
            f"C4 chatglm2-6b decoder ({layers} layers, MQA, V 65024) 6 jobs r16, M=4")
    ctx = F.Context(0)
    base = None
    for strategy in ("fifo", "minpad"):
        for padded in (True, False):
            ex = X.FusedExecutor(ctx, None, jobs(iters), max_concurrent=4, strategy=strategy, padded=padded, seed=5,
                                 model=cfg)
            if base is None:
                base = ex.layer
            else:  # every run fine-tunes the same frozen base
                js = jobs(iters)
                ex.layer = MD.MultiLoraDecoder(ctx, cfg, [j.rank for j in js], [2.0] * len(js), [j.lr for j in js],
                                               capacity=ex.layer.capacity, seed=5, frozen=base)
            ex.step()  # warm-up iteration (kernel attributes, tensor maps)
            ex.flush()
            ex.trace = X.Trace()
            trace = ex.run()
            m = trace.metrics()
            ce = {js.cfg.id: [round(js.losses[0], 4), round(js.losses[-1], 4)] for js in ex.jobs}
            print(json.dumps({"config": name,
                              "strategy": strategy, "layout": "padded" if padded else "packed",
                              **{k: round(v, 4) if isinstance(v, float) else v for k, v in m.items()},
                              "ce_first_last": ce}), flush=True)
            del ex
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
