"""Run a few MultiLoraDecoder steps (for ncu launch lists / profiles).

    python tools/decoder_step.py [--cfg chatglm2-6b] [--layers 2] [--jobs 6] [--seqs 4] [--len 512] [--steps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200 import model as MD  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="chatglm2-6b")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--jobs", type=int, default=6)
    ap.add_argument("--seqs", type=int, default=4)
    ap.add_argument("--len", type=int, default=512)
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    cfg = MD.CONFIGS[a.cfg].with_layers(a.layers)
    g = torch.Generator().manual_seed(0)
    seqs = [[torch.randint(0, cfg.vocab, (a.len,), generator=g).tolist() for _ in range(a.seqs)]
            for _ in range(a.jobs)]
    batch = MD.pack_tokens(seqs)
    m = MD.MultiLoraDecoder(F.Context(0), cfg, [16] * a.jobs, [2.0] * a.jobs, [1e-4] * a.jobs, capacity=batch.rows)
    m.set_batch(batch)
    for _ in range(a.steps):
        m.step()
    torch.cuda.synchronize()
    print("ok", m.loss.tolist())


if __name__ == "__main__":
    main()
