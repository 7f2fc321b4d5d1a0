"""Decoder-level probe: parity errors vs the torch fp32 restatement and the
step throughput of MultiLoraDecoder on a given config (B200).

    python tools/decoder_probe.py [--cfg chatglm2-6b] [--layers N] [--jobs 6] [--seqs 4] [--len 512]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import torch  # noqa: E402

from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200 import model as MD  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="chatglm2-6b")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--jobs", type=int, default=6)
    ap.add_argument("--seqs", type=int, default=4)
    ap.add_argument("--len", type=int, default=512)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--parity", action="store_true")
    a = ap.parse_args()
    cfg = MD.CONFIGS[a.cfg]
    if a.layers:
        cfg = cfg.with_layers(a.layers)
    g = torch.Generator().manual_seed(0)
    seqs = [[torch.randint(0, cfg.vocab, (a.len,), generator=g).tolist() for _ in range(a.seqs)]
            for _ in range(a.jobs)]
    batch = MD.pack_tokens(seqs)
    ctx = F.Context(0)
    t0 = time.time()
    m = MD.MultiLoraDecoder(ctx, cfg, [a.rank] * a.jobs, [2.0] * a.jobs, [1e-4] * a.jobs, capacity=batch.rows)
    init_s = time.time() - t0
    m.set_batch(batch)
    out = {"cfg": cfg.name, "layers": cfg.layers, "rows": batch.rows, "init_s": round(init_s, 1)}
    if a.parity:
        import test_gpu_decoder as T
        loss = m.forward()
        m.backward()
        torch.cuda.synchronize()
        want, grads = T.model_ref(m, batch)
        out["loss"] = loss.tolist()
        out["loss_ref"] = want.tolist()
        worst = 0.0
        roff = m.plan.rank_offsets
        for li, L in enumerate(m.layers):
            for name, p in L.proj.items():
                gA, gB = grads[(li, name)]
                for j in range(m.J):
                    r0, r = roff[j], m.ranks[j]
                    worst = max(worst, T.rel(p.dA[r0:r0 + r], gA[j]), T.rel(p.dB[:, r0:r0 + r], gB[j]))
        out["worst_grad_rel"] = worst
    for _ in range(2):
        m.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        m.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    # split: time the attention kernels alone on the same inputs
    from paper_2312_02515_b200 import model_ops as M
    L = m.layers[0]
    q, k, v = m._qkv_views(L)
    r = m.rows
    lse = L.lse.view(-1)[: cfg.heads * r].view(cfg.heads, r)
    dq, dk, dv = m._qkv_views(L, grad=True)
    e0.record()
    for _ in range(a.steps):
        m._attn_fwd(L, q, k, v, None)
        M.attn_bwd(m.layout, L.qr[:r], L.kr[:r], v, L.attn[:r], L.x1[:r], lse, dq, dk, dv, cfg.heads, cfg.kv_heads,
                   cfg.head_dim, cfg.rope_base, prerotated=True)
    e1.record()
    torch.cuda.synchronize()
    attn_ms = e0.elapsed_time(e1) / a.steps * cfg.layers
    flops = m.flops_per_step()
    out.update(ms_per_step=round(ms, 3), tokens_per_s=round(batch.real_tokens / ms * 1e3, 1),
               tflops=round(flops / ms / 1e9, 1), attn_ms_per_step=round(attn_ms, 3))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
