"""Host enqueue time per step vs device time per step (is the GPU ever starved
by the Python / ctypes launch path?).  C2 layer step and decoder steps."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200 import model as MD  # noqa: E402
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer  # noqa: E402


def probe(name, step, n=20):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    host = (time.perf_counter() - t0) / n
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / n / 1e3
    print(json.dumps({"workload": name, "host_ms_per_step": round(host * 1e3, 3), "device_ms_per_step": round(dev * 1e3, 3)}))


ctx = F.Context(0)
layer = FusedLoraLayer(ctx, LLAMA7B, [16] * 4, [2.0] * 4, [1e-4] * 4, 8192, seed=1)
layer.set_layout([j * 2048 for j in range(5)])
x = (torch.rand(8192, 4096, device="cuda") * 2 - 1).to(torch.bfloat16)
probe("c2 layer step", lambda: layer.step(x))
for cfg, L, J, n in ((MD.TINY_LLAMA, 2, 2, 64), (MD.LLAMA_7B, 4, 4, 512), (MD.CHATGLM2_6B, 4, 6, 512)):
    c = cfg.with_layers(L)
    seqs = [[list(range(1, n + 1)) for _ in range(4)] for _ in range(J)]
    b = MD.pack_tokens(seqs)
    m = MD.MultiLoraDecoder(ctx, c, [16] * J, [2.0] * J, [1e-4] * J, capacity=b.rows)
    m.set_batch(b)
    probe(f"{c.name} x{L} layers decoder step", lambda: m.step())
    del m
