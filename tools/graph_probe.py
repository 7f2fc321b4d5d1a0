"""A/B: eager layer steps vs the same step captured once in a CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_02515_b200 import fused as F
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer

dev = torch.device("cuda", 0)
ctx = F.Context(dev)
J, per = 4, 2048
layer = FusedLoraLayer(ctx, LLAMA7B, [16] * J, [2.0] * J, [1e-4, 2e-4, 5e-5, 3e-4], rows=J * per, seed=1)
layer.set_layout([j * per for j in range(J + 1)])
x = (torch.rand(J * per, 4096, device=dev) * 2 - 1).to(torch.bfloat16)
for _ in range(5):
    layer.step(x)
torch.cuda.synchronize()


def timeit(fn, n=30):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


eager = timeit(lambda: layer.step(x))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    layer.step(x)  # warm on the capture stream
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        layer.step(x)
torch.cuda.synchronize()
graphed = timeit(lambda: g.replay())
eager2 = timeit(lambda: layer.step(x))
print(f"eager {eager:.3f} ms/step, graph {graphed:.3f} ms/step, eager again {eager2:.3f} ms/step "
      f"-> {J * per / graphed * 1e3:.0f} tok/s graphed")
