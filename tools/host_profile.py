"""cProfile of the decoder step's host path (where the Python / ctypes time goes)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200 import model as MD  # noqa: E402

ctx = F.Context(0)
c = MD.LLAMA_7B.with_layers(4)
b = MD.pack_tokens([[list(range(1, 513)) for _ in range(4)] for _ in range(4)])
m = MD.MultiLoraDecoder(ctx, c, [16] * 4, [2.0] * 4, [1e-4] * 4, capacity=b.rows)
m.set_batch(b)
for _ in range(3):
    m.step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    m.step()
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
