"""Where does the e2e pass lose time against the device-resident pass?  C2 layer
step, timed with CUDA events from a rested GPU (1.5 s sleep before each pass):
  plain     layer.step(x) back to back (the headline pass)
  d2h       + every step's per-job losses copied D2H (non_blocking, pinned)
  events    + the pipelined trainer's event record/wait per step, no upload
  trainer   PipelinedTrainer: + 64 MiB H2D per step on a copy stream (the e2e pass)

    python tools/e2e_probe.py [steps] [rounds]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_02515_b200 import fused as F  # noqa: E402
from paper_2312_02515_b200.layer import LLAMA7B, FusedLoraLayer  # noqa: E402
from paper_2312_02515_b200.trainer import PipelinedTrainer  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    J, per_job = 4, 2048
    rows = J * per_job
    layer = FusedLoraLayer(ctx, LLAMA7B, [16] * J, [2.0] * J, [1e-4, 2e-4, 5e-5, 3e-4], rows, seed=1000)
    layer.set_layout([j * per_job for j in range(J + 1)])
    x_host = (torch.rand(rows, 4096) * 2 - 1).to(torch.bfloat16).pin_memory()
    x = x_host.to(dev)
    s = torch.cuda.current_stream()
    losses_host = torch.empty(steps, J, dtype=torch.float32).pin_memory()
    trainer = PipelinedTrainer(layer, rows, 4096)
    ev = [torch.cuda.Event() for _ in range(2)]

    def plain():
        for _ in range(steps):
            layer.step(x)

    def d2h():
        for i in range(steps):
            losses_host[i].copy_(layer.step(x), non_blocking=True)

    def events():
        for i in range(steps):
            s.wait_event(ev[i & 1])
            loss = layer.step(x)
            ev[i & 1].record(s)
            losses_host[i].copy_(loss, non_blocking=True)

    def train():
        trainer.run([x_host] * steps, losses_host)

    for _ in range(3):
        plain()
    train()
    torch.cuda.synchronize()
    for r in range(rounds):
        for name, fn in (("plain", plain), ("d2h", d2h), ("events", events), ("trainer", train)):
            torch.cuda.synchronize()
            time.sleep(1.5)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / steps
            print(f"round {r} {name:8s} {ms:6.3f} ms/step  {rows / ms * 1e3 / 1e6:6.3f} M tok/s", flush=True)


if __name__ == "__main__":
    main()
