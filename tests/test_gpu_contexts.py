"""One context per GPU / thread (include/mlora.h): launch attributes are opted in
per (kernel, device) under a lock, so contexts created on several devices or
driven from several threads of one process all launch correctly.  Two threads
each drive their own context (and stream) through the full layer step at the
same time; their results must be bitwise those of a single-threaded run.  With
two GPUs the second context lives on the second device."""
import threading

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def run_step(device, seed, out, key, barrier=None):
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200.layer import TINY, FusedLoraLayer
    torch.cuda.set_device(device)
    ctx = F.Context(device)
    s = torch.cuda.Stream(device=device)
    with torch.cuda.stream(s):
        layer = FusedLoraLayer(ctx, TINY, [8, 16, 32], [2.0] * 3, [1e-3] * 3, rows=600, seed=seed)
        layer.set_layout([0, 100, 350, 600])
        x = F.fill_uniform(torch.empty(600, 256, dtype=torch.bfloat16, device=device), seed + 1)
        if barrier is not None:
            barrier.wait()
        for _ in range(3):
            loss = layer.step(x)
        s.synchronize()
        out[key] = (loss.cpu().clone(), layer.proj[-1].A.p.cpu().clone(), layer.proj[0].dX.cpu().clone())


def test_two_contexts_two_threads_match_single_threaded():
    ndev = torch.cuda.device_count()
    devs = [0, 1] if ndev >= 2 else [0, 0]
    ref = {}
    for i, dv in enumerate(devs):
        run_step(dv, 10 + i, ref, i)
    got, errs = {}, []
    barrier = threading.Barrier(2)

    def worker(i):
        try:
            run_step(devs[i], 10 + i, got, i, barrier)
        except Exception as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(2):
        for a, b in zip(ref[i], got[i]):
            assert torch.equal(a, b)
