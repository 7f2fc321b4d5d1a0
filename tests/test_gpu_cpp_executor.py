"""The C++ trainer hook: the façade's real executor behind the simulator's fused
iteration (include/fusim/b200.hpp, FusedIterationExecutor) against the Python
executor, and the bf16 fused_forward behind the reference signature.

tests/cpp/executor_loop.cpp drives a run_simulation-shaped loop
(/root/reference/proj/src/sim.cpp:163-191) on the GPU through the C ABI's
one-call layer step (mlora_layer_step_timed): peek -> select -> fused_shape ->
device fuse -> fused fwd/bwd/AdamW -> commit -> IterationDone{ξ, ξ_p, jobs}
charged with the measured device time.  The Python executor
(paper_2312_02515_b200/executor.py) runs the same workload; both hosts
initialise weights and datasets with the same counter-based fill, so the two
traces must agree exactly: the event sequence, ξ, ξ_p, the jobs and their
routing order, AND every per-job loss bit for bit.
"""
import json
import os
import struct
import subprocess

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "cpp", "build")


def _binary(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        subprocess.run(["bash", os.path.join(HERE, "cpp", "build.sh")], check=True)
    return path


# the workload executor_loop.cpp hardcodes
def executor_jobs():
    from paper_2312_02515_b200.executor import JobConfig
    prio, submit = [1, 2, 1, 3, 1, 2], [0.0, 0.0, 1.0, 1.0, 2.0, 2.0]
    bs, rank = [2, 3, 2, 2, 4, 2], [8, 16, 32, 8, 16, 64]
    lr, iters = [1e-3, 2e-3, 5e-4, 1e-3, 3e-3, 1e-3], [5, 7, 4, 6, 8, 5]
    return [JobConfig(f"job{i}", [(17 * (i + 1) * (t + 3)) % 190 + 8 for t in range(6)], batch_size=bs[i],
                      rank=rank[i], lr=lr[i], scale=2.0, priority=prio[i], submit_time=submit[i], iterations=iters[i])
            for i in range(6)]


def f32_bits(v):
    return struct.unpack("<I", struct.pack("<f", v))[0]


@pytest.mark.parametrize("padded,strategy", [(False, "minpad"), (True, "minpad"), (False, "fifo")])
def test_cpp_executor_trace_matches_python_executor(padded, strategy):
    r = subprocess.run([_binary("executor_loop"), "1" if padded else "0", strategy], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    cpp, tail = lines[:-1], lines[-1]

    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200.executor import FusedExecutor
    from paper_2312_02515_b200.layer import TINY
    ctx = F.Context(0)
    ex = FusedExecutor(ctx, TINY, executor_jobs(), max_concurrent=3, strategy=strategy, padded=padded, seed=7,
                       pipelined=False)
    py = ex.run().events
    assert len(cpp) == len(py) > 0
    for c, p in zip(cpp, py):
        for key in ("total_tokens", "padding_tokens", "effective_tokens", "rows", "jobs_in_batch", "routing"):
            assert c[key] == p[key], (key, c, p)
        assert c["loss_bits"] == {k: f32_bits(v) for k, v in p["losses"].items()}, (c, p)
        assert c["duration_s"] > 0
    # every job ran to its iteration bound in both
    assert all(js.done == js.cfg.iterations for js in ex.jobs)
    # the IterationTimeModel fitted from the measured iterations (least squares, coefficients
    # >= 0) charges about their total time back; the first iteration carries the one-off
    # costs (kernel attributes, tensor maps), so the fit is loose, not exact
    fit = tail["fit"]
    assert fit["per_launch"] == 0.0 and fit["base"] >= 0.0 and fit["per_token"] >= 0.0
    charged = sum(fit["base"] + fit["per_token"] * e["total_tokens"] for e in cpp)
    assert 0.5 * tail["clock"] <= charged <= 1.5 * tail["clock"]
    # launches per fused iteration: the layer step's 22 fixed launches, plus one fixed-order
    # split reduce for each of the dA / dB groups whose token range is split (0-2 by rows),
    # plus the device fuse — independent of how many jobs are fused
    assert 23 * len(cpp) <= tail["launches"] <= 26 * len(cpp)


def test_facade_bf16_fused_forward_on_reference_golden():
    """fusim::b200::fused_forward_bf16 (tcgen05, bf16 operands, fp32 accumulation)
    on the reference's 66 golden instances (SURVEY.md §8c forward golden): per
    sequence, rel-L2 <= 1e-2 against the oracle's fused_forward (pinned to the
    reference) on the bf16-rounded inputs — the kernel's own error — and <= 5e-2
    against the reference's fp64 outputs on the raw inputs, whose extra error is
    the bf16 rounding of the inputs (the golden dims are <= 16, so a few outputs
    are small differences of rounded terms); pad rows exactly zero."""
    from oracle import mlora_oracle as O
    from oracle.golden import unpack_case

    def bf16(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).double().numpy()
    z = np.load(os.path.join(HERE, "golden", "lora_ref.npz"))
    keys = [str(k) for k in z["_index_forward"]]
    buf = [np.array([len(keys)], np.int32).tobytes()]
    shapes, rounded = [], []
    for key in keys:
        W0, ranks, As, Bs, seqs = unpack_case(z, key)
        d, k = W0.shape
        buf.append(np.array([d, k, len(ranks), *ranks, len(seqs), *[j for j, _ in seqs],
                             *[x.shape[0] for _, x in seqs]], np.int32).tobytes())
        buf += [np.ascontiguousarray(W0).tobytes(), z[key + "A_all"].tobytes(), z[key + "B_all"].tobytes(),
                z[key + "X_all"].tobytes()]
        shapes.append((d, [x.shape[0] for _, x in seqs]))
        fb = O.fuse([(j, [bf16(x)]) for j, x in seqs])
        rounded.append(O.fused_forward(bf16(W0), {j: (bf16(As[j]), bf16(Bs[j]), r) for j, r in enumerate(ranks)},
                                       fb))
    r = subprocess.run([_binary("facade_forward_io"), "--bf16"], input=b"".join(buf), capture_output=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr.decode()
    got = np.frombuffer(r.stdout, np.float64)
    off, worst, worst_raw = 0, 0.0, 0.0
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
    for key, (d, lens), want in zip(keys, shapes, rounded):
        ref_out = z[key + "out"].reshape(len(lens), -1, d)
        L = ref_out.shape[1]
        g = got[off:off + ref_out.size].reshape(ref_out.shape)
        off += ref_out.size
        for s, n in enumerate(lens):
            e, e_raw = rel(g[s, :n], want[s][:n]), rel(g[s, :n], ref_out[s, :n])
            worst, worst_raw = max(worst, e), max(worst_raw, e_raw)
            assert e <= 1e-2, (key, s, e)
            assert e_raw <= 5e-2, (key, s, e_raw)
            assert not g[s, n:L].any(), (key, s)  # pad rows come out zero
    assert off == got.size
    print(f"bf16 façade fused_forward over {len(keys)} golden instances: worst per-sequence rel-L2 {worst:.2e} "
          f"(bf16-rounded inputs), {worst_raw:.2e} (raw fp64 inputs)")
