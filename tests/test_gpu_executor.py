"""The executor behind the simulator's fused iteration, on the device: its
selection / accounting replays exactly with the oracle (reference semantics),
jobs left out of a fused batch are untouched by the optimizer, and the metrics
follow the reference's compute_metrics definitions."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import mlora_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


def make_jobs(executor_mod, packer):
    jobs = []
    ranks = [8, 16, 32, 8, 16, 4]
    for j in range(6):
        lengths = packer.sample_lengths("normal", 12, seed=100 + j, min_len=4, max_len=96, mean=16 + 12 * j,
                                        stddev=8.0)
        jobs.append(executor_mod.JobConfig(id=f"job{j}", lengths=lengths, batch_size=2 + j % 3, rank=ranks[j],
                                           lr=1e-3 * (1 + j), priority=1 + j % 2, submit_time=float(j),
                                           iterations=4))
    return jobs


@pytest.mark.parametrize("padded", [False, True])
def test_executor_replays_reference_selection(padded):
    from paper_2312_02515_b200 import executor as X
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200 import packer
    from paper_2312_02515_b200.layer import TINY

    ctx = F.Context(0)
    jobs = make_jobs(X, packer)
    ex = X.FusedExecutor(ctx, TINY, jobs, max_concurrent=3, strategy="minpad", padded=padded, seed=3,
                         pipelined=False)
    # oracle replay state
    cursors = [0] * len(jobs)
    done = [0] * len(jobs)
    while True:
        live = [i for i in range(len(jobs)) if done[i] < jobs[i].iterations]
        if not live:
            assert ex.step() is None
            break
        cands = [O.BatchCandidate(f"c{n}", O.next_candidate_batch(jobs[i].lengths, cursors[i], jobs[i].batch_size),
                                  jobs[i].priority, jobs[i].submit_time) for n, i in enumerate(live)]
        want = O.select_minpad(cands, 3)
        chosen = [live[int(c[1:])] for c in want.chosen]
        before = {j: (ex.layer.proj[0].A.p.clone(), ex.layer.proj[0].A.m.clone()) for j in range(len(jobs))}
        ev = ex.step()
        assert ev["routing"] == [jobs[i].id for i in chosen]
        shape = O.fused_shape([c.item_lengths for c in (cands[int(c[1:])] for c in want.chosen)])
        assert (ev["total_tokens"], ev["padding_tokens"]) == (shape.total_tokens, shape.padding_tokens)
        assert ev["effective_tokens"] == shape.total_tokens - shape.padding_tokens
        assert ev["rows"] == (shape.total_tokens if padded else ev["effective_tokens"])
        assert all(math.isfinite(v) for v in ev["losses"].values())
        # AdamW left every job outside the batch untouched (rows of A_cat owned by the job)
        ro = ex.layer.plan.rank_offsets
        for j in range(len(jobs)):
            p0, m0 = before[j]
            same = torch.equal(ex.layer.proj[0].A.p[ro[j]:ro[j + 1]], p0[ro[j]:ro[j + 1]]) and \
                torch.equal(ex.layer.proj[0].A.m[ro[j]:ro[j + 1]], m0[ro[j]:ro[j + 1]])
            assert same == (j not in chosen), (j, chosen)
        for i in chosen:
            b = O.next_candidate_batch(jobs[i].lengths, cursors[i], jobs[i].batch_size)
            cursors[i] = O.commit_batch(cursors[i], len(b), len(jobs[i].lengths))
            done[i] += 1
    m = ex.trace.metrics()
    xi = sum(e["total_tokens"] for e in ex.trace.events)
    xi_p = sum(e["padding_tokens"] for e in ex.trace.events)
    assert m["delta"] == pytest.approx(xi_p / xi)
    assert m["T_e"] == pytest.approx((1 - m["delta"]) * xi / m["busy_time_s"])
    assert m["iterations"] == len(ex.trace.events) and m["effective_tokens"] == xi - xi_p
    assert np.isfinite(m["effective_tokens_per_s"]) and m["effective_tokens_per_s"] > 0


def test_pipelined_executor_matches_synchronous():
    """Pipelined host packing (step t+1 selected and enqueued while step t runs,
    plan updates stream-ordered) yields the identical trace: same selections and
    accounting, bitwise-identical per-job losses."""
    from paper_2312_02515_b200 import executor as X
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200 import packer
    from paper_2312_02515_b200.layer import TINY

    ctx = F.Context(0)
    traces = []
    for pipelined in (False, True):
        ex = X.FusedExecutor(ctx, TINY, make_jobs(X, packer), max_concurrent=3, strategy="minpad", seed=9,
                             pipelined=pipelined)
        traces.append(ex.run())
    a, b = traces
    assert len(a.events) == len(b.events) > 0
    for ea, eb in zip(a.events, b.events):
        for key in ("total_tokens", "padding_tokens", "effective_tokens", "rows", "routing"):
            assert ea[key] == eb[key]
        assert ea["losses"] == eb["losses"]
