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
        # candidates carry the real job ids: the reference's tie-breaks compare them
        cands = [O.BatchCandidate(jobs[i].id, O.next_candidate_batch(jobs[i].lengths, cursors[i], jobs[i].batch_size),
                                  jobs[i].priority, jobs[i].submit_time) for i in live]
        want = O.select_minpad(cands, 3)
        pos = {jobs[i].id: n for n, i in enumerate(live)}
        chosen = [live[pos[c]] for c in want.chosen]
        before = {j: (ex.layer.proj[0].A.p.clone(), ex.layer.proj[0].A.m.clone()) for j in range(len(jobs))}
        ev = ex.step()
        assert ev["routing"] == [jobs[i].id for i in chosen]
        shape = O.fused_shape([cands[pos[c]].item_lengths for c in want.chosen])
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


@pytest.mark.parametrize("pipelined", [False, True])
def test_executor_early_stopping_on_real_losses(pipelined, tmp_path):
    """detect_stop (progress.cpp:90-124) on the device's real per-job losses: a
    job driven to overflow by a huge learning rate stops on its first
    non-finite loss, a job whose accuracy stream declines stops after
    `patience` evaluations, and both leave the fused batch while the others
    train to completion."""
    from paper_2312_02515_b200 import executor as X
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200.layer import TINY

    ctx = F.Context(0)
    jobs = [X.JobConfig(id=f"job{j}", lengths=[24, 40, 16, 32], batch_size=2, rank=8,
                        lr=(1e30 if j == 1 else 1e-3), submit_time=float(j), iterations=7) for j in range(4)]
    acc = lambda job, it, loss: 1.0 / it if job == "job2" else float(it)  # noqa: E731
    ex = X.FusedExecutor(ctx, TINY, jobs, max_concurrent=4, seed=11, pipelined=pipelined,
                         early_stopping=True, patience=2, accuracy_fn=acc, checkpoint_dir=str(tmp_path))
    trace = ex.run()
    # every job's adapter was checkpointed once, when it completed or stopped
    saved = {c["job"]: c for c in trace.checkpoints}
    assert set(saved) == {j.id for j in jobs}
    assert saved["job0"]["cause"] == "completed" and saved["job0"]["iterations"] == 7
    assert saved["job2"]["cause"] == "accuracy_decline"
    assert all((tmp_path / f"{j.id}.pt").exists() for j in jobs)
    stops = {s["job"]: s for s in trace.stops}
    assert set(stops) == {"job1", "job2"}, trace.stops
    assert stops["job1"]["cause"] == "nan_loss" and stops["job2"]["cause"] == "accuracy_decline"
    assert stops["job2"]["iteration"] == 3  # accuracies 1, 1/2, 1/3 with patience 2
    losses = {j.id: [e["losses"][j.id] for e in trace.events if j.id in e["losses"]] for j in jobs}
    assert X.detect_stop(losses["job1"]) == (stops["job1"]["iteration"], "nan_loss")
    assert all(math.isfinite(v) for v in losses["job0"] + losses["job3"])
    lag = 1 if pipelined else 0  # pipelined: the stop is seen while the next step is queued
    for jid in ("job1", "job2"):
        ran = sum(1 for e in trace.events if jid in e["routing"])
        assert ran == stops[jid]["iteration"] + lag, (jid, ran, stops[jid])
    for jid in ("job0", "job3"):
        assert sum(1 for e in trace.events if jid in e["routing"]) == 7
    r = ex.layer.plan.rank_offsets
    for p in ex.layer.proj:  # the surviving jobs' adapters never saw the diverged one
        for j in (0, 3):
            assert torch.isfinite(p.A.p[r[j]:r[j + 1]]).all() and torch.isfinite(p.B.p[:, r[j]:r[j + 1]]).all()


def test_quarantined_nan_adapter_cannot_reach_other_jobs():
    """A job whose adapter went NaN and was retired (quarantined, absent from
    the batch) leaves every output of the other jobs bitwise identical to a run
    where it never diverged — Y, per-job loss, dX, dA, dB."""
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200.layer import TINY, FusedLoraLayer

    ctx = F.Context(0)
    seg = [0, 96, 96, 200]  # job 1 absent from this batch
    outs = []
    for poison in (False, True):
        layer = FusedLoraLayer(ctx, TINY, [8, 8, 16], [2.0] * 3, [1e-3] * 3, rows=200, seed=21)
        layer.set_layout(seg)
        if poison:
            r = layer.plan.rank_offsets
            for p in layer.proj:
                p.A.p_bf16[r[1]:r[2]] = float("nan")
                p.B.p_bf16[:, r[1]:r[2]] = float("nan")
            layer.quarantine(1)
        x = torch.Generator(device="cpu").manual_seed(4)
        x = (torch.rand(200, TINY[0][2], generator=x) * 2 - 1).to(torch.bfloat16).cuda()
        loss = layer.forward_backward(x).clone()
        torch.cuda.synchronize()
        outs.append((loss, [(p.Y[:200].clone(), p.dX[:200].clone(), p.dA.clone(), p.dB.clone()) for p in layer.proj],
                     layer.plan.rank_offsets))
    (l0, t0, r), (l1, t1, _) = outs
    assert torch.equal(l0[[0, 2]], l1[[0, 2]])
    keep = [c for j in (0, 2) for c in range(r[j], r[j + 1])]
    for (y0, dx0, da0, db0), (y1, dx1, da1, db1) in zip(t0, t1):
        assert torch.equal(y0, y1) and torch.equal(dx0, dx1)
        assert torch.equal(da0[keep], da1[keep]) and torch.equal(db0[:, keep], db1[:, keep])


def test_diverged_job_leaves_other_jobs_bitwise_unchanged():
    """Without early stopping: a job driven to overflow (lr 1e30) reports a
    non-finite loss every step from its divergence on, while every other job's
    per-step loss is bitwise identical to a run in which it never diverged —
    the per-job independence of the reference (lora.cpp:168-181 computes every
    sequence with its own adapter), kept by mlora_zero_nonfinite_rows."""
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200.layer import TINY, FusedLoraLayer

    ctx = F.Context(0)
    seg = [0, 72, 144, 216, 288]
    runs = []
    for lr1 in (1e-3, 1e30):
        layer = FusedLoraLayer(ctx, TINY, [8] * 4, [2.0] * 4, [1e-3, lr1, 1e-3, 1e-3], rows=288, seed=11)
        layer.set_layout(seg)
        g = torch.Generator(device="cpu").manual_seed(3)
        losses = []
        for _ in range(5):
            x = ((torch.rand(288, TINY[0][2], generator=g) * 2 - 1).to(torch.bfloat16)).cuda()
            losses.append(layer.step(x).clone())
        torch.cuda.synchronize()
        runs.append(torch.stack(losses).cpu())
    calm, wild = runs
    assert torch.isfinite(calm).all()
    assert not torch.isfinite(wild[1:, 1]).any()            # diverged from step 2 on
    assert torch.equal(calm[:, [0, 2, 3]], wild[:, [0, 2, 3]])  # the others never noticed


def test_adapter_checkpoint_resume_is_exact(tmp_path):
    """Save every job after 3 steps, resume into a freshly initialised layer and
    continue: the next steps' per-job losses are bitwise those of the
    uninterrupted run (masters, AdamW moments and step counts all restored).
    Checkpoints are per job in the reference layout (A_j r x k, B_j d x r)."""
    from paper_2312_02515_b200 import errors as E
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200.layer import TINY, FusedLoraLayer

    ctx = F.Context(0)
    seg = [0, 100, 100, 256]  # job 1 absent: its slot must round-trip untouched too
    mk = lambda seed, W0=None: FusedLoraLayer(ctx, TINY, [8, 16, 8], [2.0, 1.0, 0.5],  # noqa: E731
                                              [1e-2, 5e-3, 2e-2], rows=256, seed=seed, W0=W0)
    g = torch.Generator().manual_seed(8)
    xs = [((torch.rand(256, 256, generator=g) * 2 - 1).to(torch.bfloat16)).cuda() for _ in range(5)]
    a = mk(1)
    a.set_layout(seg)
    for x in xs[:3]:
        a.step(x)
    paths = [str(tmp_path / f"job{j}.pt") for j in range(3)]
    for j in range(3):
        a.save_job(paths[j], j)
    want = [a.step(x).clone() for x in xs[3:]]
    b = mk(99, W0={p.name: p.W0 for p in a.proj})  # same frozen base, different initial adapters
    b.set_layout(seg)
    for j in range(3):
        b.load_job(paths[j], j)
    got = [b.step(x).clone() for x in xs[3:]]
    torch.cuda.synchronize()
    assert all(torch.equal(w, g_) for w, g_ in zip(want, got))
    st = torch.load(paths[1])
    assert tuple(st["proj"]["q"]["A"].shape) == (16, 256) and tuple(st["proj"]["q"]["B"].shape) == (256, 16)
    with pytest.raises(E.UsageError):
        b.load_job(paths[0], 1)  # rank 8 checkpoint into a rank-16 slot
    with pytest.raises(E.UsageError):
        b.load_job(paths[2], 0)  # same rank, different scale


# ---------------------------------------------------------------- decoder backend (real CE losses)
@pytest.mark.parametrize("padded", [False, True])
def test_decoder_executor_selection_accounting_and_ce(padded):
    """model=TINY_LLAMA: the same MinPad selection / ξ accounting as the layer
    backend, and the per-job losses the executor reports are the decoder's
    padding-masked CE (≈ ln V on the first visit, falling on revisits)."""
    from paper_2312_02515_b200 import executor as X
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200 import model as MD
    from paper_2312_02515_b200 import packer

    ctx = F.Context(0)
    jobs = make_jobs(X, packer)
    for j in jobs:
        j.iterations = 12
        j.lr = 5e-3
    ex = X.FusedExecutor(ctx, None, jobs, max_concurrent=3, strategy="minpad", padded=padded, seed=5,
                         pipelined=True, model=MD.TINY_LLAMA)
    cursors = [0] * len(jobs)
    done = [0] * len(jobs)
    evs = []
    while True:
        live = [i for i in range(len(jobs)) if done[i] < jobs[i].iterations]
        if not live:
            break
        cands = [O.BatchCandidate(f"c{n}", O.next_candidate_batch(jobs[i].lengths, cursors[i], jobs[i].batch_size),
                                  jobs[i].priority, jobs[i].submit_time) for n, i in enumerate(live)]
        want = O.select_minpad(cands, 3)
        chosen = [live[int(c[1:])] for c in want.chosen]
        shape = O.fused_shape([c.item_lengths for c in (cands[int(c[1:])] for c in want.chosen)])
        evs.append(([jobs[i].id for i in chosen], shape.total_tokens, shape.padding_tokens))
        ex.step()
        for i in chosen:
            b = O.next_candidate_batch(jobs[i].lengths, cursors[i], jobs[i].batch_size)
            cursors[i] = O.commit_batch(cursors[i], len(b), len(jobs[i].lengths))
            done[i] += 1
    ex.flush()
    got = [(e["routing"], e["total_tokens"], e["padding_tokens"]) for e in ex.trace.events]
    assert got == evs
    ln_v = math.log(MD.TINY_LLAMA.vocab)
    for e in ex.trace.events:
        assert all(math.isfinite(v) and 0 < v < 3 * ln_v for v in e["losses"].values())
    # each job's dataset repeats every epoch: its CE on a revisited item has fallen
    js = ex.jobs[0]
    assert js.losses[-1] < js.losses[0] - 0.1, js.losses


def test_decoder_diverged_job_is_isolated_and_stopped():
    """A job at lr 1e30 diverges (non-finite CE); AdamW's loss gate keeps its
    adapter finite, so every other job's CE stays bitwise identical to a run in
    which it trains normally; the executor stops it with nan_loss."""
    from paper_2312_02515_b200 import executor as X
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200 import model as MD

    ctx = F.Context(0)
    g = torch.Generator().manual_seed(3)
    seqs = [[torch.randint(0, 1024, (n,), generator=g).tolist() for n in (40, 17)] for _ in range(3)]
    batch = MD.pack_tokens(seqs)
    runs = []
    for lr1 in (1e-3, 1e30):
        m = MD.MultiLoraDecoder(ctx, MD.TINY_LLAMA, [8, 16, 8], [2.0] * 3, [1e-3, lr1, 2e-3],
                                capacity=batch.rows, seed=12)
        runs.append([m.step(batch).clone() for _ in range(4)])
    torch.cuda.synchronize()
    assert not math.isfinite(runs[1][-1][1].item())
    for a, b in zip(*runs):
        assert torch.equal(a[0], b[0]) and torch.equal(a[2], b[2])
    # through the executor: the diverged job is stopped on its CE, the others finish
    jobs = [X.JobConfig(id=f"j{i}", lengths=[24, 31, 9, 40], batch_size=2, rank=8, lr=lr, iterations=6)
            for i, lr in enumerate([2e-3, 1e30, 1e-3])]
    ex = X.FusedExecutor(ctx, None, jobs, max_concurrent=3, early_stopping=True, model=MD.TINY_LLAMA,
                         pipelined=False, seed=2)
    tr = ex.run()
    assert [s["job"] for s in tr.stops] == ["j1"] and tr.stops[0]["cause"] == "nan_loss"
    assert ex.jobs[0].done == 6 and ex.jobs[2].done == 6
    assert all(math.isfinite(v) for v in ex.jobs[0].losses + ex.jobs[2].losses)


def test_decoder_checkpoint_resume_is_exact(tmp_path):
    """Decoder jobs saved after 3 steps and resumed into a fresh decoder on the
    same frozen base continue with bitwise-identical per-job CE (every layer's
    adapters, AdamW moments and step counts restored; keys 'layer.proj')."""
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200 import model as MD

    ctx = F.Context(0)
    g = torch.Generator().manual_seed(21)
    seqs = [[torch.randint(0, 1024, (n,), generator=g).tolist() for n in ns] for ns in ([30, 12], [], [50])]
    batch = MD.pack_tokens(seqs)
    a = MD.MultiLoraDecoder(ctx, MD.TINY_CHATGLM2, [8, 16, 8], [2.0, 1.0, 0.5], [1e-2, 5e-3, 2e-2],
                            capacity=batch.rows, seed=5)
    for _ in range(3):
        a.step(batch)
    paths = [str(tmp_path / f"job{j}.pt") for j in range(3)]
    for j in range(3):
        a.save_job(paths[j], j)
    want = [a.step(batch).clone() for _ in range(2)]
    b = MD.MultiLoraDecoder(ctx, MD.TINY_CHATGLM2, [8, 16, 8], [2.0, 1.0, 0.5], [1e-2, 5e-3, 2e-2],
                            capacity=batch.rows, seed=77, frozen=a)
    for j in range(3):
        b.load_job(paths[j], j)
    got = [b.step(batch).clone() for _ in range(2)]
    torch.cuda.synchronize()
    assert all(torch.equal(w, g_) for w, g_ in zip(want, got))
    assert "1.h_to_4h" in torch.load(paths[0])["proj"]
