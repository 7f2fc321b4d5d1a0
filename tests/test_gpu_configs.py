"""Parity at the shapes of BASELINE.json's other configs (they are parity cases,
not bench lines):

C3 — LLaMA-13B-shaped projections, 8 jobs with heterogeneous ranks
     {8,16,32,64}x2, NormalTruncated sequence lengths with per-job means, MinPad
     choosing 4 of the 8 (so 4 adapters have empty row segments; R_pad = 256 →
     4 rank chunks).
C4 — ChatGLM2-6B shapes (multi-query attention: fused qkv 4096 → 4608; 4h → h
     13696 → 4096), 6 jobs, the reference's padded layout (pad rows zero).
Y / dX on sampled rows, dA / dB in full, against the fp64 oracle (rel-L2 1e-2).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import mlora_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def run_and_check(seg, ranks, scales, d, k, seed, rows_mask=None, nsample=192):
    from paper_2312_02515_b200 import fused as F
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    g = torch.Generator().manual_seed(seed)
    M = seg[-1]
    bf = lambda t: t.to(torch.bfloat16)
    X = bf(torch.rand(M, k, generator=g) * 2 - 1)
    dY = bf(torch.rand(M, d, generator=g) * 2 - 1)
    if rows_mask is not None:
        X[~rows_mask] = 0
        dY[~rows_mask] = 0
    W0 = bf((torch.rand(d, k, generator=g) * 2 - 1) / k ** 0.5)
    As = [bf((torch.rand(r, k, generator=g) * 2 - 1) / k ** 0.5) for r in ranks]
    Bs = [bf((torch.rand(d, r, generator=g) * 2 - 1) / r ** 0.5) for r in ranks]
    plan = F.Plan(ctx, seg, ranks, scales)
    _, _, A16, B16 = F.pack_adapters(ctx, plan, d, k, [a.float().to(dev) for a in As], [b.float().to(dev) for b in Bs])
    Y, H = F.linear_fwd(ctx, plan, X.to(dev), W0.to(dev), A16, B16)
    dX, dA, dB = F.linear_bwd(ctx, plan, dY.to(dev), X.to(dev), H, W0.to(dev), A16, B16)
    torch.cuda.synchronize()
    f64 = lambda t: t.double().cpu().numpy()
    Xn, Wn, dYn = f64(X), f64(W0), f64(dY)
    A64, B64 = [f64(a) for a in As], [f64(b) for b in Bs]
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(M, min(nsample, M), replace=False))
    job = np.searchsorted(seg, rows, side="right") - 1
    Yr, dXr = Xn[rows] @ Wn.T, dYn[rows] @ Wn
    for j in range(len(ranks)):
        sel = job == j
        if sel.any():
            Yr[sel] += scales[j] * (Xn[rows[sel]] @ A64[j].T) @ B64[j].T
            dXr[sel] += scales[j] * (dYn[rows[sel]] @ B64[j]) @ A64[j]
    assert rel(Y.float().cpu().numpy()[rows], Yr) < TOL
    assert rel(dX.float().cpu().numpy()[rows], dXr) < TOL
    ro = plan.rank_offsets
    dAn, dBn = dA.cpu().numpy(), dB.cpu().numpy()
    for j, r in enumerate(ranks):
        a, b = seg[j], seg[j + 1]
        gA, gB = dAn[ro[j]:ro[j] + r], dBn[:, ro[j]:ro[j] + r]
        if b == a:
            assert not gA.any() and not gB.any()   # jobs outside the fused batch get exactly zero
            continue
        G = scales[j] * dYn[a:b] @ B64[j]
        assert rel(gA, G.T @ Xn[a:b]) < TOL
        assert rel(gB, scales[j] * dYn[a:b].T @ (Xn[a:b] @ A64[j].T)) < TOL
    return plan


@pytest.mark.parametrize("proj", [("q", 5120, 5120), ("gate", 13824, 5120), ("down", 5120, 13824)])
def test_c3_llama13b_heterogeneous_ranks_minpad(proj):
    from paper_2312_02515_b200 import packer as P
    ranks = [8, 16, 32, 64] * 2
    means = [64, 128, 256, 512, 1024, 96, 192, 384]
    cands = []
    for j in range(8):
        lens = P.sample_lengths("normal", 4, seed=1000 + j, min_len=32, max_len=1024, mean=means[j], stddev=96.0)
        cands.append(P.Candidate(j, lens, priority=1 + j % 3, submit_time=float(j)))
    sel = P.select(cands, 4, "minpad")
    # the packer's choice is the reference's (oracle restatement, itself pinned to the reference)
    want = O.select_minpad([O.BatchCandidate(f"c{i}", c.lengths, c.priority, c.submit_time)
                            for i, c in enumerate(cands)], 4)
    assert sel.chosen == [int(c[1:]) for c in want.chosen] and sel.padding_tokens == want.padding_tokens
    chosen = set(sel.chosen)
    lay = P.layout([cands[j].lengths for j in range(8) if j in chosen], padded=False)
    seg, r, it = [0], 0, iter(lay.seg[1:])
    for j in range(8):
        if j in chosen:
            r = next(it)
        seg.append(r)
    _, d, k = proj
    plan = run_and_check(seg, ranks, [2.0] * 8, d, k, seed={"q": 1, "gate": 2, "down": 3}[proj[0]])
    assert plan.rank_padded == 256


@pytest.mark.parametrize("proj", [("qkv", 4608, 4096), ("4h_to_h", 4096, 13696)])
def test_c4_chatglm2_padded_layout(proj):
    from paper_2312_02515_b200 import packer as P
    per_job = [P.sample_lengths("uniform", 2, seed=50 + j, min_len=64, max_len=300) for j in range(6)]
    lay = P.layout(per_job, padded=True)
    mask = torch.zeros(lay.rows, dtype=torch.bool)
    for rows in lay.seq_rows:
        for r0, L in rows:
            mask[r0:r0 + L] = True
    fb_shape = O.fused_shape(per_job)
    assert (lay.total_tokens, lay.padding_tokens) == (fb_shape.total_tokens, fb_shape.padding_tokens)
    _, d, k = proj
    run_and_check(lay.seg, [16] * 6, [2.0] * 6, d, k, seed=7, rows_mask=mask)
