"""Edge cases beyond the reference's own test sizes: adapters wider than one
64-column rank chunk (r = 96, 128, 200), many jobs in one plan (J = 96), and a
single job covering the whole batch with a 1-row tail tile."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import mlora_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


def run(seg, ranks, scales, d, k, seed):
    from paper_2312_02515_b200 import fused as F
    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    g = torch.Generator().manual_seed(seed)
    bf = lambda t: t.to(torch.bfloat16)
    M = seg[-1]
    X = bf(torch.rand(M, k, generator=g) * 2 - 1)
    dY = bf(torch.rand(M, d, generator=g) * 2 - 1)
    W0 = bf((torch.rand(d, k, generator=g) * 2 - 1) / k ** 0.5)
    As = [bf((torch.rand(r, k, generator=g) * 2 - 1) / k ** 0.5) for r in ranks]
    Bs = [bf((torch.rand(d, r, generator=g) * 2 - 1) / r ** 0.5) for r in ranks]
    plan = F.Plan(ctx, seg, ranks, scales)
    _, _, A16, B16 = F.pack_adapters(ctx, plan, d, k, [a.float().to(dev) for a in As], [b.float().to(dev) for b in Bs])
    Y, H = F.linear_fwd(ctx, plan, X.to(dev), W0.to(dev), A16, B16)
    dX, dA, dB = F.linear_bwd(ctx, plan, dY.to(dev), X.to(dev), H, W0.to(dev), A16, B16)
    torch.cuda.synchronize()
    f64 = lambda t: t.double().cpu().numpy()
    A64, B64 = [f64(a) for a in As], [f64(b) for b in Bs]
    Yr = O.segmented_forward(f64(X), f64(W0), A64, B64, scales, seg)
    dXr, dAr, dBr = O.segmented_backward(f64(dY), f64(X), f64(W0), A64, B64, scales, seg)
    rel = lambda a, b: np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30)
    assert rel(Y.float().cpu().numpy(), Yr) < 1e-2
    assert rel(dX.float().cpu().numpy(), dXr) < 1e-2
    ro = plan.rank_offsets
    for j, r in enumerate(ranks):
        if seg[j + 1] == seg[j]:
            continue
        assert rel(dA.cpu().numpy()[ro[j]:ro[j] + r], dAr[j]) < 1e-2
        assert rel(dB.cpu().numpy()[:, ro[j]:ro[j] + r], dBr[j]) < 1e-2
    return plan


def test_ranks_wider_than_a_chunk():
    plan = run([0, 200, 450, 700], [96, 128, 200], [1.0, 0.5, 2.0], 384, 512, seed=1)
    assert plan.rank_padded == 96 + 128 + 208


def test_many_jobs_one_plan():
    J = 96
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 40, J)
    seg = [0] + list(np.cumsum(lens))
    ranks = list(rng.choice([4, 8, 16], J))
    run([int(s) for s in seg], [int(r) for r in ranks], [1.0] * J, 256, 192, seed=2)


def test_single_job_with_one_row_tail():
    run([0, 257], [16], [2.0], 256, 256, seed=4)


def test_plan_at_the_job_limit_with_rank_64():
    """128 jobs (the per-plan limit) of rank 64: R_pad = 8192 columns, 128 rank
    chunks; every table sized by the job limit is exercised at its bound."""
    J = 128
    rng = np.random.default_rng(5)
    lens = rng.integers(1, 24, J)
    seg = [0] + [int(x) for x in np.cumsum(lens)]
    plan = run(seg, [64] * J, [1.0] * J, 128, 128, seed=6)
    assert plan.rank_padded == 64 * J


def test_plan_over_the_job_limit_is_a_usage_error():
    from paper_2312_02515_b200 import errors as E
    from paper_2312_02515_b200 import fused as F
    ctx = F.Context(0)
    with pytest.raises(E.UsageError):
        F.Plan(ctx, list(range(130)), [8] * 129)
