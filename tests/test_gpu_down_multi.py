"""The shared-input forward down-projection (csrc/mlora_down_multi.cuh): when
several projections read the same X, mlora_down_group computes all their
H_p = s_j X A_cat_p^T in one kernel.  Its output must be BITWISE equal to the
per-projection grouped kernel (same K split, same k order, same fixed-order
partial sum), and match the fp64 restatement.  Covers NB = 2..5, several tiles
per CTA pair (ring hand-back, TMEM reuse), several 64-column rank chunks, an
empty job, K not a multiple of 64, and K = 64 (one CTA of each pair has an
empty K half)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _down(F, N, ctx, plan, X, A16s, R, shared):
    """H for every adapter: one grouped call with a shared X (multi kernel), or one call each."""
    n = len(A16s)
    outs = [torch.empty(X.shape[0], R, dtype=torch.bfloat16, device=X.device) for _ in range(n)]
    s = torch.cuda.current_stream().cuda_stream
    calls = [list(range(n))] if shared else [[i] for i in range(n)]
    for idx in calls:
        m = len(idx)
        N.check(N.lib().mlora_down_group(ctx.handle, plan.handle, m, 0, (N.i32 * m)(*[X.shape[1]] * m),
                                         (N.vp * m)(*[X.data_ptr()] * m),
                                         (N.vp * m)(*[A16s[i].data_ptr() for i in idx]),
                                         (N.vp * m)(*[outs[i].data_ptr() for i in idx]), s), ctx.handle)
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("nb,seg,ranks,k", [
    (5, [0, 6999, 6999, 20000], [64, 32, 16], 200),   # 157 m-blocks, 2 rank chunks, empty job
    (4, [0, 100, 300], [16, 8], 64),                  # num_kb = 1
    (3, [0, 129, 130, 511], [8, 8, 24], 1000),
    (2, [0, 4096, 8192], [16, 16], 4096),
])
def test_shared_input_down_matches_grouped_bitwise(nb, seg, ranks, k):
    from paper_2312_02515_b200 import _native as N
    from paper_2312_02515_b200 import fused as F

    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    scales = [0.5 + j for j in range(len(ranks))]
    plan = F.Plan(ctx, seg, ranks, scales)
    R = plan.rank_padded
    g = torch.Generator().manual_seed(nb * 1000 + k)
    M = seg[-1]
    X = (torch.rand(M, k, generator=g) * 2 - 1).to(torch.bfloat16).to(dev)
    A16s, As = [], []
    for _ in range(nb):
        A = [((torch.rand(r, k, generator=g) * 2 - 1) / k ** 0.5) for r in ranks]
        B = [torch.zeros(64, r) for r in ranks]
        _, _, A16, _ = F.pack_adapters(ctx, plan, 64, k, [a.to(dev) for a in A], [b.to(dev) for b in B])
        A16s.append(A16)
        As.append(A)
    multi = _down(F, N, ctx, plan, X, A16s, R, shared=True)
    single = _down(F, N, ctx, plan, X, A16s, R, shared=False)
    for p in range(nb):
        assert torch.equal(multi[p], single[p]), f"projection {p} differs from the grouped kernel"
    # and against fp64: H[t, roff_j : roff_j + r_j] = s_j x_t A_j^T, zero elsewhere
    ro = plan.rank_offsets
    Xd = X.double().cpu().numpy()
    for p in range(nb):
        want = np.zeros((M, R))
        for j, r in enumerate(ranks):
            a16 = A16s[p][ro[j]:ro[j] + r].double().cpu().numpy()
            want[seg[j]:seg[j + 1], ro[j]:ro[j] + r] = scales[j] * Xd[seg[j]:seg[j + 1]] @ a16.T
        got = multi[p].double().cpu().numpy()
        assert np.array_equal(got == 0, want == 0) or np.all(got[want == 0] == 0)  # block-diagonal zeros exact
        err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
        assert err < 1e-2, (p, err)


def test_shared_input_down_random_layouts_bitwise():
    """24 random layouts (1-10 jobs, ranks 1-64, empty / 1-row / straddling segments, K
    tails, NB 2-5): the rank-group narrowing of both the shared-input and the grouped
    kernel must agree bitwise and be exactly zero off the block diagonal."""
    from paper_2312_02515_b200 import _native as N
    from paper_2312_02515_b200 import fused as F

    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    rng = np.random.default_rng(2024)
    for case in range(24):
        J = int(rng.integers(1, 11))
        ranks = [int(rng.integers(1, 65)) for _ in range(J)]
        lens = [int(rng.choice([0, 1, int(rng.integers(2, 400))])) for _ in range(J)]
        if sum(lens) == 0:
            lens[0] = 37
        seg = [0]
        for n in lens:
            seg.append(seg[-1] + n)
        k = int(rng.choice([64, 200, 1000]))
        nb = int(rng.integers(2, 6))
        scales = [float(rng.uniform(0.25, 2.0)) for _ in range(J)]
        plan = F.Plan(ctx, seg, ranks, scales)
        R = plan.rank_padded
        g = torch.Generator().manual_seed(case)
        M = seg[-1]
        X = (torch.rand(M, k, generator=g) * 2 - 1).to(torch.bfloat16).to(dev)
        A16s = []
        for _ in range(nb):
            A = [((torch.rand(r, k, generator=g) * 2 - 1) / k ** 0.5) for r in ranks]
            B = [torch.zeros(64, r) for r in ranks]
            _, _, A16, _ = F.pack_adapters(ctx, plan, 64, k, [a.to(dev) for a in A], [b.to(dev) for b in B])
            A16s.append(A16)
        multi = _down(F, N, ctx, plan, X, A16s, R, shared=True)
        single = _down(F, N, ctx, plan, X, A16s, R, shared=False)
        ro = plan.rank_offsets
        for p in range(nb):
            assert torch.equal(multi[p], single[p]), (case, p, seg, ranks)
            mask = torch.zeros(M, R, dtype=torch.bool)
            for j in range(J):
                mask[seg[j]:seg[j + 1], ro[j]:ro[j] + ranks[j]] = True
            assert torch.all(multi[p].cpu()[~mask] == 0), (case, p)
            Xd = X.double().cpu().numpy()
            want = np.zeros((M, R))
            for j, r in enumerate(ranks):
                a16 = A16s[p][ro[j]:ro[j] + r].double().cpu().numpy()
                want[seg[j]:seg[j + 1], ro[j]:ro[j] + r] = scales[j] * Xd[seg[j]:seg[j + 1]] @ a16.T
            got = multi[p].double().cpu().numpy()
            err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
            assert err < 1e-2, (case, p, err)
