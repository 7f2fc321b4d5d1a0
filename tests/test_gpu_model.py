"""K4 / K5 model kernels vs fp64 numpy restatements (parity unpinned by the
reference, which has no model arithmetic).  Tolerances are stated per check."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def bf16_np(t):
    return t.float().cpu().double().numpy()


def _check_masked_ce(V, seg, seed=0):
    from paper_2312_02515_b200 import model_ops as M
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(seed)
    rows = seg[-1]
    logits = (torch.randn(rows, V, generator=g) * 3).to(torch.bfloat16)
    labels = torch.randint(0, V, (rows,), generator=g, dtype=torch.int32)
    mask = (torch.rand(rows, generator=g) > 0.25).to(torch.uint8)
    loss, dl = M.masked_ce(logits.to(dev), labels.to(dev), seg, mask.to(dev))
    loss2, dl2 = M.masked_ce(logits.to(dev), labels.to(dev), seg, mask.to(dev))
    torch.cuda.synchronize()
    assert torch.equal(loss, loss2) and torch.equal(dl, dl2)  # deterministic
    L = bf16_np(logits)
    mx = L.max(1, keepdims=True)
    lse = (mx + np.log(np.exp(L - mx).sum(1, keepdims=True)))[:, 0]
    row = lse - L[np.arange(rows), labels.numpy()]
    m = mask.numpy().astype(bool)
    for j in range(len(seg) - 1):
        sel = m[seg[j]:seg[j + 1]]
        want = row[seg[j]:seg[j + 1]][sel].mean() if sel.any() else 0.0
        assert abs(loss[j].item() - want) <= 1e-3 * max(1.0, abs(want))  # losses within 1e-3 (north star)
    P = np.exp(L - lse[:, None])
    P[np.arange(rows), labels.numpy()] -= 1.0
    cnt = np.zeros(rows)
    for j in range(len(seg) - 1):
        cnt[seg[j]:seg[j + 1]] = max(1, m[seg[j]:seg[j + 1]].sum())
    want_dl = P / cnt[:, None] * m[:, None]
    got = bf16_np(dl)
    assert np.all(got[~m] == 0)
    assert np.linalg.norm(got - want_dl) / np.linalg.norm(want_dl) < 1e-2


def test_masked_ce_per_job_mean_and_grad_c4_vocab():
    """ChatGLM2 vocabulary (V = 65024), padded fused batch with pad rows masked."""
    _check_masked_ce(65024, [0, 40, 40, 100, 128])


@pytest.mark.parametrize("V", [8, 32, 40, 1000, 32000, 1001, 70000, 75776])
def test_masked_ce_vocab_sizes(V):
    """Cluster row pass (V % 8 == 0, 32 <= V <= 74 K: 32, 40, 1000, LLaMA's 32000, 70000),
    the one-row-per-CTA vector pass (8, 75776 > 74 K) and the scalar
    path (1001: V % 8 != 0)."""
    _check_masked_ce(V, [0, 17, 17, 50, 64], seed=V)


def test_rmsnorm_fwd_bwd():
    from paper_2312_02515_b200 import model_ops as M
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(1)
    rows, h, eps = 300, 4096, 1e-6
    x = torch.randn(rows, h, generator=g).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(h, generator=g)).to(torch.bfloat16)
    dy = torch.randn(rows, h, generator=g).to(torch.bfloat16)
    y, rstd = M.rmsnorm_fwd(x.to(dev), w.to(dev), eps)
    dx, dw = M.rmsnorm_bwd(dy.to(dev), x.to(dev), w.to(dev), rstd, rows_per_block=32)
    torch.cuda.synchronize()
    X, W, DY = bf16_np(x), bf16_np(w), bf16_np(dy)
    r = 1 / np.sqrt((X * X).mean(1) + eps)
    Y = X * r[:, None] * W
    xh = X * r[:, None]
    G = DY * W
    DX = r[:, None] * (G - xh * (G * xh).mean(1, keepdims=True))
    DW = (DY * xh).sum(0)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert np.allclose(rstd.cpu().numpy(), r, rtol=1e-4)
    assert rel(bf16_np(y), Y) < 1e-2
    assert rel(bf16_np(dx), DX) < 1e-2
    assert rel(dw.cpu().numpy(), DW) < 1e-4
    # deterministic
    dx2, dw2 = M.rmsnorm_bwd(dy.to(dev), x.to(dev), w.to(dev), rstd, rows_per_block=32)
    assert torch.equal(dw, dw2) and torch.equal(dx, dx2)


def test_rope_roundtrip_and_reference():
    from paper_2312_02515_b200 import model_ops as M
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(2)
    rows, heads, hd = 257, 8, 128
    x = torch.randn(rows, heads, hd, generator=g).to(torch.bfloat16)
    pos = torch.randint(0, 4096, (rows,), generator=g, dtype=torch.int32)
    y = M.rope(x.to(dev), pos.to(dev))
    back = M.rope(y, pos.to(dev), inverse=True)
    torch.cuda.synchronize()
    X = bf16_np(x)
    half = hd // 2
    inv = 10000.0 ** (-2 * np.arange(half) / hd)
    ang = pos.numpy()[:, None].astype(np.float64) * inv[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    a, b = X[..., :half], X[..., half:]
    Y = np.concatenate([a * c - b * s, b * c + a * s], -1)
    rel = lambda p, q: np.linalg.norm(p - q) / np.linalg.norm(q)
    assert rel(bf16_np(y), Y) < 1e-2
    assert rel(bf16_np(back), X) < 1e-2  # rotation is orthogonal: backward = inverse rotation


def test_masked_ce_many_rows_per_cta_pair():
    """Several rows per CTA pair of the bulk-copy row pass (double-buffered half rows,
    pad rows interleaved so the two slots' load counts drift apart) and an empty job."""
    _check_masked_ce(4096, [0, 700, 700, 1500, 2000], seed=11)
