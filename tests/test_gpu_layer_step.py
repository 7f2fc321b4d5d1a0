"""The benchmarked step itself, end to end, against the oracle.

bench.py times FusedLoraLayer.step at C2: the seven LLaMA-7B projections of a
layer over 8192 fused rows (4 jobs x r16, s = 2, four learning rates), i.e. the
shared-input down-projection over x (q, k, v, gate, up: mlora_down_multi_kernel
with NB = 5), the grouped o / down down-projection, seven forward base GEMMs
with the fused row-sum loss, the per-job loss fused with the non-finite guard,
the 7-problem G group, seven dX GEMMs, the grouped dA / dB reductions (balanced
persistent grids; a token split + fixed-order reduce only when a group has fewer
tiles than SMs, as in the TINY edge case below) and one AdamW.  These tests run exactly that step once and check
every output it produces:

  * Y and dX of every projection on sampled rows, against the fp64 oracle
    (O.segmented_forward / O.segmented_backward: the reference's fused_forward,
    lora.cpp:160-182, and the composed-primitive backward of SURVEY.md §8c),
    chained through the layer's wiring (o <- v's Y, down <- up's Y; dY_p = Y_p
    for the loss L_j = 1/2 sum_p ||Y_p[rows of j]||^2);
  * dA_j, dB_j of every projection and job in full, against the oracle;
  * the per-job loss against 1/2 sum ||Y||^2 of a full-size fp32 PyTorch
    restatement of every projection (relative 1e-3);
  * the post-AdamW fp32 adapters against a numpy AdamW of the step's gradients,
    and their bf16 operand copies.

C3 repeats it on LLaMA-13B shapes with 8 jobs of ranks {8,16,32,64} x 2, a
MinPad-selected packed layout (half the adapters have empty segments and must
come out bitwise untouched), which takes the multi-chunk (R_pad = 256) grouped
paths.  Tolerances: rel-L2 <= 1e-2 per job (north star, bf16 operands with fp32
accumulation); losses 1e-3 relative.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import mlora_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-2
LOSS_TOL = 1e-3


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def f64(t):
    return t.double().cpu().numpy()


def sample_rows(seg, per_job, rng):
    rows = []
    for j in range(len(seg) - 1):
        a, b = seg[j], seg[j + 1]
        if b > a:
            rows.append(np.sort(rng.choice(np.arange(a, b), min(per_job, b - a), replace=False)))
    return np.concatenate(rows)


def _source_y(layer, p, rows):
    """Projection p's input as the oracle sees it: its source's Y (ChatGLM2's 4h_to_h reads
    the first p.k columns of h_to_4h's output), taken from the source, not from the layer's
    own column-slice copy."""
    base = "h_to_4h" if p.src == "h_to_4h_half" else p.src
    return next(q for q in layer.proj if q.name == base).Y[:rows, :p.k]


def run_step_and_check(shapes, ranks, scales, lrs, seg, seed):
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200.layer import FusedLoraLayer

    dev = torch.device("cuda", 0)
    ctx = F.Context(dev)
    J, rows = len(ranks), seg[-1]
    layer = FusedLoraLayer(ctx, shapes, ranks, scales, lrs, rows=rows, seed=seed)
    layer.set_layout(seg)
    g = torch.Generator().manual_seed(seed + 1)
    x = (torch.rand(rows, shapes[0][2], generator=g) * 2 - 1).to(torch.bfloat16).to(dev)
    x_host = f64(x)
    ro = layer.plan.rank_offsets
    pre = {p.name: dict(A16=p.A.p_bf16.clone(), B16=p.B.p_bf16.clone(), A=p.A.p.clone(), B=p.B.p.clone())
           for p in layer.proj}
    active = [seg[j + 1] > seg[j] for j in range(J)]
    loss = layer.step(x, active=active).clone()
    torch.cuda.synchronize()
    loss = loss.cpu().numpy()

    rng = np.random.default_rng(seed)
    srows = sample_rows(seg, 48, rng)
    sjob = np.searchsorted(seg, srows, side="right") - 1
    sseg = [int(np.searchsorted(sjob, j)) for j in range(J)] + [len(srows)]
    loss_ref = np.zeros(J)
    errs = {}
    for p in layer.proj:
        W = f64(p.W0)
        A16, B16 = f64(pre[p.name]["A16"]), f64(pre[p.name]["B16"])
        As = [A16[ro[j]:ro[j] + r] for j, r in enumerate(ranks)]
        Bs = [B16[:, ro[j]:ro[j] + r] for j, r in enumerate(ranks)]
        xin = x_host if p.src == "x" else f64(_source_y(layer, p, rows))
        Y = f64(p.Y[:rows])
        # ---- Y and dX on sampled rows (oracle: fused_forward / composed backward)
        Yr = O.segmented_forward(xin[srows], W, As, Bs, scales, sseg)
        dXr, _, _ = O.segmented_backward(Y[srows], xin[srows], W, As, Bs, scales, sseg)
        dX = f64(p.dX[:rows])
        for j in range(J):
            a, b = sseg[j], sseg[j + 1]
            if b > a:
                errs[f"{p.name}.Y{j}"] = rel(Y[srows][a:b], Yr[a:b])
                errs[f"{p.name}.dX{j}"] = rel(dX[srows][a:b], dXr[a:b])
        # ---- dA_j, dB_j in full over the job's rows (dY = Y)
        dA, dB = p.dA.cpu().numpy(), p.dB.cpu().numpy()
        dAr, dBr = O.segmented_adapter_grads(Y, xin, As, Bs, scales, seg)
        for j, r in enumerate(ranks):
            a, b = seg[j], seg[j + 1]
            gA, gB = dA[ro[j]:ro[j] + r], dB[:, ro[j]:ro[j] + r]
            if b == a:
                assert not gA.any() and not gB.any(), f"{p.name}: absent job {j} got a gradient"
                continue
            errs[f"{p.name}.dA{j}"] = rel(gA, dAr[j])
            errs[f"{p.name}.dB{j}"] = rel(gB, dBr[j])
        # ---- loss: a full-size fp32 restatement of the projection (cuBLAS, TF32 off)
        with torch.no_grad():
            prev = torch.backends.cuda.matmul.allow_tf32
            torch.backends.cuda.matmul.allow_tf32 = False
            xin_t = x.float() if p.src == "x" else _source_y(layer, p, rows).float()
            Yt = xin_t @ p.W0.float().t()
            for j, r in enumerate(ranks):
                a, b = seg[j], seg[j + 1]
                if b > a:
                    A_t = pre[p.name]["A16"][ro[j]:ro[j] + r].float()
                    B_t = pre[p.name]["B16"][:, ro[j]:ro[j] + r].float()
                    Yt[a:b] += scales[j] * (xin_t[a:b] @ A_t.t()) @ B_t.t()
            torch.backends.cuda.matmul.allow_tf32 = prev
            for j in range(J):
                a, b = seg[j], seg[j + 1]
                loss_ref[j] += 0.5 * float((Yt[a:b].double() ** 2).sum())
            errs[f"{p.name}.Y_full"] = rel(Y, Yt.double().cpu().numpy())
        # ---- AdamW (step 1, per-job lr) of the step's own gradients, numpy
        for st, grad, key, layout in ((p.A, dA, "A", 0), (p.B, dB, "B", 1)):
            p0 = pre[p.name][key].cpu().numpy().astype(np.float64)
            gr = grad.astype(np.float64)
            m = 0.1 * gr
            v = 0.001 * gr * gr
            upd = (m / 0.1) / (np.sqrt(v / 0.001) + 1e-8)
            lr_el = np.zeros_like(p0)
            for j in range(J):
                if not active[j]:
                    continue
                if layout == 0:
                    lr_el[ro[j]:ro[j + 1]] = lrs[j]
                else:
                    lr_el[:, ro[j]:ro[j + 1]] = lrs[j]
            want = p0 - lr_el * upd
            got = st.p.cpu().numpy()
            assert np.allclose(got, want, rtol=1e-5, atol=1e-7), f"{p.name}.{key}: AdamW mismatch"
            assert torch.equal(st.p_bf16, st.p.to(torch.bfloat16)), f"{p.name}.{key}: bf16 copy stale"
            for j in range(J):
                if not active[j]:  # absent jobs: master untouched bitwise
                    sl = (slice(ro[j], ro[j + 1]),) if layout == 0 else (slice(None), slice(ro[j], ro[j + 1]))
                    assert torch.equal(st.p[sl], pre[p.name][key][sl])
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    assert not bad, f"rel-L2 above {TOL}: {bad}"
    for j in range(J):
        if active[j]:
            assert abs(loss[j] - loss_ref[j]) <= LOSS_TOL * loss_ref[j], (j, loss[j], loss_ref[j])
        else:
            assert loss[j] == 0.0
    return layer, errs


def test_c2_benchmarked_step_end_to_end():
    """bench.py's C2 step, same layer, same layout (4 x 2048 rows, δ = 0)."""
    from paper_2312_02515_b200.layer import LLAMA7B
    per_job = 4 * 512
    seg = [j * per_job for j in range(5)]
    layer, errs = run_step_and_check(LLAMA7B, [16] * 4, [2.0] * 4, [1e-4, 2e-4, 5e-5, 3e-4], seg, seed=1000)
    # the step exercised the shared-input (NB = 5) and grouped kernels and the split reduce
    assert layer.plan.rank_padded == 64
    print({k: f"{v:.2e}" for k, v in sorted(errs.items()) if k.endswith("0")})


def test_c3_llama13b_minpad_step_end_to_end():
    """C3: LLaMA-13B shapes, 8 jobs, ranks {8,16,32,64} x 2, MinPad picks 4 (packed)."""
    from paper_2312_02515_b200 import packer as P
    from paper_2312_02515_b200.layer import LLAMA13B
    ranks = [8, 16, 32, 64] * 2
    means = [64, 128, 256, 512, 1024, 96, 192, 384]
    cands = [P.Candidate(j, P.sample_lengths("normal", 4, seed=1000 + j, min_len=32, max_len=1024, mean=means[j],
                                             stddev=96.0), priority=1 + j % 3, submit_time=float(j)) for j in range(8)]
    sel = P.select(cands, 4, "minpad")
    want = O.select_minpad([O.BatchCandidate(f"c{i}", c.lengths, c.priority, c.submit_time)
                            for i, c in enumerate(cands)], 4)
    assert sel.chosen == [int(c[1:]) for c in want.chosen]
    chosen = set(sel.chosen)
    seg, r = [0], 0
    for j in range(8):
        if j in chosen:
            r += sum(cands[j].lengths)
        seg.append(r)
    layer, _ = run_step_and_check(LLAMA13B, ranks, [2.0] * 8, [1e-4, 2e-4, 5e-5, 3e-4] * 2, seg, seed=2000)
    assert layer.plan.rank_padded == 256


def test_tiny_step_edge_layout():
    """TINY shapes with a 1-row job, an empty job and a 1499-row job: few tiles over a
    long token range, so the dA / dB groups take the token split (6 splits) and the
    fixed-order reduce; the empty job's adapters must come out bitwise untouched."""
    from paper_2312_02515_b200.layer import TINY
    run_step_and_check(TINY, [8, 16, 4], [2.0, 1.0, 0.5], [1e-3, 2e-3, 5e-4], [0, 1, 1, 1500], seed=77)


def test_c4_chatglm2_layer_step_column_slice():
    """ChatGLM2-6B-shaped layer (fused qkv 4096 -> 4608, dense, fused h_to_4h 4096 -> 27392,
    4h_to_h reading the first 13 696 columns of h_to_4h's output through the layer's
    column-slice copy), 3 jobs of ragged lengths: the whole step against the oracle."""
    from paper_2312_02515_b200.layer import CHATGLM2_6B
    run_step_and_check(CHATGLM2_6B, [16, 8, 32], [2.0, 1.0, 0.5], [1e-4, 2e-4, 5e-5], [0, 700, 1200, 2100], seed=91)



def test_c5_thirty_two_jobs_step():
    """C5's job count on one GPU: 32 rank-16 jobs (R_pad = 512: eight 64-column rank chunks,
    every down-projection tile narrowed to its job's group) on LLaMA-7B shapes, 64 rows
    per job: the whole step against the oracle."""
    from paper_2312_02515_b200.layer import LLAMA7B
    J = 32
    seg = [64 * j for j in range(J + 1)]
    lrs = [1e-4, 2e-4, 5e-5, 3e-4] * (J // 4)
    run_step_and_check(LLAMA7B, [16] * J, [2.0] * J, lrs, seg, seed=5)
