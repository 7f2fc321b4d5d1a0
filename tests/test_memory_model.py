"""§8f row 3: the B200 memory probes (tools/memory_probe.py → profiles/
r01_memory_samples.csv, the reference's `batch_size,seq_len,mem_gb` schema)
feed the reference's own Eq. 6 fit (fit_memory_model, memory_model.cpp, compiled
in place into oracle/_ref).  The fit must agree with an independent least-squares
fit and describe the samples to within 5 MB."""
import csv
import ctypes as C
import os

import numpy as np
import pytest

from oracle import ref

CSV = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   "r01_memory_samples.csv")


def load():
    with open(CSV) as f:
        rows = list(csv.DictReader(f))
    return (np.array([int(r["batch_size"]) for r in rows], np.int32),
            np.array([int(r["seq_len"]) for r in rows], np.int32),
            np.array([float(r["mem_gb"]) for r in rows], np.float64))


def test_reference_fit_of_b200_memory_samples():
    if not ref.available() and not ref.build():
        pytest.skip("reference checker unavailable")
    L = ref.lib()
    if not hasattr(L, "ref_fit_memory_model"):
        pytest.skip("checker built without the memory-model shim")
    bs, seq, mem = load()
    out = (C.c_double * 4)()
    fn = L.ref_fit_memory_model
    fn.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_int,
                   C.POINTER(C.c_double)]
    assert fn(len(bs), bs.ctypes.data_as(C.POINTER(C.c_int)), seq.ctypes.data_as(C.POINTER(C.c_int)),
              mem.ctypes.data_as(C.POINTER(C.c_double)), 0, out) == 0
    b0, b1, b2, rmse = list(out)
    t = bs.astype(np.float64) * seq
    A = np.stack([np.ones_like(t), t, t * seq], 1)  # Eq. 6 features (1, Bt*Ln, Bt*Ln^2)
    want, *_ = np.linalg.lstsq(A, mem, rcond=None)
    assert np.allclose([b0, b1, b2], want, rtol=1e-6, atol=1e-12)
    assert rmse < 0.005
    # activations scale linearly with tokens on this path (no attention): beta2 ~ 0
    assert abs(b2) * 8 * 1024 ** 2 < 0.01 and b1 > 0


# ---------------------------------------------------------------- the product's memory model vs the reference
def _ref_lib():
    if not ref.available() and not ref.build():
        pytest.skip("reference checker unavailable")
    L = ref.lib()
    if not hasattr(L, "ref_schedule"):
        pytest.skip("checker built without the scheduler shim")
    return L


def _ref_fit(L, samples, nonneg):
    n = len(samples)
    bs = (C.c_int * n)(*[s[0] for s in samples])
    sl = (C.c_int * n)(*[s[1] for s in samples])
    mem = (C.c_double * n)(*[s[2] for s in samples])
    out = (C.c_double * 4)()
    L.ref_fit_memory_model.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                       C.c_int, C.POINTER(C.c_double)]
    rc = L.ref_fit_memory_model(n, bs, sl, mem, 1 if nonneg else 0, out)
    return rc, list(out)


def test_product_fit_matches_reference_fit():
    """fit_memory_model (façade C++, paper_2312_02515_b200.memory) vs the reference's
    own (memory_model.cpp:76-152) on the committed B200 probes and on 200 random
    sample sets (both constraint modes, including curvature pulled negative)."""
    from paper_2312_02515_b200 import errors as E
    from paper_2312_02515_b200 import memory as MM
    L = _ref_lib()
    bs, seq, mem = load()
    samples = [(int(b), int(s), float(m)) for b, s, m in zip(bs, seq, mem)]
    rng = np.random.default_rng(5)
    sets = [samples]
    for _ in range(200):
        n = int(rng.integers(3, 14))
        b0, b1, b2 = rng.uniform(0.1, 5), rng.uniform(1e-5, 1e-3), rng.uniform(-2e-7, 2e-7)
        ss = []
        for _ in range(n):
            bt, ln = int(rng.integers(1, 9)), int(rng.choice([32, 64, 128, 256, 512, 1024]))
            u = bt * ln
            ss.append((bt, ln, max(1e-3, b0 + b1 * u + b2 * u * ln + rng.normal(0, 0.05))))
        sets.append(ss)
    checked = 0
    for ss in sets:
        for nonneg in (False, True):
            rc, want = _ref_fit(L, ss, nonneg)
            if rc != 0:
                with pytest.raises(E.FitError):
                    MM.fit_memory_model(ss, nonnegative=nonneg)
                continue
            got = MM.fit_memory_model(ss, nonnegative=nonneg)
            scale = max(abs(v) for v in want[:3])
            assert np.allclose([got.beta0, got.beta1, got.beta2], want[:3], rtol=1e-7, atol=1e-9 * scale)
            assert got.rmse == pytest.approx(want[3], rel=1e-7, abs=1e-12)
            checked += 1
    assert checked > 300


def test_product_max_packing_and_warmup_plan_bit_exact_with_reference():
    """max_packing (subset-sum DP, <= 30 items) / greedy fallback (> 30) and
    warmup_plan: the same subsets and probe lists as memory_model.cpp:181-259."""
    from paper_2312_02515_b200 import memory as MM
    L = _ref_lib()
    L.ref_max_packing.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_double, C.c_int, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int)]
    rng = np.random.default_rng(11)
    for trial in range(400):
        n = int(rng.integers(0, 36))
        quant = trial % 3 == 0  # many exact ties at the 0.01 GB grid
        items = [round(float(x), 2) if quant else float(x) for x in rng.uniform(0, 3, n)]
        budget = float(rng.uniform(0, max(1.0, sum(items) * 0.7)))
        for greedy in (0, 1):
            arr = (C.c_double * max(n, 1))(*items)
            out = (C.c_int * max(n, 1))()
            cnt = C.c_int()
            assert L.ref_max_packing(n, arr, budget, greedy, out, C.byref(cnt)) == 0
            assert MM.max_packing(items, budget, greedy=bool(greedy)) == [out[i] for i in range(cnt.value)]
    L.ref_warmup_plan.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), C.POINTER(C.c_int)]
    for bsl, lsl in [([1, 2, 4, 8], [128, 256, 512, 1024]), ([2, 2, 1], [64, 64]), ([4], [128, 256]), ([3, 1], [5])]:
        nb, nl = len(bsl), len(lsl)
        out = (C.c_int * (2 * nb * nl))()
        cnt, suff = C.c_int(), C.c_int()
        assert L.ref_warmup_plan(nb, (C.c_int * nb)(*bsl), nl, (C.c_int * nl)(*lsl), out, C.byref(cnt),
                                 C.byref(suff)) == 0
        probes, sufficient = MM.warmup_plan(bsl, lsl)
        assert probes == [(out[2 * i], out[2 * i + 1]) for i in range(cnt.value)] and sufficient == bool(suff.value)


def test_admission_matches_reference_schedule():
    """memory.admit — the executor's per-iteration admission under a budget —
    against the reference's own schedule() (scheduler.cpp:74-130, M1/M2/M3 with a
    fitted model or static footprints) on 600 random queues: the same jobs in the
    same admission order."""
    from paper_2312_02515_b200 import memory as MM
    L = _ref_lib()
    L.ref_schedule.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_int), C.POINTER(C.c_double),
                               C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_long),
                               C.POINTER(C.c_double), C.c_int, C.c_int, C.POINTER(C.c_double), C.c_double,
                               C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double)]
    rng = np.random.default_rng(17)
    names = {0: "fifo", 1: "priority", 2: "minpad"}
    for trial in range(600):
        n = int(rng.integers(1, 12))
        ids = [f"job{int(x):02d}" for x in rng.permutation(40)[:n]]
        prio = [int(rng.integers(1, 4)) for _ in range(n)]
        submit = [float(rng.integers(0, 4)) for _ in range(n)]
        bsz = [int(rng.integers(1, 5)) for _ in range(n)]
        data = [[int(x) for x in rng.integers(1, 300, int(rng.integers(1, 8)))] for _ in range(n)]
        cursor = [int(rng.integers(0, len(d))) for d in data]
        static = [float(rng.uniform(0.2, 3.0)) for _ in range(n)]
        has_model = trial % 2 == 0
        beta = [float(rng.uniform(0.05, 0.5)), float(rng.uniform(1e-5, 3e-4)), 0.0]
        floor = 0.1
        model = MM.MemoryModel(*beta) if has_model else None
        est = [model.predict_clamped(bsz[i], max(data[i]), floor) if model else static[i] for i in range(n)]
        budget = float(rng.uniform(0.3, 1.0) * sum(est))
        M = int(rng.integers(1, 5))
        strategy = trial % 3
        flat = [x for d in data for x in d]
        out = (C.c_int * n)()
        cnt, est_gb = C.c_int(), C.c_double()
        rc = L.ref_schedule(n, (C.c_char_p * n)(*[s.encode() for s in ids]), (C.c_int * n)(*prio),
                            (C.c_double * n)(*submit), (C.c_int * n)(*bsz), (C.c_int * n)(*[len(d) for d in data]),
                            (C.c_int * len(flat))(*flat), (C.c_long * n)(*cursor), (C.c_double * n)(*static),
                            strategy, 1 if has_model else 0, (C.c_double * 3)(*beta), budget, floor, M, out,
                            C.byref(cnt), C.byref(est_gb))
        assert rc == 0
        want = [out[i] for i in range(cnt.value)]
        queue = []
        for i in range(n):
            pos = cursor[i] % len(data[i])
            nb = data[i][pos:pos + min(bsz[i], len(data[i]) - pos)]
            queue.append(MM.QueuedJob(ids[i], prio[i], submit[i], nb, est[i]))
        got = MM.admit(queue, names[strategy], budget, M)
        assert got == want, (trial, names[strategy], got, want)
        assert sum(est[i] for i in got) == pytest.approx(est_gb.value)
