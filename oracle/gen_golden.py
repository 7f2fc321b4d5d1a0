"""Generate tests/golden/* from the REFERENCE itself (oracle/_ref/libfusim_ref.so,
i.e. /root/reference/proj/src/{lora,batch_select,workload}.cpp compiled in place).

Run here (where /root/reference exists):  python oracle/gen_golden.py
The fixtures are small and committed; the GPU box never needs the reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle import ref  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def rand_instance(rng, dmax=16, jmax=6, rmax=4, lmax=8, smax=3):
    """acceptance.cpp:64-114 (criterion 1) instance family."""
    d, k = int(rng.integers(1, dmax + 1)), int(rng.integers(1, dmax + 1))
    W0 = rng.uniform(-1, 1, (d, k))
    J = int(rng.integers(1, jmax + 1))
    ranks, As, Bs, seqs = [], [], [], []
    for j in range(J):
        r = min(int(rng.integers(1, rmax + 1)), d, k)
        ranks.append(r)
        As.append(rng.uniform(-1, 1, (r, k)))
        Bs.append(rng.uniform(-1, 1, (d, r)))
        for _ in range(int(rng.integers(1, smax + 1))):
            seqs.append((j, rng.uniform(-1, 1, (int(rng.integers(1, lmax + 1)), k))))
    return W0, ranks, As, Bs, seqs


def gen_forward(rng, n, prefix, arrays, **kw):
    cases = []
    for i in range(n):
        W0, ranks, As, Bs, seqs = rand_instance(rng, **kw)
        out, mask, meta = ref.fused_forward(W0, ranks, As, Bs, seqs)
        key = f"{prefix}{i}_"
        arrays[key + "W0"] = W0
        arrays[key + "ranks"] = np.array(ranks, np.int32)
        arrays[key + "A_all"] = np.concatenate([a.ravel() for a in As])
        arrays[key + "B_all"] = np.concatenate([b.ravel() for b in Bs])
        arrays[key + "seq_job"] = np.array([j for j, _ in seqs], np.int32)
        arrays[key + "seq_len"] = np.array([x.shape[0] for _, x in seqs], np.int32)
        arrays[key + "X_all"] = np.concatenate([x.ravel() for _, x in seqs])
        arrays[key + "out"] = out
        arrays[key + "mask"] = mask
        arrays[key + "meta"] = np.array([meta["max_len"], meta["sequences"], meta["total_tokens"],
                                         meta["padding_tokens"]], np.int64)
        cases.append(key)
    return cases


def gen_backward(rng, n, arrays):
    """Composed reference-primitive gradients (SURVEY.md §8c probe B)."""
    cases = []
    for i in range(n):
        d, k = int(rng.integers(2, 24)), int(rng.integers(2, 24))
        J = int(rng.integers(1, 4))
        W0 = rng.uniform(-1, 1, (d, k))
        ranks = [min(int(rng.integers(1, 5)), d, k) for _ in range(J)]
        As = [rng.uniform(-1, 1, (r, k)) for r in ranks]
        Bs = [rng.uniform(-1, 1, (d, r)) for r in ranks]
        lens = [int(rng.integers(1, 12)) for _ in range(J)]
        X = [rng.uniform(-1, 1, (L, k)) for L in lens]
        dY = [rng.uniform(-1, 1, (L, d)) for L in lens]
        # dX = fused_forward(W0^T, {A'=B^T, B'=A^T}, fuse(dY))
        outT, _, _ = ref.fused_forward(W0.T.copy(), ranks, [b.T.copy() for b in Bs], [a.T.copy() for a in As],
                                       [(j, dY[j]) for j in range(J)])
        key = f"b{i}_"
        arrays[key + "W0"] = W0
        arrays[key + "ranks"] = np.array(ranks, np.int32)
        arrays[key + "lens"] = np.array(lens, np.int32)
        for j in range(J):
            arrays[key + f"A{j}"] = As[j]
            arrays[key + f"B{j}"] = Bs[j]
            arrays[key + f"X{j}"] = X[j]
            arrays[key + f"dY{j}"] = dY[j]
            arrays[key + f"dX{j}"] = outT[j, :lens[j]]
            arrays[key + f"dA{j}"] = ref.matmul(ref.matmul(dY[j], Bs[j]).T.copy(), X[j])
            arrays[key + f"dB{j}"] = ref.matmul(dY[j].T.copy(), ref.matmul(X[j], As[j].T.copy()))
        cases.append(key)
    return cases


def gen_selection(rng, n):
    out = []
    for _ in range(n):
        cnt = int(rng.integers(1, 13))
        cands = []
        for i in range(cnt):
            items = [int(rng.integers(1, 17)) for _ in range(int(rng.integers(1, 5)))]
            cands.append((items, int(rng.integers(1, 4)), float(i if rng.random() < 0.7 else rng.integers(0, 5))))
        m = int(rng.integers(1, 7))
        rec = {"cands": cands, "m": m}
        for s in ("fifo", "priority", "minpad", "brute"):
            rec[s] = ref.select(s, cands, m)
        out.append(rec)
    return out


def main():
    if not ref.build():
        sys.exit("reference checker not available (needs /root/reference)")
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(4242)
    arrays = {}
    fwd = gen_forward(rng, 60, "f", arrays)
    med = gen_forward(rng, 6, "m", arrays, dmax=96, jmax=4, rmax=16, lmax=40, smax=3)
    bwd = gen_backward(rng, 12, arrays)
    arrays["_index_forward"] = np.array(fwd + med)
    arrays["_index_backward"] = np.array(bwd)
    np.savez_compressed(os.path.join(OUT, "lora_ref.npz"), **arrays)

    shapes = []
    for _ in range(80):
        groups = [[int(rng.integers(1, 10)) for _ in range(int(rng.integers(1, 4)))] for _ in range(int(rng.integers(1, 5)))]
        shapes.append({"groups": groups, **ref.fused_shape(groups)})
    shapes.append({"groups": [[3], [5]], **ref.fused_shape([[3], [5]])})
    shapes.append({"groups": [], **ref.fused_shape([])})

    sel = gen_selection(rng, 200)

    lengths = []
    for seed in (1, 7, 1234, 4242):
        lengths.append({"family": "uniform", "seed": seed, "min_len": 8, "max_len": 64, "count": 40,
                        "out": ref.sample_lengths("uniform", 40, seed, min_len=8, max_len=64)})
        lengths.append({"family": "normal", "seed": seed, "min_len": 32, "max_len": 512, "mean": 256.0,
                        "stddev": 96.0, "count": 40,
                        "out": ref.sample_lengths("normal", 40, seed, min_len=32, max_len=512, mean=256.0, stddev=96.0)})
        lengths.append({"family": "histogram", "seed": seed, "histogram": {"3": 2, "9": 3, "17": 1}, "count": 13,
                        "out": ref.sample_lengths("histogram", 13, seed, histogram={3: 2, 9: 3, 17: 1})})

    traces = []
    for items, bs, rounds in (([3, 5, 4], 2, 6), ([3, 5, 4], 4, 3), ([2, 9, 4, 7, 1], 3, 40), ([1], 5, 4)):
        tr, cur = ref.batch_trace(items, bs, rounds)
        traces.append({"items": items, "batch_size": bs, "rounds": rounds, "batches": tr, "final_cursor": cur})

    launches = [{"jobs": j, "fused": f, "out": list(ref.count_launches(j, f))} for j in (1, 2, 5, 32) for f in (0, 1)]

    with open(os.path.join(OUT, "host_ref.json"), "w") as f:
        json.dump({"fused_shape": shapes, "selection": sel, "sample_lengths": lengths, "batch_trace": traces,
                   "count_launches": launches}, f)
    print("wrote", OUT, sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
