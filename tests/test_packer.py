"""Host packer (C++ façade via include/fusim_c.h) vs the reference: selection,
seeded length generation and the fused-batch accounting are integer-exact."""
import json
import os

import pytest

from oracle import mlora_oracle as O
from paper_2312_02515_b200 import errors as E
from paper_2312_02515_b200 import packer as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def host_ref():
    with open(os.path.join(GOLD, "host_ref.json")) as f:
        return json.load(f)


def test_selection_matches_reference(host_ref):
    for rec in host_ref["selection"]:
        cands = [P.Candidate(i, c[0], c[1], c[2]) for i, c in enumerate(rec["cands"])]
        for name in ("fifo", "priority", "minpad", "brute"):
            r = P.select(cands, rec["m"], name)
            want = rec[name]
            assert (r.fused_max_len, r.total_sequences, r.padding_tokens) == (
                want["fused_max_len"], want["total_sequences"], want["padding_tokens"])
            assert r.chosen == want["chosen"], name


def test_sample_lengths_matches_reference(host_ref):
    for rec in host_ref["sample_lengths"]:
        kw = {k: rec[k] for k in ("min_len", "max_len", "mean", "stddev") if k in rec}
        if "histogram" in rec:
            kw["histogram"] = {int(k): v for k, v in rec["histogram"].items()}
        assert P.sample_lengths(rec["family"], rec["count"], rec["seed"], **kw) == rec["out"]


def test_layout_accounting_matches_reference(host_ref):
    for rec in host_ref["fused_shape"]:
        if not rec["groups"] or not any(rec["groups"]):
            continue
        for padded in (False, True):
            lay = P.layout(rec["groups"], padded=padded)
            assert (lay.max_len, lay.sequences, lay.total_tokens, lay.padding_tokens) == (
                rec["max_len"], rec["sequences"], rec["total_tokens"], rec["padding_tokens"])
            assert lay.rows == (rec["total_tokens"] if padded else rec["total_tokens"] - rec["padding_tokens"])
            assert lay.effective_tokens == rec["total_tokens"] - rec["padding_tokens"]


def test_layout_rows_follow_fuse_order():
    # lengths {3,5}: ξ=10, ξ_p=2, δ=0.2 (test_lora.cpp:95-109)
    lay = P.layout([[3], [5]], padded=True)
    assert (lay.total_tokens, lay.padding_tokens, lay.padding_ratio) == (10, 2, 0.2)
    assert lay.seg == [0, 5, 10] and lay.seq_rows == [[(0, 3)], [(5, 5)]]
    lay = P.layout([[3], [5]], padded=False)
    assert lay.seg == [0, 3, 8] and lay.effective_tokens == 8
    # the padded layout's mask equals fuse()'s mask
    fb = O.fuse([("a", [[[0.0]] * 6, [[0.0]] * 3]), ("b", [[[0.0]] * 2])])
    lay = P.layout([[6, 3], [2]], padded=True)
    mask = [0] * lay.rows
    for rows in lay.seq_rows:
        for r0, L in rows:
            mask[r0:r0 + L] = [1] * L
    assert mask == list(fb.mask)


def test_packer_errors():
    with pytest.raises(E.UsageError):
        P.select([P.Candidate(0, [3])], 0)
    with pytest.raises(E.ConfigError):
        P.sample_lengths("uniform", 3, 0, min_len=0, max_len=5)
    with pytest.raises(E.UsageError):
        P.layout([[3, 0]])
