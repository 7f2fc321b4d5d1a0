"""CPU oracle for the BatchFusion multi-LoRA path — TEST INFRASTRUCTURE ONLY.

A restatement of the reference algorithm (/root/reference/proj/src/lora.cpp,
batch_select.cpp, workload.cpp) in numpy (fp64, integer-exact where the
reference is integer) and plain Python.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this module, and
only as the checker or the timed CPU baseline; the product path never does.

Pinning: every function here is checked against the reference itself —
golden fixtures in tests/golden/ produced by oracle/gen_golden.py from the
reference sources compiled into oracle/_ref/libfusim_ref.so (oracle/Makefile),
plus the reference's own known-answer tests (test_lora.cpp, test_batch_select.cpp,
test_workload.cpp) restated in tests/test_oracle.py.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


# ---------------------------------------------------------------------------
# errors (errors.hpp:8-25) — the oracle raises the same classes as the product
class OracleError(RuntimeError):
    pass


class UsageError(OracleError):
    pass


class ShapeError(OracleError):
    pass


class RoutingError(OracleError):
    pass


class NumericError(OracleError):
    pass


class StateError(OracleError):
    pass


# ---------------------------------------------------------------------------
# lora.cpp
def matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """lora.cpp:19-34 (ShapeError on a.cols != b.rows).  The reference skips
    a_ik == 0 terms; with finite inputs that does not change the fp64 sum beyond
    reassociation, which numpy's BLAS also does."""
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"matmul: {a.shape[0]}x{a.shape[1]} * {b.shape[0]}x{b.shape[1]}")
    return np.asarray(a, np.float64) @ np.asarray(b, np.float64)


def max_rel_diff(a: np.ndarray, b: np.ndarray) -> float:
    """lora.cpp:51-60: inf-norm relative difference with a floor of 1."""
    if a.shape != b.shape:
        raise ShapeError("max_rel_diff: incompatible shapes")
    if a.size == 0:
        return 0.0
    denom = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
    return float(np.max(np.abs(a - b) / denom))


def validate_adapter(A: np.ndarray, B: np.ndarray, rank: int, d: int, k: int) -> None:
    """AdapterWeights::validate, lora.cpp:62-70."""
    if rank < 1:
        raise UsageError("adapter rank must be >= 1")
    if rank > min(d, k):
        raise UsageError("adapter rank exceeds min(d, k)")
    if A.shape != (rank, k):
        raise ShapeError("adapter A must be rank x k")
    if B.shape != (d, rank):
        raise ShapeError("adapter B must be d x rank")


@dataclass
class FusedShape:
    """lora.hpp:51-61"""
    max_len: int = 0
    sequences: int = 0
    total_tokens: int = 0
    padding_tokens: int = 0

    def padding_ratio(self) -> float:
        return 0.0 if self.total_tokens == 0 else self.padding_tokens / self.total_tokens


def fused_shape(per_group_lengths) -> FusedShape:
    """lora.cpp:72-85."""
    s = FusedShape()
    real = 0
    for group in per_group_lengths:
        for ln in group:
            s.max_len = max(s.max_len, int(ln))
            s.sequences += 1
            real += int(ln)
    s.total_tokens = s.sequences * s.max_len
    s.padding_tokens = s.total_tokens - real
    return s


@dataclass
class FusedBatch:
    """lora.hpp:65-82 (data as an (S*max_len, dim) fp64 array)."""
    num_sequences: int = 0
    max_len: int = 0
    dim: int = 0
    data: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))
    routing: list = field(default_factory=list)
    mask: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    total_tokens: int = 0
    padding_tokens: int = 0

    def padding_ratio(self) -> float:
        return 0.0 if self.total_tokens == 0 else self.padding_tokens / self.total_tokens

    def real_length(self, seq: int) -> int:
        """lora.cpp:87-92"""
        return int(self.mask[seq * self.max_len:(seq + 1) * self.max_len].sum())

    def sequence(self, seq: int) -> np.ndarray:
        """lora.cpp:94-100"""
        return self.data[seq * self.max_len:(seq + 1) * self.max_len].copy()


def fuse(batches) -> FusedBatch:
    """lora.cpp:114-158.  batches: list of (job_id, [seq arrays len_i x k])."""
    if len(batches) == 0:
        raise UsageError("fuse: empty batch list")
    dim = -1
    lengths = []
    num_seq = 0
    for _, seqs in batches:
        ls = []
        for s in seqs:
            s = np.asarray(s)
            if dim < 0:
                dim = s.shape[1]
            if s.shape[1] != dim:
                raise ShapeError("fuse: embedding dims differ across sequences")
            if s.shape[0] < 1:
                raise UsageError("fuse: empty sequence")
            ls.append(s.shape[0])
            num_seq += 1
        lengths.append(ls)
    if num_seq == 0:
        raise UsageError("fuse: no sequences")
    shape = fused_shape(lengths)
    fb = FusedBatch(num_sequences=num_seq, max_len=shape.max_len, dim=dim,
                    total_tokens=shape.total_tokens, padding_tokens=shape.padding_tokens)
    fb.data = np.zeros((num_seq * shape.max_len, dim), np.float64)
    fb.mask = np.zeros(num_seq * shape.max_len, np.uint8)
    s_idx = 0
    for job, seqs in batches:
        for s in seqs:
            s = np.asarray(s, np.float64)
            fb.routing.append(job)
            base = s_idx * shape.max_len
            fb.mask[base:base + s.shape[0]] = 1
            fb.data[base:base + s.shape[0]] = s
            s_idx += 1
    return fb


def lora_forward(W0, A, B, rank, x) -> np.ndarray:
    """lora.cpp:102-112 (column convention: x is k x m)."""
    d, k = W0.shape
    validate_adapter(A, B, rank, d, k)
    if x.shape[0] != k:
        raise ShapeError("lora_forward: x must be k x m")
    if not (np.isfinite(W0).all() and np.isfinite(x).all() and np.isfinite(A).all() and np.isfinite(B).all()):
        raise NumericError("lora_forward: non-finite input")
    return matmul(W0, x) + matmul(B, matmul(A, x))


def fused_forward(W0, adapters: dict, fb: FusedBatch) -> list:
    """lora.cpp:160-182.  adapters: job -> (A, B, rank).  One max_len x d
    output per sequence, parallel to routing; pad rows come out zero."""
    if W0.shape[1] != fb.dim:
        raise ShapeError("fused_forward: W0 column dim does not match batch dim")
    for job in fb.routing:
        if job not in adapters:
            raise RoutingError(f"fused_forward: no adapter for job {job}")
    W0t = W0.T
    outs = []
    for s in range(fb.num_sequences):
        xs = fb.sequence(s)
        out = matmul(xs, W0t)
        A, B, rank = adapters[fb.routing[s]]
        validate_adapter(A, B, rank, W0.shape[0], W0.shape[1])
        out = out + matmul(matmul(xs, A.T), B.T)
        outs.append(out)
    return outs


def count_launches(num_jobs: int, fused: bool) -> tuple[int, int]:
    """lora.cpp:184-189."""
    if num_jobs < 1:
        raise UsageError("count_launches: need at least one job")
    return (2 * num_jobs, 2) if fused else (4 * num_jobs, 0)


# ---------------------------------------------------------------------------
# segmented (row-packed) restatement used for device parity.  Rows of job j are
# seg[j]:seg[j+1]; the reference has no scale, so s_j is folded into B_j
# — fused_forward(W0, {A_j, s_j B_j}, ·) per row.
def segmented_forward(X, W0, As, Bs, scales, seg) -> np.ndarray:
    X = np.asarray(X, np.float64)
    W0 = np.asarray(W0, np.float64)
    Y = X @ W0.T
    for j in range(len(As)):
        a, b = seg[j], seg[j + 1]
        if b > a:
            A = np.asarray(As[j], np.float64)
            B = np.asarray(Bs[j], np.float64) * float(scales[j])
            Y[a:b] += (X[a:b] @ A.T) @ B.T
    return Y


def segmented_backward(dY, X, W0, As, Bs, scales, seg):
    """The composed reference-primitive gradients (SURVEY.md §8c probe B):
       dX   = fused_forward(W0^T, {A' = (sB)^T, B' = A^T}, dY)   = dY W0 + s (dY B) A
       dA_j = transpose(matmul(dY_j, s B_j)) @ X_j               = s (dY_j B_j)^T X_j
       dB_j = matmul(transpose(dY_j), matmul(X_j, A_j^T)) * s    = s dY_j^T (X_j A_j^T)
    """
    dY = np.asarray(dY, np.float64)
    X = np.asarray(X, np.float64)
    W0 = np.asarray(W0, np.float64)
    dX = dY @ W0
    dAs, dBs = [], []
    for j in range(len(As)):
        a, b = seg[j], seg[j + 1]
        A = np.asarray(As[j], np.float64)
        B = np.asarray(Bs[j], np.float64)
        s = float(scales[j])
        G = (dY[a:b] @ B) * s
        dX[a:b] += G @ A
        dAs.append(G.T @ X[a:b])
        dBs.append(s * (dY[a:b].T @ (X[a:b] @ A.T)))
    return dX, dAs, dBs


def segmented_adapter_grads(dY, X, As, Bs, scales, seg):
    """The adapter half of segmented_backward (same composed reference
    primitives, SURVEY.md §8c probe B) without the dense dX = dY W0 term, so
    full-size layers (8192 x 11008) are checked in seconds:
       dA_j = transpose(matmul(dY_j, s B_j)) @ X_j,  dB_j = s dY_j^T matmul(X_j, A_j^T).
    Jobs with an empty segment get exact zeros."""
    dAs, dBs = [], []
    for j in range(len(As)):
        a, b = seg[j], seg[j + 1]
        A = np.asarray(As[j], np.float64)
        B = np.asarray(Bs[j], np.float64)
        s = float(scales[j])
        dYj = np.asarray(dY[a:b], np.float64)
        Xj = np.asarray(X[a:b], np.float64)
        G = (dYj @ B) * s
        dAs.append(G.T @ Xj)
        dBs.append(s * (dYj.T @ (Xj @ A.T)))
    return dAs, dBs


# ---------------------------------------------------------------------------
# batch_select.cpp
@dataclass
class BatchCandidate:
    job_id: str
    item_lengths: list
    priority: int = 1
    submit_time: float = 0.0

    def max_len(self) -> int:
        return max(self.item_lengths, default=0)

    def token_count(self) -> int:
        return sum(self.item_lengths)


@dataclass
class SelectionResult:
    chosen: list = field(default_factory=list)
    fused_max_len: int = 0
    total_sequences: int = 0
    padding_tokens: int = 0
    padding_ratio: float = 0.0


def _urgency_key(c: BatchCandidate):
    """batch_select.cpp:10-15: priority desc, submit asc, id asc."""
    return (-c.priority, c.submit_time, c.job_id)


def score_subset(cands, subset) -> SelectionResult:
    """batch_select.cpp:40-54"""
    r = SelectionResult()
    lengths = []
    for i in subset:
        r.chosen.append(cands[i].job_id)
        lengths.append(cands[i].item_lengths)
    shape = fused_shape(lengths)
    r.fused_max_len = shape.max_len
    r.total_sequences = shape.sequences
    r.padding_tokens = shape.padding_tokens
    r.padding_ratio = shape.padding_ratio()
    return r


def select_fifo(cands, m: int) -> SelectionResult:
    """batch_select.cpp:56-64"""
    if m < 1:
        raise UsageError("select_fifo: M must be >= 1")
    order = sorted(range(len(cands)), key=lambda i: (cands[i].submit_time, cands[i].job_id))
    return score_subset(cands, order[:m])


def select_priority(cands, m: int) -> SelectionResult:
    """batch_select.cpp:66-74"""
    if m < 1:
        raise UsageError("select_priority: M must be >= 1")
    order = sorted(range(len(cands)), key=lambda i: _urgency_key(cands[i]))
    return score_subset(cands, order[:m])


def select_minpad(cands, m: int) -> SelectionResult:
    """batch_select.cpp:76-128 (exact MinPad: every candidate tried as anchor)."""
    if m < 1:
        raise UsageError("select_minpad: M must be >= 1")
    n = len(cands)
    if n == 0:
        return SelectionResult()
    want = min(m, n)
    anchor_order = sorted(range(n), key=lambda i: _urgency_key(cands[i]))
    best = None
    best_subset = []
    for anchor in anchor_order:
        L = cands[anchor].max_len()
        eligible = [i for i in range(n) if i != anchor and cands[i].max_len() <= L]
        if len(eligible) + 1 < want:
            continue

        def cost(i, L=L):
            return len(cands[i].item_lengths) * L - cands[i].token_count()

        eligible.sort(key=lambda i: (cost(i),) + _urgency_key(cands[i]))
        subset = [anchor] + eligible[:want - 1]
        padding = sum(cost(i) for i in subset)
        if best is None or padding < best:
            best = padding
            best_subset = subset
    best_subset.sort(key=lambda i: _urgency_key(cands[i]))
    return score_subset(cands, best_subset)


def brute_force_min_padding(cands, m: int) -> SelectionResult:
    """batch_select.cpp:130-159"""
    import itertools
    if m < 1:
        raise UsageError("brute_force_min_padding: M must be >= 1")
    n = len(cands)
    if n > 20:
        raise UsageError("brute_force_min_padding: too many candidates")
    if n == 0:
        return SelectionResult()
    want = min(m, n)
    best = None
    for subset in itertools.combinations(range(n), want):
        r = score_subset(cands, list(subset))
        if best is None or r.padding_tokens < best.padding_tokens:
            best = r
    return best


# ---------------------------------------------------------------------------
# workload.cpp:50-66 (peek / commit)
def next_candidate_batch(items: list, cursor: int, batch_size: int, finished: bool = False) -> list:
    if finished:
        raise StateError("job is finished; no further batches")
    n = len(items)
    pos = cursor % n
    take = min(batch_size, n - pos)
    return items[pos:pos + take]


def commit_batch(cursor: int, n_consumed: int, size: int) -> int:
    cursor += n_consumed
    return 0 if cursor >= size else cursor
