"""ctypes access to oracle/_ref/libfusim_ref.so — the reference's own lora.cpp,
batch_select.cpp and workload.cpp compiled in place by oracle/Makefile.

TEST INFRASTRUCTURE ONLY (golden-fixture generation, oracle pinning, and the
timed CPU baseline in bench.py).  `available()` is False when the library has
not been built (e.g. /root/reference absent and no prebuilt copy shipped).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libfusim_ref.so")
_lib = None

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
i64p = C.POINTER(C.c_int64)


def build() -> bool:
    """Compile the reference checker when /root/reference is present."""
    if not os.path.isdir("/root/reference/proj/src"):
        return os.path.exists(LIB_PATH)
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.exists(LIB_PATH)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _chk(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _d(a):
    a = np.ascontiguousarray(a, np.float64)
    return a, a.ctypes.data_as(dp)


def _i(a):
    a = np.ascontiguousarray(a, np.int32)
    return a, a.ctypes.data_as(ip)


def fused_shape(groups):
    sizes = [len(g) for g in groups]
    flat = [x for g in groups for x in g] or [0]
    s, sp = _i(sizes if sizes else [0])
    f, fp = _i(flat)
    ml = C.c_int()
    seq, tot, pad = C.c_int64(), C.c_int64(), C.c_int64()
    ratio = C.c_double()
    _chk(lib().ref_fused_shape(len(groups), sp, fp, C.byref(ml), C.byref(seq), C.byref(tot), C.byref(pad),
                               C.byref(ratio)))
    return dict(max_len=ml.value, sequences=seq.value, total_tokens=tot.value, padding_tokens=pad.value,
                padding_ratio=ratio.value)


def fused_forward(W0, ranks, As, Bs, seqs, has_adapter=None):
    """seqs: list of (job_index, array len x k), grouped by job in order.
    Returns (outs [S, max_len, d], mask [S*max_len], meta dict)."""
    d, k = W0.shape
    J = len(ranks)
    has = has_adapter if has_adapter is not None else [1] * J
    A_all = np.concatenate([np.asarray(a, np.float64).ravel() for a in As]) if J else np.zeros(1)
    B_all = np.concatenate([np.asarray(b, np.float64).ravel() for b in Bs]) if J else np.zeros(1)
    X_all = np.concatenate([np.asarray(x, np.float64).ravel() for _, x in seqs])
    w, wp = _d(W0)
    a, ap = _d(A_all)
    b, bp = _d(B_all)
    x, xp = _d(X_all)
    r, rp = _i(ranks)
    h, hp = _i(has)
    sj, sjp = _i([j for j, _ in seqs])
    sl, slp = _i([np.asarray(x_).shape[0] for _, x_ in seqs])
    S = len(seqs)
    max_len = int(max(sl))
    out = np.zeros((S, max_len, d), np.float64)
    mask = np.zeros(S * max_len, np.uint8)
    meta = np.zeros(4, np.int64)
    _chk(lib().ref_fused_forward_w(wp, d, k, J, rp, hp, ap, bp, S, sjp, slp, xp, out.ctypes.data_as(dp),
                                   mask.ctypes.data_as(C.POINTER(C.c_uint8)), meta.ctypes.data_as(i64p)))
    return out, mask, dict(max_len=int(meta[0]), sequences=int(meta[1]), total_tokens=int(meta[2]),
                           padding_tokens=int(meta[3]))


def matmul(a, b):
    a, ap = _d(a)
    b, bp = _d(b)
    out = np.zeros((a.shape[0], b.shape[1]), np.float64)
    _chk(lib().ref_matmul(ap, a.shape[0], a.shape[1], bp, b.shape[0], b.shape[1], out.ctypes.data_as(dp)))
    return out


def lora_forward(W0, A, B, rank, x):
    w, wp = _d(W0)
    a, ap = _d(A)
    b, bp = _d(B)
    xx, xp = _d(x)
    out = np.zeros((W0.shape[0], x.shape[1]), np.float64)
    _chk(lib().ref_lora_forward(wp, W0.shape[0], W0.shape[1], rank, ap, a.shape[0], a.shape[1], bp, b.shape[0],
                                b.shape[1], xp, xx.shape[0], xx.shape[1], out.ctypes.data_as(dp)))
    return out


def count_launches(num_jobs, fused):
    s, l = C.c_int64(), C.c_int64()
    _chk(lib().ref_count_launches(num_jobs, 1 if fused else 0, C.byref(s), C.byref(l)))
    return s.value, l.value


STRATEGY = {"fifo": 0, "priority": 1, "minpad": 2, "brute": 3}


def select(strategy, cands, m):
    """cands: list of (item_lengths, priority, submit).  Returns dict with
    chosen indices (result order), fused_max_len, total_sequences, padding_tokens, padding_ratio."""
    n = len(cands)
    counts, cp = _i([len(c[0]) for c in cands] or [0])
    flat, fp = _i([x for c in cands for x in c[0]] or [0])
    pri, pp = _i([c[1] for c in cands] or [0])
    sub, sp = _d([c[2] for c in cands] or [0.0])
    chosen = np.zeros(max(n, 1), np.int32)
    meta = np.zeros(4, np.int64)
    ratio = C.c_double()
    _chk(lib().ref_select(STRATEGY[strategy], n, cp, fp, pp, sp, m, chosen.ctypes.data_as(ip),
                          meta.ctypes.data_as(i64p), C.byref(ratio)))
    return dict(chosen=[int(x) for x in chosen[:meta[0]]], fused_max_len=int(meta[1]),
                total_sequences=int(meta[2]), padding_tokens=int(meta[3]), padding_ratio=ratio.value)


def sample_lengths(family, count, seed, min_len=1, max_len=1, mean=0.0, stddev=1.0, histogram=None):
    fam = {"uniform": 0, "normal": 1, "histogram": 2}[family]
    hist = sorted((histogram or {}).items())
    hl, hlp = _i([h[0] for h in hist] or [0])
    hc, hcp = _i([h[1] for h in hist] or [0])
    out = np.zeros(count, np.int32)
    _chk(lib().ref_sample_lengths(fam, min_len, max_len, C.c_double(mean), C.c_double(stddev), len(hist), hlp, hcp,
                                  count, C.c_uint64(seed), out.ctypes.data_as(ip)))
    return [int(x) for x in out]


def batch_trace(items, batch_size, rounds):
    it, itp = _i(items)
    sizes = np.zeros(rounds, np.int32)
    out = np.zeros(rounds * batch_size, np.int32)
    cur = C.c_int64()
    _chk(lib().ref_batch_trace(len(items), itp, batch_size, rounds, sizes.ctypes.data_as(ip), out.ctypes.data_as(ip),
                               C.byref(cur)))
    res, o = [], 0
    for s in sizes:
        res.append([int(x) for x in out[o:o + s]])
        o += s
    return res, cur.value


def detect_stop(losses, accuracies=(), patience=3):
    """fusim::detect_stop (progress.cpp:90-124): None or (iteration, cause),
    cause in {"nan_loss", "accuracy_decline"}."""
    l, lp = _d(losses or [0.0])
    a, ap = _d(accuracies or [0.0])
    it, cause = C.c_int(), C.c_int()
    rc = lib().ref_detect_stop(len(losses), lp, len(accuracies), ap, patience, C.byref(it), C.byref(cause))
    if rc == 9:
        raise RuntimeError("reference detect_stop failed")
    if rc == 0:
        return None
    return it.value, ("nan_loss", "accuracy_decline", "completed")[cause.value]


class Weights:
    """A frozen W0 marshalled once into a reference fusim::Matrix (for timing)."""

    def __init__(self, W0):
        W0 = np.ascontiguousarray(W0, np.float64)
        L = lib()
        L.ref_weights_create.restype = C.c_void_p
        L.ref_weights_create.argtypes = [dp, C.c_int, C.c_int]
        L.ref_weights_destroy.argtypes = [C.c_void_p]
        self.d, self.k = W0.shape
        self.h = L.ref_weights_create(W0.ctypes.data_as(dp), self.d, self.k)

    def __del__(self):
        try:
            lib().ref_weights_destroy(self.h)
        except Exception:
            pass


class FusedCall:
    """Pre-marshalled arguments of one reference fused_forward call (the timed unit)."""

    def __init__(self, weights: Weights, ranks, As, Bs, seqs):
        self.w = weights
        self.J = len(ranks)
        self.ranks, self.rp = _i(ranks)
        self.has, self.hp = _i([1] * self.J)
        self.A, self.ap = _d(np.concatenate([np.asarray(a, np.float64).ravel() for a in As]))
        self.B, self.bp = _d(np.concatenate([np.asarray(b, np.float64).ravel() for b in Bs]))
        self.X, self.xp = _d(np.concatenate([np.asarray(x, np.float64).ravel() for _, x in seqs]))
        self.sj, self.sjp = _i([j for j, _ in seqs])
        self.sl, self.slp = _i([np.asarray(x).shape[0] for _, x in seqs])
        self.S = len(seqs)
        self.max_len = int(max(self.sl))
        self.out = np.zeros((self.S, self.max_len, weights.d), np.float64)
        self.mask = np.zeros(self.S * self.max_len, np.uint8)
        self.meta = np.zeros(4, np.int64)
        L = lib()
        L.ref_fused_forward_h.argtypes = [C.c_void_p, C.c_int, ip, ip, dp, dp, C.c_int, ip, ip, dp, dp,
                                          C.POINTER(C.c_uint8), i64p]

    def __call__(self):
        _chk(lib().ref_fused_forward_h(self.w.h, self.J, self.rp, self.hp, self.ap, self.bp, self.S, self.sjp,
                                       self.slp, self.xp, self.out.ctypes.data_as(dp),
                                       self.mask.ctypes.data_as(C.POINTER(C.c_uint8)),
                                       self.meta.ctypes.data_as(i64p)))
        return self.out
