"""Host packer: which jobs' sequences enter the next fused batch, and where.

North-star item (5): "MinPad packing of jobs' sequences into the fused batch
runs on the host and feeds segment offsets to the kernels".  The selection
itself is the façade's C++ (libfusim_b200.so via include/fusim_c.h), i.e. the
same code the reference's own test_batch_select.cpp suite passes against, so
the Python executor and a C++ fusim user get bit-identical decisions.

Layouts:
  * packed — the kernels' rows are the real tokens only, job by job, sequence by
    sequence: job j owns rows seg[j]:seg[j+1].  No padding work at all.
  * padded — the reference FusedBatch layout (every sequence padded to the
    global max_len, lora.cpp:114-158); pad rows are zero and bitwise neutral.
Either way the reference accounting (ξ, ξ_p, δ; lora.cpp:72-85) is reported.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

from . import _native as N
from . import errors

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfusim_b200.so")
_lib = None

STRATEGIES = {"fifo": 0, "priority": 1, "minpad": 2, "brute": 3}


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run `python -m paper_2312_02515_b200._build`")
        L = C.CDLL(_LIB)
        L.fusim_c_last_error.restype = C.c_char_p
        L.fusim_c_select.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32), C.POINTER(C.c_double), C.c_int32,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        L.fusim_c_select_ids.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_char_p), C.POINTER(C.c_int32),
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                         C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        L.fusim_c_fit_memory_model.argtypes = [C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                               C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double)]
        L.fusim_c_max_packing.argtypes = [C.c_int32, C.POINTER(C.c_double), C.c_double, C.c_int32,
                                          C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.fusim_c_warmup_plan.argtypes = [C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.fusim_c_sample_lengths.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_int32,
                                             C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32, C.c_uint64,
                                             C.POINTER(C.c_int32)]
        _lib = L
    return _lib


def _chk(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().fusim_c_last_error().decode()
    raise {1: errors.UsageError, 7: errors.ConfigError, 8: errors.FitError}.get(rc, errors.Error)(msg)


@dataclass
class Candidate:
    """One job's next candidate batch (fusim::BatchCandidate)."""
    job: object
    lengths: list
    priority: int = 1
    submit_time: float = 0.0
    id: str | None = None             # the job id the reference's tie-breaks compare (default "c<index>")


@dataclass
class Selection:
    chosen: list                      # indices into the candidate list, result (urgency) order
    fused_max_len: int
    total_sequences: int
    padding_tokens: int

    @property
    def total_tokens(self) -> int:
        return self.total_sequences * self.fused_max_len

    @property
    def padding_ratio(self) -> float:
        return 0.0 if self.total_tokens == 0 else self.padding_tokens / self.total_tokens


def select(candidates: list[Candidate], m: int, strategy: str = "minpad") -> Selection:
    """fusim::select_{fifo,priority,minpad} / brute_force_min_padding on the host."""
    n = len(candidates)
    counts = (C.c_int32 * max(n, 1))(*[len(c.lengths) for c in candidates])
    flat = [int(x) for c in candidates for x in c.lengths]
    lengths = (C.c_int32 * max(len(flat), 1))(*flat)
    pri = (C.c_int32 * max(n, 1))(*[int(c.priority) for c in candidates])
    sub = (C.c_double * max(n, 1))(*[float(c.submit_time) for c in candidates])
    chosen = (C.c_int32 * max(n, 1))()
    meta = (C.c_int64 * 4)()
    if all(c.id is not None for c in candidates) and n:
        ids = (C.c_char_p * n)(*[str(c.id).encode() for c in candidates])
        _chk(lib().fusim_c_select_ids(STRATEGIES[strategy], n, ids, counts, lengths, pri, sub, m, chosen, meta))
    else:
        _chk(lib().fusim_c_select(STRATEGIES[strategy], n, counts, lengths, pri, sub, m, chosen, meta))
    return Selection([int(chosen[i]) for i in range(meta[0])], int(meta[1]), int(meta[2]), int(meta[3]))


def sample_lengths(family: str, count: int, seed: int, min_len: int = 1, max_len: int = 1, mean: float = 0.0,
                   stddev: float = 1.0, histogram: dict | None = None) -> list[int]:
    """fusim::sample_lengths with a fresh std::mt19937_64(seed)."""
    fam = {"uniform": 0, "normal": 1, "histogram": 2}[family]
    hist = sorted((histogram or {}).items())
    hl = (C.c_int32 * max(len(hist), 1))(*[h[0] for h in hist])
    hc = (C.c_int32 * max(len(hist), 1))(*[h[1] for h in hist])
    out = (C.c_int32 * count)()
    _chk(lib().fusim_c_sample_lengths(fam, min_len, max_len, mean, stddev, len(hist), hl, hc, count, seed, out))
    return list(out)


@dataclass
class FusedLayout:
    """Row layout of one fused batch for the kernels + the reference accounting."""
    seg: list                         # J+1 row offsets (job j owns rows seg[j]:seg[j+1])
    seq_rows: list = field(default_factory=list)   # per job: [(row0, length), ...] of its sequences
    max_len: int = 0
    sequences: int = 0
    total_tokens: int = 0             # ξ   (reference, padded accounting)
    padding_tokens: int = 0           # ξ_p
    effective_tokens: int = 0         # Σ real tokens
    padded: bool = False

    @property
    def rows(self) -> int:
        return self.seg[-1]

    @property
    def padding_ratio(self) -> float:
        return 0.0 if self.total_tokens == 0 else self.padding_tokens / self.total_tokens


def layout(per_job_lengths: list[list[int]], padded: bool = False) -> FusedLayout:
    """Segment offsets for a fused batch whose jobs' sequences have these lengths
    (jobs in fused order).  Accounting through mlora_fused_shape_of (integer-exact)."""
    flat = [int(x) for g in per_job_lengths for x in g]
    for x in flat:
        if x < 1:
            raise errors.UsageError("fuse: empty sequence")
    arr = (N.i32 * max(len(flat), 1))(*flat)
    shp = N.FusedShapeC()
    N.check(N.lib().mlora_fused_shape_of(arr, len(flat), C.byref(shp)))
    seg, seq_rows, r = [0], [], 0
    for g in per_job_lengths:
        rows_j = []
        for L in g:
            rows_j.append((r, int(L)))
            r += shp.max_len if padded else int(L)
        seq_rows.append(rows_j)
        seg.append(r)
    return FusedLayout(seg, seq_rows, shp.max_len, shp.sequences, shp.total_tokens, shp.padding_tokens,
                       sum(flat), padded)
