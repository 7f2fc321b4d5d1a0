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
