"""CPU-only checks of the native boundary: the C-ABI library loads, exports every
symbol include/mlora.h declares, and its host-only entry points (token
accounting, launch counting, error mapping) are integer-exact against the
reference-generated golden fixtures.  No device compute is attempted here."""
import ctypes as C
import json
import os
import subprocess

import pytest

from paper_2312_02515_b200 import _native as N
from paper_2312_02515_b200 import errors as E

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def lib():
    return N.lib()


@pytest.fixture(scope="module")
def host_ref():
    with open(os.path.join(GOLD, "host_ref.json")) as f:
        return json.load(f)


def test_library_exports_every_declared_symbol(lib):
    declared = N.exported_symbols()
    assert len(declared) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_tcgen05_and_tma():
    out = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out


def test_abi_version(lib):
    assert lib.mlora_abi_version() >= 1


def test_fused_shape_of_matches_reference(lib, host_ref):
    for rec in host_ref["fused_shape"]:
        flat = [x for g in rec["groups"] for x in g]
        arr = (C.c_int32 * max(len(flat), 1))(*flat)
        out = N.FusedShapeC()
        N.check(lib.mlora_fused_shape_of(arr, len(flat), C.byref(out)))
        assert (out.max_len, out.sequences, out.total_tokens, out.padding_tokens) == (
            rec["max_len"], rec["sequences"], rec["total_tokens"], rec["padding_tokens"])


def test_count_launches_matches_reference(lib, host_ref):
    for rec in host_ref["count_launches"]:
        s, l = C.c_int64(), C.c_int64()
        N.check(lib.mlora_count_launches(rec["jobs"], rec["fused"], C.byref(s), C.byref(l)))
        assert [s.value, l.value] == rec["out"]
    s, l = C.c_int64(), C.c_int64()
    with pytest.raises(E.UsageError):
        N.check(lib.mlora_count_launches(0, 1, C.byref(s), C.byref(l)))


def test_status_strings(lib):
    for st, name in ((0, "ok"), (1, "usage error"), (2, "shape error"), (3, "routing error"),
                     (4, "numeric error"), (6, "cuda error")):
        assert lib.mlora_status_string(st).decode() == name


def test_no_gpu_context_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = N.vp()
    with pytest.raises(E.CudaError):
        N.check(lib.mlora_ctx_create(0, C.byref(h)))
