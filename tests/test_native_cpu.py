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


def test_comm_host_entry_points(lib):
    """The native multi-GPU boundary resolves NCCL at run time; its host-only
    calls (version, unique id) work without a GPU, and argument errors map to
    the reference's UsageError before any NCCL/CUDA work."""
    v = N.i32()
    N.check(lib.mlora_comm_nccl_version(C.byref(v)))
    assert v.value >= 21800  # NCCL >= 2.18 (ncclGroup + in-place broadcast semantics)
    assert lib.mlora_comm_id_bytes() == 128
    a, b = (C.c_uint8 * 128)(), (C.c_uint8 * 128)()
    N.check(lib.mlora_comm_unique_id(C.cast(a, C.c_void_p)))
    N.check(lib.mlora_comm_unique_id(C.cast(b, C.c_void_p)))
    assert bytes(a) != bytes(b)  # fresh rendezvous id each call
    with pytest.raises(E.UsageError):
        N.check(lib.mlora_comm_unique_id(None))
    with pytest.raises(E.UsageError):
        N.check(lib.mlora_broadcast_base(None, 0, None, None, 0, None))
    assert lib.mlora_comm_rank(None) == -1 and lib.mlora_comm_size(None) == -1
    assert lib.mlora_comm_destroy(None) == 0


def test_decoder_entry_points_validate_before_device_work(lib):
    """The decoder-layer entry points reject bad arguments on the host with the
    reference's error taxonomy before touching the device (fake, never
    dereferenced device pointers; no GPU needed)."""
    fake = 1 << 20  # 16-byte aligned, never dereferenced: every call below fails validation first
    odd = fake + 2  # 2-byte aligned only
    off = (C.c_int32 * 3)()

    def desc(**kw):
        d = dict(seq_offsets=C.addressof(off), seq_lens=None, rows=128, num_seqs=2, max_len=64, heads=4,
                 kv_heads=2, head_dim=64, rope_base=10000.0, softmax_scale=0.125, flags=0)
        d.update(kw)
        return N.AttnDescC(**d)

    def st(fn, *a):
        return fn(*a)

    # attention: shape / usage taxonomy
    assert st(lib.mlora_attn_fwd, C.byref(desc(kv_heads=3)), fake, 256, fake, 128, fake, 128, fake, 256, fake,
              None) == 2
    assert st(lib.mlora_attn_fwd, C.byref(desc(head_dim=96)), fake, 384, fake, 192, fake, 192, fake, 384, fake,
              None) == 2
    assert st(lib.mlora_attn_fwd, C.byref(desc(softmax_scale=0.0)), fake, 256, fake, 128, fake, 128, fake, 256,
              fake, None) == 1
    assert st(lib.mlora_attn_fwd, C.byref(desc(flags=4)), fake, 256, fake, 128, fake, 128, fake, 256, fake,
              None) == 1
    assert st(lib.mlora_attn_fwd, None, fake, 256, fake, 128, fake, 128, fake, 256, fake, None) == 1
    assert st(lib.mlora_attn_fwd, C.byref(desc()), fake, 100, fake, 128, fake, 128, fake, 256, fake, None) == 2
    assert st(lib.mlora_attn_rope, C.byref(desc()), odd, 256, 4, fake, 256, None) == 2
    assert st(lib.mlora_attn_rope, C.byref(desc(rope_base=0.0)), fake, 256, 4, fake, 256, None) == 1
    # SwiGLU / norms / embedding
    assert st(lib.mlora_swiglu_fwd, 4, 12, fake, 12, fake, 12, fake, None) == 2          # f % 8
    assert st(lib.mlora_swiglu_fwd, 4, 16, odd, 16, fake, 16, fake, None) == 2           # misaligned slice
    assert st(lib.mlora_swiglu_bwd, 4, 16, fake, 16, fake, 16, fake, fake, 8, fake, 16, None) == 2  # ld < f
    assert st(lib.mlora_add_rmsnorm, 4, 12, fake, None, fake, 1e-6, None, fake, fake, None) == 2
    assert st(lib.mlora_add_rmsnorm, 4, 16, fake, fake, fake, 1e-6, None, fake, fake, None) == 1  # delta w/o x_out
    assert st(lib.mlora_add_rmsnorm, 4, 16, fake, None, fake, 0.0, None, fake, fake, None) == 1    # eps
    dys = (N.vp * 5)(*([fake] * 5))
    assert st(lib.mlora_rmsnorm_bwd_sum, 4, 16, 5, dys, None, fake, fake, fake, fake, None) == 1   # > 4 inputs
    assert st(lib.mlora_embed, 4, 12, 10, fake, fake, fake, None) == 1                               # h % 8
    assert st(lib.mlora_masked_ce, 2, fake, 4, 64, odd, fake, None, fake, fake, fake, None, None) == 1
