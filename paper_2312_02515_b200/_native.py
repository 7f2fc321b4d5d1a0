"""ctypes binding of the C ABI in include/mlora.h (libmlora.so, built in-tree).

This is the reference-side binding a Python maintainer would add:
plain pointers and sizes, status codes mapped onto the fusim exception types.
There is no fallback: if the shared library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import re

from . import errors

_PKG = os.path.dirname(os.path.abspath(__file__))
# MLORA_LIBRARY points the binding at another build of the same ABI (A/B runs of two builds)
LIB_PATH = os.environ.get("MLORA_LIBRARY") or os.path.join(_PKG, "libmlora.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "mlora.h")

_lib: C.CDLL | None = None

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f32 = C.c_float


class FusedShapeC(C.Structure):
    _fields_ = [("max_len", i32), ("sequences", i64), ("total_tokens", i64), ("padding_tokens", i64)]


class AttnDescC(C.Structure):
    _fields_ = [("seq_offsets", vp), ("seq_lens", vp), ("rows", i64), ("num_seqs", i32), ("max_len", i32),
                ("heads", i32), ("kv_heads", i32), ("head_dim", i32), ("rope_base", f32), ("softmax_scale", f32),
                ("flags", i32)]


class AdamGroupC(C.Structure):
    _fields_ = [("p", vp), ("g", vp), ("m", vp), ("v", vp), ("p_bf16", vp), ("rows", i64),
                ("cols", i64), ("layout", i32), ("_pad", i32)]


class LayerProjC(C.Structure):
    """mlora_layer_proj (include/mlora.h)."""
    _fields_ = [("d", i32), ("k", i32), ("src", i32), ("src_col0", i32), ("W0", vp), ("A", vp), ("B", vp),
                ("mA", vp), ("vA", vp), ("mB", vp), ("vB", vp), ("A_bf16", vp), ("B_bf16", vp), ("dA", vp),
                ("dB", vp), ("Y", vp), ("H", vp), ("G", vp), ("dX", vp), ("row_sq", vp), ("in_scratch", vp)]


class AdamHparamsC(C.Structure):
    _fields_ = [("beta1", f32), ("beta2", f32), ("eps", f32), ("weight_decay", f32)]


_SIGS = {
    "mlora_abi_version": (i32, []),
    "mlora_status_string": (C.c_char_p, [i32]),
    "mlora_last_error": (C.c_char_p, [vp]),
    "mlora_ctx_create": (i32, [i32, C.POINTER(vp)]),
    "mlora_ctx_destroy": (i32, [vp]),
    "mlora_ctx_num_sms": (i32, [vp]),
    "mlora_ctx_launch_count": (i64, [vp]),
    "mlora_free_launch_count": (i64, []),
    "mlora_ctx_set_profiling": (i32, [vp, i32]),
    "mlora_ctx_profile_read": (i32, [vp, i32, C.POINTER(i64), C.POINTER(C.c_double), i32]),
    "mlora_fused_shape_of": (i32, [C.POINTER(i32), i64, C.POINTER(FusedShapeC)]),
    "mlora_count_launches": (i32, [i32, i32, C.POINTER(i64), C.POINTER(i64)]),
    "mlora_plan_create": (i32, [vp, i32, C.POINTER(i64), C.POINTER(i32), C.POINTER(f32), vp, C.POINTER(vp)]),
    "mlora_plan_destroy": (i32, [vp]),
    "mlora_plan_update": (i32, [vp, C.POINTER(i64), vp]),
    "mlora_plan_rows": (i64, [vp]),
    "mlora_plan_rank_padded": (i32, [vp]),
    "mlora_plan_num_jobs": (i32, [vp]),
    "mlora_plan_rank_offsets": (i32, [vp, C.POINTER(i32)]),
    "mlora_linear_fwd": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp]),
    "mlora_linear_fwd_ex": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp]),
    "mlora_rowsq_blocks": (i32, [i32]),
    "mlora_loss_from_rowsq": (i32, [vp, vp, C.POINTER(vp), C.POINTER(i32), i32, vp, vp]),
    "mlora_down_group": (i32, [vp, vp, i32, i32, C.POINTER(i32), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), vp]),
    "mlora_base_fwd": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp]),
    "mlora_base_dx": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, vp, vp]),
    "mlora_grad_group": (i32, [vp, vp, i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(vp), C.POINTER(vp),
                               C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), vp]),
    "mlora_linear_bwd": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "mlora_pack_adapters": (i32, [vp, vp, i32, i32, C.POINTER(vp), C.POINTER(vp), vp, vp, vp, vp, vp]),
    "mlora_segment_sumsq_loss": (i32, [vp, vp, C.POINTER(vp), C.POINTER(i32), i32, vp, vp]),
    "mlora_zero_nonfinite_rows": (i32, [vp, vp, vp, C.POINTER(vp), C.POINTER(i32), i32, vp]),
    "mlora_fuse_rows": (i32, [vp, i32, C.POINTER(vp), C.POINTER(i64), C.POINTER(i32), i64, i32, vp, vp,
                              C.POINTER(i64), vp]),
    "mlora_adam_step": (i32, [vp, vp, C.POINTER(AdamGroupC), i32, C.POINTER(f32), C.POINTER(i32), f32, f32,
                              f32, f32, vp]),
    "mlora_adam_step_ex": (i32, [vp, vp, C.POINTER(AdamGroupC), i32, C.POINTER(f32), C.POINTER(i32), f32, f32,
                                 f32, f32, vp, vp]),
    # one fused layer step (the trainer hook) and the memory / init helpers
    "mlora_layer_create": (i32, [vp, vp, i32, C.POINTER(LayerProjC), i64, C.POINTER(vp)]),
    "mlora_layer_destroy": (i32, [vp]),
    "mlora_layer_forward_backward": (i32, [vp, vp, vp, vp]),
    "mlora_layer_step": (i32, [vp, vp, C.POINTER(f32), C.POINTER(i32), C.POINTER(AdamHparamsC), vp, vp]),
    "mlora_layer_step_timed": (i32, [vp, vp, C.POINTER(f32), C.POINTER(i32), C.POINTER(AdamHparamsC), vp, vp,
                                     C.POINTER(C.c_double), vp]),
    "mlora_malloc": (i32, [vp, C.c_size_t, C.POINTER(vp)]),
    "mlora_free": (i32, [vp, vp]),
    "mlora_memcpy": (i32, [vp, vp, vp, C.c_size_t, i32, vp]),
    "mlora_memset": (i32, [vp, vp, i32, C.c_size_t, vp]),
    "mlora_stream_sync": (i32, [vp, vp]),
    "mlora_mem_info": (i32, [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "mlora_fill_uniform": (i32, [vp, i64, i32, C.c_uint64, f32, f32, vp]),
    "mlora_ctx_timer_start": (i32, [vp, vp]),
    "mlora_ctx_timer_stop": (i32, [vp, vp, C.POINTER(C.c_double)]),
}

# Optional groups (present once the corresponding kernels are built).
_OPTIONAL = {
    "mlora_f64_gemm": (i32, [i64, i64, i64, vp, i64, i32, vp, i64, i32, vp, i64, vp]),
    "mlora_f64_add": (i32, [i64, vp, vp, vp, vp]),
    "mlora_masked_ce": (i32, [i32, vp, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp]),
    "mlora_rmsnorm_fwd": (i32, [i64, i32, vp, vp, f32, vp, vp, vp]),
    "mlora_rmsnorm_bwd": (i32, [i64, i32, vp, vp, vp, vp, vp, vp, vp, i32, vp]),
    "mlora_rope": (i32, [i64, i32, i32, vp, vp, vp, f32, i32, vp]),
    # decoder-layer kernels (model.py)
    "mlora_embed": (i32, [i64, i32, i32, vp, vp, vp, vp]),
    "mlora_add_rmsnorm": (i32, [i64, i32, vp, vp, vp, f32, vp, vp, vp, vp]),
    "mlora_rmsnorm_bwd_sum": (i32, [i64, i32, i32, C.POINTER(vp), vp, vp, vp, vp, vp, vp]),
    "mlora_swiglu_fwd": (i32, [i64, i32, vp, i64, vp, i64, vp, vp]),
    "mlora_swiglu_bwd": (i32, [i64, i32, vp, i64, vp, i64, vp, vp, i64, vp, i64, vp]),
    "mlora_attn_fwd": (i32, [C.POINTER(AttnDescC), vp, i64, vp, i64, vp, i64, vp, i64, vp, vp]),
    "mlora_attn_rope": (i32, [C.POINTER(AttnDescC), vp, i64, i32, vp, i64, vp]),
    "mlora_attn_bwd": (i32, [C.POINTER(AttnDescC), vp, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, vp, vp, i64,
                             vp, i64, vp, i64, vp]),
    # multi-GPU boundary (NCCL resolved at first use)
    "mlora_comm_id_bytes": (i32, []),
    "mlora_comm_nccl_version": (i32, [C.POINTER(i32)]),
    "mlora_comm_unique_id": (i32, [vp]),
    "mlora_comm_create": (i32, [vp, vp, i32, i32, C.POINTER(vp)]),
    "mlora_comm_destroy": (i32, [vp]),
    "mlora_comm_rank": (i32, [vp]),
    "mlora_comm_size": (i32, [vp]),
    "mlora_broadcast_base": (i32, [vp, i32, C.POINTER(vp), C.POINTER(i64), i32, vp]),
    "mlora_comm_sum_f32": (i32, [vp, vp, i64, vp]),
}


def exported_symbols() -> list[str]:
    """Every function declared in include/mlora.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(mlora_[a-z0-9_]+)\s*\(", text)) - {"mlora_status"})


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2312_02515_b200._build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in {**_SIGS}.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        for name, (res, args) in _OPTIONAL.items():
            if hasattr(L, name):
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, ctx=None) -> None:
    if status == 0:
        return
    L = lib()
    msg = L.mlora_last_error(ctx).decode() if ctx is not None else L.mlora_last_error(None).decode()
    cls = errors.STATUS_TO_ERROR.get(status, errors.Error)
    raise cls(msg or L.mlora_status_string(status).decode())


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
