"""B200-native BatchFusion multi-LoRA linear layer (ASPEN, arXiv 2312.02515).

The hot path — Y = X W0^T + s_j (X_j A_j^T) B_j^T per job row-segment, forward
and backward — runs in hand-written sm_100a kernels (tcgen05 + TMEM + TMA)
behind the C ABI in include/mlora.h.  See DESIGN.md.
"""
from . import errors  # noqa: F401

__all__ = ["errors"]
