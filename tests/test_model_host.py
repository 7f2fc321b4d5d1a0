"""Host-side logic of the decoder trainer (no GPU): fused token layout."""
import pytest

from paper_2312_02515_b200 import errors
from paper_2312_02515_b200 import model as MD


def test_pack_tokens_packed_layout():
    b = MD.pack_tokens([[[1, 2, 3], [4, 5]], [], [[6]]])
    assert b.seg == [0, 5, 5, 6]
    assert b.seq_offsets == [0, 3, 5, 6] and b.seq_lens == [3, 2, 1]
    assert b.tokens == [1, 2, 3, 4, 5, 6]
    assert b.labels == [2, 3, 0, 5, 0, 0]
    assert b.mask == [1, 1, 0, 1, 0, 0]
    assert b.real_tokens == 6 and not b.padded


def test_pack_tokens_padded_layout_matches_reference_fuse():
    """Global max_len padding, job order then sequence order (lora.cpp:114-158)."""
    b = MD.pack_tokens([[[1, 2, 3], [4, 5]], [[6]]], padded=True)
    assert b.seq_offsets == [0, 3, 6, 9] and b.seg == [0, 6, 9]
    assert b.tokens == [1, 2, 3, 4, 5, 0, 6, 0, 0]
    assert b.mask == [1, 1, 0, 1, 0, 0, 0, 0, 0]
    assert b.seq_lens == [3, 2, 1]


def test_pack_tokens_errors():
    with pytest.raises(errors.UsageError):
        MD.pack_tokens([[], []])
    with pytest.raises(errors.UsageError):
        MD.pack_tokens([[[1], []]])


def test_config_projection_shapes():
    assert [p[1:] for p in MD.CHATGLM2_6B.projections()] == [(4608, 4096), (4096, 4096), (27392, 4096),
                                                              (4096, 13696)]
    assert MD.TINY_LLAMA.head_dim == 64 and len(MD.TINY_LLAMA.projections()) == 7
    assert MD.LLAMA_13B.head_dim == 128
