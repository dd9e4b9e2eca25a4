"""The Python binding's argument checks: the C ABI sees only pointers and element
strides, so mismatched tensors must be rejected before any call -- dtype and head-dim
agreement of q / K / V, equal K and V shapes and strides, suffix_lens int32 [B], the shape,
dtype and contiguity of caller-supplied outputs, and a tree's extents.  These checks run
before the CUDA-device check, so CPU tensors exercise them here."""
import numpy as np
import pytest
import torch

import paper_2402_05099_b200 as hydra

B, Hq, Hkv, d, P, S = 3, 8, 2, 128, 40, 16
bf = torch.bfloat16


def t(*shape, dtype=bf):
    return torch.zeros(*shape, dtype=dtype)


def args():
    return dict(q=t(B, Hq, d), prefix_k=t(P, Hkv, d), prefix_v=t(P, Hkv, d), suffix_k=t(B, S, Hkv, d),
                suffix_v=t(B, S, Hkv, d), suffix_lens=torch.zeros(B, dtype=torch.int32))


def call(**over):
    a = args()
    a.update(over)
    return hydra.hydragen_attention(**a)


def test_baseline_reaches_the_device_check():
    with pytest.raises(ValueError, match="CUDA"):
        call()


@pytest.mark.parametrize("over,exc,msg", [
    (dict(prefix_k=t(P, Hkv, d, dtype=torch.float32), prefix_v=t(P, Hkv, d, dtype=torch.float32)), TypeError, "dtype"),
    (dict(suffix_v=t(B, S, Hkv, d, dtype=torch.float32)), TypeError, "dtype"),
    (dict(prefix_k=t(P, Hkv, 64), prefix_v=t(P, Hkv, 64)), ValueError, "head dim"),
    (dict(prefix_v=t(P + 1, Hkv, d)), ValueError, "equal shapes"),
    (dict(prefix_v=t(Hkv, P, d).transpose(0, 1)), ValueError, "strides"),
    (dict(suffix_k=t(B + 1, S, Hkv, d), suffix_v=t(B + 1, S, Hkv, d)), ValueError, "suffix_k"),
    (dict(suffix_k=t(B, S, 1, d), suffix_v=t(B, S, 1, d)), ValueError, "Hkv"),
    (dict(suffix_lens=torch.zeros(B, dtype=torch.int64)), ValueError, "int32"),
    (dict(suffix_lens=torch.zeros(B + 1, dtype=torch.int32)), ValueError, "int32"),
    (dict(q=t(B, 7, d)), ValueError, "multiple"),
    (dict(out=t(B, Hq, d, dtype=torch.float16)), TypeError, "out"),
    (dict(out=t(B, Hq + 1, d)), ValueError, "shape"),
    (dict(out=t(B, d, Hq).transpose(1, 2)), ValueError, "contiguous"),
    (dict(lse_out=t(B, Hq, dtype=bf), return_lse=True), TypeError, "lse_out"),
    (dict(lse_out=t(B, Hq + 2, dtype=torch.float32), return_lse=True), ValueError, "lse_out"),
])
def test_hydragen_attention_rejects(over, exc, msg):
    with pytest.raises(exc, match=msg):
        call(**over)


def test_partial_attentions_reject():
    a = args()
    with pytest.raises(TypeError):
        hydra.prefix_attn(a["q"], a["prefix_k"].float(), a["prefix_v"].float())
    with pytest.raises(TypeError, match="out"):
        hydra.prefix_attn(a["q"], a["prefix_k"], a["prefix_v"], out=t(B, Hq, d))  # bf16 partial
    with pytest.raises(ValueError, match="int32"):
        hydra.suffix_attn(a["q"], a["suffix_k"], a["suffix_v"], a["suffix_lens"].long())
    with pytest.raises(ValueError, match="batch"):
        hydra.suffix_attn(a["q"], t(B + 2, S, Hkv, d), t(B + 2, S, Hkv, d), torch.zeros(B, dtype=torch.int32))
    with pytest.raises(ValueError, match="lse_out"):
        hydra.suffix_attn(a["q"], a["suffix_k"], a["suffix_v"], a["suffix_lens"],
                          out=t(B, Hq, d, dtype=torch.float32), lse_out=t(B, Hq + 1, dtype=torch.float32))


def test_paged_rejects():
    a = args()
    pool = t(8, 16, Hkv, d)
    tab = torch.zeros(B, 2, dtype=torch.int32)
    with pytest.raises(ValueError, match="block_table"):
        hydra.suffix_attn_paged(a["q"], pool, pool, tab.long(), a["suffix_lens"])
    with pytest.raises(TypeError):
        hydra.suffix_attn_paged(a["q"], pool.float(), pool.float(), tab, a["suffix_lens"])
    with pytest.raises(ValueError, match="S_cap"):
        hydra.suffix_attn_paged(a["q"], pool, pool, tab, a["suffix_lens"], S_cap=33)


def test_combine_rejects():
    o = torch.zeros(2, 5, d)
    with pytest.raises(ValueError, match="lse"):
        hydra.combine(o, torch.zeros(2, 4))
    with pytest.raises(TypeError):
        hydra.combine(o.double(), torch.zeros(2, 5))
    with pytest.raises(ValueError, match="lse_out"):
        hydra.combine(o, torch.zeros(2, 5), lse_out=torch.zeros(4))


def test_tree_rejects_short_node_pool():
    """tree_attention checks the pooled node K/V against the tree's extents: a
    shorter node_k would otherwise be read out of bounds by the TMA maps."""
    try:
        tree = hydra.Tree([-1, 0, 0], [0, 40, 60], [40, 20, 30], [1, 2, 2])
    except hydra.HydraError:
        pytest.skip("tree creation needs a CUDA device")  # hydra_tree_create uploads its groups
    a = args()
    with pytest.raises(ValueError, match="tokens"):
        hydra.tree_attention(a["q"], tree, t(80, Hkv, d), t(80, Hkv, d), a["suffix_k"], a["suffix_v"],
                             a["suffix_lens"])
