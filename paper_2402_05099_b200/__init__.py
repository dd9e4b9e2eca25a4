"""hydra-b200: exact shared-prefix decode attention (Hydragen, arXiv 2402.05099) on B200.

All arithmetic runs in libhydra.so (hand-written sm_100a CUDA: tcgen05/TMEM/TMA
prefix kernel, split-K suffix GEMV, LSE combine); this package only marshals
torch tensors into the C ABI declared in include/hydra.h.
"""
from ._lib import HydraError, get_config, load, set_config, version  # noqa: F401
from .attn import (  # noqa: F401
    Tree,
    append_kv,
    append_kv_paged,
    attn_workspace_bytes,
    combine,
    combine_scatter,
    hydragen_attention,
    hydragen_attention_paged,
    prefix_attn,
    suffix_attn,
    suffix_attn_paged,
    tree_attention,
    tree_attention_paged,
    workspace_bytes_tree,
)
