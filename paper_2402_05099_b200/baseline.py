"""The paper's comparison point for the attention microbenchmark (§4.2): attention
computed per sequence over that sequence's OWN copy of prefix || suffix -- what a decode
kernel without prefix sharing does (the FlashAttention baseline).  It runs on this
library's own per-sequence suffix kernels (the tensor-core GEMV for GQA, the SIMT split-K
kernel otherwise), so the measured speedup isolates the method -- inter-sequence batching of
the prefix (§3.2) -- from kernel quality.  Used by `bench.py --config grid`; parity against
the oracle in tests/test_gpu_parity.py."""
from __future__ import annotations

import torch

from . import attn


def per_sequence_cache(pk: torch.Tensor, pv: torch.Tensor, sk: torch.Tensor, sv: torch.Tensor,
                       lens: torch.Tensor):
    """Every sequence's full KV: the prefix [P, Hkv, d] copied in front of its suffix
    [S_cap, Hkv, d] -> (K, V) [B, P + S_cap, Hkv, d] and lengths P + lens[b]."""
    B = sk.shape[0]
    P = pk.shape[0]
    fk = torch.cat([pk.unsqueeze(0).expand(B, *pk.shape), sk], dim=1).contiguous()
    fv = torch.cat([pv.unsqueeze(0).expand(B, *pv.shape), sv], dim=1).contiguous()
    return fk, fv, (lens + P).to(torch.int32)


def per_sequence_attention(q, fk, fv, flens, workspace=None, out=None, lse_out=None, stream=None):
    """Attention of each sequence over its own full cache (per_sequence_cache): O, LSE (f32)."""
    return attn.suffix_attn(q, fk, fv, flens, workspace=workspace, out=out, lse_out=lse_out, stream=stream)
