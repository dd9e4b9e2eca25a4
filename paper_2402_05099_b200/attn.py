"""PyTorch-facing API: tensors in, C-ABI calls out (argument marshalling only).

Every step of the computation runs in the CUDA kernels of libhydra.so; PyTorch
provides device memory and the current stream.  Names mirror the paper's App. B
pseudocode: `hydragen_attention(q, prefix_k, prefix_v, suffix_k,
suffix_v, ...)`, plus the two partial attentions, the LSE combine and tree
attention (§3.3).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import Heads, check

_DT = {torch.bfloat16: _lib.HYDRA_BF16, torch.float32: _lib.HYDRA_F32, torch.float16: _lib.HYDRA_F16}


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("hydra kernels need CUDA tensors (there is no CPU path)")


def _stream_ptr(stream: Optional[torch.cuda.Stream], device) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _heads(q: torch.Tensor, Hkv: int, scale: Optional[float]) -> Heads:
    if q.dtype not in (torch.bfloat16, torch.float32):
        raise TypeError(f"q must be bf16 or f32, got {q.dtype}")
    return Heads(q.shape[1], Hkv, q.shape[2], float(scale or 0.0), _DT[q.dtype])


def _squeeze_q(q: torch.Tensor) -> torch.Tensor:
    if q.dim() == 4:  # App. B layout [batch, nq, qheads, dim]; decode has nq == 1 (reading R8)
        if q.shape[1] != 1:
            raise ValueError("only decode (nq == 1) is supported")
        q = q[:, 0]
    if q.dim() != 3 or q.stride(-1) != 1:
        raise ValueError("q must be [B, Hq, d] with a contiguous last dim")
    return q


def _kv3(t: torch.Tensor, name: str) -> torch.Tensor:
    if t.dim() != 3 or t.stride(-1) != 1:
        raise ValueError(f"{name} must be [T, Hkv, d] with a contiguous last dim")
    return t


def _kv4(t: torch.Tensor, name: str) -> torch.Tensor:
    if t.dim() != 4 or t.stride(-1) != 1:
        raise ValueError(f"{name} must be [B, S_cap, Hkv, d] with a contiguous last dim")
    return t


def _workspace(nbytes: int, device, workspace: Optional[torch.Tensor]) -> torch.Tensor:
    if nbytes == 0:
        return workspace if workspace is not None else torch.empty(0, dtype=torch.uint8, device=device)
    if workspace is not None:
        if workspace.numel() * workspace.element_size() < nbytes:
            raise ValueError(f"workspace too small: need {nbytes} bytes")
        return workspace
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


# ------------------------------------------------------------------ partial attentions
def prefix_attn(q: torch.Tensor, prefix_k: torch.Tensor, prefix_v: torch.Tensor, scale: Optional[float] = None,
                workspace: Optional[torch.Tensor] = None, stream=None):
    """Inter-sequence batched prefix attention (§3.2): -> (O_p [B,Hq,d] f32, LSE_p [B,Hq] f32)."""
    q = _squeeze_q(q)
    prefix_k, prefix_v = _kv3(prefix_k, "prefix_k"), _kv3(prefix_v, "prefix_v")
    _require_cuda(q, prefix_k, prefix_v)
    if prefix_k.stride() != prefix_v.stride() or prefix_k.shape != prefix_v.shape:
        raise ValueError("prefix_k and prefix_v must have equal shapes and strides")
    B, Hq, d = q.shape
    P, Hkv = prefix_k.shape[0], prefix_k.shape[1]
    h = _heads(q, Hkv, scale)
    lib = _lib.load()
    o = torch.empty(B, Hq, d, dtype=torch.float32, device=q.device)
    lse = torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_PREFIX, ctypes.byref(h), B, P, 0, 0), q.device, workspace)
    check(lib.hydra_prefix_attn(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1), P, prefix_k.data_ptr(),
                                prefix_v.data_ptr(), prefix_k.stride(0), prefix_k.stride(1), o.data_ptr(),
                                lse.data_ptr(), _ptr(ws), ws.numel(), _stream_ptr(stream, q.device)),
          "hydra_prefix_attn")
    return o, lse


def suffix_attn(q: torch.Tensor, suffix_k: torch.Tensor, suffix_v: torch.Tensor, suffix_lens: torch.Tensor,
                scale: Optional[float] = None, workspace: Optional[torch.Tensor] = None, stream=None,
                out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None):
    """Per-sequence suffix attention (§3.2): -> (O_s [B,Hq,d] f32, LSE_s [B,Hq] f32)."""
    q = _squeeze_q(q)
    suffix_k, suffix_v = _kv4(suffix_k, "suffix_k"), _kv4(suffix_v, "suffix_v")
    _require_cuda(q, suffix_k, suffix_v, suffix_lens)
    if suffix_k.stride() != suffix_v.stride() or suffix_k.shape != suffix_v.shape:
        raise ValueError("suffix_k and suffix_v must have equal shapes and strides")
    if suffix_lens.dtype != torch.int32 or suffix_lens.shape != (q.shape[0],):
        raise ValueError("suffix_lens must be int32 [B]")
    B, Hq, d = q.shape
    S_cap, Hkv = suffix_k.shape[1], suffix_k.shape[2]
    h = _heads(q, Hkv, scale)
    lib = _lib.load()
    o = out if out is not None else torch.empty(B, Hq, d, dtype=torch.float32, device=q.device)
    lse = lse_out if lse_out is not None else torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    if o.dtype != torch.float32 or not o.is_contiguous() or o.numel() != B * Hq * d or not lse.is_contiguous():
        raise ValueError("out must be contiguous f32 [B, Hq, d], lse_out contiguous f32 [B, Hq]")
    ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_SUFFIX, ctypes.byref(h), B, 0, S_cap, 0), q.device,
                    workspace)
    st = suffix_k.stride()
    check(lib.hydra_suffix_attn(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1), suffix_k.data_ptr(),
                                suffix_v.data_ptr(), st[0], st[1], st[2], S_cap, suffix_lens.data_ptr(),
                                o.data_ptr(), lse.data_ptr(), _ptr(ws), ws.numel(), _stream_ptr(stream, q.device)),
          "hydra_suffix_attn")
    return o, lse


def append_kv(k_new: torch.Tensor, v_new: torch.Tensor, suffix_k: torch.Tensor, suffix_v: torch.Tensor,
              suffix_lens: torch.Tensor, stream=None):
    """Decode-loop KV append: suffix_k/v[b, lens[b]] = k/v_new[b]; lens[b] += 1,
    on the device (graph-capturable).  k_new/v_new: [B, Hkv, d] (or [B, 1, Hkv, d])."""
    if k_new.dim() == 4:
        k_new, v_new = k_new[:, 0], v_new[:, 0]
    suffix_k, suffix_v = _kv4(suffix_k, "suffix_k"), _kv4(suffix_v, "suffix_v")
    _require_cuda(k_new, v_new, suffix_k, suffix_v, suffix_lens)
    B, S_cap, Hkv, d = suffix_k.shape
    if k_new.shape != (B, Hkv, d) or v_new.shape != k_new.shape or k_new.stride() != v_new.stride():
        raise ValueError("k_new / v_new must be [B, Hkv, d] with equal strides")
    if suffix_k.stride() != suffix_v.stride():
        raise ValueError("suffix_k and suffix_v must have equal strides")
    if suffix_lens.dtype != torch.int32 or suffix_lens.shape != (B,):
        raise ValueError("suffix_lens must be int32 [B]")
    if k_new.dtype != suffix_k.dtype or v_new.dtype != suffix_v.dtype:
        raise TypeError("k_new / v_new must have the cache dtype")
    h = Heads(Hkv, Hkv, d, 0.0, _DT[suffix_k.dtype])
    st = suffix_k.stride()
    check(_lib.load().hydra_append_kv(ctypes.byref(h), B, k_new.data_ptr(), v_new.data_ptr(), k_new.stride(0),
                                      k_new.stride(1), suffix_k.data_ptr(), suffix_v.data_ptr(), st[0], st[1], st[2],
                                      S_cap, suffix_lens.data_ptr(), _stream_ptr(stream, k_new.device)),
          "hydra_append_kv")


# ------------------------------------------------------------------ paged suffix cache (hydra.h hydra_paging)
def _paging(k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor, B: int,
            S_cap: Optional[int]):
    """Validates pools [n_pages, page_size, Hkv, d] and block_table int32 [B, max_pages];
    returns (Paging, S_cap).  S_cap defaults to max_pages * page_size."""
    if k_pool.dim() != 4 or k_pool.stride(-1) != 1:
        raise ValueError("k_pool must be [n_pages, page_size, Hkv, d] with a contiguous last dim")
    if k_pool.shape != v_pool.shape or k_pool.stride() != v_pool.stride():
        raise ValueError("k_pool and v_pool must have equal shapes and strides")
    if block_table.dtype != torch.int32 or block_table.dim() != 2 or block_table.shape[0] != B \
            or block_table.stride(1) != 1:
        raise ValueError("block_table must be int32 [B, max_pages] with contiguous rows")
    _require_cuda(k_pool, v_pool, block_table)
    n_pages, page_size = k_pool.shape[0], k_pool.shape[1]
    cap = block_table.shape[1] * page_size
    S_cap = cap if S_cap is None else int(S_cap)
    pg = _lib.Paging(block_table.data_ptr(), block_table.stride(0), page_size, n_pages)
    return pg, S_cap


def suffix_attn_paged(q: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor,
                      suffix_lens: torch.Tensor, S_cap: Optional[int] = None, scale: Optional[float] = None,
                      workspace: Optional[torch.Tensor] = None, stream=None):
    """suffix_attn over a paged cache: token t of sequence b is k_pool[block_table[b, t // page_size],
    t % page_size] (reading R14).  -> (O_s [B,Hq,d] f32, LSE_s [B,Hq] f32)."""
    q = _squeeze_q(q)
    _require_cuda(q, suffix_lens)
    B, Hq, d = q.shape
    if suffix_lens.dtype != torch.int32 or suffix_lens.shape != (B,):
        raise ValueError("suffix_lens must be int32 [B]")
    pg, S_cap = _paging(k_pool, v_pool, block_table, B, S_cap)
    h = _heads(q, k_pool.shape[2], scale)
    lib = _lib.load()
    o = torch.empty(B, Hq, d, dtype=torch.float32, device=q.device)
    lse = torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_SUFFIX, ctypes.byref(h), B, 0, S_cap, 0), q.device,
                    workspace)
    st = k_pool.stride()
    check(lib.hydra_suffix_attn_paged(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1),
                                      k_pool.data_ptr(), v_pool.data_ptr(), st[0], st[1], st[2], ctypes.byref(pg),
                                      S_cap, suffix_lens.data_ptr(), o.data_ptr(), lse.data_ptr(), _ptr(ws),
                                      ws.numel(), _stream_ptr(stream, q.device)),
          "hydra_suffix_attn_paged")
    return o, lse


def append_kv_paged(k_new: torch.Tensor, v_new: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor,
                    block_table: torch.Tensor, suffix_lens: torch.Tensor, S_cap: Optional[int] = None, stream=None):
    """append_kv into a paged cache: row lens[b] % page_size of page block_table[b, lens[b] // page_size]
    receives k/v_new[b]; lens[b] += 1 on the device (graph-capturable)."""
    if k_new.dim() == 4:
        k_new, v_new = k_new[:, 0], v_new[:, 0]
    B = k_new.shape[0]
    pg, S_cap = _paging(k_pool, v_pool, block_table, B, S_cap)
    _require_cuda(k_new, v_new, suffix_lens)
    Hkv, d = k_pool.shape[2], k_pool.shape[3]
    if k_new.shape != (B, Hkv, d) or v_new.shape != k_new.shape or k_new.stride() != v_new.stride():
        raise ValueError("k_new / v_new must be [B, Hkv, d] with equal strides")
    if suffix_lens.dtype != torch.int32 or suffix_lens.shape != (B,):
        raise ValueError("suffix_lens must be int32 [B]")
    if k_new.dtype != k_pool.dtype or v_new.dtype != v_pool.dtype:
        raise TypeError("k_new / v_new must have the cache dtype")
    h = Heads(Hkv, Hkv, d, 0.0, _DT[k_pool.dtype])
    st = k_pool.stride()
    check(_lib.load().hydra_append_kv_paged(ctypes.byref(h), B, k_new.data_ptr(), v_new.data_ptr(),
                                            k_new.stride(0), k_new.stride(1), k_pool.data_ptr(), v_pool.data_ptr(),
                                            st[0], st[1], st[2], ctypes.byref(pg), S_cap, suffix_lens.data_ptr(),
                                            _stream_ptr(stream, k_new.device)),
          "hydra_append_kv_paged")


def hydragen_attention_paged(q: torch.Tensor, prefix_k: torch.Tensor, prefix_v: torch.Tensor,
                             k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor,
                             suffix_lens: torch.Tensor, S_cap: Optional[int] = None, scale: Optional[float] = None,
                             out_dtype=None, return_lse: bool = False, workspace: Optional[torch.Tensor] = None,
                             out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None,
                             stream=None, aux_stream=None):
    """hydragen_attention with the suffixes in a paged cache (pools [n_pages, page_size, Hkv, d],
    block_table int32 [B, max_pages]); the prefix stays a dense [P, Hkv, d] tensor."""
    q = _squeeze_q(q)
    prefix_k, prefix_v = _kv3(prefix_k, "prefix_k"), _kv3(prefix_v, "prefix_v")
    _require_cuda(q, prefix_k, prefix_v, suffix_lens)
    if prefix_k.stride() != prefix_v.stride():
        raise ValueError("K and V must share strides")
    B, Hq, d = q.shape
    P, Hkv = prefix_k.shape[0], prefix_k.shape[1]
    if k_pool.dim() != 4 or k_pool.shape[2] != Hkv:
        raise ValueError("k_pool must be [n_pages, page_size, Hkv, d]")
    if suffix_lens.dtype != torch.int32 or suffix_lens.shape != (B,):
        raise ValueError("suffix_lens must be int32 [B]")
    pg, S_cap = _paging(k_pool, v_pool, block_table, B, S_cap)
    h = _heads(q, Hkv, scale)
    lib = _lib.load()
    out_dtype = out_dtype or (torch.bfloat16 if q.dtype == torch.bfloat16 else torch.float32)
    if out is None:
        out = torch.empty(B, Hq, d, dtype=out_dtype, device=q.device)
    if return_lse and lse_out is None:
        lse_out = torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_ATTN, ctypes.byref(h), B, P, S_cap, 0), q.device,
                    workspace)
    ss = k_pool.stride()
    aux = None if aux_stream is None else aux_stream.cuda_stream
    check(lib.hydra_attn_paged(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1), P, prefix_k.data_ptr(),
                               prefix_v.data_ptr(), prefix_k.stride(0), prefix_k.stride(1), k_pool.data_ptr(),
                               v_pool.data_ptr(), ss[0], ss[1], ss[2], ctypes.byref(pg), S_cap,
                               suffix_lens.data_ptr(), out.data_ptr(), _DT[out.dtype], _ptr(lse_out), _ptr(ws),
                               ws.numel(), _stream_ptr(stream, q.device), aux),
          "hydra_attn_paged")
    return (out, lse_out) if return_lse else out


def combine(o_parts: torch.Tensor, lse_parts: torch.Tensor, out_dtype=torch.bfloat16, return_lse: bool = True,
            out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None, stream=None):
    """n-ary LSE combine (Eq. 5 / App. B combine_lse).

    o_parts: [n, rows, d] (f32 or f16, rows may be any leading shape flattened; parts may
    sit at any stride, e.g. slices of an all-gathered exchange buffer), lse_parts: [n, rows]
    f32.  Returns (out [rows, d] in out_dtype, lse [rows] f32).  out_dtype float16 (from f32
    parts) packs partials for a cross-GPU exchange.
    """
    _require_cuda(o_parts, lse_parts)
    n = o_parts.shape[0]
    d = o_parts.shape[-1]
    o2 = o_parts.reshape(n, -1, d)
    l2 = lse_parts.reshape(n, -1)
    rows = o2.shape[1]
    if l2.shape[1] != rows or l2.dtype != torch.float32:
        raise ValueError("lse_parts must be f32 with one value per row of each part")
    if o2.stride(2) != 1 or (rows > 1 and o2.stride(1) != d) or (rows > 1 and l2.stride(1) != 1):
        raise ValueError("parts must be row-contiguous")
    if out is None:
        out = torch.empty(rows, d, dtype=out_dtype, device=o_parts.device)
    out_dtype = out.dtype
    if out.numel() != rows * d or not out.is_contiguous():
        raise ValueError("out must be a contiguous [rows, d] tensor")
    lse = lse_out if lse_out is not None else (
        torch.empty(rows, dtype=torch.float32, device=o_parts.device) if return_lse else None)
    check(_lib.load().hydra_combine(rows, d, n, o2.data_ptr(), _DT[o2.dtype], o2.stride(0), l2.data_ptr(),
                                    l2.stride(0), out.data_ptr(), _DT[out_dtype], _ptr(lse),
                                    _stream_ptr(stream, o_parts.device)), "hydra_combine")
    return out, lse


# ------------------------------------------------------------------ whole decode-step attention
def attn_workspace_bytes(q, prefix_len: int, suffix_cap: int, Hkv: int, scale=None) -> int:
    q = _squeeze_q(q)
    h = _heads(q, Hkv, scale)
    return int(_lib.load().hydra_workspace_size(_lib.HYDRA_OP_ATTN, ctypes.byref(h), q.shape[0], prefix_len,
                                                suffix_cap, 0))


def hydragen_attention(q: torch.Tensor, prefix_k: torch.Tensor, prefix_v: torch.Tensor, suffix_k: torch.Tensor,
                       suffix_v: torch.Tensor, suffix_lens: torch.Tensor, scale: Optional[float] = None,
                       out_dtype=None, return_lse: bool = False, workspace: Optional[torch.Tensor] = None,
                       out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None,
                       stream=None, aux_stream=None):
    """App. B `hydragen_attention` for one decode step.

    q [B, Hq, d] (or [B, 1, Hq, d]); prefix_k/v [P, Hkv, d]; suffix_k/v [B, S_cap, Hkv, d];
    suffix_lens int32 [B].  Returns out [B, Hq, d] (bf16 for bf16 inputs, f32 for f32)
    and, if return_lse, the merged LSE [B, Hq].  With aux_stream the prefix kernel runs
    on it concurrently with the suffix kernel.
    """
    q = _squeeze_q(q)
    prefix_k, prefix_v = _kv3(prefix_k, "prefix_k"), _kv3(prefix_v, "prefix_v")
    suffix_k, suffix_v = _kv4(suffix_k, "suffix_k"), _kv4(suffix_v, "suffix_v")
    _require_cuda(q, prefix_k, prefix_v, suffix_k, suffix_v, suffix_lens)
    if prefix_k.stride() != prefix_v.stride() or suffix_k.stride() != suffix_v.stride():
        raise ValueError("K and V must share strides")
    B, Hq, d = q.shape
    P, Hkv = prefix_k.shape[0], prefix_k.shape[1]
    S_cap = suffix_k.shape[1]
    if suffix_k.shape[2] != Hkv or suffix_k.shape[0] != B:
        raise ValueError("suffix_k must be [B, S_cap, Hkv, d]")
    if suffix_lens.dtype != torch.int32 or suffix_lens.shape != (B,):
        raise ValueError("suffix_lens must be int32 [B]")
    h = _heads(q, Hkv, scale)
    lib = _lib.load()
    out_dtype = out_dtype or (torch.bfloat16 if q.dtype == torch.bfloat16 else torch.float32)
    if out is None:
        out = torch.empty(B, Hq, d, dtype=out_dtype, device=q.device)
    if return_lse and lse_out is None:
        lse_out = torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_ATTN, ctypes.byref(h), B, P, S_cap, 0), q.device,
                    workspace)
    ss = suffix_k.stride()
    aux = None if aux_stream is None else aux_stream.cuda_stream
    check(lib.hydra_attn(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1), P, prefix_k.data_ptr(),
                         prefix_v.data_ptr(), prefix_k.stride(0), prefix_k.stride(1), suffix_k.data_ptr(),
                         suffix_v.data_ptr(), ss[0], ss[1], ss[2], S_cap, suffix_lens.data_ptr(), out.data_ptr(),
                         _DT[out.dtype], _ptr(lse_out), _ptr(ws), ws.numel(), _stream_ptr(stream, q.device), aux),
          "hydra_attn")
    return (out, lse_out) if return_lse else out


# ------------------------------------------------------------------ tree attention (§3.3)
class Tree:
    """Sharing tree (§3.3, Fig. 2): parent[n] (root -1), node_off/node_len into the pooled
    node K/V, leaf_of_seq[b].  Validated and grouped by the C library (hydra_tree_create)."""

    def __init__(self, parent: Sequence[int], node_off: Sequence[int], node_len: Sequence[int],
                 leaf_of_seq: Sequence[int]):
        lib = _lib.load()
        self.parent = np.ascontiguousarray(parent, np.int32)
        self.node_off = np.ascontiguousarray(node_off, np.int64)
        self.node_len = np.ascontiguousarray(node_len, np.int64)
        self.leaf_of_seq = np.ascontiguousarray(leaf_of_seq, np.int32)
        self.B = int(self.leaf_of_seq.shape[0])
        handle = ctypes.c_void_p()
        check(lib.hydra_tree_create(self.parent.ctypes.data, self.node_off.ctypes.data, self.node_len.ctypes.data,
                                    len(self.parent), self.leaf_of_seq.ctypes.data, self.B, ctypes.byref(handle)),
              "hydra_tree_create")
        self._h = handle

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("tree destroyed")
        return self._h

    def depth(self) -> int:
        return int(_lib.load().hydra_tree_depth(self.handle))

    def group_size(self, node: int) -> int:
        return int(_lib.load().hydra_tree_group_size(self.handle, node))

    def destroy(self):
        if self._h is not None:
            _lib.load().hydra_tree_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def tree_attention(q: torch.Tensor, tree: Tree, node_k: torch.Tensor, node_v: torch.Tensor,
                   suffix_k: torch.Tensor, suffix_v: torch.Tensor, suffix_lens: torch.Tensor,
                   scale: Optional[float] = None, out_dtype=None, return_lse: bool = False,
                   workspace: Optional[torch.Tensor] = None, stream=None, aux_stream=None):
    """Decomposition at every tree vertex (§3.3) + suffix + n-ary combine.  With
    `aux_stream` the node attention and the suffix run concurrently on disjoint SM sets."""
    q = _squeeze_q(q)
    node_k, node_v = _kv3(node_k, "node_k"), _kv3(node_v, "node_v")
    suffix_k, suffix_v = _kv4(suffix_k, "suffix_k"), _kv4(suffix_v, "suffix_v")
    _require_cuda(q, node_k, node_v, suffix_k, suffix_v, suffix_lens)
    B, Hq, d = q.shape
    if B != tree.B:
        raise ValueError("q batch does not match the tree's sequence count")
    Hkv = node_k.shape[1]
    S_cap = suffix_k.shape[1]
    h = _heads(q, Hkv, scale)
    lib = _lib.load()
    out_dtype = out_dtype or (torch.bfloat16 if q.dtype == torch.bfloat16 else torch.float32)
    out = torch.empty(B, Hq, d, dtype=out_dtype, device=q.device)
    lse = torch.empty(B, Hq, dtype=torch.float32, device=q.device) if return_lse else None
    ws = _workspace(lib.hydra_tree_workspace_size(ctypes.byref(h), tree.handle, S_cap), q.device, workspace)
    ss = suffix_k.stride()
    check(lib.hydra_tree_attn(ctypes.byref(h), tree.handle, q.data_ptr(), q.stride(0), q.stride(1),
                              node_k.data_ptr(), node_v.data_ptr(), node_k.stride(0), node_k.stride(1),
                              suffix_k.data_ptr(), suffix_v.data_ptr(), ss[0], ss[1], ss[2], S_cap,
                              suffix_lens.data_ptr(), out.data_ptr(), _DT[out_dtype], _ptr(lse), _ptr(ws),
                              ws.numel(), _stream_ptr(stream, q.device),
                              _stream_ptr(aux_stream, q.device) if aux_stream is not None else None),
          "hydra_tree_attn")
    return (out, lse) if return_lse else out


def tree_attention_paged(q: torch.Tensor, tree: Tree, node_k: torch.Tensor, node_v: torch.Tensor,
                         k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor,
                         suffix_lens: torch.Tensor, S_cap: Optional[int] = None, scale: Optional[float] = None,
                         out_dtype=None, return_lse: bool = False, workspace: Optional[torch.Tensor] = None,
                         stream=None, aux_stream=None):
    """tree_attention with the suffixes in a paged cache (pools [n_pages, page_size, Hkv, d],
    block_table int32 [B, max_pages]; reading R14)."""
    q = _squeeze_q(q)
    node_k, node_v = _kv3(node_k, "node_k"), _kv3(node_v, "node_v")
    _require_cuda(q, node_k, node_v, suffix_lens)
    B, Hq, d = q.shape
    if B != tree.B:
        raise ValueError("q batch does not match the tree's sequence count")
    Hkv = node_k.shape[1]
    if k_pool.dim() != 4 or k_pool.shape[2] != Hkv:
        raise ValueError("k_pool must be [n_pages, page_size, Hkv, d]")
    if suffix_lens.dtype != torch.int32 or suffix_lens.shape != (B,):
        raise ValueError("suffix_lens must be int32 [B]")
    pg, S_cap = _paging(k_pool, v_pool, block_table, B, S_cap)
    h = _heads(q, Hkv, scale)
    lib = _lib.load()
    out_dtype = out_dtype or (torch.bfloat16 if q.dtype == torch.bfloat16 else torch.float32)
    out = torch.empty(B, Hq, d, dtype=out_dtype, device=q.device)
    lse = torch.empty(B, Hq, dtype=torch.float32, device=q.device) if return_lse else None
    ws = _workspace(lib.hydra_tree_workspace_size(ctypes.byref(h), tree.handle, S_cap), q.device, workspace)
    ss = k_pool.stride()
    check(lib.hydra_tree_attn_paged(ctypes.byref(h), tree.handle, q.data_ptr(), q.stride(0), q.stride(1),
                                    node_k.data_ptr(), node_v.data_ptr(), node_k.stride(0), node_k.stride(1),
                                    k_pool.data_ptr(), v_pool.data_ptr(), ss[0], ss[1], ss[2], ctypes.byref(pg),
                                    S_cap, suffix_lens.data_ptr(), out.data_ptr(), _DT[out_dtype], _ptr(lse),
                                    _ptr(ws), ws.numel(), _stream_ptr(stream, q.device),
                                    _stream_ptr(aux_stream, q.device) if aux_stream is not None else None),
          "hydra_tree_attn_paged")
    return (out, lse) if return_lse else out
