"""PyTorch-facing API: tensors in, C-ABI calls out (argument marshalling only).

Every step of the computation runs in the CUDA kernels of libhydra.so; PyTorch
provides device memory and the current stream.  Names mirror the paper's App. B
pseudocode: `hydragen_attention(q, prefix_k, prefix_v, suffix_k,
suffix_v, ...)`, plus the two partial attentions, the LSE combine and tree
attention (§3.3).

The C ABI receives only pointers and element strides, so this layer checks that the
tensors agree with each other (dtypes, head dims, shapes, strides, caller-supplied
outputs) before any call: a mismatch raises here instead of reading or writing out of
bounds on the device.  Shape and dtype checks run before the CUDA-device check, so they
are exercised by the CPU test suite.
"""
from __future__ import annotations

import contextlib
import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import Heads, check

_DT = {torch.bfloat16: _lib.HYDRA_BF16, torch.float32: _lib.HYDRA_F32, torch.float16: _lib.HYDRA_F16}


# ------------------------------------------------------------------ validation helpers
def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("hydra kernels need CUDA tensors (there is no CPU path)")
    devs = {t.device for t in ts if t is not None}
    if len(devs) > 1:
        raise ValueError(f"all tensors must be on one device, got {sorted(map(str, devs))}")


def _on(device):
    """Make `device` current for the library call (the C ABI launches on the current device)."""
    return torch.cuda.device(device) if device.type == "cuda" else contextlib.nullcontext()


def _stream_ptr(stream: Optional[torch.cuda.Stream], device) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _heads(q: torch.Tensor, Hkv: int, scale: Optional[float]) -> Heads:
    if q.dtype not in (torch.bfloat16, torch.float32):
        raise TypeError(f"q must be bf16 or f32, got {q.dtype}")
    if Hkv <= 0 or q.shape[1] % Hkv:
        raise ValueError(f"Hq={q.shape[1]} must be a positive multiple of Hkv={Hkv}")
    return Heads(q.shape[1], Hkv, q.shape[2], float(scale or 0.0), _DT[q.dtype])


def _squeeze_q(q: torch.Tensor) -> torch.Tensor:
    if q.dim() == 4:  # App. B layout [batch, nq, qheads, dim]; decode has nq == 1 (reading R8)
        if q.shape[1] != 1:
            raise ValueError("only decode (nq == 1) is supported")
        q = q[:, 0]
    if q.dim() != 3 or q.stride(-1) != 1:
        raise ValueError("q must be [B, Hq, d] with a contiguous last dim")
    return q


def _kv_pair(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, name: str, dims: int, layout: str):
    """K and V of one segment: `dims`-D, contiguous head dim, same shape and strides as each
    other (the C ABI applies K's strides to V), q's dtype and head dim."""
    if k.dim() != dims or v.dim() != dims or k.stride(-1) != 1 or v.stride(-1) != 1:
        raise ValueError(f"{name}_k / {name}_v must be {layout} with a contiguous last dim")
    if k.shape != v.shape or k.stride() != v.stride():
        raise ValueError(f"{name}_k and {name}_v must have equal shapes and strides")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError(f"{name}_k / {name}_v dtype ({k.dtype}, {v.dtype}) must equal q's ({q.dtype})")
    if k.shape[-1] != q.shape[-1]:
        raise ValueError(f"{name} head dim {k.shape[-1]} != q head dim {q.shape[-1]}")


def _check_lens(lens: torch.Tensor, B: int):
    if lens.dtype != torch.int32 or lens.shape != (B,) or (B > 1 and lens.stride(0) != 1):
        raise ValueError("suffix_lens must be a contiguous int32 [B] tensor")


def _check_out(out: torch.Tensor, shape, dtypes, name="out"):
    if out.dtype not in dtypes:
        raise TypeError(f"{name} must have dtype in {[str(d) for d in dtypes]}, got {out.dtype}")
    if tuple(out.shape) != tuple(shape) or not out.is_contiguous():
        raise ValueError(f"{name} must be a contiguous tensor of shape {tuple(shape)}, got {tuple(out.shape)}")


def _outputs(q, B, Hq, d, out, lse_out, return_lse, out_dtype):
    out_dtype = out_dtype or (torch.bfloat16 if q.dtype == torch.bfloat16 else torch.float32)
    if out is None:
        out = torch.empty(B, Hq, d, dtype=out_dtype, device=q.device)
    _check_out(out, (B, Hq, d), (torch.bfloat16, torch.float32))
    if return_lse and lse_out is None:
        lse_out = torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    if lse_out is not None:
        _check_out(lse_out, (B, Hq), (torch.float32,), "lse_out")
    return out, lse_out


def _partials(q, B, Hq, d, out, lse_out):
    o = out if out is not None else torch.empty(B, Hq, d, dtype=torch.float32, device=q.device)
    lse = lse_out if lse_out is not None else torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    _check_out(o, (B, Hq, d), (torch.float32,))
    _check_out(lse, (B, Hq), (torch.float32,), "lse_out")
    return o, lse


def _workspace(nbytes: int, device, workspace: Optional[torch.Tensor]) -> torch.Tensor:
    if workspace is not None:
        if not workspace.is_contiguous() or workspace.numel() * workspace.element_size() < nbytes:
            raise ValueError(f"workspace must be contiguous with at least {nbytes} bytes")
        return workspace
    return torch.empty(max(nbytes, 0), dtype=torch.uint8, device=device)


def _nbytes(t: torch.Tensor) -> int:
    return t.numel() * t.element_size()


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


# ------------------------------------------------------------------ partial attentions
def prefix_attn(q: torch.Tensor, prefix_k: torch.Tensor, prefix_v: torch.Tensor, scale: Optional[float] = None,
                workspace: Optional[torch.Tensor] = None, stream=None, out: Optional[torch.Tensor] = None,
                lse_out: Optional[torch.Tensor] = None):
    """Inter-sequence batched prefix attention (§3.2): -> (O_p [B,Hq,d] f32, LSE_p [B,Hq] f32)."""
    q = _squeeze_q(q)
    _kv_pair(q, prefix_k, prefix_v, "prefix", 3, "[P, Hkv, d]")
    B, Hq, d = q.shape
    P, Hkv = prefix_k.shape[0], prefix_k.shape[1]
    h = _heads(q, Hkv, scale)
    o, lse = _partials(q, B, Hq, d, out, lse_out)
    _require_cuda(q, prefix_k, prefix_v, out, lse_out, workspace)
    lib = _lib.load()
    with _on(q.device):
        ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_PREFIX, ctypes.byref(h), B, P, 0, 0), q.device,
                        workspace)
        check(lib.hydra_prefix_attn(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1), P,
                                    prefix_k.data_ptr(), prefix_v.data_ptr(), prefix_k.stride(0), prefix_k.stride(1),
                                    o.data_ptr(), lse.data_ptr(), _ptr(ws), _nbytes(ws),
                                    _stream_ptr(stream, q.device)), "hydra_prefix_attn")
    return o, lse


def suffix_attn(q: torch.Tensor, suffix_k: torch.Tensor, suffix_v: torch.Tensor, suffix_lens: torch.Tensor,
                scale: Optional[float] = None, workspace: Optional[torch.Tensor] = None, stream=None,
                out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None):
    """Per-sequence suffix attention (§3.2): -> (O_s [B,Hq,d] f32, LSE_s [B,Hq] f32)."""
    q = _squeeze_q(q)
    _kv_pair(q, suffix_k, suffix_v, "suffix", 4, "[B, S_cap, Hkv, d]")
    B, Hq, d = q.shape
    if suffix_k.shape[0] != B:
        raise ValueError(f"suffix_k batch {suffix_k.shape[0]} != q batch {B}")
    _check_lens(suffix_lens, B)
    S_cap, Hkv = suffix_k.shape[1], suffix_k.shape[2]
    h = _heads(q, Hkv, scale)
    o, lse = _partials(q, B, Hq, d, out, lse_out)
    _require_cuda(q, suffix_k, suffix_v, suffix_lens, out, lse_out, workspace)
    lib = _lib.load()
    st = suffix_k.stride()
    with _on(q.device):
        ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_SUFFIX, ctypes.byref(h), B, 0, S_cap, 0), q.device,
                        workspace)
        check(lib.hydra_suffix_attn(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1), suffix_k.data_ptr(),
                                    suffix_v.data_ptr(), st[0], st[1], st[2], S_cap, suffix_lens.data_ptr(),
                                    o.data_ptr(), lse.data_ptr(), _ptr(ws), _nbytes(ws),
                                    _stream_ptr(stream, q.device)), "hydra_suffix_attn")
    return o, lse


def append_kv(k_new: torch.Tensor, v_new: torch.Tensor, suffix_k: torch.Tensor, suffix_v: torch.Tensor,
              suffix_lens: torch.Tensor, stream=None):
    """Decode-loop KV append: suffix_k/v[b, lens[b]] = k/v_new[b]; lens[b] += 1,
    on the device (graph-capturable).  k_new/v_new: [B, Hkv, d] (or [B, 1, Hkv, d])."""
    if k_new.dim() == 4:
        k_new, v_new = k_new[:, 0], v_new[:, 0]
    if suffix_k.dim() != 4 or suffix_k.stride(-1) != 1:
        raise ValueError("suffix_k must be [B, S_cap, Hkv, d] with a contiguous last dim")
    B, S_cap, Hkv, d = suffix_k.shape
    if suffix_v.shape != suffix_k.shape or suffix_k.stride() != suffix_v.stride():
        raise ValueError("suffix_k and suffix_v must have equal shapes and strides")
    if k_new.shape != (B, Hkv, d) or v_new.shape != k_new.shape or k_new.stride() != v_new.stride() \
            or k_new.stride(-1) != 1:
        raise ValueError("k_new / v_new must be [B, Hkv, d] with equal strides")
    _check_lens(suffix_lens, B)
    if k_new.dtype != suffix_k.dtype or v_new.dtype != suffix_v.dtype or suffix_k.dtype != suffix_v.dtype:
        raise TypeError("k_new / v_new must have the cache dtype")
    if suffix_k.dtype not in (torch.bfloat16, torch.float32):
        raise TypeError("the cache must be bf16 or f32")
    _require_cuda(k_new, v_new, suffix_k, suffix_v, suffix_lens)
    h = Heads(Hkv, Hkv, d, 0.0, _DT[suffix_k.dtype])
    st = suffix_k.stride()
    with _on(k_new.device):
        check(_lib.load().hydra_append_kv(ctypes.byref(h), B, k_new.data_ptr(), v_new.data_ptr(), k_new.stride(0),
                                          k_new.stride(1), suffix_k.data_ptr(), suffix_v.data_ptr(), st[0], st[1],
                                          st[2], S_cap, suffix_lens.data_ptr(), _stream_ptr(stream, k_new.device)),
              "hydra_append_kv")


# ------------------------------------------------------------------ paged suffix cache (hydra.h hydra_paging)
def _paging(q: Optional[torch.Tensor], k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor,
            B: int, S_cap: Optional[int]):
    """Validates pools [n_pages, page_size, Hkv, d] and block_table int32 [B, max_pages];
    returns (Paging, S_cap).  S_cap defaults to max_pages * page_size."""
    if q is not None:
        _kv_pair(q, k_pool, v_pool, "pool", 4, "[n_pages, page_size, Hkv, d]")
    elif k_pool.dim() != 4 or k_pool.stride(-1) != 1 or k_pool.shape != v_pool.shape \
            or k_pool.stride() != v_pool.stride():
        raise ValueError("k_pool / v_pool must be equal [n_pages, page_size, Hkv, d] tensors, last dim contiguous")
    if block_table.dtype != torch.int32 or block_table.dim() != 2 or block_table.shape[0] != B \
            or block_table.stride(1) != 1:
        raise ValueError("block_table must be int32 [B, max_pages] with contiguous rows")
    n_pages, page_size = k_pool.shape[0], k_pool.shape[1]
    cap = block_table.shape[1] * page_size
    S_cap = cap if S_cap is None else int(S_cap)
    if S_cap > cap:
        raise ValueError(f"S_cap {S_cap} exceeds the block table's {cap} tokens")
    pg = _lib.Paging(block_table.data_ptr(), block_table.stride(0), page_size, n_pages)
    return pg, S_cap


def suffix_attn_paged(q: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor,
                      suffix_lens: torch.Tensor, S_cap: Optional[int] = None, scale: Optional[float] = None,
                      workspace: Optional[torch.Tensor] = None, stream=None, out: Optional[torch.Tensor] = None,
                      lse_out: Optional[torch.Tensor] = None):
    """suffix_attn over a paged cache: token t of sequence b is k_pool[block_table[b, t // page_size],
    t % page_size] (reading R14).  -> (O_s [B,Hq,d] f32, LSE_s [B,Hq] f32)."""
    q = _squeeze_q(q)
    B, Hq, d = q.shape
    _check_lens(suffix_lens, B)
    pg, S_cap = _paging(q, k_pool, v_pool, block_table, B, S_cap)
    h = _heads(q, k_pool.shape[2], scale)
    o, lse = _partials(q, B, Hq, d, out, lse_out)
    _require_cuda(q, k_pool, v_pool, block_table, suffix_lens, out, lse_out, workspace)
    lib = _lib.load()
    st = k_pool.stride()
    with _on(q.device):
        ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_SUFFIX, ctypes.byref(h), B, 0, S_cap, 0), q.device,
                        workspace)
        check(lib.hydra_suffix_attn_paged(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1),
                                          k_pool.data_ptr(), v_pool.data_ptr(), st[0], st[1], st[2],
                                          ctypes.byref(pg), S_cap, suffix_lens.data_ptr(), o.data_ptr(),
                                          lse.data_ptr(), _ptr(ws), _nbytes(ws), _stream_ptr(stream, q.device)),
              "hydra_suffix_attn_paged")
    return o, lse


def append_kv_paged(k_new: torch.Tensor, v_new: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor,
                    block_table: torch.Tensor, suffix_lens: torch.Tensor, S_cap: Optional[int] = None, stream=None):
    """append_kv into a paged cache: row lens[b] % page_size of page block_table[b, lens[b] // page_size]
    receives k/v_new[b]; lens[b] += 1 on the device (graph-capturable)."""
    if k_new.dim() == 4:
        k_new, v_new = k_new[:, 0], v_new[:, 0]
    B = k_new.shape[0]
    pg, S_cap = _paging(None, k_pool, v_pool, block_table, B, S_cap)
    Hkv, d = k_pool.shape[2], k_pool.shape[3]
    if k_new.shape != (B, Hkv, d) or v_new.shape != k_new.shape or k_new.stride() != v_new.stride() \
            or k_new.stride(-1) != 1:
        raise ValueError("k_new / v_new must be [B, Hkv, d] with equal strides")
    _check_lens(suffix_lens, B)
    if k_new.dtype != k_pool.dtype or v_new.dtype != v_pool.dtype or k_pool.dtype != v_pool.dtype:
        raise TypeError("k_new / v_new must have the cache dtype")
    if k_pool.dtype not in (torch.bfloat16, torch.float32):
        raise TypeError("the cache must be bf16 or f32")
    _require_cuda(k_new, v_new, k_pool, v_pool, block_table, suffix_lens)
    h = Heads(Hkv, Hkv, d, 0.0, _DT[k_pool.dtype])
    st = k_pool.stride()
    with _on(k_new.device):
        check(_lib.load().hydra_append_kv_paged(ctypes.byref(h), B, k_new.data_ptr(), v_new.data_ptr(),
                                                k_new.stride(0), k_new.stride(1), k_pool.data_ptr(),
                                                v_pool.data_ptr(), st[0], st[1], st[2], ctypes.byref(pg), S_cap,
                                                suffix_lens.data_ptr(), _stream_ptr(stream, k_new.device)),
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
    _kv_pair(q, prefix_k, prefix_v, "prefix", 3, "[P, Hkv, d]")
    B, Hq, d = q.shape
    P, Hkv = prefix_k.shape[0], prefix_k.shape[1]
    _check_lens(suffix_lens, B)
    pg, S_cap = _paging(q, k_pool, v_pool, block_table, B, S_cap)
    if k_pool.shape[2] != Hkv:
        raise ValueError(f"k_pool has {k_pool.shape[2]} KV heads, the prefix {Hkv}")
    h = _heads(q, Hkv, scale)
    out, lse_out = _outputs(q, B, Hq, d, out, lse_out, return_lse, out_dtype)
    _require_cuda(q, prefix_k, prefix_v, k_pool, v_pool, block_table, suffix_lens, out, lse_out, workspace)
    lib = _lib.load()
    ss = k_pool.stride()
    aux = None if aux_stream is None else aux_stream.cuda_stream
    with _on(q.device):
        ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_ATTN, ctypes.byref(h), B, P, S_cap, 0), q.device,
                        workspace)
        check(lib.hydra_attn_paged(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1), P,
                                   prefix_k.data_ptr(), prefix_v.data_ptr(), prefix_k.stride(0), prefix_k.stride(1),
                                   k_pool.data_ptr(), v_pool.data_ptr(), ss[0], ss[1], ss[2], ctypes.byref(pg),
                                   S_cap, suffix_lens.data_ptr(), out.data_ptr(), _DT[out.dtype], _ptr(lse_out),
                                   _ptr(ws), _nbytes(ws), _stream_ptr(stream, q.device), aux),
              "hydra_attn_paged")
    return (out, lse_out) if return_lse else out


def combine(o_parts: torch.Tensor, lse_parts: torch.Tensor, out_dtype=torch.bfloat16, return_lse: bool = True,
            out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None, stream=None,
            o_parts_f32: Optional[torch.Tensor] = None, lse_parts_f32: Optional[torch.Tensor] = None):
    """n-ary LSE combine (Eq. 5 / App. B combine_lse), hydra_combine_ex.

    o_parts: [n, rows, d] (f32 or f16; any part and row strides, head dim contiguous -- e.g.
    slices of an exchange buffer whose rows interleave O and LSE), lse_parts: [n, rows] f32
    (any strides).  Optional second group o_parts_f32 [m, rows, d] / lse_parts_f32 [m, rows]
    in f32, merged in the same pass.  out: [rows, d] with a contiguous head dim (row stride
    free); lse_out: [rows] (any stride).  Returns (out, lse).  out_dtype float16 (from f32
    parts) packs partials for a cross-GPU exchange.
    """
    d = o_parts.shape[-1]
    o2 = o_parts if o_parts.dim() == 3 else o_parts.reshape(o_parts.shape[0], -1, d)
    l2 = lse_parts if lse_parts.dim() == 2 else lse_parts.reshape(lse_parts.shape[0], -1)
    n, rows = o2.shape[0], o2.shape[1]
    if o2.dtype not in (torch.float32, torch.float16):
        raise TypeError("o_parts must be f32 or f16")
    if l2.dtype != torch.float32 or tuple(l2.shape) != (n, rows):
        raise ValueError("lse_parts must be f32 [n, rows] with one value per row of each part")
    if o2.stride(2) != 1:
        raise ValueError("the head dim of o_parts must be contiguous")
    m = 0
    if o_parts_f32 is not None:
        if o_parts_f32.dtype != torch.float32 or o_parts_f32.dim() != 3 or o_parts_f32.shape[1:] != (rows, d) \
                or o_parts_f32.stride(2) != 1:
            raise ValueError("o_parts_f32 must be f32 [m, rows, d] with a contiguous head dim")
        m = o_parts_f32.shape[0]
        if lse_parts_f32 is None or lse_parts_f32.dtype != torch.float32 or tuple(lse_parts_f32.shape) != (m, rows):
            raise ValueError("lse_parts_f32 must be f32 [m, rows]")
    if out is None:
        out = torch.empty(rows, d, dtype=out_dtype, device=o_parts.device)
    if out.dtype not in (torch.bfloat16, torch.float32, torch.float16):
        raise TypeError("out must be bf16, f32 or (from f32 parts) f16")
    out2 = out.reshape(rows, d) if out.is_contiguous() and out.numel() == rows * d else out
    if tuple(out2.shape) != (rows, d) or out2.stride(1) != 1:
        raise ValueError("out must be a [rows, d] tensor with a contiguous head dim")
    lse = lse_out if lse_out is not None else (
        torch.empty(rows, dtype=torch.float32, device=o_parts.device) if return_lse else None)
    lse2 = None
    if lse is not None:
        lse2 = lse.reshape(rows) if lse.is_contiguous() and lse.numel() == rows else lse
        if lse2.dtype != torch.float32 or tuple(lse2.shape) != (rows,):
            raise ValueError("lse_out must be an f32 tensor of one value per row")
    _require_cuda(o_parts, lse_parts, out, lse, o_parts_f32, lse_parts_f32)
    c = _lib.CombineDesc()
    c.rows, c.d, c.n_parts = rows, d, n
    c.o_parts, c.o_dtype, c.o_part_stride, c.o_row_stride = o2.data_ptr(), _DT[o2.dtype], o2.stride(0), o2.stride(1)
    c.lse_parts, c.lse_part_stride, c.lse_row_stride = l2.data_ptr(), l2.stride(0), l2.stride(1)
    if m:
        c.n_parts_f32, c.o_parts_f32 = m, o_parts_f32.data_ptr()
        c.o_f32_part_stride, c.o_f32_row_stride = o_parts_f32.stride(0), o_parts_f32.stride(1)
        c.lse_parts_f32 = lse_parts_f32.data_ptr()
        c.lse_f32_part_stride, c.lse_f32_row_stride = lse_parts_f32.stride(0), lse_parts_f32.stride(1)
    c.out, c.out_dtype, c.out_row_stride = out2.data_ptr(), _DT[out2.dtype], out2.stride(0)
    if lse2 is not None:
        c.lse_out, c.lse_out_row_stride = lse2.data_ptr(), lse2.stride(0)
    with _on(o_parts.device):
        check(_lib.load().hydra_combine_ex(ctypes.byref(c), _stream_ptr(stream, o_parts.device)), "hydra_combine_ex")
    return out, lse


def combine_scatter(o_parts: torch.Tensor, lse_parts: torch.Tensor, out_table: torch.Tensor, table_rows: int,
                    out_row_stride: int, out_dtype=torch.float16, lse_table: Optional[torch.Tensor] = None,
                    lse_row_stride: int = 1, stream=None):
    """The combine of `combine` with a scattered output (hydra_combine_ex, table_rows > 0): row r
    goes to out_table[r // table_rows] + (r % table_rows) * out_row_stride (elements of out_dtype)
    and its LSE to lse_table[r // table_rows] + (r % table_rows) * lse_row_stride (f32 elements).
    out_table / lse_table: int64 device tensors of device addresses -- e.g. other GPUs' receive
    buffers mapped through symmetric memory, so the pack of the sequence split stores each batch
    shard's rows straight into the owning GPU (paper_2402_05099_b200.dist, exchange="p2p").
    o_parts [n, rows, d] f32, lse_parts [n, rows] f32 as in `combine`."""
    d = o_parts.shape[-1]
    if o_parts.dim() != 3 or o_parts.dtype != torch.float32 or o_parts.stride(2) != 1:
        raise ValueError("o_parts must be f32 [n, rows, d] with a contiguous head dim")
    n, rows = o_parts.shape[0], o_parts.shape[1]
    if lse_parts.dtype != torch.float32 or tuple(lse_parts.shape) != (n, rows):
        raise ValueError("lse_parts must be f32 [n, rows]")
    if table_rows <= 0 or out_row_stride < d:
        raise ValueError("table_rows must be > 0 and out_row_stride >= d")
    n_tab = -(-rows // table_rows)
    for t, name in ((out_table, "out_table"), (lse_table, "lse_table")):
        if t is not None and (t.dtype != torch.int64 or t.dim() != 1 or t.numel() < n_tab or not t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous int64 tensor of >= {n_tab} device addresses")
    if out_dtype not in (torch.float16, torch.float32, torch.bfloat16):
        raise TypeError("out_dtype must be f16, f32 or bf16")
    _require_cuda(o_parts, lse_parts, out_table, lse_table)
    c = _lib.CombineDesc()
    c.rows, c.d, c.n_parts = rows, d, n
    c.o_parts, c.o_dtype, c.o_part_stride, c.o_row_stride = (o_parts.data_ptr(), _DT[o_parts.dtype],
                                                             o_parts.stride(0), o_parts.stride(1))
    c.lse_parts, c.lse_part_stride, c.lse_row_stride = lse_parts.data_ptr(), lse_parts.stride(0), lse_parts.stride(1)
    c.out_dtype, c.out_row_stride, c.lse_out_row_stride = _DT[out_dtype], out_row_stride, lse_row_stride
    c.out_table, c.table_rows = out_table.data_ptr(), table_rows
    if lse_table is not None:
        c.lse_out_table = lse_table.data_ptr()
    with _on(o_parts.device):
        check(_lib.load().hydra_combine_ex(ctypes.byref(c), _stream_ptr(stream, o_parts.device)), "hydra_combine_ex")


# ------------------------------------------------------------------ whole decode-step attention
def attn_workspace_bytes(q, prefix_len: int, suffix_cap: int, Hkv: int, scale=None) -> int:
    q = _squeeze_q(q)
    h = _heads(q, Hkv, scale)
    with _on(q.device):
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
    _kv_pair(q, prefix_k, prefix_v, "prefix", 3, "[P, Hkv, d]")
    _kv_pair(q, suffix_k, suffix_v, "suffix", 4, "[B, S_cap, Hkv, d]")
    B, Hq, d = q.shape
    P, Hkv = prefix_k.shape[0], prefix_k.shape[1]
    S_cap = suffix_k.shape[1]
    if suffix_k.shape[2] != Hkv or suffix_k.shape[0] != B:
        raise ValueError("suffix_k must be [B, S_cap, Hkv, d] with the prefix's Hkv")
    _check_lens(suffix_lens, B)
    h = _heads(q, Hkv, scale)
    out, lse_out = _outputs(q, B, Hq, d, out, lse_out, return_lse, out_dtype)
    _require_cuda(q, prefix_k, prefix_v, suffix_k, suffix_v, suffix_lens, out, lse_out, workspace)
    lib = _lib.load()
    ss = suffix_k.stride()
    aux = None if aux_stream is None else aux_stream.cuda_stream
    with _on(q.device):
        ws = _workspace(lib.hydra_workspace_size(_lib.HYDRA_OP_ATTN, ctypes.byref(h), B, P, S_cap, 0), q.device,
                        workspace)
        check(lib.hydra_attn(ctypes.byref(h), B, q.data_ptr(), q.stride(0), q.stride(1), P, prefix_k.data_ptr(),
                             prefix_v.data_ptr(), prefix_k.stride(0), prefix_k.stride(1), suffix_k.data_ptr(),
                             suffix_v.data_ptr(), ss[0], ss[1], ss[2], S_cap, suffix_lens.data_ptr(),
                             out.data_ptr(), _DT[out.dtype], _ptr(lse_out), _ptr(ws), _nbytes(ws),
                             _stream_ptr(stream, q.device), aux), "hydra_attn")
    return (out, lse_out) if return_lse else out


# ------------------------------------------------------------------ tree attention (§3.3)
class Tree:
    """Sharing tree (§3.3, Fig. 2): parent[n] (root -1), node_off/node_len into the pooled
    node K/V, leaf_of_seq[b].  Validated and grouped by the C library (hydra_tree_create).

    `prepare(num_q_heads, num_kv_heads)` uploads the node-attention work list for that head
    grouping, after which tree_attention calls with it are capturable in a CUDA graph; an
    unprepared tree is prepared by its first call outside capture."""

    def __init__(self, parent: Sequence[int], node_off: Sequence[int], node_len: Sequence[int],
                 leaf_of_seq: Sequence[int], heads: Optional[tuple] = None):
        lib = _lib.load()
        self.parent = np.ascontiguousarray(parent, np.int32)
        self.node_off = np.ascontiguousarray(node_off, np.int64)
        self.node_len = np.ascontiguousarray(node_len, np.int64)
        self.leaf_of_seq = np.ascontiguousarray(leaf_of_seq, np.int32)
        self.B = int(self.leaf_of_seq.shape[0])
        self.n_tokens = int((self.node_off + self.node_len).max()) if len(self.node_off) else 0
        self._h = None
        handle = ctypes.c_void_p()
        check(lib.hydra_tree_create(self.parent.ctypes.data, self.node_off.ctypes.data, self.node_len.ctypes.data,
                                    len(self.parent), self.leaf_of_seq.ctypes.data, self.B, ctypes.byref(handle)),
              "hydra_tree_create")
        self._h = handle
        if heads is not None:
            self.prepare(*heads)

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("tree destroyed")
        return self._h

    def prepare(self, num_q_heads: int, num_kv_heads: int, head_dim: int = 128, dtype=torch.bfloat16):
        h = Heads(num_q_heads, num_kv_heads, head_dim, 0.0, _DT[dtype])
        check(_lib.load().hydra_tree_prepare(self.handle, ctypes.byref(h)), "hydra_tree_prepare")
        return self

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


def _check_tree_inputs(q, tree, node_k, node_v):
    _kv_pair(q, node_k, node_v, "node", 3, "[T_nodes, Hkv, d]")
    if q.shape[0] != tree.B:
        raise ValueError(f"q batch {q.shape[0]} does not match the tree's {tree.B} sequences")
    if node_k.shape[0] < tree.n_tokens:
        raise ValueError(f"node_k holds {node_k.shape[0]} tokens, the tree addresses {tree.n_tokens}")


def tree_attention(q: torch.Tensor, tree: Tree, node_k: torch.Tensor, node_v: torch.Tensor,
                   suffix_k: torch.Tensor, suffix_v: torch.Tensor, suffix_lens: torch.Tensor,
                   scale: Optional[float] = None, out_dtype=None, return_lse: bool = False,
                   workspace: Optional[torch.Tensor] = None, stream=None, aux_stream=None,
                   out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None):
    """Decomposition at every tree vertex (§3.3) + suffix + n-ary combine.  With
    `aux_stream` the node attention and the suffix run concurrently on disjoint SM sets."""
    q = _squeeze_q(q)
    _check_tree_inputs(q, tree, node_k, node_v)
    _kv_pair(q, suffix_k, suffix_v, "suffix", 4, "[B, S_cap, Hkv, d]")
    B, Hq, d = q.shape
    Hkv = node_k.shape[1]
    if suffix_k.shape[0] != B or suffix_k.shape[2] != Hkv:
        raise ValueError("suffix_k must be [B, S_cap, Hkv, d] with the nodes' Hkv")
    _check_lens(suffix_lens, B)
    S_cap = suffix_k.shape[1]
    h = _heads(q, Hkv, scale)
    out, lse = _outputs(q, B, Hq, d, out, lse_out, return_lse, out_dtype)
    _require_cuda(q, node_k, node_v, suffix_k, suffix_v, suffix_lens, out, lse_out, workspace)
    lib = _lib.load()
    ss = suffix_k.stride()
    with _on(q.device):
        ws = _workspace(lib.hydra_tree_workspace_size(ctypes.byref(h), tree.handle, S_cap), q.device, workspace)
        check(lib.hydra_tree_attn(ctypes.byref(h), tree.handle, q.data_ptr(), q.stride(0), q.stride(1),
                                  node_k.data_ptr(), node_v.data_ptr(), node_k.stride(0), node_k.stride(1),
                                  suffix_k.data_ptr(), suffix_v.data_ptr(), ss[0], ss[1], ss[2], S_cap,
                                  suffix_lens.data_ptr(), out.data_ptr(), _DT[out.dtype], _ptr(lse), _ptr(ws),
                                  _nbytes(ws), _stream_ptr(stream, q.device),
                                  _stream_ptr(aux_stream, q.device) if aux_stream is not None else None),
              "hydra_tree_attn")
    return (out, lse) if return_lse else out


def tree_attention_paged(q: torch.Tensor, tree: Tree, node_k: torch.Tensor, node_v: torch.Tensor,
                         k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor,
                         suffix_lens: torch.Tensor, S_cap: Optional[int] = None, scale: Optional[float] = None,
                         out_dtype=None, return_lse: bool = False, workspace: Optional[torch.Tensor] = None,
                         stream=None, aux_stream=None, out: Optional[torch.Tensor] = None,
                         lse_out: Optional[torch.Tensor] = None):
    """tree_attention with the suffixes in a paged cache (pools [n_pages, page_size, Hkv, d],
    block_table int32 [B, max_pages]; reading R14)."""
    q = _squeeze_q(q)
    _check_tree_inputs(q, tree, node_k, node_v)
    B, Hq, d = q.shape
    Hkv = node_k.shape[1]
    _check_lens(suffix_lens, B)
    pg, S_cap = _paging(q, k_pool, v_pool, block_table, B, S_cap)
    if k_pool.shape[2] != Hkv:
        raise ValueError(f"k_pool has {k_pool.shape[2]} KV heads, the nodes {Hkv}")
    h = _heads(q, Hkv, scale)
    out, lse = _outputs(q, B, Hq, d, out, lse_out, return_lse, out_dtype)
    _require_cuda(q, node_k, node_v, k_pool, v_pool, block_table, suffix_lens, out, lse_out, workspace)
    lib = _lib.load()
    ss = k_pool.stride()
    with _on(q.device):
        ws = _workspace(lib.hydra_tree_workspace_size(ctypes.byref(h), tree.handle, S_cap), q.device, workspace)
        check(lib.hydra_tree_attn_paged(ctypes.byref(h), tree.handle, q.data_ptr(), q.stride(0), q.stride(1),
                                        node_k.data_ptr(), node_v.data_ptr(), node_k.stride(0), node_k.stride(1),
                                        k_pool.data_ptr(), v_pool.data_ptr(), ss[0], ss[1], ss[2], ctypes.byref(pg),
                                        S_cap, suffix_lens.data_ptr(), out.data_ptr(), _DT[out.dtype], _ptr(lse),
                                        _ptr(ws), _nbytes(ws), _stream_ptr(stream, q.device),
                                        _stream_ptr(aux_stream, q.device) if aux_stream is not None else None),
              "hydra_tree_attn_paged")
    return (out, lse) if return_lse else out


def workspace_bytes_tree(q: torch.Tensor, tree: Tree, Hkv: int, suffix_cap: int, scale=None) -> int:
    q = _squeeze_q(q)
    h = _heads(q, Hkv, scale)
    with _on(q.device):
        return int(_lib.load().hydra_tree_workspace_size(ctypes.byref(h), tree.handle, suffix_cap))
