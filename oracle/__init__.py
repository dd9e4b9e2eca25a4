"""fp64 CPU oracle for exact shared-prefix decode attention (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product path never imports it and
it never imports the product package; the two share only `synth` (inputs).

What it computes is the plain definition of the result Hydragen reaches exactly
(PAPER.md abstract P:7 "exact", App. A): softmax attention (Eq. 1,
P:44) with its log-sum-exp (Eq. 4) over each sequence's full,
*undecomposed* key/value set -- the concatenation of the shared prefix (or every
node on the sequence's root->leaf path, §3.3) and its own suffix.  The
heavy loop is plain C in oracle.c (fp64, two-pass softmax, OpenMP over rows).
`combine` is the paper's App. B `combine_lse` in fp64 with the
merged LSE added (reading R5); it is used only to localise failures
and in the decomposition pin, never to produce the reference result.

Every function here is pinned by tests in tests/test_oracle.py (closed forms,
invariants the paper fixes, SPEC worked examples, brute force on tiny inputs).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (plain C, -O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Seg(ctypes.Structure):
    _fields_ = [("k", ctypes.c_void_p), ("v", ctypes.c_void_p), ("len", ctypes.c_int64),
                ("st", ctypes.c_int64), ("sh", ctypes.c_int64)]


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_attention.restype = ctypes.c_int
        lib.oracle_attention.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.uint16:
        return 0  # bf16 bit patterns
    if a.dtype == np.float32:
        return 1
    raise TypeError(f"oracle inputs must be bf16 bits (uint16) or float32, got {a.dtype}")


def _estrides(a: np.ndarray):
    return [s // a.itemsize for s in a.strides]


def attention_segments(q: np.ndarray, seg_lists: Sequence[Sequence[tuple]], Hkv: int,
                       scale: Optional[float] = None, rows: Optional[np.ndarray] = None,
                       threads: int = 0):
    """Eq. 1 + Eq. 4 for each row over the concatenation of its segments.

    q: [B, Hq, d] (uint16 bf16 bits or float32; any strides, d contiguous).
    seg_lists[b]: ordered list of (K, V) array pairs of shape [len, Hkv, d] whose
      concatenation is sequence b's full key/value set (K_full = K_1 || K_2 ...).
    rows: optional int array [n, 2] of (b, h) pairs; default all B*Hq rows.
    Returns (O [n, d] float64, LSE [n] float64); with rows=None they are shaped
    [B, Hq, d] and [B, Hq].
    """
    B, Hq, d = q.shape
    if Hq % Hkv:
        raise ValueError("Hq % Hkv != 0")
    dt = _dtype_code(q)
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    max_segs = max(1, max(len(s) for s in seg_lists) if seg_lists else 1)
    segs = (_Seg * (B * max_segs))()
    nseg = np.zeros(B, np.int32)
    keep = []
    for b, lst in enumerate(seg_lists):
        nseg[b] = len(lst)
        for i, (K, V) in enumerate(lst):
            assert K.shape == V.shape and K.ndim == 3 and K.shape[1] == Hkv and K.shape[2] == d
            assert _dtype_code(K) == dt and _dtype_code(V) == dt
            ks, vs = _estrides(K), _estrides(V)
            assert ks == vs and ks[2] == 1, "K and V segments must share strides, d contiguous"
            keep += [K, V]
            segs[b * max_segs + i] = _Seg(K.ctypes.data if K.size else 0, V.ctypes.data if V.size else 0,
                                          K.shape[0], ks[0], ks[1])
    qs = _estrides(q)
    assert qs[2] == 1
    full = rows is None
    if full:
        bb, hh = np.meshgrid(np.arange(B), np.arange(Hq), indexing="ij")
        rows = np.stack([bb.ravel(), hh.ravel()], 1)
    rows = np.asarray(rows, np.int64).reshape(-1, 2)
    rb = np.ascontiguousarray(rows[:, 0], np.int64)
    rh = np.ascontiguousarray(rows[:, 1], np.int32)
    n = rows.shape[0]
    out = np.zeros((n, d), np.float64)
    lse = np.zeros(n, np.float64)
    st = _load().oracle_attention(dt, d, Hq, Hkv, float(scale), q.ctypes.data, qs[0], qs[1],
                                  n, rb.ctypes.data, rh.ctypes.data, ctypes.addressof(segs), max_segs,
                                  nseg.ctypes.data, out.ctypes.data, lse.ctypes.data, int(threads))
    if st != 0:
        raise RuntimeError(f"oracle_attention failed with status {st}")
    del keep
    if full:
        return out.reshape(B, Hq, d), lse.reshape(B, Hq)
    return out, lse


# ---------------------------------------------------------------------------
# Problem-level entry points (the workloads of synth.Problem / synth.TreeProblem)
# ---------------------------------------------------------------------------

def flat_attention(pb, rows=None, threads: int = 0):
    """Full attention over prefix || suffix[b, :lens[b]] per sequence (App. B inputs)."""
    segs = [[(pb.pk, pb.pv), (pb.sk[b, :pb.lens[b]], pb.sv[b, :pb.lens[b]])] for b in range(pb.B)]
    return attention_segments(pb.q, segs, pb.Hkv, pb.scale, rows, threads)


def prefix_only(pb, rows=None, threads: int = 0):
    """Attention over the shared prefix alone: the (O, LSE) partial of §3.2."""
    return attention_segments(pb.q, [[(pb.pk, pb.pv)]] * pb.B, pb.Hkv, pb.scale, rows, threads)


def suffix_only(pb, rows=None, threads: int = 0):
    """Attention over each sequence's own suffix alone (§3.2)."""
    segs = [[(pb.sk[b, :pb.lens[b]], pb.sv[b, :pb.lens[b]])] for b in range(pb.B)]
    return attention_segments(pb.q, segs, pb.Hkv, pb.scale, rows, threads)


def paged_rows(pool: np.ndarray, table_row: np.ndarray, page_size: int, n: int) -> np.ndarray:
    """Tokens 0..n-1 of one sequence of a paged cache, in order (reading R14):
    token t is row t % page_size of page table_row[t // page_size].  Pure indexing."""
    out = [pool[int(table_row[t // page_size]), t % page_size] for t in range(n)]
    return np.stack(out) if out else pool[:0, 0]


def suffix_only_paged(q, k_pool, v_pool, block_table, page_size, lens, Hkv, scale=None, rows=None,
                      threads: int = 0):
    """suffix_only over a paged cache: gather each suffix (paged_rows), then the definition."""
    segs = []
    for b in range(q.shape[0]):
        n = int(lens[b])
        segs.append([(paged_rows(k_pool, block_table[b], page_size, n),
                      paged_rows(v_pool, block_table[b], page_size, n))])
    return attention_segments(q, segs, Hkv, scale, rows, threads)


def flat_attention_paged(pb, pc, rows=None, threads: int = 0):
    """flat_attention with the suffixes read from a paged cache pc (synth.PagedCache)."""
    segs = []
    for b in range(pb.B):
        n = int(pb.lens[b])
        segs.append([(pb.pk, pb.pv), (paged_rows(pc.k_pool, pc.block_table[b], pc.page_size, n),
                                      paged_rows(pc.v_pool, pc.block_table[b], pc.page_size, n))])
    return attention_segments(pb.q, segs, pb.Hkv, pb.scale, rows, threads)


def tree_path(parent: np.ndarray, leaf: int) -> list:
    """Root->leaf node list by walking parent pointers (S:242-250 flatten order)."""
    out, n = [], int(leaf)
    while n >= 0:
        out.append(n)
        n = int(parent[n])
    return out[::-1]


def tree_attention(tp, rows=None, threads: int = 0):
    """Full attention over (every node on the root->leaf path, in order) || suffix (§3.3)."""
    segs = []
    for b in range(tp.B):
        lst = []
        for n in tree_path(tp.parent, tp.leaf_of_seq[b]):
            lo, L = int(tp.node_off[n]), int(tp.node_len[n])
            lst.append((tp.node_k[lo:lo + L], tp.node_v[lo:lo + L]))
        lst.append((tp.sk[b, :tp.lens[b]], tp.sv[b, :tp.lens[b]]))
        segs.append(lst)
    return attention_segments(tp.q, segs, tp.Hkv, tp.scale, rows, threads)


def tree_attention_paged(tp, pc, rows=None, threads: int = 0):
    """tree_attention with each sequence's suffix read from a paged cache pc (reading R14)."""
    segs = []
    for b in range(tp.B):
        lst = []
        for n in tree_path(tp.parent, tp.leaf_of_seq[b]):
            lo, L = int(tp.node_off[n]), int(tp.node_len[n])
            lst.append((tp.node_k[lo:lo + L], tp.node_v[lo:lo + L]))
        n_suf = int(tp.lens[b])
        lst.append((paged_rows(pc.k_pool, pc.block_table[b], pc.page_size, n_suf),
                    paged_rows(pc.v_pool, pc.block_table[b], pc.page_size, n_suf)))
        segs.append(lst)
    return attention_segments(tp.q, segs, tp.Hkv, tp.scale, rows, threads)


def combine(o1, lse1, o2, lse2):
    """App. B `combine_lse`, fp64, plus the merged LSE (reading R5).

    max_lse = max(lse1, lse2); w_i = exp(lse_i - max_lse);
    O = (o1*w1 + o2*w2) / (w1 + w2);  LSE = max_lse + ln(w1 + w2).
    The (-inf) sentinel of an empty part is the identity (reading R6).
    """
    o1, o2 = np.asarray(o1, np.float64), np.asarray(o2, np.float64)
    lse1, lse2 = np.asarray(lse1, np.float64), np.asarray(lse2, np.float64)
    max_lse = np.maximum(lse1, lse2)
    both_empty = np.isneginf(max_lse)
    safe = np.where(both_empty, 0.0, max_lse)
    w1 = np.where(np.isneginf(lse1), 0.0, np.exp(lse1 - safe))
    w2 = np.where(np.isneginf(lse2), 0.0, np.exp(lse2 - safe))
    den = w1 + w2
    with np.errstate(invalid="ignore", divide="ignore"):
        o = (o1 * w1[..., None] + o2 * w2[..., None]) / den[..., None]
        lse = safe + np.log(den)
    o = np.where(both_empty[..., None], 0.0, o)
    lse = np.where(both_empty, -np.inf, lse)
    return o, lse
