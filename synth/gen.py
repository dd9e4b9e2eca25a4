"""Seeded synthetic workloads.

Shapes follow the paper's problem statement for one decode step of one attention
layer (App. B): q[B, Hq, d] (Nq = 1 during decoding),
prefix K/V [P, Hkv, d] shared by every sequence, suffix K/V [B, S_cap, Hkv, d]
with per-sequence valid lengths lens[b] <= S_cap.  Tree workloads (P:121-135,
Fig. 2) pool every node's tokens into one [T_nodes, Hkv, d] array.

Value distributions:
  plain    : every tensor i.i.d. N(0,1)
  mixed    : K, V ~ N(0,1); each query row (b,h) is aimed at one "needle" token
             of its own sequence, q = a*k_needle + 0.5*z with
             a = target / (scale*|k_needle|^2), target = ln(N_b) + U[-2,2]
  boundary : as mixed, but the needle sits on a tile edge of the prefix
             {0,127,128,P-129,P-128,P-1} or of the suffix {0, lens[b]-1}
Suffix padding positions t >= lens[b] are poisoned with bf16/f32 NaN so that a
kernel reading past lens[b] cannot pass the parity gates.

bf16 values are produced by drawing float32 N(0,1) and rounding to bf16 with
round-to-nearest-even; both the GPU and the oracle consume the same bit patterns.
The generator is deterministic for a given seed independent of thread count:
each tensor gets its own SeedSequence([seed, stream]) which is spawned into
fixed 4 Mi-element chunks, one PCG64 stream per chunk.

No attention arithmetic lives here: the only arithmetic is drawing, rounding,
and aiming query vectors at needle keys (input construction).
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

CHUNK = 1 << 22
BF16_NAN = np.uint16(0x7FC0)
F32_NAN = np.float32("nan")

# Stream ids: fixed tensor order q, prefix_k, prefix_v, suffix_k, suffix_v, needles.
_S_Q, _S_PK, _S_PV, _S_SK, _S_SV, _S_NEEDLE = range(6)


def _threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 -> bf16 (round to nearest, ties to even); NaN -> 0x7FC0."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32)
    r = ((u >> 16) & np.uint32(1)) + np.uint32(0x7FFF)
    b = ((u + r) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        b[nan] = BF16_NAN
    return b


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns to float32."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _chunked(seed: int, stream: int, n: int, fill_chunk) -> None:
    nchunks = max(1, -(-n // CHUNK))
    children = np.random.SeedSequence([seed, stream]).spawn(nchunks)

    def work(i):
        lo, hi = i * CHUNK, min(n, (i + 1) * CHUNK)
        if lo < hi:
            g = np.random.Generator(np.random.PCG64(children[i]))
            fill_chunk(g, lo, hi)

    if nchunks == 1:
        work(0)
    else:
        with ThreadPoolExecutor(min(_threads(), nchunks)) as ex:
            list(ex.map(work, range(nchunks)))


def normal_f32(seed: int, stream: int, shape) -> np.ndarray:
    n = int(np.prod(shape)) if len(shape) else 1
    out = np.empty(n, np.float32)

    def fill(g, lo, hi):
        g.standard_normal(out=out[lo:hi], dtype=np.float32)

    _chunked(seed, stream, n, fill)
    return out.reshape(shape)


def normal_bf16_bits(seed: int, stream: int, shape) -> np.ndarray:
    """N(0,1) float32 draws rounded to bf16 bits, converted chunk by chunk."""
    n = int(np.prod(shape)) if len(shape) else 1
    out = np.empty(n, np.uint16)

    def fill(g, lo, hi):
        tmp = g.standard_normal(hi - lo, dtype=np.float32)
        out[lo:hi] = f32_to_bf16_bits(tmp)

    _chunked(seed, stream, n, fill)
    return out.reshape(shape)


def _draw(seed, stream, shape, dtype):
    return normal_bf16_bits(seed, stream, shape) if dtype == "bf16" else normal_f32(seed, stream, shape)


def _widen(a, dtype):
    return bf16_bits_to_f32(a) if dtype == "bf16" else np.asarray(a, np.float32)


def _narrow(x, dtype):
    return f32_to_bf16_bits(x) if dtype == "bf16" else np.asarray(x, np.float32)


@dataclass
class Problem:
    """One decode step of one layer with a flat shared prefix (App. B)."""

    B: int
    Hq: int
    Hkv: int
    d: int
    P: int
    S_cap: int
    dtype: str  # "bf16" (arrays hold uint16 bit patterns) or "f32"
    lens: np.ndarray  # int32 [B]
    q: np.ndarray  # [B, Hq, d]
    pk: np.ndarray  # [P, Hkv, d]
    pv: np.ndarray  # [P, Hkv, d]
    sk: np.ndarray  # [B, S_cap, Hkv, d]
    sv: np.ndarray  # [B, S_cap, Hkv, d]
    seed: int = 0
    dist: str = "plain"
    scale: float = field(default=0.0)

    def __post_init__(self):
        if not self.scale:
            self.scale = 1.0 / math.sqrt(self.d)

    @property
    def g(self) -> int:
        return self.Hq // self.Hkv

    def f32(self, name: str) -> np.ndarray:
        return _widen(getattr(self, name), self.dtype)


@dataclass
class TreeProblem:
    """One decode step with hierarchical sharing (Fig. 2 caption P:129).

    Node n owns tokens [node_off[n], node_off[n]+node_len[n]) of the pooled
    node_k/node_v arrays; parent[root] = -1; sequence b's leaf is leaf_of_seq[b].
    """

    B: int
    Hq: int
    Hkv: int
    d: int
    S_cap: int
    dtype: str
    parent: np.ndarray  # int32 [n_nodes]
    node_off: np.ndarray  # int64 [n_nodes]
    node_len: np.ndarray  # int64 [n_nodes]
    leaf_of_seq: np.ndarray  # int32 [B]
    lens: np.ndarray  # int32 [B]
    q: np.ndarray  # [B, Hq, d]
    node_k: np.ndarray  # [T_nodes, Hkv, d]
    node_v: np.ndarray
    sk: np.ndarray  # [B, S_cap, Hkv, d]
    sv: np.ndarray
    seed: int = 0
    dist: str = "plain"
    scale: float = field(default=0.0)

    def __post_init__(self):
        if not self.scale:
            self.scale = 1.0 / math.sqrt(self.d)

    @property
    def g(self) -> int:
        return self.Hq // self.Hkv

    def f32(self, name: str) -> np.ndarray:
        return _widen(getattr(self, name), self.dtype)

    def path(self, b: int) -> list:
        """Root-to-leaf node ids of sequence b (plain parent walk)."""
        out = []
        n = int(self.leaf_of_seq[b])
        while n >= 0:
            out.append(n)
            n = int(self.parent[n])
        return out[::-1]


def _aim_queries(rng, q_f32, scale, dist, lens, key_lookup, path_len_fn, boundary_fn):
    """Input construction for 'mixed'/'boundary': q = a*k_needle + 0.5*z."""
    B, Hq, d = q_f32.shape
    for b in range(B):
        npre = path_len_fn(b)
        nsuf = int(lens[b])
        ntot = npre + nsuf
        if ntot == 0:
            continue
        for h in range(Hq):
            if dist == "boundary":
                cands = boundary_fn(b)
                t = int(cands[rng.integers(len(cands))])
            else:
                use_pre = nsuf == 0 or (npre > 0 and rng.random() < 0.5)
                t = int(rng.integers(npre)) if use_pre else npre + int(rng.integers(nsuf))
            k = key_lookup(b, h, t)
            kk = float(np.dot(k.astype(np.float64), k.astype(np.float64)))
            if kk <= 0.0:
                continue
            target = math.log(ntot) + float(rng.uniform(-2.0, 2.0))
            a = target / (scale * kk)
            q_f32[b, h] = (a * k.astype(np.float64) + 0.5 * q_f32[b, h].astype(np.float64)).astype(np.float32)
    return q_f32


def _prefix_edges(P):
    return sorted({t for t in (0, 127, 128, P - 129, P - 128, P - 1) if 0 <= t < P})


def make_problem(B, Hq, Hkv, d, P, S_cap, lens=None, dtype="bf16", dist="plain", seed=0,
                 poison=True, scale=None) -> Problem:
    if Hq % Hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    if lens is None:
        lens = np.full(B, S_cap, np.int32)
    lens = np.asarray(lens, np.int32)
    assert lens.shape == (B,) and (lens >= 0).all() and (lens <= S_cap).all()
    q = _draw(seed, _S_Q, (B, Hq, d), dtype)
    pk = _draw(seed, _S_PK, (P, Hkv, d), dtype)
    pv = _draw(seed, _S_PV, (P, Hkv, d), dtype)
    sk = _draw(seed, _S_SK, (B, S_cap, Hkv, d), dtype)
    sv = _draw(seed, _S_SV, (B, S_cap, Hkv, d), dtype)
    sc = scale if scale else 1.0 / math.sqrt(d)
    g = Hq // Hkv
    if dist in ("mixed", "boundary"):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, _S_NEEDLE])))
        pkw, skw = _widen(pk, dtype), None

        def key_lookup(b, h, t):
            j = h // g
            if t < P:
                return pkw[t, j]
            return _widen(sk[b, t - P, j], dtype)

        def boundary(b):
            c = list(_prefix_edges(P))
            if lens[b] > 0:
                c += [P + 0, P + int(lens[b]) - 1]
            return c

        qf = _aim_queries(rng, _widen(q, dtype).copy(), sc, dist, lens, key_lookup, lambda b: P, boundary)
        q = _narrow(qf, dtype)
        del skw
    elif dist != "plain":
        raise ValueError(dist)
    if poison:
        for b in range(B):
            if lens[b] < S_cap:
                sk[b, lens[b]:] = BF16_NAN if dtype == "bf16" else F32_NAN
                sv[b, lens[b]:] = BF16_NAN if dtype == "bf16" else F32_NAN
    return Problem(B, Hq, Hkv, d, P, S_cap, dtype, lens, q, pk, pv, sk, sv, seed, dist, sc)


def make_tree_problem(parent, node_len, leaf_of_seq, Hq, Hkv, d, S_cap, lens=None, dtype="bf16",
                      dist="plain", seed=0, poison=True, scale=None) -> TreeProblem:
    parent = np.asarray(parent, np.int32)
    node_len = np.asarray(node_len, np.int64)
    leaf_of_seq = np.asarray(leaf_of_seq, np.int32)
    B = int(leaf_of_seq.shape[0])
    node_off = np.zeros_like(node_len)
    node_off[1:] = np.cumsum(node_len)[:-1]
    T = int(node_len.sum())
    if lens is None:
        lens = np.full(B, S_cap, np.int32)
    lens = np.asarray(lens, np.int32)
    q = _draw(seed, _S_Q, (B, Hq, d), dtype)
    nk = _draw(seed, _S_PK, (T, Hkv, d), dtype)
    nv = _draw(seed, _S_PV, (T, Hkv, d), dtype)
    sk = _draw(seed, _S_SK, (B, S_cap, Hkv, d), dtype)
    sv = _draw(seed, _S_SV, (B, S_cap, Hkv, d), dtype)
    sc = scale if scale else 1.0 / math.sqrt(d)
    tp = TreeProblem(B, Hq, Hkv, d, S_cap, dtype, parent, node_off, node_len, leaf_of_seq, lens,
                     q, nk, nv, sk, sv, seed, dist, sc)
    g = Hq // Hkv
    if dist in ("mixed", "boundary"):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, _S_NEEDLE])))
        nkw = _widen(nk, dtype)
        paths = [tp.path(b) for b in range(B)]
        path_tok = [np.concatenate([np.arange(node_off[n], node_off[n] + node_len[n]) for n in p])
                    if p else np.zeros(0, np.int64) for p in paths]

        def key_lookup(b, h, t):
            j = h // g
            npre = len(path_tok[b])
            if t < npre:
                return nkw[path_tok[b][t], j]
            return _widen(sk[b, t - npre, j], dtype)

        def boundary(b):
            c, base = [], 0
            for n in paths[b]:
                L = int(node_len[n])
                c += [base + e for e in _prefix_edges(L)]
                base += L
            if lens[b] > 0:
                c += [base, base + int(lens[b]) - 1]
            return c

        qf = _aim_queries(rng, _widen(q, dtype).copy(), sc, dist, lens, key_lookup,
                          lambda b: len(path_tok[b]), boundary)
        tp.q = _narrow(qf, dtype)
    if poison:
        for b in range(B):
            if lens[b] < S_cap:
                sk[b, lens[b]:] = BF16_NAN if dtype == "bf16" else F32_NAN
                sv[b, lens[b]:] = BF16_NAN if dtype == "bf16" else F32_NAN
    return tp


def two_level_tree(root_len, n_branches, branch_len, seqs_per_branch):
    """parent/node_len/leaf_of_seq for the C5 shape: root -> branches -> sequences."""
    parent = [-1] + [0] * n_branches
    node_len = [root_len] + [branch_len] * n_branches
    leaf = np.repeat(np.arange(1, n_branches + 1, dtype=np.int32), seqs_per_branch)
    return parent, node_len, leaf


@dataclass
class PagedCache:
    """A paged copy of a Problem's suffix caches (reading R14): token t of
    sequence b is row t % page_size of page block_table[b, t // page_size] of the pools."""

    page_size: int
    k_pool: np.ndarray  # [n_pages, page_size, Hkv, d]
    v_pool: np.ndarray
    block_table: np.ndarray  # int32 [B, max_pages]

    @property
    def n_pages(self) -> int:
        return self.k_pool.shape[0]


def paginate(pb: Problem, page_size: int, seed: int = 0, spare_pages: int = 3, map_tail: bool = True,
             unmapped: int = 2**30) -> PagedCache:
    """Scatter pb.sk/sv into page pools in a seeded random page order.

    Every sequence gets ceil(S_cap / page_size) table entries.  With map_tail=False only the
    pages covering tokens < lens[b] are mapped and the remaining entries hold `unmapped`
    (an out-of-range page id the kernels must never read).  Spare pages and page rows past
    S_cap are poisoned with NaN, as the suffix padding already is (layout only, no arithmetic).
    """
    rng = np.random.default_rng(seed)
    max_pages = -(-pb.S_cap // page_size)
    used = [max_pages if map_tail else -(-int(pb.lens[b]) // page_size) for b in range(pb.B)]
    n_pages = sum(used) + spare_pages
    perm = rng.permutation(n_pages).astype(np.int32)
    nan = BF16_NAN if pb.dtype == "bf16" else F32_NAN
    shape = (n_pages, page_size, pb.Hkv, pb.d)
    k_pool = np.full(shape, nan, dtype=pb.sk.dtype)
    v_pool = np.full(shape, nan, dtype=pb.sv.dtype)
    table = np.full((pb.B, max(1, max_pages)), unmapped, np.int32)
    nxt = 0
    for b in range(pb.B):
        for i in range(used[b]):
            page = perm[nxt]
            nxt += 1
            table[b, i] = page
            lo, hi = i * page_size, min(pb.S_cap, (i + 1) * page_size)
            k_pool[page, :hi - lo] = pb.sk[b, lo:hi]
            v_pool[page, :hi - lo] = pb.sv[b, lo:hi]
    return PagedCache(page_size, k_pool, v_pool, table)
