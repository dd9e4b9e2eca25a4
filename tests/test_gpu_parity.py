"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Gates (north_star): bf16 inputs -> max|d| <= 2e-2, mean|d| <= 2e-3 on the delivered bf16
output, plus |dLSE| <= 1e-3; fp32 reference mode -> 1e-5.  Inputs use the 'mixed' /
'boundary' needle distributions and NaN-poisoned suffix padding (SURVEY §8(c)
sensitivity analysis), sizes span several 128-token tiles with ragged tails.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from tests import nanfill as H
from tests.util import assert_parity, errors, problem_to, tree_to

hydra = pytest.importorskip("paper_2402_05099_b200")

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _reset_config():
    keys = ("prefix_impl", "prefix_splits", "suffix_splits", "prefix_ctas", "suffix_impl",
            "suffix_ctas", "overlap_prefix_ctas", "pair_cluster", "overlap_simt", "pair_item_cost")
    for k in keys:
        hydra.set_config(k, 0)
    defaults = {"prefix_variant": 9, "suffix_cb": 2, "prefix_poly": 4, "pair_poly": 0, "fuse_combine": 0,
                "combine_pdl": 1, "overlap_short": 1}  # the library defaults
    for k, v in defaults.items():
        hydra.set_config(k, v)
    yield
    for k, v in defaults.items():
        hydra.set_config(k, v)
    for k in keys:
        hydra.set_config(k, 0)


DEV = "cuda:0"


def run_flat(pb, aux=False, **kw):
    t = problem_to(pb, DEV)
    aux_stream = torch.cuda.Stream() if aux else None
    out, lse = H.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True,
                                        aux_stream=aux_stream, **kw)
    torch.cuda.synchronize()
    return out, lse


# ---------------------------------------------------------------- C1 tiny, fp32 reference mode
@pytest.mark.parametrize("Hq,Hkv", [(2, 1), (4, 2)])
@pytest.mark.parametrize("dist", ["plain", "mixed", "boundary"])
def test_tiny_fp32(Hq, Hkv, dist):
    pb = synth.make_problem(4, Hq, Hkv, 16, 32, 12, lens=[5, 8, 10, 12], dtype="f32", dist=dist, seed=1)
    out, lse = run_flat(pb)
    ref, lref = oracle.flat_attention(pb)
    assert_parity(out, ref, lse, lref, dtype="f32", what="C1")


# ---------------------------------------------------------------- prefix kernel (tcgen05)
PREFIX_SHAPES = [
    # B, Hq, Hkv, P
    (3, 4, 2, 300),     # GQA g=2, ragged tail, 1 q-tile
    (40, 8, 8, 1000),   # MHA
    (300, 4, 1, 257),   # g=4 -> 1200 stacked rows = 10 tiles, one token past a tile
    (1, 1, 1, 1),       # single row, single token
    (130, 1, 1, 128),   # exactly one KV block, 2 q-tiles (ragged rows)
    (16, 32, 8, 2048),  # Llama-3 GQA shape, g=4
]


@pytest.mark.parametrize("B,Hq,Hkv,P", PREFIX_SHAPES)
@pytest.mark.parametrize("dist", ["mixed", "boundary"])
@pytest.mark.parametrize("impl", [2, 3, 4, 5, 6, 9])
def test_prefix_tc_parity(B, Hq, Hkv, P, dist, impl):
    # 2: one-tile tcgen05 kernel, 3: persistent two-tile (128-token blocks), 4: same with 64-token
    # blocks and double-buffered scores, 5: 3 with the speculative (running-max) softmax,
    # 6: 3 with P published in two halves (default), 9: CTA-pair kernel (cta_group::2, M = 256,
    # double-buffered scores, token-split softmax; prefix_pair.cu)
    hydra.set_config("prefix_impl", min(impl, 3))
    hydra.set_config("prefix_variant", impl if impl >= 3 else 3)
    pb = synth.make_problem(B, Hq, Hkv, 128, P, 1, dtype="bf16", dist=dist, seed=3)
    t = problem_to(pb, DEV)
    o, lse = H.prefix_attn(t["q"], t["pk"], t["pv"])
    torch.cuda.synchronize()
    ref, lref = oracle.prefix_only(pb)
    assert_parity(o, ref, lse, lref, what=f"prefix {B},{Hq},{Hkv},{P}")


@pytest.mark.parametrize("splits", [1, 2, 3, 7])
def test_prefix_tc_splits(splits):
    hydra.set_config("prefix_impl", 2)
    hydra.set_config("prefix_splits", splits)
    pb = synth.make_problem(20, 8, 2, 128, 1100, 1, dtype="bf16", dist="mixed", seed=4)
    t = problem_to(pb, DEV)
    o, lse = H.prefix_attn(t["q"], t["pk"], t["pv"])
    torch.cuda.synchronize()
    ref, lref = oracle.prefix_only(pb)
    assert_parity(o, ref, lse, lref, what=f"prefix splits={splits}")


@pytest.mark.parametrize("variant,poly,steep", [(3, 0, 6), (5, 0, 6), (5, 4, 6), (5, 8, 6), (3, 4, 6), (6, 0, 6),
                                                (6, 4, 6), (9, 0, 6), (9, 4, 6), (9, 4, 60), (9, 0, 60)])
def test_prefix_tc2_growing_max(variant, poly, steep):
    """Scores that grow along the prefix: the running max is raised block after block, which
    exercises the O/l correction and, for the speculative softmax, the redo path.  The CTA-pair
    kernel raises its max only past +32 (log2 units): the steep ramp (K scaled up to 61x) makes
    it raise several times per row, in both softmax warpgroups."""
    hydra.set_config("prefix_impl", 3)
    hydra.set_config("prefix_variant", variant)
    hydra.set_config("prefix_poly", poly)
    hydra.set_config("pair_poly", poly)
    pb = synth.make_problem(300, 8, 2, 128, 2000, 1, dtype="bf16", dist="mixed", seed=11)
    ramp = (1.0 + steep * np.arange(pb.P, dtype=np.float64) / pb.P)[:, None, None]
    pb.pk = synth.gen.f32_to_bf16_bits((pb.f32("pk") * ramp).astype(np.float32))
    t = problem_to(pb, DEV)
    try:
        o, lse = H.prefix_attn(t["q"], t["pk"], t["pv"])
        torch.cuda.synchronize()
    finally:
        hydra.set_config("prefix_poly", 4)
        hydra.set_config("pair_poly", 0)
    ref, lref = oracle.prefix_only(pb)
    assert_parity(o, ref, lse, lref, what=f"prefix growing max v{variant} poly{poly} x{steep}")


@pytest.mark.parametrize("ctas", [1, 3, 7, 64, 148, 100000])
@pytest.mark.parametrize("variant", [3, 4, 5, 6, 9])
def test_prefix_tc2_stream_k_ctas(ctas, variant):
    """Stream-K piece boundaries fall inside items for most CTA counts; every piece is merged."""
    hydra.set_config("prefix_ctas", ctas)
    hydra.set_config("prefix_variant", variant)
    pb = synth.make_problem(300, 8, 2, 128, 1100, 1, dtype="bf16", dist="boundary", seed=4)
    t = problem_to(pb, DEV)
    o, lse = H.prefix_attn(t["q"], t["pk"], t["pv"])
    torch.cuda.synchronize()
    ref, lref = oracle.prefix_only(pb)
    assert_parity(o, ref, lse, lref, what=f"prefix ctas={ctas}")


@pytest.mark.parametrize("B,Hq,Hkv,P", [(1024, 40, 40, 700), (512, 32, 8, 1500), (256, 32, 4, 999), (77, 16, 1, 300),
                                        (5, 12, 4, 2000), (64, 64, 2, 129)])
@pytest.mark.parametrize("ctas,cluster", [(0, 0), (6, 0), (60, 0), (0, 1), (0, 2), (0, 4), (64, 4), (32, 2)])
def test_prefix_pair_shapes(B, Hq, Hkv, P, ctas, cluster):
    """CTA-pair kernel: MHA and GQA g = 4 / 8 / 16 / 32 (Q tiles by a 4-D TMA box of 128/g
    sequences), g = 3 (unsupported: the two-tile kernel runs instead), partial pairs (B*g not a
    multiple of 256), prefix tails inside the second token half of a block, grouped and
    ungrouped stream-K plans."""
    hydra.set_config("prefix_impl", 3)
    hydra.set_config("prefix_variant", 9)
    hydra.set_config("prefix_ctas", ctas)
    hydra.set_config("pair_cluster", cluster)  # pairs per cluster sharing K/V by multicast (0 = auto)
    pb = synth.make_problem(B, Hq, Hkv, 128, P, 1, dtype="bf16", dist="boundary", seed=B + P)
    t = problem_to(pb, DEV)
    try:
        o, lse = H.prefix_attn(t["q"], t["pk"], t["pv"])
        torch.cuda.synchronize()
    finally:
        hydra.set_config("pair_cluster", 0)
    ref, lref = oracle.prefix_only(pb)
    assert_parity(o, ref, lse, lref, what=f"pair prefix {B},{Hq},{Hkv},{P} ctas={ctas} cluster={cluster}")


@pytest.mark.parametrize("aux", [False, True])
@pytest.mark.parametrize("B,Hq,Hkv,P,S", [(40, 8, 8, 1000, 200), (24, 32, 8, 513, 33), (300, 8, 2, 2100, 300)])
def test_composite_pair_prefix(B, Hq, Hkv, P, S, aux):
    """hydra_attn with the CTA-pair prefix kernel in the sequential and the SM-partitioned schedule."""
    hydra.set_config("prefix_variant", 9)
    lens = np.random.default_rng(B + S).integers(0, S + 1, B)
    pb = synth.make_problem(B, Hq, Hkv, 128, P, S, lens=lens, dtype="bf16", dist="mixed", seed=71)
    out, lse = run_flat(pb, aux=aux)
    ref, lref = oracle.flat_attention(pb)
    assert_parity(out, ref, lse, lref, what="composite, pair prefix")


def test_prefix_simt_bf16():
    hydra.set_config("prefix_impl", 1)
    pb = synth.make_problem(9, 8, 2, 128, 333, 1, dtype="bf16", dist="mixed", seed=5)
    t = problem_to(pb, DEV)
    o, lse = H.prefix_attn(t["q"], t["pk"], t["pv"])
    torch.cuda.synchronize()
    ref, lref = oracle.prefix_only(pb)
    assert_parity(o, ref, lse, lref, what="prefix SIMT")


# ---------------------------------------------------------------- suffix kernel
@pytest.mark.parametrize("B,Hq,Hkv,d,S", [(7, 8, 8, 128, 300), (5, 16, 4, 128, 77), (6, 16, 1, 128, 40),
                                          (4, 8, 2, 64, 129), (3, 32, 2, 128, 64), (9, 12, 4, 128, 513),
                                          (8, 16, 8, 128, 200), (4, 32, 4, 128, 300)])  # g = 2, g = 8
@pytest.mark.parametrize("impl", [1, 2, 3])  # 1: SIMT split-K, 2/3: persistent tensor-core, 2 / 1 blocks per round
def test_suffix_parity(B, Hq, Hkv, d, S, impl):
    hydra.set_config("suffix_impl", min(impl, 2))
    hydra.set_config("suffix_cb", 1 if impl == 3 else 2)
    rng = np.random.default_rng(B * S)
    lens = rng.integers(0, S + 1, B)
    lens[0] = S
    pb = synth.make_problem(B, Hq, Hkv, d, 0, S, lens=lens, dtype="bf16", dist="mixed", seed=6)
    t = problem_to(pb, DEV)
    o, lse = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
    torch.cuda.synchronize()
    ref, lref = oracle.suffix_only(pb)
    assert_parity(o, ref, lse, lref, what="suffix")


@pytest.mark.parametrize("splits", [1, 2, 5])
def test_suffix_splits(splits):
    hydra.set_config("suffix_splits", splits)
    pb = synth.make_problem(6, 8, 2, 128, 0, 200, lens=[200, 3, 0, 150, 64, 1], dtype="bf16", dist="boundary",
                            seed=7)
    t = problem_to(pb, DEV)
    o, lse = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
    torch.cuda.synchronize()
    ref, lref = oracle.suffix_only(pb)
    assert_parity(o, ref, lse, lref, what=f"suffix splits={splits}")


# ---------------------------------------------------------------- composite (App. B)
COMPOSITE = [
    (4, 8, 1, 128, 300, 40),     # paper microbenchmark head shape (8 q / 1 kv), ragged
    (32, 32, 32, 128, 700, 64),  # CodeLlama-7b head shape (MHA)
    (24, 32, 8, 128, 513, 33),   # Llama-3 GQA
    (5, 4, 2, 64, 100, 20),      # d=64 (SIMT prefix)
]


@pytest.mark.parametrize("B,Hq,Hkv,d,P,S", COMPOSITE)
@pytest.mark.parametrize("dist", ["mixed", "boundary"])
@pytest.mark.parametrize("aux", [False, True])
def test_composite_parity(B, Hq, Hkv, d, P, S, dist, aux):
    rng = np.random.default_rng(P + S)
    lens = rng.integers(S // 2, S + 1, B)
    pb = synth.make_problem(B, Hq, Hkv, d, P, S, lens=lens, dtype="bf16", dist=dist, seed=8)
    out, lse = run_flat(pb, aux=aux)
    ref, lref = oracle.flat_attention(pb)
    assert out.dtype == torch.bfloat16
    assert_parity(out, ref, lse, lref, what="composite")


@pytest.mark.parametrize("B,Hq,Hkv,P,S,impls", [
    (40, 8, 8, 1000, 200, (3, 2)), (24, 32, 8, 513, 33, (3, 2)), (300, 8, 2, 2100, 300, (3, 1)),
    (33, 4, 1, 700, 129, (2, 2)), (64, 40, 40, 300, 0, (0, 0)), (5, 8, 2, 129, 140, (2, 1))])
@pytest.mark.parametrize("aux", [False, True])
def test_fused_combine_matches_separate_combine(B, Hq, Hkv, P, S, impls, aux):
    """The Eq. 5 merge fused into the kernel epilogues (fused.cuh: the writer of a row's last
    part merges it) against the separate combine launch (fuse_combine = 0): the same parts
    merged in the same order, so the outputs are bitwise equal -- for the persistent and the
    one-tile prefix kernels, both suffix kernels, both schedules, ragged and empty suffixes.
    fuse_combine = 2 forces the arrival-counter protocol in the SM-partitioned schedule too."""
    pi, si = impls
    hydra.set_config("prefix_variant", 6)  # the fused protocol's stream-K piece plan (not the CTA-pair kernel)
    hydra.set_config("prefix_impl", pi)
    hydra.set_config("suffix_impl", si)
    lens = np.random.default_rng(B + P).integers(0, S + 1, B)
    if S:
        lens[0] = 0
    pb = synth.make_problem(B, Hq, Hkv, 128, P, max(S, 1), lens=lens, dtype="bf16", dist="mixed", seed=61)
    res = []
    for fuse in (1, 2, 0):  # sequential only, counters in both schedules, never (default)
        hydra.set_config("fuse_combine", fuse)
        res.append(run_flat(pb, aux=aux))
    hydra.set_config("fuse_combine", 0)
    (a, la), (c, lc), (b, lb) = res
    ref, lref = oracle.flat_attention(pb)
    assert_parity(a, ref, la, lref, what="fused")
    assert_parity(c, ref, lc, lref, what="fused, counters")
    assert torch.equal(a, b) and torch.equal(la, lb), (a.float() - b.float()).abs().max()
    assert torch.equal(c, b) and torch.equal(lc, lb), (c.float() - b.float()).abs().max()


@pytest.mark.parametrize("k", [1, 50, 100, 147])
@pytest.mark.parametrize("B,Hq,Hkv,P,S", [(40, 8, 8, 1000, 200), (24, 32, 8, 513, 33)])
def test_composite_sm_partitioned(k, B, Hq, Hkv, P, S):
    """Persistent prefix (k CTAs) || persistent tensor-core suffix (SMs - k CTAs) on two streams."""
    hydra.set_config("prefix_impl", 3)
    hydra.set_config("suffix_impl", 2)
    hydra.set_config("overlap_prefix_ctas", k)
    rng = np.random.default_rng(k)
    lens = rng.integers(0, S + 1, B)
    pb = synth.make_problem(B, Hq, Hkv, 128, P, S, lens=lens, dtype="bf16", dist="boundary", seed=17)
    out, lse = run_flat(pb, aux=True)
    ref, lref = oracle.flat_attention(pb)
    assert_parity(out, ref, lse, lref, what=f"partitioned k={k}")


@pytest.mark.parametrize("B,Hq,Hkv,P,S", [(64, 8, 8, 4096, 300), (40, 16, 16, 2100, 129), (300, 4, 4, 4200, 64)])
def test_composite_simt_dependent(B, Hq, Hkv, P, S):
    """SM-partitioned schedule with the SIMT suffix (MHA) as the programmatic dependent of a
    prefix on a few persistent CTAs (overlap_simt forced; shapes with >= 8 blocks per prefix CTA at
    32 CTAs, the persistent kernel's minimum): the suffix grid's CTAs run beside the
    prefix and only its last CTA waits for the prefix grid -- the combine after it must still
    see every prefix part (ragged lens, NaN-poisoned padding, NaN-filled outputs)."""
    hydra.set_config("overlap_simt", 1)
    try:
        rng = np.random.default_rng(B)
        lens = rng.integers(0, S + 1, B)
        pb = synth.make_problem(B, Hq, Hkv, 128, P, S, lens=lens, dtype="bf16", dist="boundary", seed=46)
        out, lse = run_flat(pb, aux=True)
        assert hydra.get_config("last_overlap_simt") == 1 and hydra.get_config("last_overlap_k") >= 32
    finally:
        hydra.set_config("overlap_simt", 0)
    ref, lref = oracle.flat_attention(pb)
    assert_parity(out, ref, lse, lref, what=f"SIMT-dependent overlap B={B} H={Hq}")


@pytest.mark.parametrize("key,val", [("pair_item_cost", 5), ("pair_item_cost", 40), ("combine_pdl", 0)])
@pytest.mark.parametrize("B,Hq,Hkv,P,S", [(256, 32, 4, 5000, 100), (96, 16, 16, 3000, 200)])
def test_composite_optional_schedules(key, val, B, Hq, Hkv, P, S):
    """Schedule options that are off by default stay correct: cost-balanced stream-K group
    boundaries of the CTA-pair prefix (its pieces cut units unevenly; the slot count must cover
    them) and the combine as a programmatic dependent of the suffix kernel."""
    hydra.set_config(key, val)
    try:
        rng = np.random.default_rng(B + val)
        lens = rng.integers(0, S + 1, B)
        pb = synth.make_problem(B, Hq, Hkv, 128, P, S, lens=lens, dtype="bf16", dist="mixed", seed=47)
        out, lse = run_flat(pb)
        out2, lse2 = run_flat(pb, aux=True)
    finally:
        hydra.set_config(key, {"combine_pdl": 1}.get(key, 0))  # back to the library default
    ref, lref = oracle.flat_attention(pb)
    assert_parity(out, ref, lse, lref, what=f"{key}={val} sequential")
    assert_parity(out2, ref, lse2, lref, what=f"{key}={val} overlapped")


@pytest.mark.parametrize("k", [16, 64, 128])
@pytest.mark.parametrize("B,Hq,Hkv,P,S", [(256, 32, 4, 6000, 128), (120, 16, 4, 3000, 96), (64, 16, 8, 2500, 40),
                                         (120, 16, 4, 3000, 200)])
def test_composite_short_suffix_on_share(k, B, Hq, Hkv, P, S):
    """SM-partitioned schedule with the short-suffix kernel on the suffix's SM share (overlap_short,
    the default for short GQA suffixes): 3 x (SMs - k) short CTAs as the prefix's programmatic
    dependent, ragged lens with NaN-poisoned padding, NaN-filled outputs."""
    hydra.set_config("overlap_prefix_ctas", k)
    rng = np.random.default_rng(k + B)
    lens = rng.integers(0, S + 1, B)
    pb = synth.make_problem(B, Hq, Hkv, 128, P, S, lens=lens, dtype="bf16", dist="boundary", seed=48)
    out, lse = run_flat(pb, aux=True)
    assert hydra.get_config("last_overlap_k") > 0
    ref, lref = oracle.flat_attention(pb)
    assert_parity(out, ref, lse, lref, what=f"short suffix on the share k={k} g={Hq // Hkv}")


def test_composite_auto_overlap_small_shard():
    """A 5-KV-head shard (C3 on 8 GPUs, scaled down): too few prefix blocks for 148 persistent
    CTAs but enough for the automatic SM split, which must pick the persistent kernel for its
    own CTA count."""
    rng = np.random.default_rng(31)
    lens = rng.integers(64, 129, 256)
    pb = synth.make_problem(256, 5, 5, 128, 8192, 128, lens=lens, dtype="bf16", dist="mixed", seed=31)
    out, lse = run_flat(pb, aux=True)
    assert hydra.get_config("last_overlap_k") > 0
    ref, lref = oracle.flat_attention(pb)
    assert_parity(out, ref, lse, lref, what="auto overlap, 5-head shard")


@pytest.mark.parametrize("ctas", [1, 5, 148])
@pytest.mark.parametrize("cb", [1, 2])
def test_suffix_tc_ctas_and_ragged(ctas, cb):
    hydra.set_config("suffix_impl", 2)
    hydra.set_config("suffix_cb", cb)
    hydra.set_config("suffix_ctas", ctas)
    lens = [0, 1, 127, 128, 129, 255, 256, 300, 17, 0, 384]
    pb = synth.make_problem(len(lens), 8, 1, 128, 0, 384, lens=lens, dtype="bf16", dist="boundary", seed=18)
    t = problem_to(pb, DEV)
    o, lse = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
    torch.cuda.synchronize()
    ref, lref = oracle.suffix_only(pb)
    assert_parity(o, ref, lse, lref, what=f"suffix tc ctas={ctas} cb={cb}")


def test_suffix_tc_ragged_repeat():
    """Many ragged items with NaN-poisoned padding, repeated: the PV warp must zero the padded V
    rows of exactly the landed tile (a parity wait run ahead of the V ring once zeroed the wrong
    phase's tile and let NaN through, intermittently)."""
    hydra.set_config("suffix_impl", 2)
    lens = np.arange(600) % 301
    pb = synth.make_problem(600, 4, 4, 128, 0, 300, lens=lens, dtype="bf16", dist="boundary", seed=18)
    t = problem_to(pb, DEV)
    ref, lref = oracle.suffix_only(pb)
    for _ in range(8):
        o, lse = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
        torch.cuda.synchronize()
        assert_parity(o, ref, lse, lref, what="suffix tc ragged repeat")


@pytest.mark.parametrize("g", [2, 4, 8])
@pytest.mark.parametrize("ctas", [0, 1, 7])
def test_suffix_short_ragged(g, ctas):
    """Short-suffix kernel (suffix_short.cu, S_cap <= 256): ragged lens incl. 0, 1, 127, 128,
    129 and 256 with NaN-poisoned padding (V rows past lens[b] must be zeroed), every GQA width
    it takes, a grid of all resident CTAs (0), one CTA walking every item, and 7 (items dealt
    unevenly).  Same arithmetic as the persistent tensor-core kernel with 2-block rounds: the
    two agree bit for bit."""
    hydra.set_config("suffix_impl", 3)
    hydra.set_config("suffix_ctas", ctas)
    lens = [0, 1, 127, 128, 129, 255, 256, 200, 17, 0, 64, 128, 1]
    Hkv = 2
    pb = synth.make_problem(len(lens), g * Hkv, Hkv, 128, 0, 256, lens=lens, dtype="bf16", dist="boundary", seed=40 + g)
    t = problem_to(pb, DEV)
    o, lse = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
    torch.cuda.synchronize()
    ref, lref = oracle.suffix_only(pb)
    assert_parity(o, ref, lse, lref, what=f"suffix short g={g} ctas={ctas}")
    hydra.set_config("suffix_impl", 2)
    hydra.set_config("suffix_ctas", 0)
    o2, lse2 = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(lse, lse2), (o - o2).abs().max()


def test_suffix_short_two_block_jump_and_repeat():
    """Scores that jump between the two blocks of an item (the round max must cover both),
    many items (3 CTAs per SM, several items per CTA), repeated 6x on NaN-filled outputs."""
    hydra.set_config("suffix_impl", 3)
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 257, 700)
    pb = synth.make_problem(700, 32, 4, 128, 0, 256, lens=lens, dtype="bf16", dist="mixed", seed=44)
    ramp = np.ones((pb.S_cap, 1, 1))
    ramp[128:] = 9.0  # block 2 of every item scores ~9x higher
    pb.sk = synth.gen.f32_to_bf16_bits((pb.f32("sk") * ramp[None]).astype(np.float32))
    t = problem_to(pb, DEV)
    ref, lref = oracle.suffix_only(pb)
    for _ in range(6):
        o, lse = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
        torch.cuda.synchronize()
        assert_parity(o, ref, lse, lref, what="suffix short two-block jump")


@pytest.mark.parametrize("B,Hq,Hkv,P,S", [(256, 32, 4, 1500, 128), (96, 32, 8, 700, 100), (50, 16, 8, 300, 40),
                                         (96, 32, 8, 700, 200)])
def test_composite_short_suffix_auto(B, Hq, Hkv, P, S):
    """The automatic choice (suffix_impl 0) routes short GQA suffixes to the short kernel, in
    the sequential schedule as a programmatic dependent of the prefix: whole step vs oracle."""
    rng = np.random.default_rng(B)
    lens = rng.integers(0, S + 1, B)
    pb = synth.make_problem(B, Hq, Hkv, 128, P, S, lens=lens, dtype="bf16", dist="mixed", seed=45)
    out, lse = run_flat(pb)
    ref, lref = oracle.flat_attention(pb)
    assert_parity(out, ref, lse, lref, what=f"short-suffix composite B={B} g={Hq // Hkv}")


def test_composite_f32_output_is_tighter():
    pb = synth.make_problem(16, 8, 2, 128, 600, 50, dtype="bf16", dist="mixed", seed=9)
    out, lse = run_flat(pb, out_dtype=torch.float32)
    ref, _ = oracle.flat_attention(pb)
    mx, mean, _ = errors(out, ref)
    assert mx <= 5e-3 and mean <= 5e-4, (mx, mean)


@pytest.mark.parametrize("P,lens", [(0, [5, 0, 9]), (200, [0, 0, 0]), (0, [0, 0, 0]), (1, [0, 1, 17]),
                                    (129, [128, 127, 1])])
def test_edge_cases(P, lens):
    pb = synth.make_problem(3, 4, 2, 128, P, 17 if max(lens) <= 17 else 128, lens=lens, dtype="bf16",
                            dist="mixed", seed=10)
    out, lse = run_flat(pb)
    ref, lref = oracle.flat_attention(pb)
    if P == 0 and max(lens) == 0:  # no keys at all: out = 0, lse = -inf (reading R6)
        assert (out.float() == 0).all() and torch.isneginf(lse).all()
        return
    assert_parity(out, ref, lse, lref, what=f"edge P={P} lens={lens}")


def test_determinism_bitwise():
    pb = synth.make_problem(64, 8, 2, 128, 1500, 100, dtype="bf16", dist="mixed", seed=11)
    a, la = run_flat(pb)
    b, lb = run_flat(pb)
    assert torch.equal(a, b) and torch.equal(la, lb)


def test_lens_out_of_range_is_clamped():
    """lens[b] outside [0, S_cap] violates the documented precondition; the release kernels
    clamp it (hydra.h): lens > S_cap attends all S_cap rows, lens < 0 none -- never a read
    past the cache (both suffix kernels)."""
    pb = synth.make_problem(4, 8, 2, 128, 100, 32, lens=[32, 0, 5, 32], dtype="bf16", dist="mixed", seed=3)
    ref, lref = oracle.flat_attention(pb)
    for impl in (1, 2):
        hydra.set_config("suffix_impl", impl)
        t = problem_to(pb, DEV)
        t["lens"].copy_(torch.tensor([40, -3, 5, 1 << 30], dtype=torch.int32))
        out, lse = H.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True)
        torch.cuda.synchronize()
        assert_parity(out, ref, lse, lref, what=f"clamped lens impl={impl}")


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("B,P,S", [(32, 1024, 64), (7, 300, 129)])
def test_per_sequence_baseline_parity(impl, B, P, S):
    """The microbenchmark's comparison path (bench.py --config grid; P:160 / P:177-192): each
    sequence attends over its own copy of prefix || suffix with the per-sequence kernels --
    the same attention, so it must match the oracle like the Hydragen path does."""
    from paper_2402_05099_b200 import baseline

    hydra.set_config("suffix_impl", impl)
    lens = np.random.default_rng(B).integers(0, S + 1, B)
    pb = synth.make_problem(B, 8, 1, 128, P, S, lens=lens, dtype="bf16", dist="mixed", seed=50)
    t = problem_to(pb, DEV)
    fk, fv, flens = baseline.per_sequence_cache(t["pk"], t["pv"], t["sk"], t["sv"], t["lens"])
    o, l = H.suffix_attn(t["q"], fk, fv, flens)
    torch.cuda.synchronize()
    ref, lref = oracle.flat_attention(pb)
    assert_parity(o, ref, l, lref, what=f"per-sequence baseline impl={impl}")


# ---------------------------------------------------------------- tree (§3.3)
@pytest.mark.parametrize("impl", [0, 1, 2])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_tree_parity(impl, dtype):
    if dtype == "f32" and impl == 0:
        pytest.skip("f32 always runs the SIMT path")
    hydra.set_config("prefix_impl", impl)
    parent, node_len, leaf = synth.two_level_tree(300, 3, 150, 5)
    # add a third level under branch 1 to exercise depth > 2 and ragged paths
    parent = list(parent) + [1]
    node_len = list(node_len) + [70]
    leaf = np.array(leaf)
    leaf[:5] = 4  # branch 1's sequences now sit one level deeper
    d = 128
    tp = synth.make_tree_problem(parent, node_len, leaf, 8, 2, d, 40, lens=np.arange(15) % 41, dtype=dtype,
                                 dist="mixed", seed=13)
    t = tree_to(tp, DEV)
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
    assert tree.depth() == 3 and tree.group_size(0) == 15 and tree.group_size(4) == 5
    out, lse = H.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"],
                                    return_lse=True)
    torch.cuda.synchronize()
    ref, lref = oracle.tree_attention(tp)
    assert_parity(out, ref, lse, lref, dtype=dtype, what=f"tree impl={impl}")
    tree.destroy()


@pytest.mark.parametrize("k", [1, 37, 147])
@pytest.mark.parametrize("per,g", [(300, 1), (100, 4)])
def test_tree_sm_partitioned(k, per, g):
    """Tree node attention on k SMs (aux stream) || tensor-core suffix on the other SMs."""
    hydra.set_config("prefix_impl", 3)
    hydra.set_config("suffix_impl", 2)
    hydra.set_config("overlap_prefix_ctas", k)
    parent, node_len, leaf = synth.two_level_tree(300, 2, 200, per)
    tp = synth.make_tree_problem(parent, node_len, leaf, 4 * g, 4, 128, 300, dtype="bf16", dist="boundary",
                                 seed=23, lens=np.arange(2 * per) % 301)
    t = tree_to(tp, DEV)
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
    out, lse = H.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"],
                                    return_lse=True, aux_stream=torch.cuda.Stream())
    torch.cuda.synchronize()
    assert hydra.get_config("last_overlap_k") == k
    ref, lref = oracle.tree_attention(tp)
    assert_parity(out, ref, lse, lref, what=f"tree partitioned k={k}")
    tree.destroy()


def test_tree_first_use_is_captured_in_a_graph():
    """A prepared tree's attention is a pure launch sequence (hydra.h): its FIRST call can be
    captured in a CUDA graph (the paper's CUDA-graph requirement), and the replay is
    exact; an unprepared tree refuses capture with nothing launched."""
    parent, node_len, leaf = synth.two_level_tree(300, 3, 150, 40)
    tp = synth.make_tree_problem(parent, node_len, leaf, 8, 2, 128, 64, lens=np.arange(120) % 65, dtype="bf16",
                                 dist="mixed", seed=33)
    t = tree_to(tp, DEV)
    ref, lref = oracle.tree_attention(tp)
    cold = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
    out = torch.full((120, 8, 128), float("nan"), dtype=torch.bfloat16, device=DEV)
    lse = torch.full((120, 8), float("nan"), dtype=torch.float32, device=DEV)
    ws = H.nan_bytes(hydra.workspace_bytes_tree(t["q"], cold, 2, 64), DEV)
    g = torch.cuda.CUDAGraph()
    with pytest.raises(hydra.HydraError, match="prepare"):
        with torch.cuda.graph(g):
            hydra.tree_attention(t["q"], cold, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"], out=out,
                                 lse_out=lse, workspace=ws)
    cold.destroy()
    torch.cuda.synchronize()
    for aux in (None, torch.cuda.Stream()):
        tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq, heads=(8, 2))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):  # the tree's first call
            hydra.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"], out=out,
                                 lse_out=lse, workspace=ws, aux_stream=aux)
        for _ in range(2):
            out.fill_(float("nan")); lse.fill_(float("nan")); ws.fill_(0xFF)
            g.replay()
            torch.cuda.synchronize()
            assert_parity(out, ref, lse, lref, what=f"captured tree aux={aux is not None}")
        del g
        tree.destroy()


def test_one_level_tree_equals_flat():
    pb = synth.make_problem(20, 8, 2, 128, 400, 30, dtype="bf16", dist="mixed", seed=14)
    t = problem_to(pb, DEV)
    tree = hydra.Tree([-1], [0], [pb.P], np.zeros(pb.B, np.int32))
    a = H.tree_attention(t["q"], tree, t["pk"], t["pv"], t["sk"], t["sv"], t["lens"])
    b = H.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"])
    torch.cuda.synchronize()
    ref, _ = oracle.flat_attention(pb)
    assert_parity(a, ref, what="one-level tree")
    assert_parity(b, ref, what="flat")


# ---------------------------------------------------------------- combine as a standalone op
def test_combine_f16_parts_and_identity():
    rng = np.random.default_rng(15)
    n, rows, d = 3, 50, 128
    o = rng.standard_normal((n, rows, d))
    l = rng.uniform(-5, 5, (n, rows))
    l[1, :10] = -np.inf  # empty parts are skipped
    ref_o, ref_l = o[0], l[0]
    for i in range(1, n):
        ref_o, ref_l = oracle.combine(ref_o, ref_l, o[i], l[i])
    ot = torch.tensor(o, dtype=torch.float16, device=DEV)
    lt = torch.tensor(l, dtype=torch.float32, device=DEV)
    out, lse = H.combine(ot, lt, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref16 = ot.cpu().double().numpy()  # the exact fp16 values the kernel read
    l32 = lt.cpu().double().numpy()
    ro, rl = ref16[0], l32[0]
    for i in range(1, n):
        ro, rl = oracle.combine(ro, rl, ref16[i], l32[i])
    np.testing.assert_allclose(out.cpu().numpy(), ro, atol=2e-6)
    np.testing.assert_allclose(lse.cpu().numpy(), rl, atol=2e-6)


# ---------------------------------------------------------------- multi-GPU layer, kernel side
def test_seqsplit_single_rank_nccl():
    """dist.seqsplit_attention on a 1-rank NCCL group: f16 packing of the prefix partials,
    all-gather, strided combine of the gathered parts, suffix, final combine."""
    import socket

    import torch.distributed as tdist
    from paper_2402_05099_b200 import dist as hdist

    if not tdist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        pb = synth.make_problem(24, 32, 8, 128, 700, 40, dtype="bf16", dist="mixed", seed=31)
        t = problem_to(pb, DEV)
        for ex in (torch.float16, torch.float32):
            out, lse = hdist.seqsplit_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"],
                                                exchange_dtype=ex, return_lse=True)
            torch.cuda.synchronize()
            ref, lref = oracle.flat_attention(pb)
            assert_parity(out, ref, lse, lref, what=f"seqsplit {ex}")
    finally:
        tdist.destroy_process_group()


def test_seqsplit_single_rank_p2p():
    """exchange="p2p" on a 1-rank NCCL group: the pack stores into the (symmetric-memory) receive
    buffer through the output table, then the device barrier and the merge -- the multi-rank
    data path with the one GPU this environment has (skipped if symmetric memory is missing)."""
    import socket

    import torch.distributed as tdist
    from paper_2402_05099_b200 import dist as hdist

    if not tdist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                 device_id=torch.device(DEV))
    try:
        pb = synth.make_problem(24, 32, 8, 128, 700, 40, dtype="bf16", dist="mixed", seed=33)
        t = problem_to(pb, DEV)
        try:
            out, lse = hdist.seqsplit_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"],
                                                exchange="p2p", return_lse=True)
        except (RuntimeError, NotImplementedError) as e:
            pytest.skip(f"symmetric memory unavailable: {e}")
        torch.cuda.synchronize()
        ref, lref = oracle.flat_attention(pb)
        assert_parity(out, ref, lse, lref, what="seqsplit p2p")
        a2a = hdist.seqsplit_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], exchange="alltoall")
        assert torch.equal(out, a2a)
    finally:
        hdist.release_plans()
        tdist.destroy_process_group()


@pytest.mark.parametrize("rows,table_rows,edt", [(1000, 256, torch.float16), (777, 100, torch.float32),
                                                  (64, 64, torch.bfloat16)])
def test_combine_scatter_matches_combine(rows, table_rows, edt):
    """hydra_combine_ex with an output table (the p2p pack): rows scattered over several buffers
    with interleaved (O | LSE) rows equal the dense combine bit for bit, and nothing outside the
    addressed rows is written."""
    g = torch.Generator(device=DEV)
    g.manual_seed(rows)
    d = 128
    o = torch.randn(3, rows, d, device=DEV, generator=g)
    lse = torch.randn(3, rows, device=DEV, generator=g)
    lse[1, ::7] = -float("inf")
    ref, lref = hydra.combine(o, lse, out_dtype=edt)
    n_tab = -(-rows // table_rows)
    esz = torch.empty((), dtype=edt).element_size()
    row_bytes = (d * esz + 4 + 15) // 16 * 16
    bufs = [torch.full((table_rows * row_bytes + 64,), 0x7F, dtype=torch.uint8, device=DEV) for _ in range(n_tab)]
    otab = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    ltab = torch.tensor([b.data_ptr() + d * esz for b in bufs], dtype=torch.int64, device=DEV)
    hydra.combine_scatter(o, lse, otab, table_rows, row_bytes // esz, out_dtype=edt, lse_table=ltab,
                          lse_row_stride=row_bytes // 4)
    torch.cuda.synchronize()
    for t, b in enumerate(bufs):
        r0, r1 = t * table_rows, min(rows, (t + 1) * table_rows)
        n = r1 - r0
        got_o = b[:n * row_bytes].view(n, row_bytes)[:, :d * esz].contiguous().view(edt).view(n, d)
        got_l = b[:n * row_bytes].view(n, row_bytes)[:, d * esz:d * esz + 4].contiguous().view(torch.float32).view(n)
        assert torch.equal(got_o, ref[r0:r1]) and torch.equal(got_l, lref[r0:r1])
        assert bool((b[n * row_bytes:] == 0x7F).all()), "stores past the table's rows"


@pytest.mark.parametrize("impl", [0, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("per,g", [(300, 1), (100, 4)])
def test_tree_large_groups(impl, per, g):
    """Groups with > 128 and > 256 stacked rows: both query tiles of a pair and several pairs
    per node (the persistent kernel's task mode), on root and branch nodes."""
    hydra.set_config("prefix_impl", min(impl, 3))
    hydra.set_config("prefix_variant", impl if impl >= 3 else 3)
    parent, node_len, leaf = synth.two_level_tree(300, 2, 200, per)
    tp = synth.make_tree_problem(parent, node_len, leaf, 4 * g, 4, 128, 24, dtype="bf16", dist="boundary", seed=19)
    t = tree_to(tp, DEV)
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
    out, lse = H.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"],
                                    return_lse=True)
    torch.cuda.synchronize()
    ref, lref = oracle.tree_attention(tp)
    assert_parity(out, ref, lse, lref, what=f"tree large groups impl={impl} per={per} g={g}")
    tree.destroy()


@pytest.mark.parametrize("splits", [2, 3, 5])
@pytest.mark.parametrize("g", [1, 4, 8])
def test_suffix_tc_split_k(splits, g):
    """Tensor-core suffix with split-K over tokens (512-token-or-longer suffixes on few items):
    ragged lengths that end inside, at, and before split boundaries, empty splits, empty
    sequences; partials combined by the library."""
    hydra.set_config("suffix_impl", 2)
    hydra.set_config("suffix_splits", splits)
    try:
        B, Hkv, S = 6, 2, 700
        lens = [700, 0, 1, 128, 256 + 5, 511]
        pb = synth.make_problem(B, Hkv * g, Hkv, 128, 0, S, lens=lens, dtype="bf16", dist="mixed", seed=40 + g)
        t = problem_to(pb, DEV)
        o, l = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
        torch.cuda.synchronize()
        ref, lref = oracle.suffix_only(pb)
        assert_parity(o, ref, l, lref, what=f"suffix_tc split-K s={splits} g={g}")
    finally:
        hydra.set_config("suffix_splits", 0)
        hydra.set_config("suffix_impl", 0)


def test_suffix_gqa_long_suffix_auto():
    """Auto policy: GQA, 512 items on 148 SMs, 2048-token suffixes -> the tensor-core kernel on
    the full chip; sampled rows vs the oracle, and the paged call gives the same bits."""
    B, Hq, Hkv, S = 128, 32, 4, 2048
    rng = np.random.default_rng(3)
    lens = rng.integers(1500, S + 1, B).astype(np.int32)
    pb = synth.make_problem(B, Hq, Hkv, 128, 0, S, lens=lens, dtype="bf16", dist="mixed", seed=77)
    t = problem_to(pb, DEV)
    o, l = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
    torch.cuda.synchronize()
    rows = np.array([(b, h) for b in (0, 1, 63, 127) for h in (0, 7, 8, 31)])
    ref, lref = oracle.suffix_only(pb, rows=rows)
    assert_parity(o[rows[:, 0], rows[:, 1]], ref, l[rows[:, 0], rows[:, 1]], lref, what="auto split long suffix")
    pc = synth.paginate(pb, 64, seed=2)
    kp, vp = (torch.from_numpy(x).view(torch.bfloat16).to(DEV) for x in (pc.k_pool, pc.v_pool))
    o2, l2 = H.suffix_attn_paged(t["q"], kp, vp, torch.from_numpy(pc.block_table).to(DEV), t["lens"], S_cap=S)
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(l, l2)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("rows", [1, 7, 33, 1001])
def test_combine_part_counts_and_odd_rows(n, rows):
    """The combine kernels for 2 / 4 / 8 parts at two rows per warp: odd row counts (a warp's
    second row past the end), all-empty rows, NaN in an empty part's unwritten slot."""
    rng = np.random.default_rng(n * 1000 + rows)
    o = rng.standard_normal((n, rows, 128))
    l = rng.uniform(-6, 6, (n, rows))
    l[0, ::3] = -np.inf
    if n > 1:
        l[:, rows // 2] = -np.inf  # every part empty for this row
        o[1, l[1] == -np.inf] = np.nan  # garbage in slots the combine must not read
        l[1, ::2] = -np.inf
        o[1, l[1] == -np.inf] = np.nan
    o_ref = np.where(np.isneginf(l)[..., None], 0.0, o)  # an empty part is the (0, -inf) sentinel (R6)
    ref_o, ref_l = o_ref[0], l[0]
    for i in range(1, n):
        ref_o, ref_l = oracle.combine(ref_o, ref_l, o_ref[i], l[i])
    ot = torch.tensor(o, dtype=torch.float32, device=DEV)
    lt = torch.tensor(l, dtype=torch.float32, device=DEV)
    out, lse = H.combine(ot, lt, out_dtype=torch.float32)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.isfinite(got).all()
    np.testing.assert_allclose(got, ref_o, atol=2e-5)
    np.testing.assert_array_equal(np.isneginf(lse.cpu().numpy()), np.isneginf(ref_l))
    fin = np.isfinite(ref_l)
    np.testing.assert_allclose(lse.cpu().numpy()[fin], ref_l[fin], atol=2e-5)
