"""Pins for the fp64 oracle (oracle/): it is checked against things other than itself.

Each test names the passage or mathematical fact that fixes the expected value:
closed forms, SPEC worked examples (tests/golden/spec_examples.json), invariants
the paper states (App. A decomposition exactness, query independence P:114),
and 50-digit brute force on tiny inputs.  A plausible oracle bug (dropped term,
wrong sign, transposed operand, wrong head map, wrong scale, wrong log base,
reading past lens) fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def f32(a):
    return np.ascontiguousarray(np.asarray(a, np.float32))


def one_row(q, K, V, scale=None):
    """Attention of a single query q[d] over K[N,d], V[N,d] (Hq = Hkv = 1)."""
    q = f32(q).reshape(1, 1, -1)
    K = f32(K).reshape(len(K), 1, -1)
    V = f32(V).reshape(len(V), 1, -1)
    o, l = oracle.attention_segments(q, [[(K, V)]], 1, scale)
    return o[0, 0], l[0, 0]


# ----------------------------------------------------------------- SPEC examples
def test_spec_zero_query():
    e = GOLD["zero_query_two_keys"]
    o, l = one_row(e["q"], e["k"], e["v"])
    np.testing.assert_allclose(o, e["out"], rtol=0, atol=1e-15)
    assert abs(l - e["lse"]) < 1e-15


def test_spec_single_key():
    e = GOLD["single_key"]
    o, l = one_row(e["q"], e["k"], e["v"])
    np.testing.assert_array_equal(o, e["out"])  # singleton softmax: weight exactly 1
    assert abs(l - e["lse"]) < 1e-15  # natural log over SCALED scores: 2/sqrt(2)


def test_spec_softmax_uniform_and_large():
    # scores [0,0]: d=1, scale=1, q=0 ; scores [1000,1000]: q=1000, k=1 (max-shift needed)
    for key, qv in (("softmax_uniform", 0.0), ("softmax_large", 1000.0)):
        e = GOLD[key]
        V = [[1.0], [4.0]]
        o, l = one_row([qv], [[1.0], [1.0]], V, scale=1.0)
        assert abs(l - e["lse"]) < 1e-12
        assert abs(o[0] - (e["probs"][0] * 1.0 + e["probs"][1] * 4.0)) < 1e-15


def test_spec_combine_examples():
    for key in ("combine_example", "combine_equal_lse", "combine_empty"):
        e = GOLD[key]
        l2 = -math.inf if e["lse2"] == "-inf" else e["lse2"]
        o, l = oracle.combine(np.array([e["out1"]]), np.array([e["lse1"]]), np.array([e["out2"]]), np.array([l2]))
        if key == "combine_empty":
            np.testing.assert_array_equal(o[0], e["out"])  # bit-for-bit identity
            assert l[0] == e["lse"]
        else:
            np.testing.assert_allclose(o[0], e["out"], rtol=0, atol=1e-15)
            assert abs(l[0] - e["lse"]) < 1e-15


def test_spec_log_add_exp_value():
    e = GOLD["log_add_exp"]
    _, l = oracle.combine(np.zeros((1, 1)), np.array([e["a"]]), np.zeros((1, 1)), np.array([e["b"]]))
    assert abs(l[0] - e["value"]) < 1e-14


# ----------------------------------------------------------------- closed forms
def test_identical_keys_give_mean_of_values():
    rng = np.random.default_rng(1)
    d, N = 16, 37
    q = rng.standard_normal(d).astype(np.float32)
    k = rng.standard_normal(d).astype(np.float32)
    V = rng.standard_normal((N, d)).astype(np.float32)
    o, l = one_row(q, np.tile(k, (N, 1)), V)
    s = float(np.dot(q.astype(np.float64), k.astype(np.float64))) / math.sqrt(d)
    np.testing.assert_allclose(o, V.astype(np.float64).mean(0), rtol=0, atol=1e-14)
    assert abs(l - (s + math.log(N))) < 1e-13


def test_two_key_closed_form_weights_one_quarter_three_quarters():
    # d=4, scale=1/sqrt(4)=1/2, q=(2,0,0,0) => s_t = K[t,0]; scores 0 and ln3 => weights 1/4, 3/4
    ln3 = np.float32(math.log(3.0))
    K = [[0, 5, -1, 2], [ln3, -5, 7, 1]]
    V = [[4.0, 0.0, -8.0, 1.0], [0.0, 8.0, 4.0, 1.0]]
    o, l = one_row([2, 0, 0, 0], K, V)
    e = math.exp(float(ln3))  # = 3 up to the fp32 rounding of ln 3
    w2 = e / (1 + e)
    np.testing.assert_allclose(o, (1 - w2) * np.array(V[0]) + w2 * np.array(V[1]), rtol=0, atol=1e-14)
    assert abs(l - math.log(1 + e)) < 1e-15
    assert abs(w2 - 0.75) < 1e-7


def test_constant_values_weights_sum_to_one():
    pb = synth.make_problem(3, 4, 2, 32, 50, 9, lens=[9, 0, 4], dtype="f32", dist="mixed", seed=3)
    pb.pv[:] = 1.5
    pb.sv[:] = 1.5
    o, _ = oracle.flat_attention(pb)
    np.testing.assert_allclose(o, 1.5, rtol=0, atol=1e-14)


def test_gqa_head_map_floor():
    # Hq=4, Hkv=2: heads 0,1 -> kv head 0 ; heads 2,3 -> kv head 1 (reading R3)
    pb = synth.make_problem(2, 4, 2, 8, 6, 3, dtype="f32", seed=5)
    pb.pv[:, 0] = 1.0
    pb.pv[:, 1] = 2.0
    pb.sv[:, :, 0] = 1.0
    pb.sv[:, :, 1] = 2.0
    o, _ = oracle.flat_attention(pb)
    np.testing.assert_allclose(o[:, :2], 1.0, atol=1e-14)
    np.testing.assert_allclose(o[:, 2:], 2.0, atol=1e-14)


def test_shift_invariance_exact_integers():
    # K -> K + u shifts every score by scale*q.u: O unchanged, LSE shifted (max-subtraction pin)
    rng = np.random.default_rng(7)
    d, N = 8, 21
    q = rng.integers(-3, 4, d).astype(np.float32)
    K = rng.integers(-3, 4, (N, d)).astype(np.float32)
    V = rng.standard_normal((N, d)).astype(np.float32)
    u = rng.integers(-20, 21, d).astype(np.float32)
    o1, l1 = one_row(q, K, V)
    o2, l2 = one_row(q, K + u, V)
    np.testing.assert_allclose(o2, o1, rtol=0, atol=1e-13)
    assert abs((l2 - l1) - float(q @ u) / math.sqrt(d)) < 1e-12


def test_linearity_in_values():
    rng = np.random.default_rng(8)
    d, N = 16, 30
    q, K = rng.standard_normal(d), rng.standard_normal((N, d))
    V1, V2 = rng.integers(-4, 5, (N, d)), rng.integers(-4, 5, (N, d))
    o1, _ = one_row(q, K, V1)
    o2, _ = one_row(q, K, V2)
    o3, _ = one_row(q, K, V1 + V2)
    np.testing.assert_allclose(o3, o1 + o2, rtol=0, atol=1e-13)


def test_mpmath_brute_force_tiny():
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 50
    rng = np.random.default_rng(11)
    for trial in range(4):
        d, N = int(rng.integers(1, 6)), int(rng.integers(1, 5))
        q = rng.standard_normal(d).astype(np.float32) * 3
        K = rng.standard_normal((N, d)).astype(np.float32) * 3
        V = rng.standard_normal((N, d)).astype(np.float32)
        o, l = one_row(q, K, V)
        sc = 1 / mp.sqrt(d)
        s = [sc * mp.fsum(mp.mpf(float(q[i])) * mp.mpf(float(K[t, i])) for i in range(d)) for t in range(N)]
        den = mp.fsum(mp.e ** x for x in s)
        for i in range(d):
            ref = mp.fsum(mp.e ** s[t] * mp.mpf(float(V[t, i])) for t in range(N)) / den
            assert abs(float(ref) - o[i]) <= 1e-13 * (1 + abs(float(ref)))
        assert abs(float(mp.log(den)) - l) <= 1e-13 * (1 + abs(l))


# ----------------------------------------------------------------- paper invariants
@pytest.mark.parametrize("B,Hq,Hkv,d,P,S", [(4, 2, 1, 16, 32, 12), (3, 8, 2, 64, 0, 9), (2, 4, 4, 32, 17, 1)])
@pytest.mark.parametrize("dist", ["plain", "mixed"])
def test_decomposition_matches_undecomposed(B, Hq, Hkv, d, P, S, dist):
    """App. A: combine(SDP(K1), SDP(K2)) == SDP(K1 || K2)."""
    lens = np.random.default_rng(B * 100 + P).integers(0, S + 1, B)
    for dtype in ("bf16", "f32"):
        pb = synth.make_problem(B, Hq, Hkv, d, P, S, lens=lens, dtype=dtype, dist=dist, seed=2)
        of, lf = oracle.flat_attention(pb)
        op, lp = oracle.prefix_only(pb)
        os_, ls = oracle.suffix_only(pb)
        oc, lc = oracle.combine(op, lp, os_, ls)
        np.testing.assert_allclose(oc, of, rtol=0, atol=1e-12)
        fin = np.isfinite(lf)
        np.testing.assert_allclose(lc[fin], lf[fin], rtol=0, atol=1e-12)
        assert (np.isneginf(lc) == np.isneginf(lf)).all()


def test_chunked_seven_segments_equal_monolith():
    """seven length-1 segments vs the length-7 monolith (iterated Eq. 5)."""
    rng = np.random.default_rng(4)
    d = 16
    q = f32(rng.standard_normal((1, 1, d)))
    K = f32(rng.standard_normal((7, 1, d)))
    V = f32(rng.standard_normal((7, 1, d)))
    om, lm = oracle.attention_segments(q, [[(K, V)]], 1)
    o, l = None, None
    for t in range(7):
        ot, lt = oracle.attention_segments(q, [[(K[t:t + 1], V[t:t + 1])]], 1)
        o, l = (ot, lt) if o is None else oracle.combine(o, l, ot, lt)
    np.testing.assert_allclose(o, om, atol=1e-14)
    np.testing.assert_allclose(l, lm, atol=1e-14)


def test_kv_permutation_and_batch_equivariance():
    """Queries are independent and attention is a set operation over KV rows."""
    pb = synth.make_problem(5, 4, 2, 16, 23, 7, lens=[7, 3, 0, 5, 1], dtype="f32", dist="mixed", seed=9)
    o, l = oracle.flat_attention(pb)
    perm = np.random.default_rng(0).permutation(pb.P)
    pb2 = synth.make_problem(5, 4, 2, 16, 23, 7, lens=[7, 3, 0, 5, 1], dtype="f32", dist="mixed", seed=9)
    pb2.pk, pb2.pv = np.ascontiguousarray(pb.pk[perm]), np.ascontiguousarray(pb.pv[perm])
    o2, l2 = oracle.flat_attention(pb2)
    np.testing.assert_allclose(o2, o, atol=1e-13)
    np.testing.assert_allclose(l2, l, atol=1e-13)
    bp = np.array([3, 0, 4, 1, 2])
    pb2 = synth.make_problem(5, 4, 2, 16, 23, 7, lens=[7, 3, 0, 5, 1], dtype="f32", dist="mixed", seed=9)
    pb2.q, pb2.sk, pb2.sv, pb2.lens = pb.q[bp].copy(), pb.sk[bp].copy(), pb.sv[bp].copy(), pb.lens[bp].copy()
    o3, l3 = oracle.flat_attention(pb2)
    np.testing.assert_array_equal(o3, o[bp])
    np.testing.assert_array_equal(l3, l[bp])


def test_one_token_prefix_reduces_to_ordinary_attention():
    """P = 1: prefix part is (v0, s0); composite = plain attention over 1+lens tokens."""
    pb = synth.make_problem(3, 2, 1, 16, 1, 5, lens=[5, 2, 0], dtype="f32", seed=12)
    op, lp = oracle.prefix_only(pb)
    for b in range(3):
        for h in range(2):
            np.testing.assert_array_equal(op[b, h], pb.pv[0, 0].astype(np.float64))
            s0 = float(pb.q[b, h].astype(np.float64) @ pb.pk[0, 0].astype(np.float64)) / 4.0
            assert abs(lp[b, h] - s0) < 1e-14
    o, l = oracle.flat_attention(pb)
    # lens=0 sequence: the result is exactly the single prefix value row
    np.testing.assert_array_equal(o[2, 0], pb.pv[0, 0].astype(np.float64))


def test_empty_sets_and_empty_parts():
    pb = synth.make_problem(3, 2, 1, 16, 0, 4, lens=[4, 0, 2], dtype="bf16", seed=13)
    o, l = oracle.flat_attention(pb)
    assert np.isneginf(l[1]).all() and (o[1] == 0).all()  # no keys at all: sentinel (R6)
    os_, ls = oracle.suffix_only(pb)
    np.testing.assert_array_equal(o, os_)  # empty prefix == suffix-only
    pb = synth.make_problem(3, 2, 1, 16, 9, 4, lens=[0, 0, 0], dtype="bf16", seed=13)
    o, l = oracle.flat_attention(pb)
    op, lp = oracle.prefix_only(pb)
    np.testing.assert_array_equal(o, op)  # zero-length suffixes == prefix attention


def test_poisoned_padding_is_never_read():
    pb = synth.make_problem(4, 2, 1, 16, 32, 12, lens=[5, 8, 10, 12], dtype="bf16", seed=1)
    assert (pb.sk[0, 5:] == synth.BF16_NAN).all()
    o, l = oracle.flat_attention(pb)
    assert np.isfinite(o).all() and np.isfinite(l).all()


def test_strided_query_view():
    pb = synth.make_problem(3, 4, 2, 16, 10, 4, dtype="f32", seed=14)
    big = np.zeros((3, 8, 16), np.float32)
    big[:, ::2] = pb.q
    o1, l1 = oracle.attention_segments(pb.q, [[(pb.pk, pb.pv)]] * 3, 2)
    o2, l2 = oracle.attention_segments(big[:, ::2], [[(pb.pk, pb.pv)]] * 3, 2)
    np.testing.assert_array_equal(o1, o2)


def test_row_subset_matches_full():
    pb = synth.make_problem(6, 4, 2, 16, 20, 5, dtype="bf16", dist="mixed", seed=15)
    o, l = oracle.flat_attention(pb)
    rows = np.array([[5, 3], [0, 0], [2, 1]])
    os_, ls = oracle.flat_attention(pb, rows=rows)
    for i, (b, h) in enumerate(rows):
        np.testing.assert_array_equal(os_[i], o[b, h])
        assert ls[i] == l[b, h]


# ----------------------------------------------------------------- combine (App. B vs Eq. 5)
def test_stabilized_combine_equals_raw_eq5():
    """App. B's max-shifted combine equals raw Eq. 5 when exp does not overflow."""
    rng = np.random.default_rng(21)
    o1, o2 = rng.standard_normal((50, 8)), rng.standard_normal((50, 8))
    l1, l2 = rng.uniform(-30, 30, 50), rng.uniform(-30, 30, 50)
    o, l = oracle.combine(o1, l1, o2, l2)
    raw = (o1 * np.exp(l1)[:, None] + o2 * np.exp(l2)[:, None]) / (np.exp(l1) + np.exp(l2))[:, None]
    np.testing.assert_allclose(o, raw, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(l, np.log(np.exp(l1) + np.exp(l2)), rtol=1e-12, atol=1e-12)


def test_combine_extreme_lse_finite_and_assoc_comm():
    rng = np.random.default_rng(22)
    o = [rng.standard_normal((20, 4)) for _ in range(3)]
    l = [rng.uniform(-1e4, 1e4, 20) for _ in range(3)]
    ab, lab = oracle.combine(o[0], l[0], o[1], l[1])
    assert np.isfinite(ab).all() and np.isfinite(lab).all()
    ba, lba = oracle.combine(o[1], l[1], o[0], l[0])
    np.testing.assert_allclose(ab, ba, atol=1e-12)
    x1, lx1 = oracle.combine(ab, lab, o[2], l[2])
    bc, lbc = oracle.combine(o[1], l[1], o[2], l[2])
    x2, lx2 = oracle.combine(o[0], l[0], bc, lbc)
    np.testing.assert_allclose(x1, x2, atol=1e-12)
    np.testing.assert_allclose(lx1, lx2, rtol=1e-12)


# ----------------------------------------------------------------- tree (§3.3)
def test_tree_path_walk():
    # Fig. 2 shape: root 0 -> problems 1,2 ; deeper 3 under 1
    parent = np.array([-1, 0, 0, 1])
    assert oracle.tree_path(parent, 3) == [0, 1, 3]
    assert oracle.tree_path(parent, 2) == [0, 2]
    assert oracle.tree_path(parent, 0) == [0]


def test_one_level_tree_equals_flat():
    B = 5
    tp = synth.make_tree_problem([-1], [40], np.zeros(B, np.int32), 4, 2, 16, 6, lens=[6, 1, 0, 3, 6],
                                 dtype="bf16", dist="mixed", seed=30)
    pb = synth.Problem(B, 4, 2, 16, 40, 6, "bf16", tp.lens, tp.q, tp.node_k, tp.node_v, tp.sk, tp.sv)
    o1, l1 = oracle.tree_attention(tp)
    o2, l2 = oracle.flat_attention(pb)
    np.testing.assert_array_equal(o1, o2)
    np.testing.assert_array_equal(l1, l2)


def test_tree_equals_explicit_flattening_and_path_lengths():
    parent, node_len, leaf = [-1, 0, 0, 1], [16, 8, 8, 5], np.array([3, 3, 2, 2, 1], np.int32)
    tp = synth.make_tree_problem(parent, node_len, leaf, 4, 2, 16, 4, lens=[2, 4, 0, 1, 3], dtype="f32",
                                 dist="mixed", seed=31)
    o, l = oracle.tree_attention(tp)
    # Explicit concatenation by token ranges: node tokens are pooled in node order.
    ranges = {3: [(0, 16), (16, 24), (32, 37)], 2: [(0, 16), (24, 32)], 1: [(0, 16), (16, 24)]}
    for b in range(5):
        K = np.concatenate([tp.node_k[a:z] for a, z in ranges[int(leaf[b])]] + [tp.sk[b, :tp.lens[b]]])
        V = np.concatenate([tp.node_v[a:z] for a, z in ranges[int(leaf[b])]] + [tp.sv[b, :tp.lens[b]]])
        assert len(K) == sum(z - a for a, z in ranges[int(leaf[b])]) + tp.lens[b]  # path sum + suffix
        ob, lb = oracle.attention_segments(tp.q[b:b + 1], [[(K, V)]], 2)
        np.testing.assert_allclose(ob[0], o[b], atol=1e-14)
        np.testing.assert_allclose(lb[0], l[b], atol=1e-14)


# ---------------------------------------------------------------- paged suffix cache (reading R14)
def test_paged_rows_hand_example():
    """Hand-laid pool: page_size 2, sequence table [2, 0] -> tokens are (page 2, row 0),
    (page 2, row 1), (page 0, row 0) -- the expected rows are written out, not computed."""
    pool = np.arange(3 * 2 * 1 * 2, dtype=np.float32).reshape(3, 2, 1, 2)  # value = 4*page + 2*row + i
    got = oracle.paged_rows(pool, np.array([2, 0], np.int32), 2, 3)
    want = np.array([[[8, 9]], [[10, 11]], [[0, 1]]], np.float32)
    assert np.array_equal(got, want)
    assert oracle.paged_rows(pool, np.array([1], np.int32), 2, 0).shape == (0, 1, 2)


@pytest.mark.parametrize("page_size,map_tail", [(8, True), (16, False), (64, True), (256, False)])
def test_paged_suffix_equals_contiguous(page_size, map_tail):
    """Reading R14: paging only moves rows, so the paged oracle reproduces the contiguous
    suffix result bit for bit (same rows, same order, same fp64 arithmetic), with unmapped
    table entries past lens[b] and NaN-poisoned spare pages never read."""
    pb = synth.make_problem(5, 4, 2, 32, 0, 70, lens=[0, 1, 8, 69, 70], dtype="bf16", dist="mixed", seed=7)
    pc = synth.paginate(pb, page_size, seed=3, map_tail=map_tail)
    o_ref, l_ref = oracle.suffix_only(pb)
    o, l = oracle.suffix_only_paged(pb.q, pc.k_pool, pc.v_pool, pc.block_table, page_size, pb.lens, pb.Hkv,
                                    pb.scale)
    assert np.array_equal(o, o_ref) and np.array_equal(l, l_ref)
    assert np.isneginf(l[0]).all() and (o[0] == 0).all()  # empty suffix sentinel (R6)


def test_paged_flat_attention_equals_contiguous():
    pb = synth.make_problem(3, 8, 2, 16, 40, 33, lens=[33, 5, 17], dtype="f32", dist="mixed", seed=9)
    pc = synth.paginate(pb, 8, seed=1)
    o_ref, l_ref = oracle.flat_attention(pb)
    o, l = oracle.flat_attention_paged(pb, pc)
    assert np.array_equal(o, o_ref) and np.array_equal(l, l_ref)


def test_paginate_is_a_permutation_of_the_suffix_rows():
    """The synthetic paged layout holds every suffix row exactly once (layout check of synth)."""
    pb = synth.make_problem(4, 2, 2, 16, 0, 20, lens=[20, 3, 0, 11], dtype="bf16", seed=2)
    pc = synth.paginate(pb, 8, seed=5, spare_pages=2)
    ids = pc.block_table[pc.block_table < pc.n_pages]
    assert len(set(ids.tolist())) == ids.size == 4 * 3 and pc.n_pages == 14
    for b in range(pb.B):
        for t in range(pb.S_cap):
            assert np.array_equal(pc.k_pool[pc.block_table[b, t // 8], t % 8], pb.sk[b, t], equal_nan=False) \
                or np.isnan(synth.bf16_bits_to_f32(pb.sk[b, t])).all()


def test_paged_tree_equals_contiguous_tree():
    parent, node_len, leaf = synth.two_level_tree(20, 2, 9, 2)
    tp = synth.make_tree_problem(parent, node_len, leaf, 4, 2, 16, 24, lens=[24, 0, 7, 16], dtype="bf16",
                                 dist="mixed", seed=4)
    pc = synth.paginate(tp, 8, seed=6, map_tail=False)
    o_ref, l_ref = oracle.tree_attention(tp)
    o, l = oracle.tree_attention_paged(tp, pc)
    assert np.array_equal(o, o_ref) and np.array_equal(l, l_ref)
