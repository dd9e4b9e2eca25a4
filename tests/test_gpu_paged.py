"""Paged suffix cache (SURVEY §8(f) NEXT-4 "growable or paged cache"; reading R14):
hydra_suffix_attn_paged / hydra_attn_paged / hydra_append_kv_paged against the fp64 oracle
over the same pages (oracle.suffix_only_paged / flat_attention_paged), on both suffix kernels
(SIMT split-K and the TMA-fed tensor-core kernel), page sizes 8..256, shuffled page order,
NaN-poisoned spare pages and out-of-range table entries past lens[b]."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import nanfill as H
from tests.util import assert_parity, problem_to, to_torch

hydra = pytest.importorskip("paper_2402_05099_b200")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _reset():
    keys = ("suffix_impl", "suffix_ctas", "overlap_prefix_ctas")
    for k in keys:
        hydra.set_config(k, 0)
    yield
    for k in keys:
        hydra.set_config(k, 0)


def paged_to(pc, dtype):
    return (to_torch(pc.k_pool, dtype, DEV), to_torch(pc.v_pool, dtype, DEV),
            torch.from_numpy(pc.block_table).to(DEV))


CASES = [  # (B, Hq, Hkv, d, S_cap, lens, dtype)
    (6, 8, 8, 128, 300, [300, 0, 1, 127, 128, 129], "bf16"),   # MHA, ragged around a 128-token tile
    (5, 32, 4, 128, 520, [520, 17, 256, 300, 8], "bf16"),     # g = 8
    (4, 4, 2, 64, 90, [90, 0, 33, 64], "bf16"),               # d = 64 (SIMT only)
    (3, 4, 2, 128, 70, [70, 9, 40], "f32"),                   # fp32 reference mode
]


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("page_size", [8, 16, 64, 128, 256])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_suffix_paged_parity(impl, page_size, case):
    B, Hq, Hkv, d, S, lens, dt = CASES[case]
    pb = synth.make_problem(B, Hq, Hkv, d, 0, S, lens=lens, dtype=dt, dist="mixed", seed=11 + case)
    pc = synth.paginate(pb, page_size, seed=page_size, map_tail=False)
    t = problem_to(pb, DEV)
    kp, vp, tab = paged_to(pc, dt)
    hydra.set_config("suffix_impl", impl)  # 2 = tensor-core kernel where supported (bf16, d = 128)
    o, l = H.suffix_attn_paged(t["q"], kp, vp, tab, t["lens"], S_cap=S)
    torch.cuda.synchronize()
    ref, lref = oracle.suffix_only_paged(pb.q, pc.k_pool, pc.v_pool, pc.block_table, page_size, pb.lens, Hkv,
                                         pb.scale)
    assert_parity(o, ref, l, lref, dtype=dt, what=f"paged suffix impl={impl} ps={page_size} case={case}")
    # paging moves rows only: the contiguous call over the same data gives the same bits
    o2, l2 = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(l, l2)


@pytest.mark.parametrize("aux", [False, True])
@pytest.mark.parametrize("page_size", [16, 128])
def test_attn_paged_parity(aux, page_size):
    """Whole decode step (prefix || paged suffix -> combine), with the SM-partitioned overlap
    (tensor-core suffix on a share of the SMs) when aux: B*Hkv = 1024 items."""
    B, Hq, Hkv, d, P, S = 128, 32, 8, 128, 4096, 300
    rng = np.random.default_rng(5)
    lens = rng.integers(0, S + 1, B).astype(np.int32)
    lens[:3] = [0, S, 1]
    pb = synth.make_problem(B, Hq, Hkv, d, P, S, lens=lens, dtype="bf16", dist="mixed", seed=21)
    pc = synth.paginate(pb, page_size, seed=2)
    t = problem_to(pb, DEV)
    kp, vp, tab = paged_to(pc, "bf16")
    side = torch.cuda.Stream() if aux else None
    if aux:  # force the SM split (the planner runs this small prefix sequentially)
        hydra.set_config("overlap_prefix_ctas", 48)
    out, lse = H.hydragen_attention_paged(t["q"], t["pk"], t["pv"], kp, vp, tab, t["lens"], S_cap=S,
                                              return_lse=True, aux_stream=side)
    torch.cuda.synchronize()
    if aux:
        assert hydra.get_config("last_overlap_k") > 0
    ref, lref = oracle.flat_attention_paged(pb, pc)
    assert_parity(out, ref, lse, lref, what=f"paged attn aux={aux} ps={page_size}")
    out2, lse2 = H.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True,
                                          aux_stream=side)
    torch.cuda.synchronize()
    assert torch.equal(out, out2) and torch.equal(lse, lse2)


def test_append_kv_paged_exact():
    """Row lens[b] % page_size of page table[b][lens[b] // page_size] receives the new token,
    bit-exactly; every other pool row is unchanged; full sequences are left alone."""
    B, Hkv, d, S, ps = 4, 2, 128, 32, 8
    lens0 = [0, 7, 8, 32]
    pb = synth.make_problem(B, 4, Hkv, d, 0, S, lens=lens0, dtype="bf16", seed=4)
    pc = synth.paginate(pb, ps, seed=9)
    kp, vp, tab = paged_to(pc, "bf16")
    lens = torch.tensor(lens0, dtype=torch.int32, device=DEV)
    g = torch.Generator(device=DEV).manual_seed(0)
    k_new = torch.randn(B, Hkv, d, device=DEV, generator=g).bfloat16()
    v_new = torch.randn(B, Hkv, d, device=DEV, generator=g).bfloat16()
    k0, v0 = kp.clone(), vp.clone()
    hydra.append_kv_paged(k_new, v_new, kp, vp, tab, lens, S_cap=S)
    torch.cuda.synchronize()
    want_k, want_v = k0.clone(), v0.clone()
    for b, L in enumerate(lens0):
        if L < S:
            page = int(pc.block_table[b, L // ps])
            want_k[page, L % ps] = k_new[b]
            want_v[page, L % ps] = v_new[b]
    bits = lambda x: x.view(torch.int16)  # NaN-safe bitwise comparison
    assert torch.equal(bits(kp), bits(want_k)) and torch.equal(bits(vp), bits(want_v))
    assert lens.cpu().tolist() == [1, 8, 9, 32]


def test_paged_decode_loop_in_one_graph():
    """append (paged) + attention (paged) captured in one CUDA graph and replayed; each step
    matches the oracle over the pool as it stands after that step's append."""
    B, Hq, Hkv, d, P, S, ps = 6, 8, 2, 128, 200, 48, 16
    lens0 = np.array([0, 15, 16, 31, 47, 5], np.int32)
    pb = synth.make_problem(B, Hq, Hkv, d, P, S, lens=lens0, dtype="bf16", dist="mixed", seed=8)
    pc = synth.paginate(pb, ps, seed=4)
    t = problem_to(pb, DEV)
    kp, vp, tab = paged_to(pc, "bf16")
    steps = 3
    gk = torch.Generator(device=DEV).manual_seed(2)
    new_k = [torch.randn(B, Hkv, d, device=DEV, generator=gk).bfloat16() for _ in range(steps)]
    new_v = [torch.randn(B, Hkv, d, device=DEV, generator=gk).bfloat16() for _ in range(steps)]
    k_in, v_in = torch.empty_like(new_k[0]), torch.empty_like(new_v[0])
    out = torch.empty(B, Hq, d, dtype=torch.bfloat16, device=DEV)
    lse = torch.empty(B, Hq, dtype=torch.float32, device=DEV)
    ws = torch.empty(hydra.attn_workspace_bytes(t["q"], P, S, Hkv), dtype=torch.uint8, device=DEV)

    def step():
        hydra.append_kv_paged(k_in, v_in, kp, vp, tab, t["lens"], S_cap=S)
        H.hydragen_attention_paged(t["q"], t["pk"], t["pv"], kp, vp, tab, t["lens"], S_cap=S, out=out,
                                       lse_out=lse, workspace=ws)

    state = [x.clone() for x in (kp, vp, t["lens"])]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for x, x0 in zip((kp, vp, t["lens"]), state):
        x.copy_(x0)
    torch.cuda.synchronize()
    for i in range(steps):
        k_in.copy_(new_k[i])
        v_in.copy_(new_v[i])
        out.fill_(float("nan")); lse.fill_(float("nan")); ws.fill_(0xFF)  # unwritten rows fail
        graph.replay()
        torch.cuda.synchronize()
        lens = t["lens"].cpu().numpy().astype(np.int32)
        assert (lens == np.minimum(lens0 + i + 1, S)).all()
        cur_pb = synth.Problem(B, Hq, Hkv, d, P, S, "bf16", lens, pb.q, pb.pk, pb.pv, pb.sk, pb.sv, scale=pb.scale)
        cur_pc = synth.PagedCache(ps, kp.view(torch.int16).cpu().numpy().view(np.uint16),
                                  vp.view(torch.int16).cpu().numpy().view(np.uint16), pc.block_table)
        ref, lref = oracle.flat_attention_paged(cur_pb, cur_pc)
        assert_parity(out, ref, lse, lref, what=f"paged decode step {i}")


@pytest.mark.parametrize("aux", [False, True])
def test_tree_paged_parity(aux):
    """Tree attention (§3.3) with the suffixes in 16-token pages; with aux the node attention and
    the tensor-core suffix run on disjoint SM sets."""
    from tests.util import tree_to

    parent, node_len, leaf = synth.two_level_tree(300, 2, 200, 40)
    tp = synth.make_tree_problem(parent, node_len, leaf, 16, 4, 128, 200, dtype="bf16", dist="mixed", seed=31,
                                 lens=np.arange(80) * 7 % 201)
    pc = synth.paginate(tp, 16, seed=8, map_tail=False)
    t = tree_to(tp, DEV)
    kp, vp, tab = paged_to(pc, "bf16")
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
    if aux:
        hydra.set_config("suffix_impl", 2)
        hydra.set_config("overlap_prefix_ctas", 32)
    out, lse = H.tree_attention_paged(t["q"], tree, t["node_k"], t["node_v"], kp, vp, tab, t["lens"],
                                          S_cap=tp.S_cap, return_lse=True,
                                          aux_stream=torch.cuda.Stream() if aux else None)
    torch.cuda.synchronize()
    ref, lref = oracle.tree_attention_paged(tp, pc)
    assert_parity(out, ref, lse, lref, what=f"tree paged aux={aux}")
    out2, lse2 = H.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"],
                                      return_lse=True, aux_stream=torch.cuda.Stream() if aux else None)
    torch.cuda.synchronize()
    assert torch.equal(out, out2) and torch.equal(lse, lse2)
    tree.destroy()


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("edge", ["one_seq", "all_empty", "page_gt_cap", "ragged_cap", "wide_table", "shared_pages"])
def test_suffix_paged_edges(impl, edge):
    """Degenerate paged layouts: a single sequence, every suffix empty, one page larger than the
    whole capacity, S_cap not a multiple of the page size, a block table wider than needed, and
    two sequences mapping the same physical pages (prefix-sharing caches do this)."""
    B, Hq, Hkv, d, S, ps = 4, 8, 2, 128, 150, 16
    lens = [150, 3, 77, 128]
    if edge == "one_seq":
        B, lens = 1, [150]
    elif edge == "all_empty":
        lens = [0, 0, 0, 0]
    elif edge == "page_gt_cap":
        ps = 256
    elif edge == "ragged_cap":
        S, lens = 150, [150, 149, 1, 145]
    pb = synth.make_problem(B, Hq, Hkv, d, 0, S, lens=lens, dtype="bf16", dist="mixed", seed=5)
    pc = synth.paginate(pb, ps, seed=3)
    table = pc.block_table
    if edge == "wide_table":
        table = np.concatenate([table, np.full((B, 5), 2**30, np.int32)], axis=1)
    if edge == "shared_pages":  # sequence 1 reads sequence 0's pages (and therefore its rows)
        table = table.copy()
        table[1] = table[0]
    t = problem_to(pb, DEV)
    kp, vp, _ = paged_to(pc, "bf16")
    tab = torch.from_numpy(np.ascontiguousarray(table)).to(DEV)
    hydra.set_config("suffix_impl", impl)
    o, l = H.suffix_attn_paged(t["q"], kp, vp, tab, t["lens"], S_cap=S)
    torch.cuda.synchronize()
    ref, lref = oracle.suffix_only_paged(pb.q, pc.k_pool, pc.v_pool, table, ps, pb.lens, Hkv, pb.scale)
    assert_parity(o, ref, l, lref, what=f"paged edge {edge} impl={impl}")
