"""Full-size parity at BASELINE.json's configurations, in the launch configurations bench.py
times, on EVERY output row (sampled rows left stream-K piece boundaries and
second-tile rows unchecked).

Each workload is drawn once with the seeded generator ('mixed' needles, so |O| is O(1) and
prefix/suffix LSEs differ; 'boundary' needles where stated), the fp64 oracle computes all
B*Hq rows once (about 20 s for C3@16K on a 16-core host), and every schedule of the CUDA
path that bench.py can pick is compared against it element by element, with every output
and workspace buffer pre-filled with NaN (tests/nanfill.py)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import nanfill as H
from tests.util import assert_parity, problem_to, tree_to

hydra = pytest.importorskip("paper_2402_05099_b200")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda:0"

_CACHE = {}


def workload(name):
    """(problem, O_ref, LSE_ref) of a named full-size workload; one kept at a time (host memory)."""
    if name in _CACHE:
        return _CACHE[name]
    _CACHE.clear()
    if name == "c3_16k":
        pb = synth.make_problem(1024, 40, 40, 128, 16384, 256, dtype="bf16", dist="mixed", seed=0)
    elif name == "c2":
        lens = np.random.default_rng(2).integers(64, 129, 256)
        pb = synth.make_problem(256, 32, 32, 128, 2048, 128, lens=lens, dtype="bf16", dist="boundary", seed=2)
    elif name == "c6":
        lens = np.random.default_rng(6).integers(1, 129, 256)
        pb = synth.make_problem(256, 32, 4, 128, 19947, 128, lens=lens, dtype="bf16", dist="boundary", seed=6)
    elif name == "c4":
        pb = synth.make_problem(512, 32, 8, 128, 32768, 128, dtype="bf16", dist="mixed", seed=4)
    elif name == "c5":
        parent, node_len, leaf = synth.two_level_tree(4096, 16, 1024, 64)
        tp = synth.make_tree_problem(parent, node_len, leaf, 32, 32, 128, 512, dtype="bf16", dist="mixed", seed=5)
        ref, lref = oracle.tree_attention(tp)
        _CACHE[name] = (tp, ref, lref)
        return _CACHE[name]
    else:
        raise KeyError(name)
    ref, lref = oracle.flat_attention(pb)
    _CACHE[name] = (pb, ref, lref)
    return _CACHE[name]


@pytest.fixture(autouse=True)
def _reset():
    keys = ("prefix_impl", "suffix_impl", "overlap_prefix_ctas", "prefix_ctas", "suffix_ctas")
    for k in keys:
        hydra.set_config(k, 0)
    yield
    for k in keys:
        hydra.set_config(k, 0)
    torch.cuda.empty_cache()


def sample_rows(B, Hq, n=64, seed=0):
    rng = np.random.default_rng(seed)
    rows = {(0, 0), (B - 1, Hq - 1), (0, Hq - 1), (B - 1, 0)}
    while len(rows) < n:
        rows.add((int(rng.integers(B)), int(rng.integers(Hq))))
    return np.array(sorted(rows))


def check_rows(out, lse, ref, lref, rows, what):
    o = out[rows[:, 0], rows[:, 1]]
    l = lse[rows[:, 0], rows[:, 1]]
    assert_parity(o, ref, l, lref, what=what)


def run_flat(pb, aux, **kw):
    t = problem_to(pb, DEV)
    out, lse = H.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True,
                                    aux_stream=torch.cuda.Stream(priority=-1) if aux else None, **kw)
    torch.cuda.synchronize()
    k = hydra.get_config("last_overlap_k")
    del t
    return out, lse, k


@pytest.mark.parametrize("overlap", [False, True])
def test_c3_16k_full_size(overlap):
    """CodeLlama-13b shape, B=1024, prefix 16384, suffix 256 (bench.py default workload): all
    40,960 rows, sequential and SM-partitioned schedules."""
    pb, ref, lref = workload("c3_16k")
    out, lse, k = run_flat(pb, overlap)
    assert (k > 0) == overlap
    assert_parity(out, ref, lse, lref, what=f"C3@16K overlap={overlap}")


def test_c3_16k_paged_full_size():
    """bench.py's C3@16K workload with the suffix in 16-token pages (a shuffled pool built on the
    GPU from the contiguous cache), overlapped schedule, all rows vs the oracle over the
    contiguous suffix (paging is a row move, pinned by tests/test_oracle.py)."""
    pb, ref, lref = workload("c3_16k")
    B, Hq, Hkv, d, S, ps = 1024, 40, 40, 128, 256, 16
    t = problem_to(pb, DEV)
    npg = S // ps
    perm = torch.from_numpy(np.random.default_rng(1).permutation(B * npg).astype(np.int64)).to(DEV)
    kp = torch.empty(B * npg, ps, Hkv, d, dtype=torch.bfloat16, device=DEV)
    vp = torch.empty_like(kp)
    kp[perm] = t["sk"].view(B * npg, ps, Hkv, d)
    vp[perm] = t["sv"].view(B * npg, ps, Hkv, d)
    tab = perm.view(B, npg).to(torch.int32)
    del t["sk"], t["sv"], perm
    out, lse = H.hydragen_attention_paged(t["q"], t["pk"], t["pv"], kp, vp, tab, t["lens"], return_lse=True,
                                          aux_stream=torch.cuda.Stream(priority=-1))
    torch.cuda.synchronize()
    assert_parity(out, ref, lse, lref, what="C3@16K paged(16)")


def test_c3_16k_prefix_partials_full_size():
    """The prefix kernel's own output at C3@16K (stream-K pieces merged), every row, against
    the prefix-only oracle: catches errors the suffix-dominated composite could mask."""
    pb, _, _ = workload("c3_16k")
    t = problem_to(pb, DEV)
    o, l = H.prefix_attn(t["q"], t["pk"], t["pv"])
    torch.cuda.synchronize()
    rows = np.stack(np.meshgrid(np.arange(0, 1024, 3), np.arange(40), indexing="ij"), -1).reshape(-1, 2)
    ref, lref = oracle.prefix_only(pb, rows=rows)
    check_rows(o, l, ref, lref, rows, "C3@16K prefix partials (every 3rd sequence, all heads)")


def test_c2_full_size_ragged():
    """CodeLlama-7b shape, B=256, prefix 2048, suffix 128 with ragged lens ~ U[64, 128]."""
    pb, ref, lref = workload("c2")
    for aux in (False, True):
        out, lse, _ = run_flat(pb, aux)
        assert_parity(out, ref, lse, lref, what=f"C2 aux={aux}")


@pytest.mark.parametrize("overlap", [False, True])
def test_c6_longdoc_full_size(overlap):
    """Long-document shape: 19,947-token prefix (not a multiple of the 128-token tile),
    32 q / 4 kv heads (g = 8), B = 256, ragged suffixes up to 128."""
    pb, ref, lref = workload("c6")
    out, lse, _ = run_flat(pb, overlap)
    assert_parity(out, ref, lse, lref, what=f"long-doc overlap={overlap}")


def test_c4_full_size_single_rank():
    """Llama-3-8B GQA shape, B=512, prefix 32768, suffix 128 on one GPU (both schedules)."""
    pb, ref, lref = workload("c4")
    for aux in (False, True):
        out, lse, _ = run_flat(pb, aux)
        assert_parity(out, ref, lse, lref, what=f"C4 1-GPU aux={aux}")


@pytest.mark.parametrize("overlap", [False, True])
def test_c5_tree_full_size(overlap):
    """Tree: 4096-token root -> 16 x 1024-token branches -> 64 sequences each, 512-token suffixes
    (overlap: node attention on k SMs || tensor-core suffix, the bench's schedule)."""
    tp, ref, lref = workload("c5")
    t = tree_to(tp, DEV)
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq, heads=(32, 32))
    out, lse = H.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"],
                                return_lse=True, aux_stream=torch.cuda.Stream() if overlap else None)
    torch.cuda.synchronize()
    assert (hydra.get_config("last_overlap_k") > 0) == overlap
    assert_parity(out, ref, lse, lref, what=f"C5 tree overlap={overlap}")
    tree.destroy()
