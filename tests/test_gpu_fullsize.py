"""Full-size parity at BASELINE.json's configurations, in the launch configuration bench.py
times, on sampled output rows the oracle computes one by one.

Each test draws the whole workload with the seeded generator ('mixed' needles, so |O| is
O(1) and prefix/suffix LSEs differ), runs the CUDA path exactly as bench.py launches it,
and compares ~64 sampled (sequence, head) rows -- including the first and last sequence
and first/last head -- against the fp64 oracle (same gates as tests/test_gpu_parity.py)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.util import assert_parity, problem_to, tree_to

hydra = pytest.importorskip("paper_2402_05099_b200")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda:0"


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


@pytest.mark.parametrize("overlap", [False, True])
def test_c3_16k_full_size(overlap):
    """CodeLlama-13b shape, B=1024, prefix 16384, suffix 256 (bench.py default workload)."""
    pb = synth.make_problem(1024, 40, 40, 128, 16384, 256, dtype="bf16", dist="mixed", seed=0)
    t = problem_to(pb, DEV)
    aux = torch.cuda.Stream(priority=-1) if overlap else None
    out, lse = hydra.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True,
                                        aux_stream=aux)
    torch.cuda.synchronize()
    rows = sample_rows(1024, 40)
    ref, lref = oracle.flat_attention(pb, rows=rows)
    check_rows(out, lse, ref, lref, rows, f"C3@16K overlap={overlap}")


def test_c2_full_size_ragged():
    """CodeLlama-7b shape, B=256, prefix 2048, suffix 128 with ragged lens ~ U[64, 128]."""
    lens = np.random.default_rng(2).integers(64, 129, 256)
    pb = synth.make_problem(256, 32, 32, 128, 2048, 128, lens=lens, dtype="bf16", dist="boundary", seed=2)
    t = problem_to(pb, DEV)
    out, lse = hydra.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True)
    torch.cuda.synchronize()
    rows = sample_rows(256, 32)
    ref, lref = oracle.flat_attention(pb, rows=rows)
    check_rows(out, lse, ref, lref, rows, "C2")


@pytest.mark.parametrize("overlap", [False, True])
def test_c6_longdoc_full_size(overlap):
    """Long-document shape: 19,947-token prefix (not a multiple of the 128-token tile),
    32 q / 4 kv heads (g = 8), B = 256, ragged suffixes up to 128."""
    lens = np.random.default_rng(6).integers(1, 129, 256)
    pb = synth.make_problem(256, 32, 4, 128, 19947, 128, lens=lens, dtype="bf16", dist="boundary", seed=6)
    t = problem_to(pb, DEV)
    aux = torch.cuda.Stream(priority=-1) if overlap else None
    out, lse = hydra.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True,
                                        aux_stream=aux)
    torch.cuda.synchronize()
    rows = sample_rows(256, 32)
    ref, lref = oracle.flat_attention(pb, rows=rows)
    check_rows(out, lse, ref, lref, rows, f"long-doc overlap={overlap}")


def test_c4_full_size_single_rank_seqsplit():
    """Llama-3-8B GQA shape, B=512, prefix 32768, suffix 128, through dist.seqsplit_attention (1 rank)."""
    import socket

    import torch.distributed as tdist
    from paper_2402_05099_b200 import dist as hdist

    pb = synth.make_problem(512, 32, 8, 128, 32768, 128, dtype="bf16", dist="mixed", seed=4)
    t = problem_to(pb, DEV)
    if not tdist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        out, lse = hdist.seqsplit_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True)
        torch.cuda.synchronize()
    finally:
        tdist.destroy_process_group()
    rows = sample_rows(512, 32)
    ref, lref = oracle.flat_attention(pb, rows=rows)
    check_rows(out, lse, ref, lref, rows, "C4 seq-split")


@pytest.mark.parametrize("overlap", [False, True])
def test_c5_tree_full_size(overlap):
    """Tree: 4096-token root -> 16 x 1024-token branches -> 64 sequences each, 512-token suffixes
    (overlap: node attention on k SMs || tensor-core suffix, the bench's schedule)."""
    parent, node_len, leaf = synth.two_level_tree(4096, 16, 1024, 64)
    tp = synth.make_tree_problem(parent, node_len, leaf, 32, 32, 128, 512, dtype="bf16", dist="mixed", seed=5)
    t = tree_to(tp, DEV)
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
    out, lse = hydra.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"],
                                    return_lse=True, aux_stream=torch.cuda.Stream() if overlap else None)
    torch.cuda.synchronize()
    assert (hydra.get_config("last_overlap_k") > 0) == overlap
    rows = sample_rows(1024, 32)
    ref, lref = oracle.tree_attention(tp, rows=rows)
    check_rows(out, lse, ref, lref, rows, "C5 tree")
    tree.destroy()
