"""GPU stress: repeated runs of the concurrent (SM-partitioned) paths with NaN-poisoned padding.

Races between the warps of the persistent kernels show up intermittently, so each case runs
several times and every run must pass the parity gate (an earlier V-ring race produced NaN
in about 1 run in 15).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import nanfill as H
from tests.util import assert_parity, problem_to, tree_to

hydra = pytest.importorskip("paper_2402_05099_b200")

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _reset_config():
    keys = ("prefix_impl", "suffix_impl", "overlap_prefix_ctas", "prefix_ctas", "suffix_ctas")
    for k in keys:
        hydra.set_config(k, 0)
    yield
    for k in keys:
        hydra.set_config(k, 0)


@pytest.mark.parametrize("per,g,k", [(300, 1, 1), (300, 1, 37), (100, 4, 1)])
def test_tree_partitioned_repeat(per, g, k):
    hydra.set_config("prefix_impl", 3)
    hydra.set_config("suffix_impl", 2)
    hydra.set_config("overlap_prefix_ctas", k)
    parent, node_len, leaf = synth.two_level_tree(300, 2, 200, per)
    tp = synth.make_tree_problem(parent, node_len, leaf, 4 * g, 4, 128, 300, dtype="bf16", dist="boundary",
                                 seed=23, lens=np.arange(2 * per) % 301)
    t = tree_to(tp, DEV)
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
    ref, lref = oracle.tree_attention(tp)
    aux = torch.cuda.Stream()
    for _ in range(6):
        out, lse = H.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"],
                                        return_lse=True, aux_stream=aux)
        torch.cuda.synchronize()
        assert_parity(out, ref, lse, lref, what=f"tree partitioned k={k} (repeat)")
    tree.destroy()


def test_flat_partitioned_repeat():
    hydra.set_config("prefix_impl", 3)
    hydra.set_config("suffix_impl", 2)
    hydra.set_config("overlap_prefix_ctas", 72)
    lens = np.arange(512) % 257
    pb = synth.make_problem(512, 8, 8, 128, 1500, 256, lens=lens, dtype="bf16", dist="boundary", seed=29)
    t = problem_to(pb, DEV)
    ref, lref = oracle.flat_attention(pb)
    aux = torch.cuda.Stream()
    for _ in range(6):
        out, lse = H.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True,
                                            aux_stream=aux)
        torch.cuda.synchronize()
        assert_parity(out, ref, lse, lref, what="flat partitioned (repeat)")
