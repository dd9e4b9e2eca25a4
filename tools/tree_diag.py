import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2402_05099_b200 as hydra
from tests.util import tree_to, errors
def run(root, nbr, blen, per, S, H, impl=0, splits=0, rows=48):
    hydra.set_config("prefix_impl", impl); hydra.set_config("prefix_splits", splits)
    parent, node_len, leaf = synth.two_level_tree(root, nbr, blen, per)
    tp = synth.make_tree_problem(parent, node_len, leaf, H, H, 128, S, dtype="bf16", dist="mixed", seed=5)
    t = tree_to(tp, "cuda:0")
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
    out, lse = hydra.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"], return_lse=True)
    torch.cuda.synchronize()
    B = tp.B
    rng = np.random.default_rng(0)
    rr = np.array(sorted({(int(rng.integers(B)), int(rng.integers(H))) for _ in range(rows)}))
    ref, lref = oracle.tree_attention(tp, rows=rr)
    mx, mean, _ = errors(out[rr[:, 0], rr[:, 1]], ref)
    le = float(np.abs(lse[rr[:, 0], rr[:, 1]].cpu().numpy() - lref).max())
    bad = sorted({int(b) for (b, h), e in zip(rr, np.abs(out[rr[:, 0], rr[:, 1]].float().cpu().numpy() - ref).max(1)) if e > 2e-2})
    print(f"root={root} nbr={nbr} blen={blen} per={per} S={S} H={H} impl={impl} splits={splits}: max={mx:.3e} lse={le:.3e} bad_seqs={bad[:10]}", flush=True)
    tree.destroy()
run(4096, 16, 1024, 64, 512, 32)
run(4096, 16, 1024, 64, 512, 32, impl=2)
run(4096, 16, 1024, 64, 512, 32, impl=1)
run(4096, 16, 1024, 64, 512, 32, impl=3, splits=1)
run(4096, 16, 1024, 64, 64, 32)
run(1024, 16, 256, 64, 64, 32)
run(4096, 4, 1024, 64, 64, 8)
run(4096, 16, 1024, 16, 64, 8)
run(1024, 2, 256, 300, 64, 4)
run(512, 16, 128, 64, 64, 4)
