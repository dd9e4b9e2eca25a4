import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2402_05099_b200 as hydra
from tests.util import tree_to
def run(parent, node_len, leaf, H=4, S=16, impl=3, tag=""):
    hydra.set_config("prefix_impl", impl)
    tp = synth.make_tree_problem(parent, node_len, leaf, H, H, 128, S, dtype="bf16", dist="mixed", seed=5)
    t = tree_to(tp, "cuda:0")
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
    out, lse = hydra.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"], return_lse=True)
    torch.cuda.synchronize()
    ref, lref = oracle.tree_attention(tp)
    err = np.abs(out.float().cpu().numpy() - ref).max(axis=(1, 2))
    bad = np.nonzero(err > 2e-2)[0]
    print(f"{tag}: B={tp.B} nbad={len(bad)} first={bad[:6].tolist()} last={bad[-3:].tolist()}", flush=True)
    tree.destroy()
B = 256
run([-1], [512], np.zeros(B, np.int32), tag="root only B=256")
run([-1], [512], np.zeros(1024, np.int32), tag="root only B=1024")
run([-1, 0, 0, 0, 0], [0, 128, 128, 128, 128], np.repeat(np.arange(1, 5), 64).astype(np.int32), tag="empty root, 4 branches x64")
run([-1, 0, 0], [0, 128, 128], np.repeat(np.arange(1, 3), 300).astype(np.int32), tag="empty root, 2 branches x300")
run([-1, 0, 0, 0, 0], [256, 128, 128, 128, 128], np.repeat(np.arange(1, 5), 64).astype(np.int32), tag="root 256 + 4 branches x64")
run([-1, 0, 0, 0, 0], [256, 128, 128, 128, 128], np.repeat(np.arange(1, 5), 64).astype(np.int32), impl=2, tag="TC1 root 256 + 4 branches x64")
