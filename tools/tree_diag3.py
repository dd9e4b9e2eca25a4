import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2402_05099_b200 as hydra
from tests.util import tree_to, problem_to
B, H, P, S = 256, 1, 512, 16
tp = synth.make_tree_problem([-1], [P], np.zeros(B, np.int32), H, H, 128, S, dtype="bf16", dist="mixed", seed=5)
t = tree_to(tp, "cuda:0")
ref, lref = oracle.tree_attention(tp)
hydra.set_config("prefix_impl", 3)
for splits in (1, 2, 4):
    for ctas in (1, 2, 148):
        hydra.set_config("prefix_splits", splits); hydra.set_config("prefix_ctas", ctas)
        tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
        out, lse = hydra.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"], return_lse=True)
        torch.cuda.synchronize()
        err = np.abs(out.float().cpu().numpy() - ref).max(axis=(1, 2))
        bad = np.nonzero(err > 2e-2)[0]
        lerr = np.abs(lse.cpu().numpy() - lref).max(axis=1)
        print(f"splits={splits} ctas={ctas}: nbad={len(bad)} first={bad[:4].tolist()} last={bad[-2:].tolist()} lse_err_bad={lerr[bad[:3]].tolist() if len(bad) else []}", flush=True)
        tree.destroy()
# same data via the flat path
pb = synth.Problem(B, H, H, 128, P, S, "bf16", tp.lens, tp.q, tp.node_k, tp.node_v, tp.sk, tp.sv)
tt = problem_to(pb, "cuda:0")
hydra.set_config("prefix_splits", 0); hydra.set_config("prefix_ctas", 0)
out = hydra.hydragen_attention(tt["q"], tt["pk"], tt["pv"], tt["sk"], tt["sv"], tt["lens"])
torch.cuda.synchronize()
err = np.abs(out.float().cpu().numpy() - ref).max(axis=(1, 2))
print("flat TC2: nbad", int((err > 2e-2).sum()))
