import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2402_05099_b200 as hydra
from tests.util import tree_to
B, H, P, S = 256, 1, 512, 16
tp = synth.make_tree_problem([-1], [P], np.zeros(B, np.int32), H, H, 128, S, lens=np.zeros(B, np.int32), dtype="bf16", dist="mixed", seed=5)
t = tree_to(tp, "cuda:0")
ref, lref = oracle.tree_attention(tp)
hydra.set_config("prefix_impl", 3)
tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
out, lse = hydra.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"], return_lse=True)
torch.cuda.synchronize()
o = out.float().cpu().numpy()[:, 0]; l = lse.cpu().numpy()[:, 0]
R = ref[:, 0]; L = lref[:, 0]
for i in (0, 1, 127, 128, 129, 200, 255):
    d = np.abs(R - o[i]).max(axis=1)
    j = int(d.argmin())
    print(f"row {i}: err vs own {np.abs(R[i]-o[i]).max():.3e}; best match ref row {j} (err {d[j]:.3e}); lse {l[i]:.4f} own {L[i]:.4f} match-lse {L[j]:.4f}", flush=True)
