"""Stress: repeated tree (SM-partitioned) and ragged tensor-core suffix runs with NaN-poisoned
padding, counting parity failures (caught an intermittent V-ring race; diagnostics)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth
import paper_2402_05099_b200 as hydra
from tests.util import tree_to, problem_to, errors
DEV = "cuda:0"
fails = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    for (per, g, k, impl) in [(300, 1, 1, 2), (300, 1, 37, 2), (100, 4, 1, 2)]:
        hydra.set_config("prefix_impl", 3); hydra.set_config("suffix_impl", impl); hydra.set_config("overlap_prefix_ctas", k)
        parent, node_len, leaf = synth.two_level_tree(300, 2, 200, per)
        tp = synth.make_tree_problem(parent, node_len, leaf, 4 * g, 4, 128, 300, dtype="bf16", dist="boundary",
                                     seed=23, lens=np.arange(2 * per) % 301)
        t = tree_to(tp, DEV)
        tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
        out, lse = hydra.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"],
                                        return_lse=True, aux_stream=torch.cuda.Stream())
        torch.cuda.synchronize()
        ref, lref = oracle.tree_attention(tp)
        o = out.float().cpu().numpy(); l = lse.cpu().numpy()
        e = np.abs(o - ref); le = np.abs(l - lref)
        bad = (e.max() > 2e-2) or (np.nanmax(le) > 1e-3) or not np.isfinite(o).all()
        if bad:
            fails += 1
            idx = np.argwhere(np.abs(o - ref).max(axis=2) > 2e-2)
            print(f"it={it} per={per} g={g} k={k}: max|dO|={e.max():.3e} max|dL|={np.nanmax(le):.3e} nbad_rows={len(idx)} first={idx[:5].tolist()} finite={np.isfinite(o).all()}", flush=True)
        tree.destroy()
# also the flat path with cb=2 suffix TC only, many times
hydra.set_config("overlap_prefix_ctas", 0); hydra.set_config("prefix_impl", 0); hydra.set_config("suffix_impl", 2)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    lens = np.arange(600) % 301
    pb = synth.make_problem(600, 4, 4, 128, 0, 300, lens=lens, dtype="bf16", dist="boundary", seed=18)
    tt = problem_to(pb, DEV)
    o, l = hydra.suffix_attn(tt["q"], tt["sk"], tt["sv"], tt["lens"])
    torch.cuda.synchronize()
    ref, lref = oracle.suffix_only(pb)
    e = np.abs(o.cpu().numpy() - ref)
    if e.max() > 2e-2 or not np.isfinite(o.cpu().numpy()).all():
        print(f"suffix it={it}: max|dO|={e.max():.3e}", flush=True)
print("fails", fails)
