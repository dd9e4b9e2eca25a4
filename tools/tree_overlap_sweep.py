"""C5 tree: node attention on k SMs || tensor-core suffix, step time vs k (diagnostics)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2402_05099_b200 as hydra
from tests.util import tree_to
ks = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "15,24,32,48,64").split(",")]
dev = torch.device("cuda:0")
parent, node_len, leaf = synth.two_level_tree(4096, 16, 1024, 64)
tp = synth.make_tree_problem(parent, node_len, leaf, 32, 32, 128, 512, dtype="bf16", dist="plain", seed=5)
t = tree_to(tp, "cuda:0")
tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq)
aux = torch.cuda.Stream(priority=-1)
def timeit(fn, iters=20):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr): fn()
    for _ in range(3): gr.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): gr.replay()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / iters, 4)
run = lambda a=None: hydra.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], t["lens"], aux_stream=a)
print(json.dumps(dict(what="sequential", ms=timeit(lambda: run()))))
print(json.dumps(dict(what="auto", ms=timeit(lambda: run(aux)), k=hydra.get_config("last_overlap_k"))))
for k in ks:
    hydra.set_config("overlap_prefix_ctas", k)
    ms = timeit(lambda: run(aux))
    # node attention alone on k SMs (empty suffix: lens = 0)
    z = torch.zeros_like(t["lens"])
    hydra.set_config("prefix_ctas", k)
    msp = timeit(lambda: hydra.tree_attention(t["q"], tree, t["node_k"], t["node_v"], t["sk"], t["sv"], z))
    hydra.set_config("prefix_ctas", 0)
    print(json.dumps(dict(k=k, overlap=ms, nodes_alone_on_k=msp)), flush=True)
hydra.set_config("overlap_prefix_ctas", 0)
