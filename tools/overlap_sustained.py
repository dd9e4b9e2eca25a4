"""Sustained (power-capped) overlap step time vs prefix CTA count k at C3 (diagnostics).
Each k: ~1.5 s of back-to-back replays, median of the second half.
    python tools/overlap_sustained.py [k,k,...]
"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2402_05099_b200 as hydra
ks = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "56,60,64,68,72,76,80").split(",")]
B, H, P, S = int(os.environ.get("B", 1024)), int(os.environ.get("H", 40)), int(os.environ.get("P", 16384)), int(os.environ.get("S", 256))
HKV = int(os.environ.get("HKV", H))
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(P, HKV, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(P, HKV, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(B, S, HKV, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(B, S, HKV, 128, device=dev, generator=g).bfloat16()
lens = torch.full((B,), S, dtype=torch.int32, device=dev)
ws = torch.empty(hydra.attn_workspace_bytes(q, P, S, HKV) * 4, dtype=torch.uint8, device=dev)
out = torch.empty(B, H, 128, dtype=torch.bfloat16, device=dev)
aux = torch.cuda.Stream(priority=-1)
def graph(fn):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr): fn()
    return gr
graphs = {}
hydra.set_config("pair_cluster", int(os.environ.get("CLUSTER", 0)))
if os.environ.get("POLY") is not None:
    hydra.set_config("prefix_poly", int(os.environ["POLY"]))
for k in ks:
    hydra.set_config("overlap_prefix_ctas", k)
    graphs[k] = graph(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws, aux_stream=aux))
hydra.set_config("overlap_prefix_ctas", 0)
graphs["seq"] = graph(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws))
# warm to the power cap first
t_end = time.time() + 1.5
while time.time() < t_end:
    for _ in range(50): graphs["seq"].replay()
    torch.cuda.synchronize()
for k, gr in graphs.items():
    times = []
    t_end = time.time() + 1.5
    while time.time() < t_end:
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): gr.replay()
        e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 20)
    n = len(times)
    print(json.dumps(dict(k=k, ms_first=round(float(np.median(times[:2])), 4), ms_sustained=round(float(np.median(times[n // 2:])), 4))), flush=True)
