"""Prefix/suffix overlap experiment at a bench workload: stage count x suffix unroll."""
import os, sys, json, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_05099_b200 as hydra

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=16384); ap.add_argument("--S", type=int, default=256)
ap.add_argument("--B", type=int, default=1024); ap.add_argument("--H", type=int, default=40)
ap.add_argument("--Hkv", type=int, default=0)
ap.add_argument("--grid", default="2:4,2:8,3:4,3:8")
a = ap.parse_args()
Hkv = a.Hkv or a.H
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(a.B, a.H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(a.P, Hkv, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(a.P, Hkv, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(a.B, a.S, Hkv, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(a.B, a.S, Hkv, 128, device=dev, generator=g).bfloat16()
lens = torch.full((a.B,), a.S, dtype=torch.int32, device=dev)
ws = torch.empty(hydra.attn_workspace_bytes(q, a.P, a.S, Hkv) * 2, dtype=torch.uint8, device=dev)
out = torch.empty(a.B, a.H, 128, dtype=torch.bfloat16, device=dev)
aux = torch.cuda.Stream(priority=-1)

def graph_ms(fn, iters=30):
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
    return e0.elapsed_time(e1) / iters

for cfg in a.grid.split(","):
    st, un = map(int, cfg.split(":"))
    hydra.set_config("prefix_stages", st); hydra.set_config("suffix_unroll", un)
    r = dict(stages=st, unroll=un,
             prefix=graph_ms(lambda: hydra.prefix_attn(q, pk, pv, workspace=ws)),
             suffix=graph_ms(lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws)),
             seq=graph_ms(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws)),
             overlap=graph_ms(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws, aux_stream=aux)))
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
