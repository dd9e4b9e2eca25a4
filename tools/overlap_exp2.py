"""SM-partitioned overlap sweep: persistent prefix (k CTAs) || tensor-core suffix (148-k CTAs)."""
import os, sys, json, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_05099_b200 as hydra
ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=16384); ap.add_argument("--S", type=int, default=256)
ap.add_argument("--B", type=int, default=1024); ap.add_argument("--H", type=int, default=40)
ap.add_argument("--Hkv", type=int, default=0); ap.add_argument("--ks", default="0,60,70,80,90,100,110")
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
kvb = 2 * a.B * a.S * Hkv * 256
for impl in (1, 2):
    hydra.set_config("suffix_impl", impl)
    for c in ([148, 96, 64, 48, 32] if impl == 2 else [148]):
        hydra.set_config("suffix_ctas", c)
        ms = graph_ms(lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws))
        print(json.dumps(dict(what="suffix", impl=impl, ctas=c, ms=round(ms, 4), gbs=round(kvb / ms / 1e6, 1))), flush=True)
hydra.set_config("suffix_ctas", 0)
hydra.set_config("suffix_impl", 0)
for k in [int(x) for x in a.ks.split(",")]:
    hydra.set_config("overlap_prefix_ctas", k)
    ms_o = graph_ms(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws, aux_stream=aux))
    print(json.dumps(dict(what="overlap", k=k, ms=round(ms_o, 4))), flush=True)
hydra.set_config("overlap_prefix_ctas", 0)
ms_s = graph_ms(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws))
print(json.dumps(dict(what="sequential", ms=round(ms_s, 4))), flush=True)
