"""Run-to-run variance of the SM-partitioned overlap vs its parts (diagnostics)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_05099_b200 as hydra
k = int(sys.argv[1]) if len(sys.argv) > 1 else 48
B, H, P, S = 1024, 40, 16384, 256
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(P, H, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(P, H, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(B, S, H, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(B, S, H, 128, device=dev, generator=g).bfloat16()
lens = torch.full((B,), S, dtype=torch.int32, device=dev)
ws = torch.empty(hydra.attn_workspace_bytes(q, P, S, H) * 2, dtype=torch.uint8, device=dev)
out = torch.empty(B, H, 128, dtype=torch.bfloat16, device=dev)
aux = torch.cuda.Stream(priority=-1)
def graph(fn):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr): fn()
    return gr
def t(gr, iters=10):
    gr.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): gr.replay()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / iters, 4)
hydra.set_config("prefix_ctas", k)
g_pre = graph(lambda: hydra.prefix_attn(q, pk, pv, workspace=ws))
hydra.set_config("prefix_ctas", 0)
hydra.set_config("suffix_impl", 2); hydra.set_config("suffix_ctas", 148 - k)
g_suf = graph(lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws))
hydra.set_config("suffix_impl", 0); hydra.set_config("suffix_ctas", 0)
hydra.set_config("overlap_prefix_ctas", k)
g_ov = graph(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws, aux_stream=aux))
hydra.set_config("overlap_prefix_ctas", 0)
g_seq = graph(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws))
rows = {"prefix_k": [], "suffix_rest": [], "overlap": [], "sequential": []}
for rep in range(6):
    rows["prefix_k"].append(t(g_pre)); rows["suffix_rest"].append(t(g_suf))
    rows["overlap"].append(t(g_ov)); rows["sequential"].append(t(g_seq))
for kk, v in rows.items():
    print(json.dumps({"k": k, "what": kk, "ms": v}))
