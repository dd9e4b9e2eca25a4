"""SM-partitioned overlap at C3@16K: step time vs prefix CTA count k (diagnostics).
    python tools/overlap_sweep.py [k,k,...] [variant]
"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_05099_b200 as hydra
ks = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "48,56,60,64,68,72,76").split(",")]
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 3
B, H, P, S = int(os.environ.get("B", 1024)), int(os.environ.get("H", 40)), int(os.environ.get("P", 16384)), int(os.environ.get("S", 256))
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
PAGED = int(os.environ.get("PAGED", 0))  # page size: the suffix in a shuffled page pool
if PAGED:
    perm = torch.randperm(B * (S // PAGED), device=dev, generator=g)
    kp = torch.empty(B * (S // PAGED), PAGED, H, 128, dtype=torch.bfloat16, device=dev); vp = torch.empty_like(kp)
    kp[perm] = sk.view(-1, PAGED, H, 128); vp[perm] = sv.view(-1, PAGED, H, 128)
    tab = perm.view(B, -1).to(torch.int32)
    suffix_call = lambda: hydra.suffix_attn_paged(q, kp, vp, tab, lens, workspace=ws)
    attn_call = lambda **kw: hydra.hydragen_attention_paged(q, pk, pv, kp, vp, tab, lens, out=out, workspace=ws, **kw)
else:
    suffix_call = lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws)
    attn_call = lambda **kw: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws, **kw)
hydra.set_config("prefix_variant", variant)
def graph(fn):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr): fn()
    return gr
def t(gr, iters=20):
    for _ in range(3): gr.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): gr.replay()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / iters, 4)
for k in ks:
    hydra.set_config("prefix_ctas", k)
    tp = t(graph(lambda: hydra.prefix_attn(q, pk, pv, workspace=ws)))
    hydra.set_config("prefix_ctas", 0)
    hydra.set_config("suffix_impl", 2); hydra.set_config("suffix_ctas", 148 - k)
    ts = t(graph(suffix_call))
    hydra.set_config("suffix_impl", 0); hydra.set_config("suffix_ctas", 0)
    hydra.set_config("overlap_prefix_ctas", k)
    to = t(graph(lambda: attn_call(aux_stream=aux)))
    hydra.set_config("overlap_prefix_ctas", 0)
    print(json.dumps(dict(k=k, variant=variant, prefix_alone=tp, suffix_alone=ts, overlap=to)), flush=True)
hydra.set_config("overlap_prefix_ctas", 0)
ts = t(graph(lambda: attn_call()))
print(json.dumps(dict(what="sequential", ms=ts)))
to = t(graph(lambda: attn_call(aux_stream=aux)))
print(json.dumps(dict(what="auto", k=hydra.get_config("last_overlap_k"), ms=to)))
hydra.set_config("prefix_variant", 6)
