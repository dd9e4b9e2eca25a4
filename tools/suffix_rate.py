"""Tensor-core suffix kernel: streaming rate vs CTA count and blocks per softmax round (diagnostics)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_05099_b200 as hydra
B, H, S = int(os.environ.get("B", 1024)), int(os.environ.get("H", 40)), int(os.environ.get("S", 256))
Hkv = int(os.environ.get("HKV", H))
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
lens = torch.full((B,), S, dtype=torch.int32, device=dev)
ws = torch.empty(hydra.attn_workspace_bytes(q, 0, S, Hkv) * 2 + (1 << 20), dtype=torch.uint8, device=dev)
def graph_ms(fn, iters=20):
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
kvb = 2 * B * S * Hkv * 256
hydra.set_config("suffix_impl", 2)
hydra.set_config("tc_debug_variant", int(os.environ.get("DEBUG", 0)))
ctas_list = [int(x) for x in os.environ.get("CTAS", "148,120,100,92,80,64,48,32,16").split(",")]
for cb in (1, 2):
    hydra.set_config("suffix_cb", cb)
    for c in ctas_list:
        hydra.set_config("suffix_ctas", c)
        ms = graph_ms(lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws))
        print(json.dumps(dict(cb=cb, ctas=c, ms=round(ms, 4), gbs=round(kvb / ms / 1e6, 1),
                              gbs_per_sm=round(kvb / ms / 1e6 / c, 1))), flush=True)
hydra.set_config("suffix_impl", 0); hydra.set_config("suffix_ctas", 0); hydra.set_config("tc_debug_variant", 0); hydra.set_config("suffix_cb", 2)
