"""Suffix GB/s and prefix TFLOP/s versus the number of SMs (CUDA green contexts).

Decides the SM split for overlapping the HBM-bound suffix with the tensor-bound prefix.
"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_05099_b200 as hydra
from torch.cuda.green_contexts import GreenContext

dev = torch.device("cuda:0")
B, H, P, S = 1024, 40, 16384, 256
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(P, H, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(P, H, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(B, S, H, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(B, S, H, 128, device=dev, generator=g).bfloat16()
lens = torch.full((B,), S, dtype=torch.int32, device=dev)
ws = torch.empty(hydra.attn_workspace_bytes(q, P, S, H), dtype=torch.uint8, device=dev)
sbytes = 2 * B * S * H * 128 * 2
pflops = 4.0 * B * H * P * 128

def timeit(fn, stream, iters=10):
    with torch.cuda.stream(stream):
        fn(); fn()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters): fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters

res = []
for k in [8, 16, 32, 48, 64, 72, 80, 96, 112, 128, 148]:
    try:
        gc = GreenContext.create(k, 0)
        st = gc.Stream()
    except Exception as e:
        print("gc", k, "failed", e); continue
    ms_s = timeit(lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws, stream=st), st)
    ms_p = timeit(lambda: hydra.prefix_attn(q, pk, pv, workspace=ws, stream=st), st, iters=3)
    r = dict(sms=k, suffix_ms=round(ms_s, 4), suffix_gbs=round(sbytes / ms_s / 1e6, 1),
             prefix_ms=round(ms_p, 4), prefix_tflops=round(pflops / ms_p / 1e9, 1))
    print(json.dumps(r), flush=True)
    res.append(r)
