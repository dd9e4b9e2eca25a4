"""Tensor-core suffix alone on the full chip for the C3 / C4 / C6 / C2 suffix shapes (diagnostics)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

SH = {"c3": (1024, 40, 40, 256), "c4": (512, 32, 8, 128), "c6": (256, 32, 4, 128), "c2": (256, 32, 32, 128)}
if os.environ.get("SHAPES"):  # name:B,H,HKV,S;...
    SH = {k: tuple(int(x) for x in v.split(",")) for k, v in (e.split(":") for e in os.environ["SHAPES"].split(";"))}
dev = torch.device("cuda:0")
ctas = int(os.environ.get("CTAS", 0))
for name, (B, H, HKV, S) in SH.items():
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
    sk = torch.randn(B, S, HKV, 128, device=dev, generator=g).bfloat16()
    sv = torch.randn(B, S, HKV, 128, device=dev, generator=g).bfloat16()
    lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    ws = torch.empty(hydra.attn_workspace_bytes(q, 1, S, HKV) * 2, dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    hydra.set_config("suffix_impl", 2)
    hydra.set_config("suffix_ctas", ctas)
    fn = lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws)
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    byt = 2 * B * S * HKV * 256
    print(json.dumps(dict(shape=name, ms=round(ms, 4), tbs=round(byt / ms / 1e9, 2))), flush=True)
    hydra.set_config("suffix_impl", 0)
    hydra.set_config("suffix_ctas", 0)
    del q, sk, sv, ws, flush
    torch.cuda.empty_cache()
