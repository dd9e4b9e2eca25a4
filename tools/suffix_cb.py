"""Tensor-core suffix: blocks per softmax round (suffix_cb 1 / 2) vs suffix shape (diagnostics)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for (B, Hq, Hkv, S, ctas) in [(256, 32, 4, 128, 148), (512, 32, 8, 128, 148), (1024, 40, 40, 256, 76),
                              (128, 32, 4, 2048, 148), (1024, 32, 32, 512, 76)]:
    q = torch.randn(B, Hq, 128, device=dev, generator=g).bfloat16()
    sk = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
    sv = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
    lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    res = {}
    for cb in (1, 2):
        hydra.set_config("suffix_impl", 2)
        hydra.set_config("suffix_ctas", ctas)
        hydra.set_config("suffix_cb", cb)
        hydra.suffix_attn(q, sk, sv, lens)
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hydra.suffix_attn(q, sk, sv, lens)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        ms = tot / 20
        res[f"cb{cb}"] = [round(ms * 1e3, 1), round(2 * B * S * Hkv * 256 / ms / 1e6)]
    print(json.dumps(dict(shape=[B, Hq, Hkv, S], ctas=ctas, us_gbs=res)), flush=True)
for k in ("suffix_impl", "suffix_ctas"):
    hydra.set_config(k, 0)
hydra.set_config("suffix_cb", 2)
