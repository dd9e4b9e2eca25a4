"""Prefix kernels across shapes: automatic choice vs forced kernel / CTA count (diagnostics).

L2 flushed before every launch; TFLOP/s = 4 B Hq P d / time."""
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
SHAPES = [(256, 32, 4, 19947), (512, 32, 8, 32768), (256, 32, 32, 2048), (16, 32, 8, 8192), (64, 40, 40, 4096),
          (1024, 40, 40, 1024), (128, 32, 8, 16384)]
if os.environ.get("SHAPES"):
    SHAPES = [tuple(int(x) for x in sh.split("x")) for sh in os.environ["SHAPES"].split(",")]
for (B, Hq, Hkv, P) in SHAPES:
    q = torch.randn(B, Hq, 128, device=dev, generator=g).bfloat16()
    pk = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    pv = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flops = 4.0 * B * Hq * P * 128
    res = {}
    for name, cfg in [("auto", {}), ("tc1", {"prefix_impl": 2}), ("tc2_148", {"prefix_impl": 3}), ("auto2", {}),
                      ("tc2_120", {"prefix_impl": 3, "prefix_ctas": 120}),
                      ("tc2_96", {"prefix_impl": 3, "prefix_ctas": 96}), ("simt", {"prefix_impl": 1})]:
        for k, v in cfg.items():
            hydra.set_config(k, v)
        try:
            hydra.prefix_attn(q, pk, pv, workspace=ws)
            torch.cuda.synchronize()
            tot = 0.0
            for _ in range(10):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                hydra.prefix_attn(q, pk, pv, workspace=ws)
                e1.record()
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
            ms = tot / 10
            res[name] = [round(ms * 1e3, 1), round(flops / ms / 1e9, 1)]
        except Exception as e:  # noqa: BLE001 -- diagnostics: report and go on
            res[name] = str(e)[:60]
        for k in cfg:
            hydra.set_config(k, 0)
    print(json.dumps(dict(shape=[B, Hq, Hkv, P], us_tflops=res)), flush=True)
