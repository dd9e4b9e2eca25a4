"""Prefix kernel alone: time per launch and TFLOP/s for prefix_variant values on the C3 / C4 / C6
prefix shapes (diagnostics).   python tools/prefix_ab.py [variants] [shapes]
    variants: comma list (default 6,9); "9p2" = variant 9 with pair_poly 2 (testing build for 2 / 3); shapes: c3,c4,c6,c2 (default all)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

variants = (sys.argv[1] if len(sys.argv) > 1 else "6,9").split(",")  # prefix_variant values, or t1 (one-tile kernel)
SH = {"c3": (1024, 40, 40, 16384), "c4": (512, 32, 8, 32768), "c6": (256, 32, 4, 19947), "c2": (256, 32, 32, 2048)}
shapes = (sys.argv[2] if len(sys.argv) > 2 else "c3,c4,c6,c2").split(",")
ctas = int(os.environ.get("CTAS", 0))
dev = torch.device("cuda:0")
for name in shapes:
    B, Hq, Hkv, P = SH[name]
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    q = torch.randn(B, Hq, 128, device=dev, generator=g).bfloat16()
    pk = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    pv = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    ws = torch.empty(hydra.attn_workspace_bytes(q, P, 1, Hkv) * 4, dtype=torch.uint8, device=dev)
    flops = 4.0 * B * Hq * P * 128
    ref = None
    for v in variants:
        vv, _, poly = v.partition("p")
        hydra.set_config("prefix_impl", 2 if v == "t1" else 3)
        hydra.set_config("prefix_variant", 9 if v == "t1" else int(vv))
        hydra.set_config("prefix_poly", int(poly) if poly else 4)
        hydra.set_config("pair_poly", int(poly) if poly else 0)
        hydra.set_config("prefix_ctas", ctas)
        hydra.set_config("pair_cluster", int(os.environ.get("CLUSTER", 0)))
        fn = lambda: hydra.prefix_attn(q, pk, pv, workspace=ws)
        o, lse = fn()
        torch.cuda.synchronize()
        if ref is None:
            ref = (o.float(), lse)
            diff = 0.0
        else:
            diff = float((o.float() - ref[0]).abs().max())
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(json.dumps(dict(shape=name, variant=v, ms=round(ms, 4), tflops=round(flops / ms / 1e9, 1),
                              max_diff_vs_first=diff)), flush=True)
    hydra.set_config("prefix_variant", 6)
    hydra.set_config("prefix_impl", 0)
    del q, pk, pv, ws
    torch.cuda.empty_cache()
