"""Step time of hydragen_attention per schedule (sequential / SM-partitioned) and combine mode
(fuse_combine 0 / 1 / 2) on several shapes (diagnostics).
    python tools/fuse_ab.py [shape,...]      shapes: c3_16k c3_1k c2 c4 c6
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

SHAPES = {"c3_16k": (1024, 40, 40, 16384, 256), "c3_1k": (1024, 40, 40, 1024, 256), "c2": (256, 32, 32, 2048, 128),
          "c4": (512, 32, 8, 32768, 128), "c6": (256, 32, 4, 19947, 128)}
names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(SHAPES)
dev = torch.device("cuda:0")
aux = torch.cuda.Stream(priority=-1)


def graph(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    return gr


def t(gr, iters=30):
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / iters, 4)


for name in names:
    B, Hq, Hkv, P, S = SHAPES[name]
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    q = torch.randn(B, Hq, 128, device=dev, generator=g).bfloat16()
    pk = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    pv = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    sk = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
    sv = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
    lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    ws = torch.empty(hydra.attn_workspace_bytes(q, P, S, Hkv) * 2, dtype=torch.uint8, device=dev)
    out = torch.empty(B, Hq, 128, dtype=torch.bfloat16, device=dev)
    res = dict(shape=name)
    for fuse in (0, 1, 2):
        hydra.set_config("fuse_combine", fuse)
        for sched in ("seq", "overlap"):
            kw = dict(aux_stream=aux) if sched == "overlap" else {}
            res[f"{sched}_f{fuse}"] = t(graph(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out,
                                                                             workspace=ws, **kw)))
            if sched == "overlap":
                res["k"] = hydra.get_config("last_overlap_k")
    hydra.set_config("fuse_combine", 0)
    print(json.dumps(res), flush=True)
    del q, pk, pv, sk, sv, ws, out
    torch.cuda.empty_cache()
