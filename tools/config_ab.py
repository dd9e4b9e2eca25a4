"""Step time of hydragen_attention (sequential and SM-partitioned) for values of one config key
on several shapes (diagnostics).   KEY=seq_pdl VALUES=0,1 [EXTRA=k=v,..] [FLUSH=1] python tools/config_ab.py [shape,...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

SHAPES = {"c3_16k": (1024, 40, 40, 16384, 256), "c3_1k": (1024, 40, 40, 1024, 256), "c2": (256, 32, 32, 2048, 128),
          "c4": (512, 32, 8, 32768, 128), "c6": (256, 32, 4, 19947, 128)}
names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(SHAPES)
key = os.environ.get("KEY", "seq_pdl")
values = [int(v) for v in os.environ.get("VALUES", "0,1").split(",")]
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


FLUSH = os.environ.get("FLUSH") == "1"  # L2 flushed (write + read) before every timed replay
if FLUSH:
    fw = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    fr = torch.zeros(512 << 20, dtype=torch.uint8, device=dev)
for kv in filter(None, os.environ.get("EXTRA", "").split(",")):  # other keys held fixed: k=v,...
    k_, v_ = kv.split("=")
    hydra.set_config(k_, int(v_))


def t(gr, iters=50):
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    if FLUSH:
        ts = []
        for _ in range(iters):
            fw.zero_()
            fr.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gr.replay()
            e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        return round(sorted(a.elapsed_time(b) for a, b in ts)[iters // 2], 4)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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
    res = dict(shape=name, key=key)
    old = hydra.get_config(key)
    for v in values:
        hydra.set_config(key, v)
        for sched in ("seq", "overlap"):
            kw = dict(aux_stream=aux) if sched == "overlap" else {}
            res[f"{sched}_{v}"] = t(graph(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out,
                                                                           workspace=ws, **kw)))
    hydra.set_config(key, old)
    print(json.dumps(res), flush=True)
    del q, pk, pv, sk, sv, ws, out
    torch.cuda.empty_cache()
