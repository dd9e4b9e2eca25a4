"""Step time with one step per CUDA graph (replayed K times) vs M steps captured in one graph (replayed
K/M times): the per-graph launch cost at each step boundary (diagnostics).
    python tools/graph_chunk_ab.py [shape,...]      M=8 K=400"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

SHAPES = {"c3_16k": (1024, 40, 40, 16384, 256), "c2": (256, 32, 32, 2048, 128), "c4": (512, 32, 8, 32768, 128),
          "c6": (256, 32, 4, 19947, 128)}
M, K = int(os.environ.get("M", 8)), int(os.environ.get("K", 400))
dev = torch.device("cuda:0")
aux = torch.cuda.Stream(priority=-1)
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else list(SHAPES)):
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
    step = lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws, aux_stream=aux)

    def graph(n):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(n):
                step()
        return gr

    res = {"shape": name}
    for n in (1, M):
        gr = graph(n)
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K // n):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        res[f"ms_per_step_graph_of_{n}"] = round(e0.elapsed_time(e1) / (K // n * n), 5)
        del gr
    print(json.dumps(res), flush=True)
    del q, pk, pv, sk, sv, ws, out
    torch.cuda.empty_cache()
