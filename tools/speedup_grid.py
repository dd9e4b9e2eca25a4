"""Attention microbenchmark in the style of the paper's §4.2 (App. D.2).

Shape: 8 query heads, 1 KV head, d = 128 (CodeLlama-34b per GPU under 8-way TP).
Hydragen = hydra.hydragen_attention (tcgen05 prefix + suffix + combine).  Baseline =
per-sequence attention over each sequence's own full KV (prefix copied into every
sequence, as in the paper's FlashAttention baseline), run with the same split-K
decode kernel the suffix uses.  Timing: CUDA graph per call, L2 flushed by writing a
256 MiB buffer before every replay (the paper uses 128 MiB on A100's 40 MB L2), mean
over the timed replays.  Output: one JSON line per grid point and a summary.

    python tools/speedup_grid.py [--out profiles/r1_speedup_grid.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="32,128,512,1024")
ap.add_argument("--prefixes", default="1024,4096,16384")
ap.add_argument("--suffixes", default="64,256")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--out", default="")
a = ap.parse_args()
dev = torch.device("cuda:0")
Hq, Hkv, d = 8, 1, 128
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def graph_ms(fn, iters):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    tot = 0.0
    for i in range(iters + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            tot += e0.elapsed_time(e1)
    return tot / iters


rows = []
gen = torch.Generator(device=dev)
gen.manual_seed(0)
for P in [int(x) for x in a.prefixes.split(",")]:
    for S in [int(x) for x in a.suffixes.split(",")]:
        for B in [int(x) for x in a.batches.split(",")]:
            full_bytes = B * (P + S) * Hkv * d * 2 * 2
            if full_bytes > 60e9:
                continue
            q = torch.randn(B, Hq, d, device=dev, generator=gen).bfloat16()
            pk = torch.randn(P, Hkv, d, device=dev, generator=gen).bfloat16()
            pv = torch.randn(P, Hkv, d, device=dev, generator=gen).bfloat16()
            sk = torch.randn(B, S, Hkv, d, device=dev, generator=gen).bfloat16()
            sv = torch.randn(B, S, Hkv, d, device=dev, generator=gen).bfloat16()
            lens = torch.full((B,), S, dtype=torch.int32, device=dev)
            ws = torch.empty(hydra.attn_workspace_bytes(q, P, S, Hkv), dtype=torch.uint8, device=dev)
            out = torch.empty(B, Hq, d, dtype=torch.bfloat16, device=dev)
            t_h = graph_ms(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws), a.iters)
            # baseline: every sequence owns a full copy of prefix || suffix
            fk = torch.cat([pk.unsqueeze(0).expand(B, P, Hkv, d), sk], dim=1).contiguous()
            fv = torch.cat([pv.unsqueeze(0).expand(B, P, Hkv, d), sv], dim=1).contiguous()
            flens = torch.full((B,), P + S, dtype=torch.int32, device=dev)
            hydra.set_config("suffix_impl", 1)
            wsb = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
            t_b = graph_ms(lambda: hydra.suffix_attn(q, fk, fv, flens, workspace=wsb), a.iters)
            hydra.set_config("suffix_impl", 0)
            r = dict(B=B, prefix=P, suffix=S, hydragen_ms=round(t_h, 4), per_sequence_ms=round(t_b, 4),
                     speedup=round(t_b / t_h, 2))
            print(json.dumps(r), flush=True)
            rows.append(r)
            del fk, fv, q, pk, pv, sk, sv, ws, wsb
            torch.cuda.empty_cache()
summary = {"shape": "8 q heads / 1 kv head / d=128 (paper §4.2)", "max_speedup": max(r["speedup"] for r in rows),
           "rows": rows}
print(json.dumps({"max_speedup": summary["max_speedup"]}))
if a.out:
    json.dump(summary, open(a.out, "w"), indent=1)
