"""Suffix kernel alone: CUDA-event time of one graph replay vs the kernel's own span (first CTA
start to last CTA end, %globaltimer, config key step_timer), L2 flushed (write + read) before
each replay (diagnostics).     IMPL=2|3 SHAPES="name:B,H,HKV,S;..." python tools/suffix_span.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

SH = {"c6": (256, 32, 4, 128), "c6r": (256, 32, 4, 64), "c4": (512, 32, 8, 128)}
if os.environ.get("SHAPES"):
    SH = {k: tuple(int(x) for x in v.split(",")) for k, v in (e.split(":") for e in os.environ["SHAPES"].split(";"))}
dev = torch.device("cuda:0")
fw = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
fr = torch.zeros(512 << 20, dtype=torch.uint8, device=dev)
for name, (B, H, HKV, S) in SH.items():
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
    sk = torch.randn(B, S, HKV, 128, device=dev, generator=g).bfloat16()
    sv = torch.randn(B, S, HKV, 128, device=dev, generator=g).bfloat16()
    lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    ws = torch.empty(hydra.attn_workspace_bytes(q, 1, S, HKV) * 2, dtype=torch.uint8, device=dev)
    timer = torch.zeros(4, dtype=torch.int64, device=dev)
    init = torch.tensor([-1, 0, -1, 0], dtype=torch.int64, device=dev)
    for impl in [int(x) for x in os.environ.get("IMPL", "2,3").split(",")]:
        hydra.set_config("suffix_impl", impl)
        hydra.set_config("step_timer", timer.data_ptr())
        call = lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws)
        call()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            call()
        torch.cuda.current_stream().wait_stream(st)
        with torch.cuda.graph(gr):
            call()
        ev, span = [], []
        for _ in range(20):
            timer.copy_(init)
            fw.zero_()
            fr.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gr.replay()
            e1.record()
            torch.cuda.synchronize()
            t = [int(v) & 0xFFFFFFFFFFFFFFFF for v in timer.tolist()]
            ev.append(e0.elapsed_time(e1) * 1e3)
            span.append((t[3] - t[2]) * 1e-3)
        ev.sort()
        span.sort()
        byt = 2 * B * S * HKV * 256
        print(json.dumps(dict(shape=name, impl=impl, event_us=round(ev[10], 1), span_us=round(span[10], 1),
                              span_tbs=round(byt / span[10] / 1e6, 2))), flush=True)
        hydra.set_config("step_timer", 0)
        hydra.set_config("suffix_impl", 0)
        del gr
    del q, sk, sv, ws
    torch.cuda.empty_cache()
