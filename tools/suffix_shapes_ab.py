"""Tensor-core suffix alone (IMPL=2 persistent kernel, 3 short-suffix kernel) on the full chip for the C3 / C4 / C6 / C2 suffix shapes (diagnostics)."""
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
    flush_r = torch.zeros(512 << 20, dtype=torch.uint8, device=dev)
    write_only = os.environ.get("FLUSH") == "w"  # the old write-only flush (leaves L2 dirty)
    hydra.set_config("suffix_impl", int(os.environ.get("IMPL", 2)))  # 2 persistent, 3 short-suffix kernel
    hydra.set_config("suffix_ctas", ctas)
    call = lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws)
    call()
    torch.cuda.synchronize()
    # CUDA graph of the call: no Python marshalling inside the timed region (the 512-MB flush
    # before each replay runs longer than the host needs to enqueue the replay)
    gr = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        call()
    torch.cuda.current_stream().wait_stream(st)
    with torch.cuda.graph(gr):
        call()
    fn = gr.replay
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.zero_()
        if not write_only:
            flush_r.sum()  # evict the dirty flush lines before the timed region
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
    del q, sk, sv, ws, flush, flush_r, gr
    torch.cuda.empty_cache()
