"""Paged vs contiguous suffix streaming rate at the C3 shape (diagnostics; no oracle).

For each page size, the contiguous [B, S, Hkv, 128] caches are scattered into a shuffled page
pool and hydra_suffix_attn_paged is timed (CUDA graph, events) on the SIMT kernel (all SMs)
and on the tensor-core kernel (CTAS SMs, default 76 = the overlapped step's share)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

B, H, S = int(os.environ.get("B", 1024)), int(os.environ.get("H", 40)), int(os.environ.get("S", 256))
Hkv = int(os.environ.get("HKV", H))
CTAS = [int(x) for x in os.environ.get("CTAS", "76,148").split(",")]
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
lens = torch.full((B,), S, dtype=torch.int32, device=dev)
ws = torch.empty(hydra.attn_workspace_bytes(q, 0, S, Hkv) * 2 + (1 << 20), dtype=torch.uint8, device=dev)


def graph_ms(fn, iters=30):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


kvb = 2 * B * S * Hkv * 256
hydra.set_config("tc_debug_variant", int(os.environ.get("DEBUG", 0)))  # 256 = drain only (invalid results)
for ps in [0] + [int(x) for x in os.environ.get("PS", "8,16,32,64,128,256").split(",")]:
    if ps:
        npg = S // ps
        # PERM=0: pages in sequence order (the contiguous layout, through the block table);
        # PERM=2: pages shuffled within each sequence only
        mode = int(os.environ.get("PERM", 1))
        if mode == 0:
            perm = torch.arange(B * npg, device=dev)
        elif mode == 2:
            perm = (torch.arange(B, device=dev)[:, None] * npg +
                    torch.argsort(torch.rand(B, npg, device=dev, generator=g), dim=1)).reshape(-1)
        else:
            perm = torch.randperm(B * npg, device=dev, generator=g)
        if mode == 3:  # the contiguous caches themselves as the pools, identity table
            perm = torch.arange(B * npg, device=dev)
            kp, vp = sk.view(B * npg, ps, Hkv, 128), sv.view(B * npg, ps, Hkv, 128)
        else:
            kp = torch.empty(B * npg, ps, Hkv, 128, dtype=torch.bfloat16, device=dev)
            vp = torch.empty_like(kp)
            kp[perm] = sk.view(B * npg, ps, Hkv, 128)
            vp[perm] = sv.view(B * npg, ps, Hkv, 128)
        tab = perm.view(B, npg).to(torch.int32)
        fn = lambda: hydra.suffix_attn_paged(q, kp, vp, tab, lens, workspace=ws)
    else:
        fn = lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws)
    for impl, ctas in [(1, 0)] + [(2, c) for c in CTAS]:
        hydra.set_config("suffix_impl", impl)
        hydra.set_config("suffix_ctas", ctas)
        ms = graph_ms(fn)
        print(json.dumps(dict(perm=int(os.environ.get("PERM", 1)), page_size=ps or "contiguous", impl="simt" if impl == 1 else "tc", ctas=ctas or 148,
                              ms=round(ms, 4), gbs=round(kvb / ms / 1e6, 1))), flush=True)
hydra.set_config("suffix_impl", 0)
hydra.set_config("suffix_ctas", 0)
hydra.set_config("tc_debug_variant", 0)
