import os, sys, json
sys.path.insert(0, "/root/repo")
import torch
import paper_2402_05099_b200 as hydra
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for (B, Hq, Hkv, P) in [(16, 32, 8, 8192), (64, 40, 40, 4096), (8, 32, 8, 32768)]:
    q = torch.randn(B, Hq, 128, device=dev, generator=g).bfloat16()
    pk = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    pv = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    ws = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    res = {}
    for sp in [0, 2, 4, 8, 16, 32, 64]:
        hydra.set_config("prefix_splits", sp)
        for _ in range(3): hydra.prefix_attn(q, pk, pv, workspace=ws)
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); hydra.prefix_attn(q, pk, pv, workspace=ws); e1.record(); torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        res[sp] = round(tot / 10 * 1e3, 1)
    hydra.set_config("prefix_splits", 0)
    print(json.dumps(dict(shape=[B, Hq, Hkv, P], us_by_splits=res, kv_mb=round(2 * P * Hkv * 256 / 1e6, 1))), flush=True)
