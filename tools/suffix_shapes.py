import os, sys, json
sys.path.insert(0, "/root/repo")
import torch
import paper_2402_05099_b200 as hydra
sys.path.insert(0, "/root/repo/tools")
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(0)
for (B, Hq, Hkv, S) in [(8, 32, 32, 4096), (4, 40, 40, 8192), (64, 32, 32, 1024), (2, 32, 32, 16384), (16, 32, 32, 512), (256, 32, 32, 128), (1024, 40, 40, 256), (128, 40, 40, 128)]:
    q = torch.randn(B, Hq, 128, device=dev, generator=g).bfloat16()
    sk = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
    sv = torch.randn(B, S, Hkv, 128, device=dev, generator=g).bfloat16()
    lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    ws = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    def t(fn, iters=20):
        fn(); torch.cuda.synchronize()
        tot = 0.0
        for _ in range(iters):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / iters
    kvb = 2 * B * S * Hkv * 256
    res = {}
    for impl, sp, ctas in [(0, 0, 0), (1, 0, 0), (1, 1, 0), (1, 2, 0), (1, 4, 0), (2, 0, 148), (2, 0, 76), (2, 2, 148), (2, 4, 148), (2, 8, 148)]:
        hydra.set_config("suffix_impl", impl); hydra.set_config("suffix_splits", sp); hydra.set_config("suffix_ctas", ctas)
        ms = t(lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws))
        res[f"impl{impl}_sp{sp}_c{ctas}"] = (round(ms * 1000, 1), round(kvb / ms / 1e6))
    print(json.dumps(dict(shape=[B, Hq, Hkv, S], us_gbs=res)), flush=True)
for k in ("suffix_impl", "suffix_splits", "suffix_ctas"): hydra.set_config(k, 0)
