"""LSE combine kernel rate at the C3 size (B*Hq = 40960 rows, d = 128) vs part count (diagnostics)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(0)
rows, d = 40960, 128
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for n in (2, 3, 4, 6):
    o = torch.randn(n, rows, d, device=dev, generator=g)
    lse = torch.randn(n, rows, device=dev, generator=g)
    lse[0, ::7] = -float("inf")
    out = torch.empty(rows, d, dtype=torch.bfloat16, device=dev)
    lo = torch.empty(rows, dtype=torch.float32, device=dev)
    hydra.combine(o, lse, out=out, lse_out=lo)
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hydra.combine(o, lse, out=out, lse_out=lo)
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    us = tot / 20 * 1e3
    nbytes = n * rows * (d + 1) * 4 + rows * (d * 2 + 4)
    print(json.dumps(dict(parts=n, us=round(us, 1), gbs=round(nbytes / us / 1e3, 1))), flush=True)
