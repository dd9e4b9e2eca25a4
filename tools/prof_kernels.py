"""Run the hot kernels at a bench workload for ncu captures (not a benchmark)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2402_05099_b200 as hydra

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=1024); ap.add_argument("--Hq", type=int, default=40)
ap.add_argument("--Hkv", type=int, default=40); ap.add_argument("--P", type=int, default=16384)
ap.add_argument("--S", type=int, default=256); ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--what", default="prefix", choices=["prefix", "suffix", "attn"])
ap.add_argument("--splits", type=int, default=0)
ap.add_argument("--suffix-impl", type=int, default=0)
ap.add_argument("--prefix-impl", type=int, default=0)
ap.add_argument("--suffix-ctas", type=int, default=0)
ap.add_argument("--prefix-ctas", type=int, default=0)
ap.add_argument("--paged", type=int, default=0, help="suffix in a shuffled page pool of this page size")
a = ap.parse_args()
dev = torch.device("cuda:0")
hydra.set_config("prefix_splits", a.splits)
hydra.set_config("suffix_impl", a.suffix_impl)
hydra.set_config("prefix_impl", a.prefix_impl)
hydra.set_config("suffix_ctas", a.suffix_ctas)
hydra.set_config("prefix_ctas", a.prefix_ctas)
S = a.S if a.what != "prefix" else 1
# plain N(0,1) on device is enough for profiling (values do not change the work)
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(a.B, a.Hq, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(a.P, a.Hkv, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(a.P, a.Hkv, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(a.B, S, a.Hkv, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(a.B, S, a.Hkv, 128, device=dev, generator=g).bfloat16()
lens = torch.full((a.B,), S, dtype=torch.int32, device=dev)
ws = torch.empty(hydra.attn_workspace_bytes(q, a.P, S, a.Hkv), dtype=torch.uint8, device=dev)
if a.paged:
    npg = S // a.paged
    perm = torch.randperm(a.B * npg, device=dev, generator=g)
    kp = torch.empty(a.B * npg, a.paged, a.Hkv, 128, dtype=torch.bfloat16, device=dev)
    vp = torch.empty_like(kp)
    kp[perm] = sk.view(-1, a.paged, a.Hkv, 128)
    vp[perm] = sv.view(-1, a.paged, a.Hkv, 128)
    tab = perm.view(a.B, npg).to(torch.int32)
for _ in range(a.iters):
    if a.what == "prefix":
        hydra.prefix_attn(q, pk, pv, workspace=ws)
    elif a.what == "suffix" and a.paged:
        hydra.suffix_attn_paged(q, kp, vp, tab, lens, workspace=ws)
    elif a.what == "suffix":
        hydra.suffix_attn(q, sk, sv, lens, workspace=ws)
    else:
        hydra.hydragen_attention(q, pk, pv, sk, sv, lens, workspace=ws)
torch.cuda.synchronize()
print("done")
