"""Bring-up diagnostic for the tcgen05 prefix kernel: prefix parity per debug variant."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2402_05099_b200 as hydra
from tests.util import problem_to, errors, lse_err

for variant in (0, 1):
    hydra.set_config("tc_debug_variant", variant)
    for (B, Hq, Hkv, P) in [(3, 4, 2, 300), (130, 1, 1, 128), (40, 8, 8, 1000)]:
        pb = synth.make_problem(B, Hq, Hkv, 128, P, 1, dtype="bf16", dist="mixed", seed=3)
        t = problem_to(pb, "cuda:0")
        o, lse = hydra.prefix_attn(t["q"], t["pk"], t["pv"])
        torch.cuda.synchronize()
        ref, lref = oracle.prefix_only(pb)
        mx, mean, fin = errors(o, ref)
        try:
            le = lse_err(lse, lref)
        except AssertionError as e:
            le = str(e)
        print(f"variant={variant} B={B} Hq={Hq} Hkv={Hkv} P={P}: max={mx:.3e} mean={mean:.3e} finite={fin} lse={le}", flush=True)
