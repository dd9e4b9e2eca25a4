import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2402_05099_b200 as hydra
from tests.util import problem_to
hydra.set_config("suffix_impl", 2)
lens = [0, 1, 127, 128, 129, 255, 256, 300, 17, 0, 384]
for Hq in (1, 8):
    for dist in ("plain", "boundary"):
        pb = synth.make_problem(len(lens), Hq, 1, 128, 0, 384, lens=lens, dtype="bf16", dist=dist, seed=18)
        t = problem_to(pb, "cuda:0")
        ref, lref = oracle.suffix_only(pb)
        for ctas in (1, 2, 3, 4, 5, 6, 11):
            hydra.set_config("suffix_ctas", ctas)
            o, lse = hydra.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
            torch.cuda.synchronize()
            err = np.abs(o.cpu().numpy() - ref).max(axis=2)  # [B, Hq]
            l_ = lse.cpu().numpy(); lerr = np.where(np.isneginf(lref) & np.isneginf(l_), 0.0, np.abs(l_ - lref))
            bad = [(b, h, round(float(err[b, h]), 4), round(float(lerr[b, h]), 4)) for b in range(len(lens)) for h in range(Hq) if err[b, h] > 2e-2 or lerr[b, h] > 1e-3]
            print(f"Hq={Hq} dist={dist} ctas={ctas} bad={bad[:12]}", flush=True)
