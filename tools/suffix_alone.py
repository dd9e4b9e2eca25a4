"""The C3@16K suffix alone on SUFFIX_CTAS SMs (tensor-core kernel), for ncu (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2402_05099_b200 as hydra

B, H, S = 1024, 40, 256
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(B, S, H, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(B, S, H, 128, device=dev, generator=g).bfloat16()
lens = torch.full((B,), S, dtype=torch.int32, device=dev)
hydra.set_config("suffix_impl", 2)
hydra.set_config("suffix_ctas", int(os.environ.get("SUFFIX_CTAS", 84)))
for _ in range(3):
    hydra.suffix_attn(q, sk, sv, lens)
torch.cuda.synchronize()
print("ok")
