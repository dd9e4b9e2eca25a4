"""Launch the persistent prefix kernel a few times at one shape (for ncu metric captures).

    python tools/prefix_one.py [poly] [debug] [B H Hkv P]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_05099_b200 as hydra
dev = torch.device("cuda:0")
poly = int(sys.argv[1]) if len(sys.argv) > 1 else 0
debug = int(sys.argv[2]) if len(sys.argv) > 2 else 0
B, H, Hkv, P = (int(x) for x in sys.argv[3:7]) if len(sys.argv) > 6 else (1024, 40, 40, 16384)
hydra.set_config("prefix_impl", 3); hydra.set_config("prefix_poly", poly); hydra.set_config("tc_debug_variant", debug)
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
ws = torch.empty(hydra.attn_workspace_bytes(q, P, 1, Hkv), dtype=torch.uint8, device=dev)
for _ in range(3):
    hydra.prefix_attn(q, pk, pv, workspace=ws)
torch.cuda.synchronize()
