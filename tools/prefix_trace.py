"""CTA-0 event timeline of the persistent prefix kernel (diagnostics).

Rows (clock64 per block): 3t+0 softmax_t starts waiting for S, 3t+1 S_t ready, 3t+2 P_t
published, 6+t MMA thread saw P_t, 8+t softmax_t exps done (before the PV wait), 10+t S in
registers, 12+t row max done.
    python tools/prefix_trace.py [poly] [variant] [B H Hkv P]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2402_05099_b200 as hydra
dev = torch.device("cuda:0")
poly = int(sys.argv[1]) if len(sys.argv) > 1 else 0
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 3
B, H, Hkv, P = (int(x) for x in sys.argv[3:7]) if len(sys.argv) > 6 else (1024, 40, 40, 16384)
N = 1024
tr = torch.zeros(14 * N, dtype=torch.int64, device=dev)
hydra.set_config("prefix_impl", 3); hydra.set_config("prefix_poly", poly); hydra.set_config("prefix_variant", variant)
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
ws = torch.empty(hydra.attn_workspace_bytes(q, P, 1, Hkv), dtype=torch.uint8, device=dev)
for _ in range(3):
    hydra.prefix_attn(q, pk, pv, workspace=ws)
torch.cuda.synchronize()
hydra.set_config("prefix_trace", tr.data_ptr())
hydra.prefix_attn(q, pk, pv, workspace=ws)
torch.cuda.synchronize()
hydra.set_config("prefix_trace", 0)
T = tr.view(14, N).cpu().numpy().astype(np.int64)
n = int(min((T[1] > 0).sum(), (T[4] > 0).sum()))
t0 = T[T > 0].min()
T = T - t0
lo, hi = n // 4, 3 * n // 4  # steady state
print(f"blocks per tile traced: {n}")
for t in (0, 1):
    w_s = T[3 * t + 1, lo:hi] - T[3 * t + 0, lo:hi]         # waiting for S
    sm = T[8 + t, lo:hi] - T[3 * t + 1, lo:hi]              # ld + max + exps
    pvw = T[3 * t + 2, lo:hi] - T[8 + t, lo:hi]             # PV wait + correction + st + arrive
    per = np.diff(T[3 * t + 1, lo:hi])                       # S ready -> next S ready
    mma = T[3 * t + 1, lo + 1:hi + 1] - T[6 + t, lo:hi]     # MMA saw P(n) -> S(n+1) ready (v3)
    rx = T[6 + t, lo:hi] - T[3 * t + 2, lo:hi]               # P published -> MMA thread saw it
    ldw = T[10 + t, lo:hi] - T[3 * t + 1, lo:hi]
    mxw = T[12 + t, lo:hi] - T[10 + t, lo:hi]
    exw = T[8 + t, lo:hi] - T[12 + t, lo:hi]
    print(f"tile {t}: tmem-ld {np.median(ldw):.0f}  max {np.median(mxw):.0f}  exps(+pp wait) {np.median(exw):.0f}")
    print(f"tile {t}: period {np.median(per):.0f}  waitS {np.median(w_s):.0f}  softmax {np.median(sm):.0f}  "
          f"pv-wait+st {np.median(pvw):.0f}  mma-react {np.median(rx):.0f}  P->S(n+1) {np.median(mma):.0f}")
off = T[4, lo:hi] - T[1, lo:hi]
print(f"S1 ready - S0 ready (same n): median {np.median(off):.0f}")
for k in range(lo, lo + 4):
    print(k, " ".join(f"{T[r, k]:>9d}" for r in range(14)))
