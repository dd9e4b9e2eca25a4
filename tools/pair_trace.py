"""Cluster-0 event timeline of the CTA-pair prefix kernel (testing build; diagnostics).
    HYDRA_TESTING=1 python tools/pair_trace.py [poly] [B Hq Hkv P]
Per block (median over the steady state): S ready -> registers -> max -> exps -> P arrived for
both token halves of the leader, the MMA thread's view, and the block period."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2402_05099_b200 as hydra

assert hydra.get_config("testing_build") == 1, "run with HYDRA_TESTING=1"
dev = torch.device("cuda:0")
poly = int(sys.argv[1]) if len(sys.argv) > 1 else 0
B, H, Hkv, P = (int(x) for x in sys.argv[2:6]) if len(sys.argv) > 5 else (1024, 40, 40, 16384)
N, R = 1024, 44
tr = torch.zeros(R * N, dtype=torch.int64, device=dev)
hydra.set_config("prefix_impl", 3)
hydra.set_config("prefix_poly", poly)
hydra.set_config("pair_poly", poly)
hydra.set_config("prefix_variant", 9)
hydra.set_config("tc_debug_variant", int(os.environ.get("TC_DEBUG", 0)))
g = torch.Generator(device=dev)
g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
ws = torch.empty(hydra.attn_workspace_bytes(q, P, 1, Hkv) * 2, dtype=torch.uint8, device=dev)
for _ in range(3):
    hydra.prefix_attn(q, pk, pv, workspace=ws)
torch.cuda.synchronize()
hydra.set_config("prefix_trace", tr.data_ptr())
hydra.prefix_attn(q, pk, pv, workspace=ws)
torch.cuda.synchronize()
hydra.set_config("prefix_trace", 0)
hydra.set_config("tc_debug_variant", 0)
T = tr.view(R, N).cpu().numpy().astype(np.int64)
t0 = T[T > 0].min()
T = np.where(T > 0, T - t0, 0)
med = lambda a: float(np.median(a)) if len(a) else float("nan")
# WG a (rows 0-5) takes the even blocks of an item, WG b (rows 6-11) the odd ones
for x, base in (("a", 0), ("b", 6)):
    idx = np.nonzero(T[base + 5] > 0)[0]
    idx = idx[len(idx) // 4: 3 * len(idx) // 4]
    r = lambda k: T[base + k, idx]
    mrow = T[15 + (3 if x == "b" else 0), idx]
    print(f"WG {x}: row max {med(mrow - r(2)):.0f}  wait for m(n-1) + decide {med(r(3) - mrow):.0f}")
    print(f"WG {x} ({len(idx)} blocks): waitS {med(r(1) - r(0)):.0f}  ld {med(r(2) - r(1)):.0f}  max+m(n-1) {med(r(3) - r(2)):.0f}  "
          f"exps {med(r(4) - r(3)):.0f}  st+arrive {med(r(5) - r(4)):.0f}  S->P {med(r(5) - r(1)):.0f}  "
          f"own-block period {med(np.diff(r(1))):.0f}")
# per block (any WG): P arrival time = max over the two WGs' rows 5 (one of them is 0)
Parr = np.maximum(T[5], T[11])
idx = np.nonzero((Parr > 0) & (T[12] > 0))[0]
idx = idx[len(idx) // 4: 3 * len(idx) // 4]
print(f"block period (S ready n -> n+1): {med(np.diff(np.maximum(T[1], T[7])[idx])):.0f}")
print(f"MMA per block n, relative to P(n) arrival: saw P(+V) {med(T[12, idx] - Parr[idx]):.0f}  PV issued {med(T[19, idx] - Parr[idx]):.0f}"
      f"  K(n+3) seen {med(T[22, idx + 3] - Parr[idx]):.0f}  S(n+3) issued {med(T[14, idx + 3] - Parr[idx]):.0f}"
      f"  S(n+3) ready {med(np.maximum(T[1], T[7])[idx + 3] - Parr[idx]):.0f}")
W = T[23:31, idx]
print("per-warp P arrival relative to the earliest of the 8 (leader q0-3, peer q0-3):",
      " ".join(f"{med(W[i] - W.min(axis=0)):.0f}" for i in range(8)), "  MMA saw P - last arrival",
      f"{med(T[12, idx] - W.max(axis=0)):.0f}")
C = tr.view(-1)[40 * N: 44 * N].view(1024, 4).cpu().numpy().astype(np.int64)
n_cta = int((C[:, 0] > 0).sum())
C = C[:n_cta]
t0 = C[:, 0].min()
us = lambda x: (x - t0) / 1000.0
print(f"CTAs: {n_cta}; entry spread {us(C[:,0]).max():.2f} us, setup done median {np.median(us(C[:,1])):.2f} us, "
      f"softmax done min/median/max {us(C[:,2]).min():.2f}/{np.median(us(C[:,2])):.2f}/{us(C[:,2]).max():.2f} us, "
      f"exit max {us(C[:,3]).max():.2f} us")
if os.environ.get("PER_CTA"):
    done = us(C[:, 2])
    for w in range(0, n_cta, 2):
        print(f"cta {w:3d} worker {w // 2:3d} softmax done {done[w]:7.2f} us  exit {us(C[w, 3]):7.2f}")
E = T[32:35]
ne = int((E[2] > 0).sum())
if ne:
    print("items of WG a (leader): ordy wait begin -> O landed -> epilogue stores done; next item's first S ready")
    S1 = T[1]
    firsts = [int(np.nonzero(S1 > E[2, i])[0].min()) if (S1 > E[2, i]).any() else -1 for i in range(ne)]
    for i in range(ne):
        nxt = S1[firsts[i]] - E[2, i] if firsts[i] >= 0 else -1
        print(f"  item {i}: wait ordy {E[1, i] - E[0, i]}  epilogue {E[2, i] - E[1, i]}  -> next block's S ready +{nxt}")
if ne:
    print("Q issued (row 36) / Q seen late by the MMA thread (row 37), per item; S issued (row 14) of the items' first blocks")
    for i in range(min(4, int((T[36] > 0).sum()))):
        print(f"  item {i}: Q issued {T[36, i]}  Q seen-late {T[37, i]}  epilogue(i-1) end {E[2, i - 1] if i > 0 else 0}")
    idx14 = np.nonzero(T[14] > 0)[0]
    print("  S issued around item starts:", [(int(k), int(T[14, k])) for k in idx14[:4]], "...")
if ne and os.environ.get("RAW_EPI"):
    e_end = E[2, 0]
    ks = np.nonzero((T[14] > 0))[0]
    # the blocks around item 0's end: S issued (row 14), WG a S wait begin / ready (rows 0, 1), WG b (6, 7)
    for k in range(max(0, 124), 136):
        print(f"gs {k}: S issued {T[14, k] - e_end:8d}  a: wait {T[0, k] - e_end if T[0, k] else 0:8d} ready {T[1, k] - e_end if T[1, k] else 0:8d}"
              f"  b: wait {T[6, k] - e_end if T[6, k] else 0:8d} ready {T[7, k] - e_end if T[7, k] else 0:8d}  PV issued {T[19, k] - e_end if T[19, k] else 0:8d}")
    print("epilogue item 0 (rel. its end): ordy wait", E[0, 0] - e_end, " O landed", E[1, 0] - e_end,
          " (m,l) exchanged", T[35, 0] - e_end, " chunk0 in regs", T[31, 0] - e_end, " chunk0 stored", T[38, 0] - e_end, " chunk1 stored", T[39, 0] - e_end)
