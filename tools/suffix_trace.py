"""CTA-0 timeline of the tensor-core suffix kernel (diagnostics; see the trace rows in suffix_tc.cu).

    python tools/suffix_trace.py [cb] [ctas]      (C3 shape: B=1024, 40 MHA heads, S=256)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2402_05099_b200 as hydra
cb = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 16
B, H, S = int(os.environ.get("B", 1024)), int(os.environ.get("H", 40)), int(os.environ.get("S", 256))
HKV = int(os.environ.get("HKV", H))  # KV heads (GQA when < H)
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(B, S, HKV, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(B, S, HKV, 128, device=dev, generator=g).bfloat16()
lens = torch.full((B,), S, dtype=torch.int32, device=dev)
PAGED = int(os.environ.get("PAGED", 0))  # page size: the same caches through the paged path (identity table)
if PAGED:
    tab = torch.arange(B * (S // PAGED), device=dev, dtype=torch.int32).view(B, S // PAGED)
    kp, vp = sk.view(-1, PAGED, HKV, 128), sv.view(-1, PAGED, HKV, 128)
    call = lambda: hydra.suffix_attn_paged(q, kp, vp, tab, lens)
else:
    call = lambda: hydra.suffix_attn(q, sk, sv, lens)
N = 1024
tr = torch.zeros(16, N, dtype=torch.int64, device=dev)
hydra.set_config("suffix_impl", 2); hydra.set_config("suffix_ctas", ctas); hydra.set_config("suffix_cb", cb)
hydra.set_config("tc_debug_variant", int(os.environ.get("DEBUG", 0)))
for _ in range(2):
    call()
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
st = torch.cuda.Stream(); st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    call()
torch.cuda.current_stream().wait_stream(st)
with torch.cuda.graph(gr):
    call()
for _ in range(3):
    gr.replay()
ga, gb_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ga.record()
for _ in range(20):
    gr.replay()
gb_.record()
torch.cuda.synchronize()
gms = ga.elapsed_time(gb_) / 20
print(f"graph-replayed (no trace): {gms * 1e3:.1f} us = {2 * B * S * HKV * 256 / gms / 1e9:.0f} GB/s")
del gr
hydra.set_config("suffix_trace", tr.data_ptr())
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); call(); e1.record()
torch.cuda.synchronize()
hydra.set_config("suffix_trace", 0); hydra.set_config("tc_debug_variant", 0); hydra.set_config("suffix_impl", 0); hydra.set_config("suffix_ctas", 0); hydra.set_config("suffix_cb", 2)
ms = e0.elapsed_time(e1)
print(f"cb={cb} ctas={ctas} ms={ms:.3f} GB/s/SM={2*B*S*HKV*256/ms/1e6/ctas:.1f}")
t = tr.cpu().numpy().astype(np.float64)
nc = min(ctas, N)
ct = t[13:16, :nc]
t0 = ct[0].min()
print("CTA spans (us from the first CTA entry): entry max %.2f, setup done median %.2f max %.2f, exit min %.2f median %.2f max %.2f"
      % ((ct[0].max() - t0) / 1e3, np.median(ct[1] - t0) / 1e3, (ct[1].max() - t0) / 1e3, (ct[2].min() - t0) / 1e3,
         np.median(ct[2] - t0) / 1e3, (ct[2].max() - t0) / 1e3))
names = ["sm_wait0", "s_full", "ld", "max", "p_arrive", "epi0", "epi1", "mma_S", "mma_PV", "tma_K", "tma_V"]
lo, hi = 50, 400  # steady-state window (rounds / blocks)
def med(x): return float(np.median(x)) if len(x) else float("nan")
r = np.arange(lo, hi)
print("per round (median cycles):")
print("  round period        ", med(np.diff(t[1, lo:hi])))
print("  wait for S          ", med(t[1, r] - t[0, r]))
print("  TMEM load           ", med(t[2, r] - t[1, r]))
print("  cross-warp max      ", med(t[3, r] - t[2, r]))
print("  exp + P^T + arrive  ", med(t[4, r] - t[3, r]))
print("  S commit -> s_full seen", med(t[1, r] - t[7, r]))
print("  p_arrive -> PV commit  ", med(t[8, r] - t[4, r]))
e = np.arange(20, 150)
print("  epilogue            ", med(t[6, e] - t[5, e]), " period", med(np.diff(t[5, 20:150])))
bpr = cb
blk = np.arange(lo * bpr, hi * bpr)
blk = np.arange(lo * bpr, hi * bpr)
print("  K latency (TMA issue -> landed seen)", med(t[11, blk] - t[9, blk]), " V latency", med(t[12, blk] - t[10, blk]))
print("per block: K TMA period", med(np.diff(t[9, lo * bpr:hi * bpr])), " V TMA period", med(np.diff(t[10, lo * bpr:hi * bpr])))
# K TMA issue of the round's first block -> S commit of that round
first = np.arange(lo, hi) * bpr
print("  K TMA (first blk of round) -> S commit", med(t[7, r] - t[9, first]))
print("  V TMA (last blk of round) -> PV commit", med(t[8, r] - t[10, first + bpr - 1]))
if os.environ.get("RAW"):
    base = t[9, 100 * bpr]
    print("round: Ktma Vtma Kseen Vseen Scommit s_full_seen p_arrive PVcommit   (cb=1; cycles rel. to K TMA of round 100)")
    for rr in range(100, 116):
        b0 = rr * bpr
        print(f"{rr:4d}: " + " ".join(f"{x - base:8.0f}" for x in (t[9, b0], t[10, b0], t[11, b0], t[12, b0], t[7, rr], t[1, rr], t[4, rr], t[8, rr])))
if os.environ.get("FIRST"):
    n = int(os.environ["FIRST"])
    base = t[9, 0]
    print(f"first {n} rounds/blocks/items of CTA 0 (cycles rel. to the first K TMA):")
    print("idx:  Ktma  Vtma Kseen Vseen Scommit sm_wait0 s_full ld  max  p_arrive PVcommit ofree0 ofree1")
    for i in range(n):
        print(f"{i:3d}: " + " ".join(f"{x - base:6.0f}" for x in (t[9, i], t[10, i], t[11, i], t[12, i], t[7, i], t[0, i], t[1, i],
                                                              t[2, i], t[3, i], t[4, i], t[8, i], t[5, i], t[6, i])))
