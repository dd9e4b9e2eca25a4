"""Per-CTA globaltimer timeline of the persistent prefix kernel: start skew, setup, first S,
compute end, exit -- where the fixed per-call overhead goes (diagnostics).
    python tools/prefix_cta_timeline.py [B H Hkv P]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2402_05099_b200 as hydra
B, H, Hkv, P = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (256, 32, 4, 19947)
dev = torch.device("cuda:0")
N = 1024
tr = torch.zeros(16 * N, dtype=torch.int64, device=dev)
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
ws = torch.empty(hydra.attn_workspace_bytes(q, P, 1, Hkv), dtype=torch.uint8, device=dev)
hydra.set_config("prefix_impl", 3)
for _ in range(3):
    hydra.prefix_attn(q, pk, pv, workspace=ws)
torch.cuda.synchronize()
hydra.set_config("prefix_trace", tr.data_ptr())
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); hydra.prefix_attn(q, pk, pv, workspace=ws); e1.record()
torch.cuda.synchronize()
hydra.set_config("prefix_trace", 0); hydra.set_config("prefix_impl", 0)
T8 = tr.view(16, N).cpu().numpy()[14:].reshape(-1)[:256 * 8].reshape(256, 8).astype(np.float64)
T8 = T8[T8[:, 0] > 0]
t0 = T8[:, 0].min()
T = (T8[:, :5] - t0) / 1e3  # us
print(f"call (events) {e0.elapsed_time(e1) * 1e3:.1f} us; CTAs {len(T)}")
for name, col in (("entry", 0), ("setup done", 1), ("first S", 2), ("compute done", 3), ("exit", 4)):
    c = T[:, col]
    print(f"  {name:13s} min {c.min():7.1f}  median {np.median(c):7.1f}  max {c.max():7.1f} us")
act = T[:, 3] - T[:, 2]
o = np.argsort(T[:, 3])
print("  compute done, sorted (CTA: us):", " ".join(f"{int(i)}:{T[i, 3]:.0f}" for i in o[::max(1, len(o) // 24)]))
two = T8[:, 7] > 0
if two.any():
    X = (T8[two] - t0) / 1e3
    print(f"  CTAs with a 2nd item: {int(two.sum())}; last P(1st) -> epilogue done {np.median(X[:, 6] - X[:, 5]):.1f} us, "
          f"epilogue done -> first S(2nd) {np.median(X[:, 7] - X[:, 6]):.1f} us (median)")
print("  slowest 8:", " ".join(f"{int(i)}:{T[i, 3]:.0f}" for i in o[-8:]))
print(f"  first S -> compute done: min {act.min():.1f} median {np.median(act):.1f} max {act.max():.1f} us")
