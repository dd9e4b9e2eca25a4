"""Power draw and SM clock of each part of the C3@16K step run back to back for ~2 s (diagnostics).
    python tools/power_profile.py [k]
"""
import os, sys, json, subprocess, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2402_05099_b200 as hydra
dev = torch.device("cuda:0")
B, H, P, S = 1024, 40, int(os.environ.get("P", 16384)), 256
k = int(sys.argv[1]) if len(sys.argv) > 1 else 60
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(P, H, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(P, H, 128, device=dev, generator=g).bfloat16()
sk = torch.randn(B, S, H, 128, device=dev, generator=g).bfloat16()
sv = torch.randn(B, S, H, 128, device=dev, generator=g).bfloat16()
lens = torch.full((B,), S, dtype=torch.int32, device=dev)
ws = torch.empty(hydra.attn_workspace_bytes(q, P, S, H) * 2, dtype=torch.uint8, device=dev)
out = torch.empty(B, H, 128, dtype=torch.bfloat16, device=dev)
aux = torch.cuda.Stream(priority=-1)
def cap(fn, cfg):
    for kk, vv in cfg.items(): hydra.set_config(kk, vv)
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr): fn()
    for kk in cfg: hydra.set_config(kk, 0)
    return gr
full = lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws, aux_stream=aux)
seq = lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws)
pre = lambda: hydra.prefix_attn(q, pk, pv, workspace=ws)
suf = lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws)
cases = [("overlap k=%d" % k, cap(full, {"overlap_prefix_ctas": k})),
         ("sequential", cap(seq, {})),
         ("prefix 148 SMs", cap(pre, {})),
         ("prefix %d SMs" % k, cap(pre, {"prefix_ctas": k})),
         ("suffix SIMT 148 SMs", cap(suf, {"suffix_impl": 1})),
         ("suffix TC 148 SMs", cap(suf, {"suffix_impl": 2})),
         ("suffix TC %d SMs" % (148 - k), cap(suf, {"suffix_impl": 2, "suffix_ctas": 148 - k}))]
for name, gr in cases:
    time.sleep(3)
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "50"],
                           stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    t_end = time.time() + 2.0
    times = []
    while time.time() < t_end:
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): gr.replay()
        e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 20)
    smi.terminate()
    rows = [l.split(",") for l in smi.stdout.read().strip().splitlines() if l.strip()]
    clk = np.array([float(r[0]) for r in rows]); pw = np.array([float(r[1]) for r in rows])
    n = len(times)
    print(json.dumps(dict(case=name, ms_first=round(float(np.median(times[:3])), 4), ms_last=round(float(np.median(times[n // 2:])), 4),
                          sm_mhz=float(np.median(clk[len(clk) // 2:])), power_w=round(float(np.median(pw[len(pw) // 2:])), 1),
                          power_max=round(float(pw.max()), 1))), flush=True)
