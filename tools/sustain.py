"""Per-chunk step time over a long run (power-cap behaviour), overlap vs sequential."""
import os, sys, json, subprocess, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_05099_b200 as hydra
dev = torch.device("cuda:0")
B, H, P, S = 1024, 40, 16384, 256
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
def cap(fn):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr): fn()
    return gr
k = int(sys.argv[1]) if len(sys.argv) > 1 else 0
hydra.set_config("overlap_prefix_ctas", k)
for name, gr in (("overlap", cap(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws, aux_stream=aux))),
                 ("sequential", cap(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws)))):
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    res = []
    for chunk in range(30):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): gr.replay()
        e1.record(); torch.cuda.synchronize()
        res.append(round(e0.elapsed_time(e1) / 20, 4))
    smi.terminate(); lines = smi.stdout.read().strip().splitlines()
    print(name, res, flush=True)
    print(name, "clock/power samples:", lines[::max(1, len(lines)//10)], flush=True)
    torch.cuda.synchronize()
    import time; time.sleep(5)
