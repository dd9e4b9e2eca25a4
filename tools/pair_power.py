"""Sustained power / clock / time of the CTA-pair prefix kernel at C3@16K with parts switched off
(testing build timing experiments: tc_debug_variant 4 = no K/V TMA after the ring fill, 2 = no
softmax math).  HYDRA_TESTING=1 python tools/pair_power.py"""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2402_05099_b200 as hydra

dev = torch.device("cuda:0")
B, H, P = 1024, 40, 16384
g = torch.Generator(device=dev)
g.manual_seed(0)
q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
pk = torch.randn(P, H, 128, device=dev, generator=g).bfloat16()
pv = torch.randn(P, H, 128, device=dev, generator=g).bfloat16()
ws = torch.empty(hydra.attn_workspace_bytes(q, P, 1, H) * 2, dtype=torch.uint8, device=dev)


def cap(dbg):
    if dbg:
        hydra.set_config("tc_debug_variant", dbg)
    fn = lambda: hydra.prefix_attn(q, pk, pv, workspace=ws)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    if dbg:
        hydra.set_config("tc_debug_variant", 0)
    return gr


cases = [("prefix", 0, 0), ("no K/V TMA", 4, 0), ("no softmax", 2, 0), ("prefix again", 0, 0)]
if os.environ.get("CLUSTERS"):
    cases = [(f"cluster {c}", 0, int(c)) for c in os.environ["CLUSTERS"].split(",")]
for name, dbg, clu in cases:
    hydra.set_config("pair_cluster", clu)
    gr = cap(dbg)
    time.sleep(2)
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    t_end = time.time() + 2.0
    times = []
    while time.time() < t_end:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 20)
    smi.terminate()
    rows = [l.split(",") for l in smi.stdout.read().strip().splitlines() if l.strip()]
    clk = np.array([float(r[0]) for r in rows])
    pw = np.array([float(r[1]) for r in rows])
    n = len(times)
    print(json.dumps(dict(case=name, ms_first=round(float(np.median(times[:3])), 4),
                          ms_sustained=round(float(np.median(times[n // 2:])), 4),
                          sm_mhz=float(np.median(clk[len(clk) // 2:])), power_w=round(float(np.median(pw[len(pw) // 2:])), 1))),
          flush=True)
