"""Time the prefix kernels (v1 one-tile, v3 persistent two-tile) at bench shapes."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_05099_b200 as hydra
dev = torch.device("cuda:0")
def run(B, H, Hkv, P, impl, ctas=0, iters=20, poly=0, variant=3):
    hydra.set_config("prefix_impl", impl); hydra.set_config("prefix_ctas", ctas); hydra.set_config("prefix_poly", poly)
    hydra.set_config("prefix_variant", variant)
    g = torch.Generator(device=dev); g.manual_seed(0)
    q = torch.randn(B, H, 128, device=dev, generator=g).bfloat16()
    pk = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    pv = torch.randn(P, Hkv, 128, device=dev, generator=g).bfloat16()
    ws = torch.empty(hydra.attn_workspace_bytes(q, P, 1, Hkv), dtype=torch.uint8, device=dev)
    fn = lambda: hydra.prefix_attn(q, pk, pv, workspace=ws)
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr): fn()
    for _ in range(3): gr.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): gr.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    fl = 4.0 * B * H * P * 128
    print(json.dumps(dict(B=B, H=H, Hkv=Hkv, P=P, impl=impl, ctas=ctas, poly=poly, variant=variant, ms=round(ms, 4), tflops=round(fl / ms / 1e9, 1))), flush=True)
mode = sys.argv[1] if len(sys.argv) > 1 else "variants"
if mode == "variants":
    for variant in (3, 4):
        run(1024, 40, 40, 16384, 3, variant=variant)
        run(512, 32, 8, 32768, 3, variant=variant)
        run(1024, 40, 40, 4096, 3, variant=variant)
elif mode == "split":
    for variant, poly in ((3, 0), (6, 0), (6, 4), (3, 0), (6, 0)):
        run(1024, 40, 40, 16384, 3, poly=poly, variant=variant)
        run(512, 32, 8, 32768, 3, poly=poly, variant=variant)
    hydra.set_config("prefix_poly", 0); hydra.set_config("prefix_variant", 3)
elif mode == "v8":
    for variant, poly in ((6, 0), (8, 0), (8, 8), (8, 4), (8, 3), (6, 4)):
        run(1024, 40, 40, 16384, 3, variant=variant, poly=poly)
        run(512, 32, 8, 32768, 3, variant=variant, poly=poly)
    hydra.set_config("prefix_poly", 0)
    hydra.set_config("prefix_variant", 6)
elif mode == "longdoc":
    for P in (19947, 39894, 79788):
        run(256, 32, 4, P, 3, variant=6, poly=4)
    run(512, 32, 8, 32768, 3, variant=6, poly=4)
    run(256, 32, 8, 32768, 3, variant=6, poly=4)
    run(1024, 5, 5, 16384, 3, variant=6, poly=4)
    run(1024, 40, 40, 16384, 3, variant=6, poly=4)
elif mode == "spec":
    for variant, poly in ((3, 0), (5, 0), (5, 8), (5, 4), (3, 4)):
        run(1024, 40, 40, 16384, 3, poly=poly, variant=variant)
        run(512, 32, 8, 32768, 3, poly=poly, variant=variant)
    hydra.set_config("prefix_poly", 0)
elif mode == "poly":
    for poly in (0, 8, 4, 3, -1):  # -1: timing experiment, no exp at all
        run(1024, 40, 40, 16384, 3, poly=poly)
        run(512, 32, 8, 32768, 3, poly=poly)
    hydra.set_config("prefix_poly", 0)
elif mode == "debug":
    hydra.set_config("tc_debug_variant", 2)
    print("debug: softmax math skipped (timing only)")
    run(1024, 40, 40, 16384, 3, variant=3)
    run(512, 32, 8, 32768, 3, variant=3)
    hydra.set_config("tc_debug_variant", 0)
elif mode == "feed":
    for dbg, poly in ((4, 0), (6, 0), (4, -1)):
        hydra.set_config("tc_debug_variant", dbg)
        print(f"debug={dbg} poly={poly} (timing only: 4 = no K/V TMA after the fill, 2 = no softmax math)")
        run(1024, 40, 40, 16384, 3, poly=poly)
        run(512, 32, 8, 32768, 3, poly=poly)
    hydra.set_config("tc_debug_variant", 0); hydra.set_config("prefix_poly", 0)
