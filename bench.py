#!/usr/bin/env python
"""bench.py -- decode-attention queries/s for shared-prefix attention (Hydragen) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3_16k] [--impl hydra|reference]

One "step" = the whole hot path for one decode step of one attention layer over the
configured batch: batched prefix attention (tcgen05) + per-sequence suffix attention +
LSE combine, i.e. App. B `hydragen_attention`.  The unit is one
decode query = one sequence's new token across all query heads.

Default workload: BASELINE.json configs[2] at its headline point -- CodeLlama-13b head
shape (40 q / 40 kv heads, d = 128), batch 1024, shared prefix 16384 tokens, suffix 256
tokens, bf16 K/V/Q with fp32 accumulation.  For N > 1 (torchrun) the KV heads are sharded
across ranks (40/N each, no collective): the batch and total work are fixed -> strong
scaling; value = B / max-over-ranks step time.

Inputs come from the seeded generator (`synth`, 'mixed' needle distribution), are
resident in HBM for `value`, and total 5.7 GB per step (> 126 MB L2), so no L2 flush is
needed between steps (stated in config.l2).  Timing: CUDA graph of one step, W warm-up
replays, K timed replays between CUDA events after a barrier + synchronize.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c3_16k": dict(B=1024, Hq=40, Hkv=40, d=128, P=16384, S=256,
                   name="CodeLlama-13b attention shape (40 q / 40 kv heads, d=128), B=1024, prefix 16384, suffix 256"),
    "c3_1k": dict(B=1024, Hq=40, Hkv=40, d=128, P=1024, S=256,
                  name="CodeLlama-13b attention shape (40 q / 40 kv heads, d=128), B=1024, prefix 1024, suffix 256"),
    "c2": dict(B=256, Hq=32, Hkv=32, d=128, P=2048, S=128,
               name="CodeLlama-7b attention shape (32 q / 32 kv heads, d=128), B=256, prefix 2048, suffix 128"),
    "c4_1gpu": dict(B=512, Hq=32, Hkv=8, d=128, P=32768, S=128,
                    name="Llama-3-8B GQA attention shape (32 q / 8 kv, d=128), B=512, prefix 32768, suffix 128"),
    # prefix sequence split across ranks + NCCL all-gather of (O fp16, LSE) (dist.seqsplit_attention)
    "c4": dict(B=512, Hq=32, Hkv=8, d=128, P=32768, S=128, kind="seqsplit",
               name="Llama-3-8B GQA attention shape (32 q / 8 kv, d=128), B=512, prefix 32768 split along the "
                    "sequence across ranks with one NCCL all-to-all of packed (O fp16, LSE) rows, suffix 128"),
    # the paper's long-document shape (P:198, 19,947-token document,
    # Yi-6B-200k-like heads 32 q / 4 kv); suffix length assumed 128 (the paper gives none)
    "c6_longdoc": dict(B=256, Hq=32, Hkv=4, d=128, P=19947, S=128,
                       name="long-document shape (Yi-6B-like 32 q / 4 kv heads, d=128), B=256, prefix 19947, "
                            "suffix 128 (assumed)"),
    # SURVEY §8(f) NEXT-2 on N GPUs: the long document's prefix split along the sequence (4 KV
    # heads cap head sharding at 4 GPUs); B sweep with --batch-sweep 64,256,1024
    "c6_seqsplit": dict(B=256, Hq=32, Hkv=4, d=128, P=19947, S=128, kind="seqsplit",
                        name="long-document shape (Yi-6B-like 32 q / 4 kv heads, d=128), B=256, prefix 19947 split "
                             "along the sequence across ranks with one NCCL all-to-all of packed (O fp16, LSE) rows, "
                             "suffix 128 (assumed)"),
    # the paper's attention microbenchmark grid (§4.2, App. D.2
    # P:547): 8 q / 1 kv heads, d=128; Hydragen vs per-sequence attention over each sequence's
    # own copy of prefix || suffix (paper_2402_05099_b200.baseline); one JSON line per point
    "grid": dict(B=1024, Hq=8, Hkv=1, d=128, P=16384, S=256, kind="grid",
                 batches=(32, 128, 512, 1024), prefixes=(1024, 4096, 16384), suffixes=(64, 256),
                 name="attention microbenchmark grid (paper §4.2): 8 q / 1 kv heads, d=128"),
    # two-level sharing tree (tree_attention)
    "c5": dict(B=1024, Hq=32, Hkv=32, d=128, P=4096, S=512, kind="tree", branches=16, branch_len=1024,
               name="tree sharing: 4096-token root -> 16 branches x 1024 tokens -> 64 sequences each with 512-token "
                    "suffixes, CodeLlama-7b attention shape (32 MHA heads, d=128)"),
}


# DRAM bytes (read + write) per launch from one `ncu --set full` capture of the kernel at this
# config (profiles/r1b_ncu_full_*.csv: dram__bytes_read.sum + dram__bytes_write.sum)
NCU_TRAFFIC = {
    ("c3_16k", "decode_attn_kernel"): 5379746000 + 6668800,    # profiles/r1o_suffix_decode_raw.csv
    ("c3_16k", "suffix_tc_kernel"): 5379274000 + 25441024,     # profiles/r1o_suffix_tc_76_raw.csv (76 CTAs, k = 72)
    ("c3_16k", "prefix_tc2_kernel"): 355092736 + 21645312,     # profiles/r1o_prefix_tc2_raw.csv (variant 6, poly 4)
    ("c3_16k", "prefix_pair_kernel"): 349904640 + 21081600,    # profiles/r2u_pair_c3_raw.csv (variant 9, pair_poly 0)
    ("c6_longdoc", "suffix_short_kernel"): 69250560 + 1515264,  # profiles/r2u_suffix_short_c6_raw.csv
    ("c4_1gpu", "suffix_short_kernel"): 272669952 + 13087232,   # profiles/r2u_suffix_short_c4_raw.csv
    ("c4_1gpu", "prefix_pair_kernel"): 138497792 + 8392704,     # profiles/r3_pair_c4_raw.csv
    ("c6_longdoc", "prefix_pair_kernel"): 43016448 + 1049600,   # profiles/r3_pair_c6_raw.csv
    ("c3_16k", "suffix_tc_kernel@84"): 5379332000 + 26637568,  # profiles/r2_suffix_tc_84_raw.csv (84 CTAs, k = 64)
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3_16k", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="hydra", choices=["hydra", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="target CPU time of the oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--paged-page-size", type=int, default=16,
                    help="also time the step with the suffix in a paged cache of this page size (0 = skip)")
    ap.add_argument("--batch-sweep", default="",
                    help="comma-separated batch sizes: one JSON line per B (seqsplit and flat configs)")
    ap.add_argument("--overlap-k", type=int, default=0,
                    help="force the SM split of the overlapped step (prefix CTAs; 0 = the library's planner)")
    ap.add_argument("--exchange", default="alltoall", choices=["alltoall", "allgather", "p2p"],
                    help="sequence-split exchange (seqsplit configs)")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """SM clock, power and throttle reasons sampled during the timed region: NVML every 5 ms from
    a thread (enough samples inside a 20-ms loop), else nvidia-smi every 50 ms."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    PERIOD_S = 0.005

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.nvml = None
        self.stop = threading.Event()
        self.t = None

    def _nvml_loop(self):
        nv, h = self.nvml
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.lines.append(", ".join([str(sm), str(mx), "%.2f" % pw] +
                                            ["Active" if r & bb else "Not Active" for bb in bits]))
            except Exception:
                pass
            self.stop.wait(self.PERIOD_S)

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nvml = (nv, nv.nvmlDeviceGetHandleByIndex(self.index))
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes ~0.1-0.5 s to print its first sample: wait for it, so a short timed
            # region is sampled at the 50 ms period instead of falling into the start-up gap
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.t.join(1.0)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, busy_floor=0.0):
        sm, pw, mx, reasons = [], [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in list(self.lines):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            try:
                pw.append(float(parts[2]))
            except ValueError:
                pass
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None,
                "source": "nvml (5 ms)" if self.nvml else "nvidia-smi (50 ms)"}


L2_BYTES = 126 * 1024 * 1024  # B200 L2

# Test-only: HYDRA_BENCH_SHARED_GPU=1 lets N ranks share the visible GPU(s) (rank -> device
# LOCAL_RANK % count) over a gloo process group, so the N-rank code path (self-launch, head
# shard / sequence split, barriers, max over ranks, the JSON line) runs on a 1-GPU box
# (tests/test_gpu_bench_multirank.py).  Head-shard ranks never wait on one another's kernels;
# the line is marked and its numbers are not measurements.
SHARED_GPU = os.environ.get("HYDRA_BENCH_SHARED_GPU") == "1"


def rank_device(torch):
    """(world, rank, local device index) of this process; sets the current CUDA device."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARED_GPU:
        local %= max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    return world, rank, local


def mark_shared(line):
    if SHARED_GPU and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        line["shared_gpu_test"] = ("ranks share one GPU over gloo (HYDRA_BENCH_SHARED_GPU=1): a test of the "
                                   "N-rank code path, not a measurement")
    return line


class L2Flush:
    """Evicts the step's inputs from L2 between timed steps: writes a 2 x L2 buffer, then reads
    another 2 x L2 buffer.  The read matters: after a write-only flush L2 holds ~126 MB of DIRTY
    lines, and the timed step that follows pays their write-back to HBM (measured: a fixed
    ~15-19 us on every short step, e.g. the C6 suffix, tools/suffix_shapes_ab.py); after the
    read L2 holds clean, unrelated lines only."""

    DESC = "L2 flushed before every timed step (2 x 126 MB written, then another 2 x 126 MB read: no dirty line left)"

    def __init__(self, torch, dev, nbytes=None):
        n = nbytes or 2 * L2_BYTES
        self.w = torch.empty(n, dtype=torch.uint8, device=dev)
        self.r = torch.zeros(n, dtype=torch.uint8, device=dev)

    def __call__(self):
        self.w.zero_()
        self.r.sum()


def l2_flush_buffer(torch, dev, input_bytes):
    """An L2Flush to run between timed steps when the step's inputs would otherwise stay
    L2-resident (e.g. a rank's shard at 8 GPUs); None when inputs > 2x L2."""
    if input_bytes >= 2 * L2_BYTES:
        return None
    return L2Flush(torch, dev)


# per-step statistics of the last timed_steps call (the median next to the mean it returns)
LAST_TIMING = {}


def timed_steps(torch, run, k, flush):
    """(Python's garbage collector is paused for the loop: a collection while the host enqueues a
    short step's replays showed up as a 1.8 ms gap in one step of a C2 run.)"""
    import gc

    gc_on = gc.isenabled()
    gc.disable()
    try:
        return _timed_steps(torch, run, k, flush)
    finally:
        if gc_on:
            gc.enable()


def _timed_steps(torch, run, k, flush):
    """Device time of k steps (ms per step, the mean).  Without `flush`: k back-to-back steps
    between the first and the last of k+1 events (an event before every step also gives each
    step's own time: median / min / max in LAST_TIMING).  With `flush` (an L2Flush): L2 is
    flushed before every step and only the steps themselves are timed (one event pair
    per step, summed)."""
    if flush is None:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
        evs[0].record()
        for i in range(k):
            run()
            evs[i + 1].record()
        torch.cuda.synchronize()
        per = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(k))
        LAST_TIMING.update(median_ms=per[k // 2], min_ms=per[0], max_ms=per[-1], n=k, flushed=False)
        return evs[0].elapsed_time(evs[-1]) / k
    evs = []
    for _ in range(k):
        flush()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        c.record()
        evs.append((a, c))
    torch.cuda.synchronize()
    per = sorted(a.elapsed_time(c) for a, c in evs)
    LAST_TIMING.update(median_ms=per[k // 2], min_ms=per[0], max_ms=per[-1], n=k, flushed=True)
    return sum(per) / k


def make_timer(torch, dist, dev, world, flush=None):
    """CUDA-graph capture and device timing (CUDA events, barrier, max over ranks)."""

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            fn()  # eager warm-up outside capture
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize(dev)
        return g

    def time_fn(run, k, w):
        for _ in range(w):
            run()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ms = timed_steps(torch, run, k, flush)
        if world > 1:
            dist.barrier()
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    return capture, time_fn


def base_line(args, cfg, world, ms, B, dtype="bf16"):
    return {
        "metric": "decode-attn queries/s and % of bf16 TC peak; prefix 16K, batch 1024, 1/2/4/8 GPU",
        "value": round(B / (ms * 1e-3), 1), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (seeded PCG64 N(0,1) K/V rounded to bf16, 'mixed' needle queries)",
    }


def run_tree(args, cfg):
    """C5: two-level sharing tree through hydra.tree_attention (one GPU; replicas for N > 1)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2402_05099_b200 as hydra

    world, rank, local = rank_device(torch)
    dev = torch.device("cuda", local)
    if world > 1:
        init_dist(torch, dist, dev, world, rank)
    B, Hq, Hkv, d, S = cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["d"], cfg["S"]
    nbr, blen = cfg["branches"], cfg["branch_len"]
    if Hkv % world:
        raise SystemExit("Hkv not divisible by world")
    Hq_r, Hkv_r = Hq // world, Hkv // world
    parent, node_len, leaf = synth.two_level_tree(cfg["P"], nbr, blen, B // nbr)
    tp = synth.make_tree_problem(parent, node_len, leaf, Hq_r, Hkv_r, d, S, dtype="bf16", dist="mixed",
                                 seed=args.seed + rank)
    t = lambda a: torch.from_numpy(a).view(torch.bfloat16).to(dev)
    q, nk, nv, sk, sv = t(tp.q), t(tp.node_k), t(tp.node_v), t(tp.sk), t(tp.sv)
    lens = torch.from_numpy(tp.lens.astype(np.int32)).to(dev)
    tree = hydra.Tree(tp.parent, tp.node_off, tp.node_len, tp.leaf_of_seq, heads=(Hq_r, Hkv_r))
    capture, time_fn = make_timer(torch, dist, dev, world)
    aux = torch.cuda.Stream(priority=-1)
    # node attention on k SMs || tensor-core suffix on the rest (aux stream), or sequential:
    # whichever is faster on a short probe
    g_over = capture(lambda: hydra.tree_attention(q, tree, nk, nv, sk, sv, lens, aux_stream=aux))
    k_over = int(hydra.get_config("last_overlap_k"))
    g_seq = capture(lambda: hydra.tree_attention(q, tree, nk, nv, sk, sv, lens))
    probe = max(3, min(20, args.steps // 5))
    ms_over, ms_seq = time_fn(g_over.replay, probe, 2), time_fn(g_seq.replay, probe, 2)
    g = g_over if ms_over <= ms_seq else g_seq
    with ClockSampler(local) as clk:
        ms = time_fn(g.replay, args.steps, args.warmup)
    g_suf = capture(lambda: hydra.suffix_attn(q, sk, sv, lens))
    ms_suf = time_fn(g_suf.replay, max(5, args.steps // 4), 3)
    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    suffix_bytes = 2 * int(tp.lens.sum()) * Hkv_r * d * 2 + B * Hq_r * d * 2
    # every node's K/V attended by the stacked queries of its group (§3.3): 4 d per (row, token)
    flops = 4.0 * Hq_r * d * sum(int(node_len[n]) * tree.group_size(n) for n in range(len(node_len)))
    line = base_line(args, cfg, world, ms, B)
    line["config"] = {"workload": args.config, "description": cfg["name"], "B": B, "Hq": Hq, "Hkv": Hkv, "d": d,
                      "root_len": cfg["P"], "branches": nbr, "branch_len": blen, "suffix_len": S,
                      "parallelism": f"kv-head shard x{world}" if world > 1 else "1 GPU",
                      "l2": "no flush: %.2f GB of inputs per step > 126 MB L2" % (suffix_bytes / 1e9)}
    line["roofline"] = {"bound": "hbm", "kernel": "suffix split-K GEMV (decode_attn_kernel)",
                        "achieved": round(suffix_bytes / (ms_suf * 1e-3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(suffix_bytes / (ms_suf * 1e-3) / 1e9 / hbm, 4), "traffic": None,
                        "algorithmic_bytes_per_launch": suffix_bytes, "launch_ms": round(ms_suf, 5)}
    line["tree_prefix_flops_per_step"] = flops
    line["schedule"] = {"overlap": bool(ms_over <= ms_seq), "prefix_ctas": k_over, "ms_overlap_probe": round(ms_over, 5),
                        "ms_sequential_probe": round(ms_seq, 5)}
    line["clocks"] = clk.summary()
    line["gpu_launches"] = args.steps * 4
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        n = 2
        bb, hh = np.meshgrid(np.arange(n), np.arange(Hq_r), indexing="ij")
        t0 = time.time()
        oracle.tree_attention(tp, rows=np.stack([bb.ravel(), hh.ravel()], 1))
        dt = time.time() - t0
        n2 = int(max(1, min(B, n * args.cpu_seconds / max(dt, 1e-3))))
        bb, hh = np.meshgrid(np.arange(n2), np.arange(Hq_r), indexing="ij")
        t0 = time.time()
        oracle.tree_attention(tp, rows=np.stack([bb.ravel(), hh.ravel()], 1))
        dt2 = time.time() - t0
        line["cpu_baseline"] = {"value": round(n2 / dt2, 3), "unit": "queries/s", "cores": oracle.max_threads(),
                                "kind": "oracle", "sample": f"first {n2} of {B} sequences x all heads, {dt2:.1f} s"}
    if not args.no_e2e:
        pinned = [x.pin_memory() for x in (torch.from_numpy(tp.q).view(torch.bfloat16),
                                             torch.from_numpy(tp.sk).view(torch.bfloat16),
                                             torch.from_numpy(tp.sv).view(torch.bfloat16))]
        h2d = sum(x.numel() * x.element_size() for x in pinned)
        hout = torch.empty(B, Hq_r, d, dtype=torch.bfloat16).pin_memory()

        def one():
            for src, dst in zip(pinned, (q, sk, sv)):
                dst.copy_(src, non_blocking=True)
            hout.copy_(hydra.tree_attention(q, tree, nk, nv, sk, sv, lens), non_blocking=True)

        ms_e = time_fn(one, args.e2e_steps, 1)
        line["e2e"] = {"value": round(B / (ms_e * 1e-3), 1), "unit": "queries/s", "h2d_bytes_per_step": int(h2d),
                       "d2h_bytes_per_step": int(hout.numel() * 2), "ms_per_step": round(ms_e, 3),
                       "note": "tree node K/V stay resident (shared across steps); q and suffix K/V copied per step"}
    if rank == 0:
        print(json.dumps(mark_shared(line)), flush=True)
    if world > 1:
        dist.barrier()


def init_dist(torch, dist, dev, world, rank):
    """NCCL process group for N ranks (torchrun env), or a 1-rank group for N = 1."""
    if dist.is_initialized():
        return
    if world > 1:
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    else:
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        dist.init_process_group("nccl", device_id=dev, init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)


def run_seqsplit(args, cfg):
    """C4 / C6 on N ranks: prefix split along the sequence, one packed all-to-all + Eq. 5 merge
    (dist.SeqSplit), suffix of each rank's batch shard on a side stream during the exchange."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2402_05099_b200 as hydra
    from paper_2402_05099_b200 import dist as hdist

    world, rank, local = rank_device(torch)
    dev = torch.device("cuda", local)
    init_dist(torch, dist, dev, world, rank)
    B, Hq, Hkv, d, P, S = cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["d"], cfg["P"], cfg["S"]
    p0, p1 = hdist.shard_range(P, world, rank)
    b0, b1 = hdist.batch_shard(B, world, rank)
    # every rank draws the same q; its own prefix shard and batch-shard suffixes (seeded per rank)
    pq = synth.make_problem(B, Hq, Hkv, d, 0, 0, dtype="bf16", seed=args.seed)
    pr = synth.make_problem(max(1, b1 - b0), Hq, Hkv, d, p1 - p0, S, dtype="bf16", seed=args.seed + 1 + rank)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).to(dev)
    q, pk, pv, sk, sv = t(pq.q), t(pr.pk), t(pr.pv), t(pr.sk)[:b1 - b0], t(pr.sv)[:b1 - b0]
    lens = torch.from_numpy(pr.lens.astype(np.int32)).to(dev)[:b1 - b0]
    in_bytes = sum(x.numel() * x.element_size() for x in (q, pk, pv, sk, sv))
    flush = l2_flush_buffer(torch, dev, in_bytes)  # a rank's shard fits in L2 at 8 GPUs
    capture, time_fn = make_timer(torch, dist, dev, world, flush=flush)
    plan = hdist.SeqSplit(B, Hq, d, device=dev, exchange=args.exchange)
    fn = lambda: plan(q, pk, pv, sk, sv, lens)
    try:
        g = capture(fn)
        run, graphed = g.replay, True
    except Exception:  # NCCL capture unsupported here: time eagerly
        run, graphed = fn, False
    with ClockSampler(local) as clk:
        ms = time_fn(run, args.steps, args.warmup)
    # the phases alone (same buffers, CUDA graphs where possible): prefix, suffix, exchange
    kk = max(5, args.steps // 4)
    ms_pre = time_fn(capture(lambda: hydra.prefix_attn(q, pk, pv, out=plan.o_p, lse_out=plan.l_p)).replay, kk, 3)
    ms_suf = (time_fn(capture(lambda: hydra.suffix_attn(q[b0:b1], sk, sv, lens, out=plan.o_s[0].view(b1 - b0, Hq, d),
                                                         lse_out=plan.l_s[0].view(b1 - b0, Hq))).replay, kk, 3)
              if b1 > b0 else 0.0)
    try:
        ms_ex = time_fn(capture(plan._collective).replay, kk, 3)
    except Exception:
        ms_ex = time_fn(plan._collective, kk, 3)
    pk_ = peaks()
    flops = 4.0 * B * Hq * (p1 - p0) * d
    tc = float(pk_.get("bf16_tflops", 1590.0))
    line = base_line(args, cfg, world, ms, B)
    line["config"] = {"workload": args.config, "description": cfg["name"], "B": B, "Hq": Hq, "Hkv": Hkv, "d": d,
                      "prefix_len": P, "suffix_len": S, "parallelism": f"prefix sequence split x{world}",
                      "prefix_tokens_per_rank": p1 - p0, "batch_shard": [b0, b1],
                      "exchange": f"one NCCL {args.exchange} of packed rows [O fp16 | LSE f32 | pad] "
                                  f"({plan.row_bytes} B per row), merged with the suffix part in one combine",
                      "exchange_bytes_sent_per_rank": plan.exchange_bytes(), "cuda_graph": graphed,
                      "l2": ("no flush: %.2f GB of inputs per rank > 2 x 126 MB L2" % (in_bytes / 1e9)) if flush is None
                      else L2Flush.DESC + ": %.3f GB of inputs per rank" % (in_bytes / 1e9)}
    line["roofline"] = {"bound": "tensor", "kernel": prefix_kernel_name(hydra, Hq // Hkv) + ", this rank's prefix shard",
                        "achieved": round(flops / (ms_pre * 1e-3) / 1e12, 1), "peak": tc, "unit": "TFLOP/s",
                        "frac": round(flops / (ms_pre * 1e-3) / 1e12 / tc, 4), "traffic": None,
                        "algorithmic_flops_per_launch": flops, "launch_ms": round(ms_pre, 5)}
    line["phases_alone_ms"] = {"prefix": round(ms_pre, 5), "suffix": round(ms_suf, 5), "exchange": round(ms_ex, 5),
                               "sum": round(ms_pre + ms_suf + ms_ex, 5), "step": round(ms, 5),
                               "note": "each phase timed alone (max over ranks); the step overlaps the suffix "
                                       "with the exchange on a side stream"}
    line["clocks"] = clk.summary()
    line["gpu_launches"] = args.steps * 5  # prefix (+ -inf fill), pack, suffix, merge; + NCCL's own kernel
    if rank == 0:
        print(json.dumps(mark_shared(line)), flush=True)
    dist.barrier()
    hdist.release_plans()
    del plan


def run_grid(args, cfg):
    """NEXT-1: speedup of Hydragen attention over per-sequence attention on the paper's
    microbenchmark shape, App. D.2 protocol: CUDA graph per call, the L2 flushed (L2Flush: a
    2 x L2 write, then a 2 x L2 read) before every timed replay, mean and median over the timed replays."""
    import numpy as np
    import torch

    import synth
    import paper_2402_05099_b200 as hydra
    from paper_2402_05099_b200 import baseline

    if int(os.environ.get("RANK", "0")) != 0:
        return  # one GPU's microbenchmark: other ranks idle
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    Hq, Hkv, d = cfg["Hq"], cfg["Hkv"], cfg["d"]
    flush = L2Flush(torch, dev)
    iters, warm = max(5, args.steps), max(3, args.warmup)

    def graph_times(fn):
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        for _ in range(warm):
            g.replay()
        evs = []
        for _ in range(iters):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize(dev)
        t = [a.elapsed_time(b) for a, b in evs]
        return statistics.mean(t), statistics.median(t)

    best = None
    for P in cfg["prefixes"]:
        for S in cfg["suffixes"]:
            for B in cfg["batches"]:
                pb = synth.make_problem(B, Hq, Hkv, d, P, S, dtype="bf16", dist="mixed", seed=args.seed)
                t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).to(dev)
                q, pk, pv, sk, sv = t(pb.q), t(pb.pk), t(pb.pv), t(pb.sk), t(pb.sv)
                lens = torch.from_numpy(pb.lens.astype(np.int32)).to(dev)
                ws = torch.empty(hydra.attn_workspace_bytes(q, P, S, Hkv), dtype=torch.uint8, device=dev)
                out = torch.empty(B, Hq, d, dtype=torch.bfloat16, device=dev)
                h_mean, h_med = graph_times(lambda: hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out,
                                                                             workspace=ws))
                fk, fv, flens = baseline.per_sequence_cache(pk, pv, sk, sv, lens)
                o_b = torch.empty(B, Hq, d, dtype=torch.float32, device=dev)
                l_b = torch.empty(B, Hq, dtype=torch.float32, device=dev)
                h = hydra._lib.Heads(Hq, Hkv, d, 0.0, hydra._lib.HYDRA_BF16)
                import ctypes

                wsb = torch.empty(max(1, hydra.load().hydra_workspace_size(hydra._lib.HYDRA_OP_SUFFIX, ctypes.byref(h), B,
                                                                           0, P + S, 0)), dtype=torch.uint8, device=dev)
                b_mean, b_med = graph_times(lambda: baseline.per_sequence_attention(q, fk, fv, flens, workspace=wsb,
                                                                                    out=o_b, lse_out=l_b))
                line = {"metric": "Hydragen attention speedup over per-sequence attention (paper §4.2 microbenchmark)",
                        "value": round(b_mean / h_mean, 3), "unit": "x", "higher_is_better": True, "n_gpus": 1,
                        "steps": iters, "warmup": warm, "dtype": "bf16",
                        "data": "synthetic (seeded PCG64 N(0,1) K/V rounded to bf16, 'mixed' needle queries)",
                        "config": {"workload": "grid", "B": B, "Hq": Hq, "Hkv": Hkv, "d": d, "prefix_len": P,
                                   "suffix_len": S, "l2": L2Flush.DESC},
                        "hydragen_ms": {"mean": round(h_mean, 5), "median": round(h_med, 5)},
                        "per_sequence_ms": {"mean": round(b_mean, 5), "median": round(b_med, 5)},
                        "speedup_median": round(b_med / h_med, 3),
                        "baseline": "each sequence attends over its own copy of prefix || suffix with this library's "
                                    "per-sequence kernels (paper_2402_05099_b200.baseline; P:160)",
                        "timing": "App. D.2 (P:547): CUDA graph per call, L2 flushed before every replay, "
                                  f"{warm} warm-up and {iters} timed replays, mean and median"}
                print(json.dumps(mark_shared(line)), flush=True)
                if best is None or line["value"] > best["value"]:
                    best = line
                del fk, fv, q, pk, pv, sk, sv, ws, wsb, o_b, l_b, out
                torch.cuda.empty_cache()
    print(json.dumps({"metric": "max Hydragen attention speedup over per-sequence attention (paper §4.2; paper: "
                                ">16x on A100, P:27)", "value": best["value"], "unit": "x",
                      "at": best["config"]}), flush=True)


def self_launch(args):
    """`bench.py --gpus N` without a torchrun environment: start N ranks with torchrun on this node
    (one per GPU) and pass their output through; fail loudly when fewer GPUs are visible."""
    import socket

    import torch

    n = torch.cuda.device_count()
    if n < args.gpus and not (SHARED_GPU and n >= 1):
        print(json.dumps({"error": f"--gpus {args.gpus} requested but {n} CUDA device(s) visible"}), flush=True)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE={world}")
    cfg = dict(CONFIGS[args.config])
    batches = [int(x) for x in args.batch_sweep.split(",") if x.strip()] or [cfg["B"]]
    kind = cfg.get("kind")
    for B in batches:
        c = dict(cfg, B=B)
        if B != cfg["B"]:
            c["name"] = cfg["name"].replace("B=%d" % cfg["B"], "B=%d" % B)
        if kind == "grid":
            run_grid(args, c)
            break
        if kind == "tree":
            run_tree(args, c)
        elif kind == "seqsplit":
            run_seqsplit(args, c)
        else:
            run_flat(args, c)
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()


def run_flat(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2402_05099_b200 as hydra

    world, rank, local = rank_device(torch)
    dev = torch.device("cuda", local)
    if world > 1:
        init_dist(torch, dist, dev, world, rank)

    B, Hq, Hkv, d, P, S = cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["d"], cfg["P"], cfg["S"]
    if Hkv % world:
        raise SystemExit(f"Hkv={Hkv} is not divisible by {world} GPUs (head sharding)")
    Hq_r, Hkv_r = Hq // world, Hkv // world

    t_gen = time.time()
    pb = synth.make_problem(B, Hq_r, Hkv_r, d, P, S, dtype="bf16", dist="mixed", seed=args.seed + rank)
    t_gen = time.time() - t_gen

    def host(a):
        return torch.from_numpy(a).view(torch.bfloat16)

    hq, hpk, hpv, hsk, hsv = (host(pb.q), host(pb.pk), host(pb.pv), host(pb.sk), host(pb.sv))
    hlens = torch.from_numpy(pb.lens.astype(np.int32))
    q, pk, pv, sk, sv = (t.to(dev) for t in (hq, hpk, hpv, hsk, hsv))
    lens = hlens.to(dev)
    ws = torch.empty(hydra.attn_workspace_bytes(q, P, S, Hkv_r), dtype=torch.uint8, device=dev)
    out = torch.empty(B, Hq_r, d, dtype=torch.bfloat16, device=dev)
    aux = torch.cuda.Stream(device=dev, priority=-1)
    in_bytes = sum(x.numel() * x.element_size() for x in (q, pk, pv, sk, sv))
    flush = l2_flush_buffer(torch, dev, in_bytes)  # only when this rank's inputs fit in 2x L2

    def step(overlap: bool):
        hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws, aux_stream=aux if overlap else None)

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            fn()  # eager warm-up outside capture
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize(dev)
        return g

    def time_graph(g, k, w):
        for _ in range(w):
            g.replay()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ms = timed_steps(torch, g.replay, k, flush)
        if world > 1:
            dist.barrier()
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # Prefix phase (north_star: >= 60% of bf16 tensor peak), measured before the step loop:
    # burst = 20 replays on a cool GPU (against the burst cuBLAS figure); sustained = replays
    # back to back for ~1 s (against the sustained cuBLAS figure, itself a seconds-long loop
    # under the 1 kW power cap).
    g_pre = capture(lambda: hydra.prefix_attn(q, pk, pv, workspace=ws))
    ms_pre_burst = time_graph(g_pre, 20, 3)
    # the prefix KERNEL alone (prefix_attn also merges the kernel's stream-K pieces with a combine
    # launch): the persistent kernel's own span (config key step_timer), 20 graph replays
    pre_span = []
    tmr = torch.zeros(4, dtype=torch.int64, device=dev)
    tmr_init = torch.tensor([-1, 0, -1, 0], dtype=torch.int64, device=dev)
    try:
        hydra.set_config("step_timer", tmr.data_ptr())
        g_span = capture(lambda: hydra.prefix_attn(q, pk, pv, workspace=ws))
    finally:
        hydra.set_config("step_timer", 0)
    for _ in range(20):
        tmr.copy_(tmr_init)
        g_span.replay()
        torch.cuda.synchronize(dev)
        t4 = [int(v) & 0xFFFFFFFFFFFFFFFF for v in tmr.tolist()]
        if t4[1] > 0 and t4[0] != 0xFFFFFFFFFFFFFFFF:
            pre_span.append((t4[1] - t4[0]) * 1e-6)
    del g_span
    ms_pre_span = statistics.median(pre_span) if pre_span else None
    n_sus = max(20, int(1000.0 / max(ms_pre_burst, 1e-3)))
    with ClockSampler(local) as clk_pre:
        ms_pre_sus = time_graph(g_pre, n_sus, 0)
    clocks_pre = clk_pre.summary()

    # pick the step variant (prefix || suffix on disjoint SMs, or sequential) on a short probe
    if args.overlap_k > 0:
        hydra.set_config("overlap_prefix_ctas", args.overlap_k)
    g_over = capture(lambda: step(True))
    k_over = int(hydra.get_config("last_overlap_k"))  # SM split chosen for the overlapped step
    ov_simt = bool(hydra.get_config("last_overlap_simt"))  # ... with the SIMT suffix as the prefix's dependent
    g_seq = capture(lambda: step(False))
    probe = max(3, min(20, args.steps // 5))
    ms_over = time_graph(g_over, probe, 2)
    ms_seq = time_graph(g_seq, probe, 2)
    overlap = ms_over <= ms_seq
    g_main = g_over if overlap else g_seq

    with ClockSampler(local) as clk:
        ms = time_graph(g_main, args.steps, args.warmup)
    clocks = clk.summary()
    step_stats = {k: (round(v, 5) if isinstance(v, float) else v) for k, v in LAST_TIMING.items()}
    # the same step with L2 flushed (256 MB written) before every timed step: the inputs
    # already exceed L2, so this should match the back-to-back figure
    flush_buf = L2Flush(torch, dev)
    ms_flushed = timed_steps(torch, g_main.replay, max(10, min(50, args.steps // 4)), flush_buf)
    del flush_buf

    # Flatness (north_star: total time at B=1024 should drop < 15% when the prefix grows
    # from 1K to 16K): the same suffixes with the prefix cut to its first 1024 tokens,
    # timed the same way (best of the two schedules).
    flat = None
    if P > 1024:
        P1 = 1024
        pk1, pv1 = pk[:P1], pv[:P1]
        ws1 = torch.empty(hydra.attn_workspace_bytes(q, P1, S, Hkv_r), dtype=torch.uint8, device=dev)

        def step1(overlap: bool):
            hydra.hydragen_attention(q, pk1, pv1, sk, sv, lens, out=out, workspace=ws1,
                                     aux_stream=aux if overlap else None)

        ms1 = min(time_graph(capture(lambda: step1(True)), args.steps, args.warmup),
                  time_graph(capture(lambda: step1(False)), args.steps, args.warmup))
        q1, q16 = B / (ms1 * 1e-3), B / (ms * 1e-3)
        flat = {"prefix_1k_queries_per_s": round(q1, 1), "prefix_%d_queries_per_s" % P: round(q16, 1),
                "drop": round(1.0 - q16 / q1, 4), "target_drop": 0.15, "ms_prefix_1k": round(ms1, 5)}

    # Each kernel's duration INSIDE the timed step: the library records CUDA events around the
    # prefix (on its stream) and the suffix launches of hydra_attn; the same step graph as the
    # timed loop is captured with those event nodes and replayed (synchronised per replay to
    # read the events), so the suffix is timed concurrently with the prefix, as in the step.
    # In the SM-partitioned schedule both kernels run on one stream (the suffix is a programmatic
    # dependent launch), so no event can sit between them: the persistent kernels record their
    # own span instead (config key step_timer: min CTA start / max CTA end, %globaltimer ns).
    ev_keys = ("ev_prefix_begin", "ev_prefix_end", "ev_suffix_begin", "ev_suffix_end")
    evs = [torch.cuda.Event(enable_timing=True) for _ in ev_keys]
    for e in evs:
        e.record()
    torch.cuda.synchronize(dev)
    M = 8  # steps per timer graph: each step records into its own slots, the M run back to back
    timer = torch.zeros(M, 4, dtype=torch.int64, device=dev)
    timer_init = torch.tensor([-1, 0, -1, 0], dtype=torch.int64, device=dev).repeat(M, 1)  # UINT64_MAX, 0
    use_timer = overlap and k_over > 0
    try:
        if use_timer:
            def steps_timed():
                for i in range(M):
                    hydra.set_config("step_timer", timer[i].data_ptr())
                    step(overlap)
            g_ev = capture(steps_timed)
        else:
            for key, e in zip(ev_keys, evs):
                hydra.set_config(key, e.cuda_event)
            g_ev = capture(lambda: step(overlap))
        for _ in range(3):
            g_ev.replay()
        torch.cuda.synchronize(dev)
        pre_in, suf_in = [], []
        for _ in range(max(10, min(50, args.steps // 4)) // (M if use_timer else 1) + 1):
            if use_timer:
                timer.copy_(timer_init)  # stream-ordered before the replay: no host sync
            g_ev.replay()
            torch.cuda.synchronize(dev)
            if use_timer:
                for row in timer.tolist():
                    t = [int(v) & 0xFFFFFFFFFFFFFFFF for v in row]
                    pre_in.append((t[1] - t[0]) * 1e-6)
                    suf_in.append((t[3] - t[2]) * 1e-6)
            else:
                pre_in.append(evs[0].elapsed_time(evs[1]))
                suf_in.append(evs[2].elapsed_time(evs[3]))
    finally:
        hydra.set_config("step_timer", 0)
        for key in ev_keys:
            hydra.set_config(key, 0)
    del g_ev
    ms_pre_in, ms_suf_in = statistics.mean(pre_in), statistics.mean(suf_in)
    in_step_how = ("inside the step: the kernel's own span (min CTA start to max CTA end, %%globaltimer), the "
                   "prefix on its SM share concurrently, in graphs of %d back-to-back steps, mean of %d steps"
                   % (M, len(suf_in))) if use_timer else (
                   "inside the step: CUDA events recorded by hydra_attn around the suffix launch, in the step "
                   "graph of the timed loop, mean of %d replays" % len(suf_in))

    # The same step with the suffixes in a paged cache (hydra_attn_paged, R14): the
    # contiguous caches scattered into a shuffled page pool, the same schedule as g_main.
    paged = None
    if args.paged_page_size > 0 and S % args.paged_page_size == 0:
        ps = args.paged_page_size
        npg = S // ps
        perm = torch.from_numpy(np.random.default_rng(args.seed + 7).permutation(B * npg).astype(np.int64)).to(dev)
        kp = torch.empty(B * npg, ps, Hkv_r, d, dtype=torch.bfloat16, device=dev)
        vp = torch.empty_like(kp)
        kp[perm] = sk.view(B * npg, ps, Hkv_r, d)
        vp[perm] = sv.view(B * npg, ps, Hkv_r, d)
        tab = perm.view(B, npg).to(torch.int32)
        del perm
        g_pg = capture(lambda: hydra.hydragen_attention_paged(q, pk, pv, kp, vp, tab, lens, out=out, workspace=ws,
                                                              aux_stream=aux if overlap else None))
        ms_pg = time_graph(g_pg, args.steps, args.warmup)
        paged = {"page_size": ps, "pages": B * npg, "layout": "shuffled page pool, block table [B, %d]" % npg,
                 "queries_per_s": round(B / (ms_pg * 1e-3), 1), "ms_per_step": round(ms_pg, 5),
                 "vs_contiguous": round(ms / ms_pg, 4)}
        del g_pg, kp, vp, tab
        torch.cuda.empty_cache()

    # per-kernel timing on their own (roofline of the dominant kernel and the prefix phase)
    # (the composite's workspace holds (prefix + suffix) split partials, enough for either alone)
    kk = max(5, args.steps // 4)
    g_suf = capture(lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws))
    ms_pre = time_graph(g_pre, kk, 3)  # after the step loop: GPU warm, power-capped
    ms_suf = time_graph(g_suf, kk, 3)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    in_step = None
    short_share = Hq // Hkv in (2, 4, 8) and S <= 256  # the short-suffix kernel on the suffix's share
    if overlap and k_over > 0 and short_share:
        pass  # its share cannot be isolated for an "alone" timing: the in-step spans below stand
    elif overlap and k_over > 0 and ov_simt:
        # prefix on k persistent CTAs, the SIMT suffix (full grid) its programmatic dependent: the
        # dominant kernel stays the SIMT suffix (timed inside the step by its span below)
        try:
            hydra.set_config("prefix_ctas", k_over)
            ms_pre_k = time_graph(capture(lambda: hydra.prefix_attn(q, pk, pv, workspace=ws)), kk, 3)
        finally:
            hydra.set_config("prefix_ctas", 0)
        in_step = {"prefix_ctas": k_over, "suffix": "SIMT kernel, full grid, programmatic dependent of the prefix",
                   "ms_prefix": round(ms_pre_k, 5), "ms_suffix": round(ms_suf, 5)}
    elif overlap and k_over > 0:
        # the kernels as the overlapped step runs them: prefix on k SMs || tensor-core suffix on
        # the other SMs (timed one at a time, so without the other's HBM/L2/power interference)
        try:
            hydra.set_config("prefix_ctas", k_over)
            ms_pre_k = time_graph(capture(lambda: hydra.prefix_attn(q, pk, pv, workspace=ws)), kk, 3)
            hydra.set_config("prefix_ctas", 0)
            hydra.set_config("suffix_impl", 2)
            hydra.set_config("suffix_ctas", sms - k_over)
            ms_suf_k = time_graph(capture(lambda: hydra.suffix_attn(q, sk, sv, lens, workspace=ws)), kk, 3)
        finally:
            for key in ("prefix_ctas", "suffix_impl", "suffix_ctas"):
                hydra.set_config(key, 0)
        in_step = {"prefix_ctas": k_over, "suffix_ctas": sms - k_over, "ms_prefix": round(ms_pre_k, 5),
                   "ms_suffix": round(ms_suf_k, 5)}

    pk_meas = peaks()
    hbm = float(pk_meas.get("hbm_gbs", 6650.0))
    tc_burst = float(pk_meas.get("bf16_tflops", 1590.0))
    tc_sust = float(pk_meas.get("bf16_tflops_sustained", 1400.0))
    peak_src = "MEASURED_PEAKS.json" if pk_meas else "fallback (B200_PROFILING.md)"

    lens_sum = int(pb.lens.sum())
    suffix_bytes = 2 * lens_sum * Hkv_r * d * 2 + B * Hq_r * d * 2  # K+V valid rows + q (bf16)
    prefix_flops = 4.0 * B * Hq_r * P * d
    prefix_bytes = 2 * P * Hkv_r * d * 2
    total_bytes = suffix_bytes + prefix_bytes + B * Hq_r * d * 2  # + bf16 output
    suf_gbs = suffix_bytes / (ms_suf * 1e-3) / 1e9
    pre_tflops = prefix_flops / (ms_pre * 1e-3) / 1e12
    pre_burst = prefix_flops / (ms_pre_burst * 1e-3) / 1e12
    pre_sus = prefix_flops / (ms_pre_sus * 1e-3) / 1e12
    t_roof = max(prefix_flops / (tc_burst * 1e12), total_bytes / (hbm * 1e9))

    value = B / (ms * 1e-3)
    line = {
        "metric": "decode-attn queries/s and % of bf16 TC peak; prefix 16K, batch 1024, 1/2/4/8 GPU",
        "value": round(value, 1),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 5),
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded PCG64 N(0,1) K/V rounded to bf16, 'mixed' needle queries)",
        "config": {"workload": args.config, "description": cfg["name"], "B": B, "Hq": Hq, "Hkv": Hkv, "d": d,
                   "prefix_len": P, "suffix_len": S, "parallelism": f"kv-head shard x{world}" if world > 1 else "1 GPU",
                   "heads_per_gpu": Hq_r, "overlap_prefix_suffix": overlap,
                   "schedule": ("sequential" if not (overlap and k_over > 0) else
                                "prefix on %d CTAs, SIMT suffix its programmatic dependent (full grid)" % k_over if ov_simt else
                                "prefix on %d CTAs || short-suffix kernel (3 CTAs per SM) on the other SMs" % k_over
                                if Hq // Hkv in (2, 4, 8) and S <= 256 else
                                "prefix on %d CTAs || tensor-core suffix on the other SMs" % k_over),
                   "l2": (f"no flush: {in_bytes / 1e9:.2f} GB of inputs per step > 2 x 126 MB L2" if flush is None else
                          L2Flush.DESC + f": {in_bytes / 1e9:.3f} GB of inputs per rank"),
                   "timing": "CUDA graph of one step, CUDA events over K replays, max over ranks"},
        "roofline": {"bound": "hbm", "kernel": (("suffix_short_kernel (tensor-core GEMV, 3 CTAs per SM; GQA g = %d; the sequential schedule's suffix)"
                                                 if Hq // Hkv in (2, 4, 8) and S <= 256 else
                                                 "suffix_tc_kernel (tensor-core GEMV, all SMs; GQA g = %d; the sequential schedule's suffix)") % (Hq // Hkv)
                                                if Hq // Hkv >= 2 else
                                                "suffix split-K GEMV (decode_attn_kernel, all SMs; the sequential schedule's dominant kernel)"),
                     "achieved": round(suf_gbs, 1), "peak": hbm, "unit": "GB/s", "frac": round(suf_gbs / hbm, 4),
                     "traffic": NCU_TRAFFIC.get((args.config, ("suffix_short_kernel" if Hq // Hkv in (2, 4, 8) and S <= 256 else
                                                               "suffix_tc_kernel") if Hq // Hkv >= 2 else "decode_attn_kernel")),
                     "algorithmic_bytes_per_launch": suffix_bytes,
                     "launch_ms": round(ms_suf, 5), "peak_source": peak_src + " (STREAM copy)",
                     "frac_of_nominal_7700": round(suf_gbs / 7700.0, 4),
                     "note": "read-only stream vs a read+write copy peak: can read a little above 1.0"},
        "prefix_phase": {"bound": "tensor", "kernel": prefix_kernel_name(hydra, Hq // Hkv),
                         "achieved": round(pre_burst, 1), "unit": "TFLOP/s", "peak": tc_burst,
                         "frac": round(pre_burst / tc_burst, 4), "launch_ms": round(ms_pre_burst, 5),
                         "timed": "burst: 20 graph replays on a cool GPU, before the step loop",
                         "sustained": {"achieved": round(pre_sus, 1), "peak": tc_sust,
                                       "frac": round(pre_sus / tc_sust, 4), "launch_ms": round(ms_pre_sus, 5),
                                       "replays": n_sus, "clocks": clocks_pre,
                                       "timed": "back-to-back replays for ~1 s vs the sustained cuBLAS loop"},
                         "after_step_loop": {"achieved": round(pre_tflops, 1), "launch_ms": round(ms_pre, 5)},
                         "frac_of_spec_2250": round(pre_burst / 2250.0, 4), "flops_per_launch": prefix_flops,
                         "kernel_span": ({"launch_ms": round(ms_pre_span, 5),
                                          "achieved": round(prefix_flops / (ms_pre_span * 1e-3) / 1e12, 1),
                                          "frac": round(prefix_flops / (ms_pre_span * 1e-3) / 1e12 / tc_burst, 4),
                                          "timed": "the kernel's own span (first CTA start to last CTA end), median of 20 "
                                                   "graph replays; launch_ms above also holds the combine of its pieces"}
                                         if ms_pre_span else None),
                         "traffic": NCU_TRAFFIC.get((args.config, prefix_kernel_name(hydra, Hq // Hkv).split()[0])),
                         "algorithmic_bytes_per_launch": prefix_bytes},
        "step_roofline": {"t_roof_ms": round(t_roof * 1e3, 5), "frac": round(t_roof * 1e3 / ms, 4),
                          "ms_sequential": round(ms_seq, 5), "ms_overlap": round(ms_over, 5)},
        "step_time": dict(step_stats, mean_ms=round(ms, 5), ms_l2_flushed=round(ms_flushed, 5),
                          note="per-step events inside the back-to-back timed loop; ms_l2_flushed: L2Flush "
                               "before each of its steps, only the steps timed"),
        "clocks": clocks,
        # prefix, suffix, combine (+ the -inf fill of the partial slots, which the CTA-pair prefix
        # kernel does itself)
        "gpu_launches": args.steps * (3 if prefix_kernel_name(hydra, Hq // Hkv).startswith("prefix_pair") else 4),
    }
    if flat:
        line["flatness"] = flat
    if paged:
        line["paged_suffix"] = paged
    if clocks.get("power_w"):
        # board power (nvidia-smi power.draw, median over the timed region) x step time
        j = clocks["power_w"] * ms * 1e-3
        line["energy"] = {"board_power_w": clocks["power_w"], "joules_per_step": round(j, 5),
                          "queries_per_joule": round(B / j, 1), "samples": clocks["samples"]}
    if in_step and not ov_simt:
        # the overlapped step's dominant kernel: the tensor-core suffix on (SMs - k) SMs
        b_k = suffix_bytes / (in_step["ms_suffix"] * 1e-3) / 1e9
        f_k = prefix_flops / (in_step["ms_prefix"] * 1e-3) / 1e12
        # it is the step's dominant kernel, so it becomes `roofline`; the SIMT kernel of the
        # sequential schedule stays reported as `roofline_sequential`
        line["roofline_sequential"] = line["roofline"]
        line["roofline"] = {
            "bound": "hbm", "kernel": "suffix_tc_kernel on %d SMs (prefix on %d SMs), the overlapped step's dominant kernel"
            % (sms - k_over, k_over),
            "achieved": round(b_k, 1), "peak": hbm, "unit": "GB/s", "frac": round(b_k / hbm, 4),
            "traffic": NCU_TRAFFIC.get((args.config, "suffix_tc_kernel@%d" % (sms - k_over)),
                                       NCU_TRAFFIC.get((args.config, "suffix_tc_kernel"))),
            "algorithmic_bytes_per_launch": suffix_bytes,
            "launch_ms": in_step["ms_suffix"], "peak_source": peak_src + " (STREAM copy)",
            "frac_of_nominal_7700": round(b_k / 7700.0, 4),
            "timed": "alone on its SM share (CUDA graph, events), after the step loop",
            "prefix_tflops_on_k_sms": round(f_k, 1), "prefix_launch_ms_on_k_sms": in_step["ms_prefix"]}

    if in_step and ov_simt:
        line["overlap_parts_alone"] = in_step
    # the dominant kernel's figure as it runs inside the step (events on its own stream);
    # the kernel timed alone stays as `alone`
    suf_in_gbs = suffix_bytes / (ms_suf_in * 1e-3) / 1e9
    rl = line["roofline"]
    rl["alone"] = {"achieved": rl["achieved"], "frac": rl["frac"], "launch_ms": rl["launch_ms"],
                   "timed": rl.get("timed", "alone on the full chip (CUDA graph, events), after the step loop")}
    rl.update({"achieved": round(suf_in_gbs, 1), "frac": round(suf_in_gbs / hbm, 4), "launch_ms": round(ms_suf_in, 5),
               "frac_of_nominal_7700": round(suf_in_gbs / 7700.0, 4),
               "timed": in_step_how,
               "prefix_in_step_ms": round(ms_pre_in, 5),
               "prefix_in_step_tflops": round(prefix_flops / (ms_pre_in * 1e-3) / 1e12, 1),
               "share_of_step": round(ms_suf_in / ms, 4)})
    if ms_pre_in > ms_suf_in:
        # the prefix is the step's dominant kernel (C4, C6): it becomes `roofline` (tensor-bound, timed
        # inside the step, against the sustained bf16 figure); the suffix figure stays as roofline_suffix
        line["roofline_suffix"] = line["roofline"]
        pre_in_tf = prefix_flops / (ms_pre_in * 1e-3) / 1e12
        pname = prefix_kernel_name(hydra, Hq // Hkv)
        line["roofline"] = {
            "bound": "tensor", "kernel": pname + ", the step's dominant kernel",
            "achieved": round(pre_in_tf, 1), "peak": tc_sust, "unit": "TFLOP/s", "frac": round(pre_in_tf / tc_sust, 4),
            "traffic": NCU_TRAFFIC.get((args.config, pname.split()[0])),
            "algorithmic_flops_per_launch": prefix_flops, "algorithmic_bytes_per_launch": prefix_bytes,
            "launch_ms": round(ms_pre_in, 5), "peak_source": peak_src + " (sustained cuBLAS bf16 loop)",
            "timed": in_step_how.replace("around the suffix launch", "around the prefix launch"),
            "share_of_step": round(ms_pre_in / ms, 4), "frac_of_spec_2250": round(pre_in_tf / 2250.0, 4),
            "frac_of_burst_peak": round(pre_in_tf / tc_burst, 4),
            "alone": {"achieved": round(pre_burst, 1), "peak": tc_burst, "frac": round(pre_burst / tc_burst, 4),
                      "launch_ms": round(ms_pre_burst, 5), "timed": "burst: 20 graph replays on a cool GPU"}}

    if not args.no_e2e:
        line["e2e"] = e2e_leg(args, hydra, torch, dev, world, (hq, hpk, hpv, hsk, hsv, hlens),
                              (q, pk, pv, sk, sv, lens), ws, out, B)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(pb, args.cpu_seconds)
    line["gen_seconds"] = round(t_gen, 1)
    if rank == 0:
        print(json.dumps(mark_shared(line)), flush=True)
    if world > 1:
        dist.barrier()


def prefix_kernel_name(hydra, g):
    if hydra.get_config("prefix_variant") == 9 and 128 % g == 0:
        return "prefix_pair_kernel (CTA-pair cta_group::2 tcgen05, persistent, all SMs)"
    return "prefix_tc2_kernel (persistent tcgen05, all SMs)"


def e2e_leg(args, hydra, torch, dev, world, host_t, dev_t, ws, out, B):
    """Same metric through the public API with HOST inputs: H2D of every input + compute + D2H of out."""
    import torch.distributed as dist

    pinned = [t.pin_memory() for t in host_t]
    h2d = sum(t.numel() * t.element_size() for t in pinned)
    hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    d2h = hout.numel() * hout.element_size()
    q, pk, pv, sk, sv, lens = dev_t

    def one():
        for src, dst in zip(pinned, dev_t):
            dst.copy_(src, non_blocking=True)
        hydra.hydragen_attention(q, pk, pv, sk, sv, lens, out=out, workspace=ws)
        hout.copy_(out, non_blocking=True)

    one()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.e2e_steps):
        one()
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / args.e2e_steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": round(B / (ms * 1e-3), 1), "unit": "queries/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 3), "steps": args.e2e_steps}


def cpu_baseline(pb, target_s: float):
    """The fp64 oracle (oracle/), as it stands, on a bounded sample of the same workload."""
    import numpy as np

    import oracle

    cores = oracle.max_threads()
    Hq = pb.Hq

    def rows_for(nseq):
        bb, hh = np.meshgrid(np.arange(nseq), np.arange(Hq), indexing="ij")
        return np.stack([bb.ravel(), hh.ravel()], 1)

    n = 2
    t0 = time.time()
    oracle.flat_attention(pb, rows=rows_for(n))
    dt = time.time() - t0
    n2 = int(max(1, min(pb.B, math.floor(n * target_s / max(dt, 1e-3)))))
    t0 = time.time()
    oracle.flat_attention(pb, rows=rows_for(n2))
    dt2 = time.time() - t0
    return {"value": round(n2 / dt2, 3), "unit": "queries/s", "cores": cores, "kind": "oracle",
            "sample": f"first {n2} of {pb.B} sequences x all {Hq} heads (prefix {pb.P} + suffix {pb.S_cap} tokens), "
                      f"fp64 two-pass, {dt2:.1f} s",
            "cpu_model": cpu_model()}


def reference_arm(args):
    """--impl reference: the fp64 CPU oracle timed on this box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import numpy as np

    import oracle
    import synth

    cfg = dict(CONFIGS[args.config])
    B, Hq, Hkv, d, P, S = cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["d"], cfg["P"], cfg["S"]
    budget = 150.0  # seconds for the whole --steps K --warmup W run
    per_step = budget / max(1, args.steps + args.warmup)
    tree = cfg.get("kind") == "tree"

    def problem(n):
        if tree:  # same root / branch lengths, n sequences spread over the branches
            per = max(1, -(-n // cfg["branches"]))
            parent, node_len, leaf = synth.two_level_tree(P, cfg["branches"], cfg["branch_len"], per)
            return synth.make_tree_problem(parent, node_len, leaf, Hq, Hkv, d, S, dtype="bf16", dist="mixed",
                                           seed=args.seed)
        return synth.make_problem(n, Hq, Hkv, d, P, S, dtype="bf16", dist="mixed", seed=args.seed)

    run_oracle = oracle.tree_attention if tree else oracle.flat_attention
    # calibrate the sample size on a small problem of the same shape
    cal = problem(2)
    t0 = time.time()
    run_oracle(cal)
    per_seq = (time.time() - t0) / cal.B
    nseq = int(max(1, min(B, per_step / max(per_seq, 1e-6))))
    pb = problem(nseq)
    nseq = pb.B
    for _ in range(args.warmup):
        run_oracle(pb)
    t0 = time.time()
    for _ in range(args.steps):
        run_oracle(pb)
    dt = (time.time() - t0) / max(1, args.steps)
    value = nseq / dt
    cores = oracle.max_threads()
    line = {
        "metric": "decode-attn queries/s and % of bf16 TC peak; prefix 16K, batch 1024, 1/2/4/8 GPU",
        "value": round(value, 3), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded PCG64 N(0,1) K/V rounded to bf16, 'mixed' needle queries)",
        "config": {"workload": args.config, "description": cfg["name"], "B": B, "Hq": Hq, "Hkv": Hkv, "d": d,
                   "prefix_len": P, "suffix_len": S},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 3), "unit": "queries/s", "cores": cores, "kind": "oracle",
                         "sample": f"{nseq} of {B} sequences x all {Hq} heads per step, fp64 two-pass",
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 3), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
