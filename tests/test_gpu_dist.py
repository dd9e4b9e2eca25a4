"""The multi-GPU layer through the CUDA kernels, in N processes (one per rank).

The round's GPU boxes have one B200, so the ranks share cuda:0 and talk over gloo; the
sequence split then stages its one all-to-all through pinned host memory (dist.py), every
other step -- prefix, pack, suffix on the side stream, merge -- runs the library's kernels
in both ranks.  Each rank compares its own output rows with the fp64 oracle element by
element (same gates as the single-GPU parity tests):
  * sequence split (C4-like GQA shape and the paper's long-document shape P:198 at full size,
    P:557's motivation), all-to-all and all-gather exchanges, fp16 and fp32 exchange rows;
  * KV-head sharding: each rank's head slice passed as strided views, no copy.
Head-shard invariance (SURVEY §8(c) pin): with a head-separable schedule (one-tile prefix
kernel, fixed KV splits) every head's output is bitwise the one the 1-GPU call produces."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {  # name: (B, Hq, Hkv, d, P, S, dist, seed)
    "gqa": (24, 32, 8, 128, 700, 40, "mixed", 31),
    "mha_ragged": (30, 8, 8, 128, 1100, 300, "boundary", 32),
    "longdoc_full": (256, 32, 4, 128, 19947, 128, "boundary", 6),
}


def _worker(rank, world, port, case, mode, exchange, edt, outdir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist

    import oracle
    import synth
    from paper_2402_05099_b200 import dist as hdist
    from tests import nanfill as H
    from tests.util import assert_parity, problem_to

    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, Hq, Hkv, d, P, S, dist_, seed = CASES[case]
        lens = np.random.default_rng(seed).integers(1, S + 1, B)
        pb = synth.make_problem(B, Hq, Hkv, d, P, S, lens=lens, dtype="bf16", dist=dist_, seed=seed)
        t = problem_to(pb, "cuda:0")
        if mode == "seqsplit":
            p0, p1 = hdist.shard_range(P, world, rank)
            b0, b1 = hdist.batch_shard(B, world, rank)
            plan = hdist.SeqSplit(B, Hq, d, device="cuda:0", exchange_dtype=edt, exchange=exchange)
            # NaN in every plan buffer: rows a kernel leaves unwritten fail parity
            for buf in (plan.o_p, plan.l_p, plan.o_s, plan.l_s, plan.out, plan.lse):
                buf.fill_(float("nan"))
            plan.send.fill_(0xFF)
            plan.recv.fill_(0xFF)
            for rep in range(2):  # the second call reuses the plan's buffers
                out, lse = plan(t["q"], t["pk"][p0:p1], t["pv"][p0:p1], t["sk"][b0:b1], t["sv"][b0:b1],
                                t["lens"][b0:b1], return_lse=True, check_range=True)
                torch.cuda.synchronize()
            assert out.shape == (b1 - b0, Hq, d)
            if b1 > b0:
                rows = np.stack(np.meshgrid(np.arange(b0, b1), np.arange(Hq), indexing="ij"), -1).reshape(-1, 2)
                ref, lref = oracle.flat_attention(pb, rows=rows)
                assert_parity(out.reshape(-1, d), ref, lse.reshape(-1), lref,
                              what=f"rank {rank} seq-split {case} {exchange} {edt}")
        else:  # KV-head shard: this rank's slice of the full tensors, strided, no copy
            (h0, h1), (j0, j1) = hdist.head_shard(Hq, Hkv, world, rank)
            out = H.nan((B, h1 - h0, d), torch.bfloat16, "cuda:0")
            hdist.head_sharded_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], world=world,
                                         rank=rank, out=out)
            torch.cuda.synchronize()
            rows = np.stack(np.meshgrid(np.arange(B), np.arange(h0, h1), indexing="ij"), -1).reshape(-1, 2)
            ref, _ = oracle.flat_attention(pb, rows=rows)
            assert_parity(out.reshape(-1, d), ref, what=f"rank {rank} head shard {case}")
        open(os.path.join(outdir, f"ok{rank}"), "w").write("ok")
    finally:
        tdist.destroy_process_group()


def _spawn(world, case, mode, exchange="alltoall", edt=torch.float16):
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), case, mode, exchange, edt, td), nprocs=world, join=True)
        for r in range(world):
            assert os.path.exists(os.path.join(td, f"ok{r}")), f"rank {r} did not finish"


@pytest.mark.parametrize("case,world,exchange,edt", [
    ("gqa", 2, "alltoall", torch.float16),
    ("gqa", 2, "alltoall", torch.float32),
    ("gqa", 3, "allgather", torch.float16),
    ("mha_ragged", 2, "alltoall", torch.float16),
])
def test_seqsplit_cuda_ranks(case, world, exchange, edt):
    _spawn(world, case, "seqsplit", exchange, edt)


@pytest.mark.slow
def test_seqsplit_longdoc_full_size_world2():
    """The paper's long-document shape (19,947-token prefix, 32 q / 4 kv heads) at full
    size, prefix split across 2 ranks: every row of each rank's batch shard."""
    _spawn(2, "longdoc_full", "seqsplit")


@pytest.mark.parametrize("world", [2, 4])
def test_head_shard_cuda_ranks(world):
    _spawn(world, "gqa", "heads")


def test_head_shard_bitwise_invariance():
    """SURVEY §8(c) "head-shard invariance": with a schedule that treats heads independently
    (one-tile tcgen05 prefix kernel with a fixed KV split count; tensor-core suffix, one item
    per (sequence, KV head)), a rank's head slice -- passed as strided views of the full
    tensors -- reproduces the 1-GPU output of those heads bit for bit, at 2, 4 and 8 shards."""
    import synth
    import paper_2402_05099_b200 as hydra
    from paper_2402_05099_b200 import dist as hdist
    from tests.util import problem_to

    B, Hq, Hkv, d, P, S = 40, 32, 8, 128, 900, 200
    pb = synth.make_problem(B, Hq, Hkv, d, P, S, lens=np.arange(B) * 5 % (S + 1), dtype="bf16", dist="mixed",
                            seed=44)
    t = problem_to(pb, "cuda:0")
    try:
        hydra.set_config("prefix_impl", 2)
        hydra.set_config("prefix_splits", 3)
        hydra.set_config("suffix_impl", 2)
        full = hydra.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"])
        for world in (2, 4, 8):
            for rank in range(world):
                (h0, h1), _ = hdist.head_shard(Hq, Hkv, world, rank)
                part = hdist.head_sharded_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"],
                                                    world=world, rank=rank)
                torch.cuda.synchronize()
                assert torch.equal(part, full[:, h0:h1]), f"world {world} rank {rank} differs from 1 GPU"
    finally:
        for k in ("prefix_impl", "prefix_splits", "suffix_impl"):
            hydra.set_config(k, 0)
