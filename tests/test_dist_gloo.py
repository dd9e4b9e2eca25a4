"""Multi-GPU layer on CPU: world size 2 over gloo.

The orchestration in paper_2402_05099_b200/dist.py (shard ranges, the packed (O, LSE)
exchange block, all-gather, strided combine of the gathered parts, suffix of the batch
shard) is exercised with reference ops built on the fp64 oracle in place of the CUDA
kernels.  The result of every rank must equal the oracle's undecomposed attention of its
batch-shard rows (App. A decomposition across ranks)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _np(t: torch.Tensor):
    t = t.contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


class OracleOps:
    """fp64 oracle stand-ins for the kernel calls (test infrastructure)."""

    def prefix(self, q, k, v, scale=None, out=None, lse_out=None):
        B = q.shape[0]
        o, l = oracle.attention_segments(_np(q), [[(_np(k), _np(v))]] * B, k.shape[1], scale)
        o, l = torch.from_numpy(o).float(), torch.from_numpy(l).float()
        if out is None:
            return o, l
        out.copy_(o)
        lse_out.copy_(l)
        return out, lse_out

    def suffix(self, q, k, v, lens, scale=None, out=None, lse_out=None):
        kn, vn = _np(k), _np(v)
        segs = [[(kn[b, :int(lens[b])], vn[b, :int(lens[b])])] for b in range(q.shape[0])]
        o, l = oracle.attention_segments(_np(q), segs, k.shape[2], scale)
        out.copy_(torch.from_numpy(o).float())
        lse_out.copy_(torch.from_numpy(l).float())
        return out, lse_out

    def combine(self, o_parts, lse_parts, out_dtype=torch.bfloat16, out=None, lse_out=None, o_parts_f32=None,
                lse_parts_f32=None):
        o = o_parts.double().numpy()
        l = lse_parts.double().numpy()
        if o_parts_f32 is not None:  # the second (f32) part group is merged in the same pass
            o = np.concatenate([o, o_parts_f32.double().numpy()])
            l = np.concatenate([l, lse_parts_f32.double().numpy()])
        ro, rl = o[0], l[0]
        for i in range(1, o.shape[0]):
            ro, rl = oracle.combine(ro, rl, o[i], l[i])
        if out is None:
            out = torch.empty(ro.shape, dtype=out_dtype)
        out.copy_(torch.from_numpy(ro).to(out.dtype).view(out.shape))
        if lse_out is None:
            lse_out = torch.empty(rl.shape, dtype=torch.float32)
        lse_out.copy_(torch.from_numpy(rl).float().view(lse_out.shape))
        return out, lse_out

    def attention(self, q, pk, pv, sk, sv, lens, scale=None, out=None):
        B = q.shape[0]
        segs = [[(_np(pk), _np(pv)), (_np(sk)[b, :int(lens[b])], _np(sv)[b, :int(lens[b])])] for b in range(B)]
        o, _ = oracle.attention_segments(_np(q), segs, pk.shape[1], scale)
        return torch.from_numpy(o).float()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, exchange, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2402_05099_b200 import dist as hdist

    try:
        lens_all = [12, 0, 5, 12, 1, 7, 3]
        # world 3: unequal batch shards (3, 3, 1 rows); world 4: B = 5 leaves rank 3 without sequences
        B = {2: 6, 3: 7, 4: 5}[world]
        Hq, Hkv, d, P, S = 8, 2, 32, 90, 12
        pb = synth.make_problem(B, Hq, Hkv, d, P, S, lens=lens_all[:B], dtype="bf16", dist="mixed", seed=21)
        tt = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16)
        q, pk, pv, sk, sv = tt(pb.q), tt(pb.pk), tt(pb.pv), tt(pb.sk), tt(pb.sv)
        lens = torch.from_numpy(pb.lens.astype(np.int32))
        ref, lref = oracle.flat_attention(pb)
        ops = OracleOps()
        if mode.startswith("seqsplit"):
            p0, p1 = hdist.shard_range(P, world, rank)
            b0, b1 = hdist.batch_shard(B, world, rank)
            out, lse = hdist.seqsplit_attention(q, pk[p0:p1], pv[p0:p1], sk[b0:b1], sv[b0:b1], lens[b0:b1],
                                                exchange_dtype=exchange, out_dtype=torch.float32, ops=ops,
                                                return_lse=True,
                                                exchange="allgather" if mode.endswith("ag") else "alltoall")
            err = float(np.abs(out.double().numpy() - ref[b0:b1]).max()) if b1 > b0 else 0.0
            lerr = float(np.abs(lse.double().numpy() - lref[b0:b1]).max()) if b1 > b0 else 0.0
            tol = 1e-6 if exchange == torch.float32 else 4e-3
            assert out.shape == (b1 - b0, Hq, d)
            assert err <= tol, f"rank {rank}: seq-split max err {err}"
            assert lerr <= 1e-6, f"rank {rank}: lse err {lerr}"
        else:
            out = hdist.head_sharded_attention(q, pk, pv, sk, sv, lens, ops=ops, world=world, rank=rank)
            # gather the head shards and compare the full output
            full = [torch.empty_like(out) for _ in range(world)]
            dist.all_gather(full, out)
            full = torch.cat(full, dim=1)
            err = float(np.abs(full.double().numpy() - ref).max())
            assert err <= 1e-6, f"rank {rank}: head-shard err {err}"
        open(os.path.join(outdir, f"ok{rank}"), "w").write(str(err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,exchange,world", [("seqsplit-a2a", torch.float32, 2), ("seqsplit-a2a", torch.float16, 2),
                                                 ("seqsplit-a2a", torch.float16, 3), ("seqsplit-ag", torch.float16, 2),
                                                 ("seqsplit-a2a", torch.float16, 4), ("seqsplit-ag", torch.float16, 3),
                                                 ("heads", torch.float16, 2)])
def test_world_gloo(mode, exchange, world):
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), mode, exchange, td), nprocs=world, join=True)
        for r in range(world):
            assert os.path.exists(os.path.join(td, f"ok{r}"))


def test_shard_ranges_partition():
    from paper_2402_05099_b200 import dist as hdist

    for n in (0, 1, 7, 32768, 40):
        for w in (1, 2, 3, 8):
            rs = [hdist.shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    assert hdist.head_shard(40, 40, 8, 3) == ((15, 20), (15, 20))
    assert hdist.head_shard(32, 8, 4, 1) == ((8, 16), (2, 4))
    with pytest.raises(ValueError):
        hdist.head_shard(40, 40, 3, 0)
    assert hdist.exchange_layout(128, torch.float16) == (272, 256)  # O f16 | LSE f32 | pad: 16-B rows
    assert hdist.exchange_layout(128, torch.float32) == (528, 512)
    assert [hdist.batch_shard(7, 3, r) for r in range(3)] == [(0, 3), (3, 6), (6, 7)]
    assert [hdist.batch_shard(5, 4, r) for r in range(4)] == [(0, 2), (2, 4), (4, 5), (5, 5)]
