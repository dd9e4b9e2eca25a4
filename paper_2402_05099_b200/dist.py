"""Multi-GPU layer: one process per GPU, torch.distributed (NCCL) for the plumbing.

Two ways the shared-prefix decode attention shards:

* **KV-head sharding** (`head_shard`, `head_sharded_attention`): rank r owns KV heads
  [r*Hkv/N, (r+1)*Hkv/N) and their g*Hkv/N query heads, with their prefix and suffix
  K/V slices.  There is no collective: this is the tensor-parallel layout of the paper's
  end-to-end runs; the output stays head-sharded for the output projection.  The
  library takes strided tensors, so a rank's head slice of full-width tensors is passed
  without a copy.

* **Prefix sequence split** (`SeqSplit`, `seqsplit_attention`), for a very long prefix with
  few KV heads (Yi-6B has 4 KV heads, so head sharding stops at 4 GPUs): rank r owns
  prefix tokens [r*P/N, (r+1)*P/N) for all heads and the batch shard `batch_shard(B, N, r)`
  of the suffixes.  Per decode step each rank
    1. attends all B*g stacked queries to its prefix shard (tcgen05 prefix kernel),
    2. packs every row's (O, LSE) into one exchange buffer with ONE combine launch: rows of
       [O (fp16, d) | LSE (f32) | pad] (272 B at d = 128), batch shard c's rows contiguous,
    3. exchanges it with ONE all-to-all (NCCL over NVLink / NVSwitch): every rank receives
       only the N pieces of its own batch shard's rows -- B*Hq*272 bytes per rank in total,
       1/N of what an all-gather moves (`exchange="allgather"` is kept for comparison).
       With `exchange="p2p"` there is no collective: the receive buffers live in symmetric
       memory (torch.distributed._symmetric_memory), the pack of step 2 stores batch shard c's
       rows straight into rank c's buffer over NVLink (hydra_combine_ex with an output
       table of peer addresses: the computation and the transfer are one kernel), and a
       device-side barrier orders those stores before the merge,
    4. meanwhile runs suffix attention for its batch shard on a second stream (it needs no
       prefix data), so the suffix overlaps the exchange,
    5. merges the N received prefix pieces and its suffix part in ONE Eq. 5 combine launch
       (hydra_combine_ex: f16 parts read in place from the received rows + one f32 part).
  fp16 (not bf16) carries the exchanged O: |O_r| <= max|V| for a normalised partial, and
  fp16's 11-bit mantissa keeps the delivered bf16 output inside the parity gate (SURVEY
  §8(c)); an |O_r| beyond fp16's range (|V| > 65504) is detected after the pack and raises
  (`exchange_dtype=torch.float32` moves 528-byte rows instead).

With a gloo process group and CUDA tensors (the CPU-side tests of the CUDA path: two ranks
sharing one GPU), the exchange is staged through pinned host memory; with NCCL the whole
step, exchange included, is CUDA-graph capturable.  All buffers belong to the `SeqSplit`
plan and are allocated once.  The kernel calls go through an `ops` object (default: the
CUDA library), so the orchestration is also exercised by world-size-2/3 gloo tests on CPU
with fp64 oracle ops.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous near-equal split of range(n) across `world` ranks (prefix tokens, heads)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def batch_shard(B: int, world: int, rank: int) -> Tuple[int, int]:
    """Batch shard of the sequence split: ceil(B/N) sequences per rank, so every rank's rows
    form one contiguous slot of the exchange buffer (the last ranks may hold fewer, or none)."""
    mb = -(-B // world)
    return min(B, rank * mb), min(B, (rank + 1) * mb)


def head_shard(Hq: int, Hkv: int, world: int, rank: int):
    """(q-head range, kv-head range) owned by `rank` under KV-head sharding."""
    if Hkv % world:
        raise ValueError(f"Hkv={Hkv} is not divisible by world={world}")
    g = Hq // Hkv
    j0, j1 = shard_range(Hkv, world, rank)
    return (j0 * g, j1 * g), (j0, j1)


class KernelOps:
    """The CUDA library (libhydra.so) as used by the multi-GPU layer."""

    def __init__(self):
        from . import attn

        self._a = attn

    def prefix(self, q, k, v, scale=None, out=None, lse_out=None):
        return self._a.prefix_attn(q, k, v, scale=scale, out=out, lse_out=lse_out)

    def suffix(self, q, k, v, lens, scale=None, out=None, lse_out=None):
        return self._a.suffix_attn(q, k, v, lens, scale=scale, out=out, lse_out=lse_out)

    def combine(self, o_parts, lse_parts, out_dtype=torch.bfloat16, out=None, lse_out=None, o_parts_f32=None,
                lse_parts_f32=None):
        return self._a.combine(o_parts, lse_parts, out_dtype=out_dtype, out=out, lse_out=lse_out,
                               o_parts_f32=o_parts_f32, lse_parts_f32=lse_parts_f32)

    def combine_scatter(self, o_parts, lse_parts, out_table, table_rows, out_row_stride, out_dtype, lse_table,
                        lse_row_stride):
        return self._a.combine_scatter(o_parts, lse_parts, out_table, table_rows, out_row_stride,
                                       out_dtype=out_dtype, lse_table=lse_table, lse_row_stride=lse_row_stride)

    def attention(self, q, pk, pv, sk, sv, lens, scale=None, out=None):
        return self._a.hydragen_attention(q, pk, pv, sk, sv, lens, scale=scale, out=out)


def head_sharded_attention(q, pk, pv, sk, sv, lens, scale=None, ops=None, world: Optional[int] = None,
                           rank: Optional[int] = None, out=None):
    """Attention for one rank's KV-head shard (no communication).

    With world/rank None the tensors are this rank's shard already.  Otherwise they hold all
    heads and the rank's slice (q[:, h0:h1], K/V[..., j0:j1, :]) is passed as strided views --
    no copy -- and the output [B, (h1-h0), d] is that rank's head slice."""
    ops = ops or KernelOps()
    if world is not None:
        (h0, h1), (j0, j1) = head_shard(q.shape[1], pk.shape[1], world, rank)
        q, pk, pv, sk, sv = q[:, h0:h1], pk[:, j0:j1], pv[:, j0:j1], sk[:, :, j0:j1], sv[:, :, j0:j1]
    return ops.attention(q, pk, pv, sk, sv, lens, scale=scale, out=out)


def exchange_layout(d: int, exchange_dtype=torch.float16):
    """Bytes of one exchanged row [O (d, exchange_dtype) | LSE (f32) | pad to 16 B] and the LSE's
    offset in it."""
    esz = torch.empty((), dtype=exchange_dtype).element_size()
    return (d * esz + 4 + 15) // 16 * 16, d * esz


class SeqSplit:
    """Plan and buffers of the prefix sequence split for one rank (see the module docstring).

    B, Hq, d: the whole batch's query shape (q is replicated on every rank).  Calling the
    plan with this rank's prefix shard and batch-shard suffixes returns this rank's output
    rows [nb, Hq, d] (and LSEs)."""

    def __init__(self, B: int, Hq: int, d: int, group: Optional[dist.ProcessGroup] = None, device=None,
                 exchange_dtype=torch.float16, out_dtype=torch.bfloat16, exchange: str = "alltoall", ops=None):
        if exchange not in ("alltoall", "allgather", "p2p"):
            raise ValueError("exchange must be 'alltoall', 'allgather' or 'p2p'")
        self.ops = ops or KernelOps()
        self.group = group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.B, self.Hq, self.d = B, Hq, d
        self.dev = torch.device(device) if device is not None else torch.device("cpu")
        self.edt, self.out_dtype, self.exchange = exchange_dtype, out_dtype, exchange
        self.b0, self.b1 = batch_shard(B, self.world, self.rank)
        self.nb = self.b1 - self.b0
        self.mb = -(-B // self.world)
        self.row_bytes, lse_off = exchange_layout(d, exchange_dtype)
        esz = torch.empty((), dtype=exchange_dtype).element_size()
        slot_rows = self.mb * Hq
        self.slot_rows = slot_rows
        W = self.world
        # exchange buffers: slot c (rows of batch shard c) at rows [c*slot_rows, (c+1)*slot_rows)
        self.send = torch.zeros(W * slot_rows * self.row_bytes, dtype=torch.uint8, device=self.dev)
        n_recv = W * W * slot_rows if exchange == "allgather" else W * slot_rows
        self.symm = None
        if exchange == "p2p":
            # receive buffer in symmetric memory: every rank maps every peer's over NVLink, and the
            # pack kernel stores each batch shard's rows straight into the owner's buffer at
            # piece [my rank] -- the exchange is the pack's own stores, ordered by a barrier
            try:
                import torch.distributed._symmetric_memory as symm_mem
            except ImportError as e:  # pragma: no cover - depends on the torch build
                raise RuntimeError("exchange='p2p' needs torch.distributed._symmetric_memory") from e
            if self.dev.type != "cuda":
                raise ValueError("exchange='p2p' needs CUDA tensors")
            self.recv = symm_mem.empty(n_recv * self.row_bytes, dtype=torch.uint8, device=self.dev)
            self.recv.zero_()
            self.symm = symm_mem.rendezvous(self.recv, group if group is not None else dist.group.WORLD)
            peer_base = [self.symm.get_buffer(p, (n_recv * self.row_bytes,), torch.uint8).data_ptr()
                         for p in range(W)]
            delta = self.recv.data_ptr() - peer_base[self.rank]  # the tensor's offset in its allocation
            peer_base = [b + delta for b in peer_base]
            mine = self.rank * slot_rows * self.row_bytes  # my piece in every peer's buffer
            self.out_table = torch.tensor([b + mine for b in peer_base], dtype=torch.int64, device=self.dev)
            self.lse_table = torch.tensor([b + mine + lse_off for b in peer_base], dtype=torch.int64,
                                          device=self.dev)
        else:
            self.recv = torch.zeros(n_recv * self.row_bytes, dtype=torch.uint8, device=self.dev)
        re, rf = self.row_bytes // esz, self.row_bytes // 4
        self.send_o = self.send.view(exchange_dtype).view(W * slot_rows, re)[:B * Hq, :d]
        self.send_l = self.send.view(torch.float32).view(W * slot_rows, rf)[:B * Hq, lse_off // 4]
        if exchange != "allgather":  # piece p = my rows as computed by rank p
            ro = self.recv.view(exchange_dtype).view(W, slot_rows, re)
            rl = self.recv.view(torch.float32).view(W, slot_rows, rf)
            self.recv_o, self.recv_l = ro[:, :self.nb * Hq, :d], rl[:, :self.nb * Hq, lse_off // 4]
        else:  # rank p's whole send buffer at [p]; my rows start at b0*Hq
            ro = self.recv.view(exchange_dtype).view(W, W * slot_rows, re)
            rl = self.recv.view(torch.float32).view(W, W * slot_rows, rf)
            r0, r1 = self.b0 * Hq, self.b1 * Hq
            self.recv_o, self.recv_l = ro[:, r0:r1, :d], rl[:, r0:r1, lse_off // 4]
        self.o_p = torch.empty(B, Hq, d, dtype=torch.float32, device=self.dev)
        self.l_p = torch.empty(B, Hq, dtype=torch.float32, device=self.dev)
        self.o_s = torch.empty(1, max(self.nb, 1) * Hq, d, dtype=torch.float32, device=self.dev)
        self.l_s = torch.empty(1, max(self.nb, 1) * Hq, dtype=torch.float32, device=self.dev)
        self.out = torch.empty(max(self.nb, 1) * Hq, d, dtype=out_dtype, device=self.dev)
        self.lse = torch.empty(max(self.nb, 1) * Hq, dtype=torch.float32, device=self.dev)
        self.cuda = self.dev.type == "cuda"
        backend = dist.get_backend(group)
        self.staged = self.cuda and backend != "nccl" and exchange != "p2p"  # gloo: stage on the host
        if self.staged:
            self.h_send = torch.empty(self.send.numel(), dtype=torch.uint8).pin_memory()
            self.h_recv = torch.empty(self.recv.numel(), dtype=torch.uint8).pin_memory()
        if self.cuda:
            self.side = torch.cuda.Stream(device=self.dev)
            self.ev_packed = torch.cuda.Event()
            self.ev_suffix = torch.cuda.Event()
        self.overflow = None

    def exchange_bytes(self) -> int:
        """Bytes this rank sends per step (its slots for the other ranks)."""
        return (self.world - 1) * self.slot_rows * self.row_bytes if self.exchange != "allgather" else \
            (self.world - 1) * self.send.numel()

    def _collective(self):
        if self.exchange == "p2p":
            # every rank's stores into my buffer (and mine into theirs) are complete and visible
            self.symm.barrier(channel=0)
            return
        if self.staged:
            self.h_send.copy_(self.send)
            hs, hr = self.h_send, self.h_recv
        else:
            hs, hr = self.send, self.recv
        if self.exchange == "alltoall":
            dist.all_to_all_single(hr, hs, group=self.group)
        else:
            dist.all_gather_into_tensor(hr, hs, group=self.group)
        if self.staged:
            self.recv.copy_(self.h_recv)

    def __call__(self, q, pk_shard, pv_shard, sk_local, sv_local, lens_local, scale=None, return_lse=False,
                 check_range: bool = False):
        B, Hq, d = self.B, self.Hq, self.d
        if tuple(q.shape) != (B, Hq, d):
            raise ValueError(f"q must be [{B}, {Hq}, {d}] (the plan's shape)")
        if sk_local.shape[0] != self.nb:
            raise ValueError(f"this rank's batch shard holds {self.nb} sequences (batch_shard), got {sk_local.shape[0]}")
        ops = self.ops
        # 1. prefix pieces of all B*Hq rows over the local prefix shard
        ops.prefix(q, pk_shard, pv_shard, scale=scale, out=self.o_p, lse_out=self.l_p)
        # 2. one pack: (O f16 | LSE f32) rows, batch shard c's rows in slot c -- with p2p the pack
        #    stores batch shard c's rows straight into rank c's receive buffer (piece [my rank])
        if self.exchange == "p2p":
            esz = torch.empty((), dtype=self.edt).element_size()
            ops.combine_scatter(self.o_p.view(1, B * Hq, d), self.l_p.view(1, B * Hq), self.out_table,
                                self.slot_rows, self.row_bytes // esz, self.edt, self.lse_table, self.row_bytes // 4)
        else:
            ops.combine(self.o_p.view(1, B * Hq, d), self.l_p.view(1, B * Hq), out_dtype=self.edt, out=self.send_o,
                        lse_out=self.send_l)
        if check_range and self.edt == torch.float16:
            self.overflow = (~torch.isfinite(self.recv_o if self.exchange == "p2p" else self.send_o)).any()
        cur = torch.cuda.current_stream(self.dev) if self.cuda else None
        # 4. suffix of the local batch shard on the side stream, overlapping the exchange
        if self.nb > 0:
            if self.cuda:
                self.ev_packed.record(cur)
                self.side.wait_event(self.ev_packed)
                with torch.cuda.stream(self.side):
                    ops.suffix(q[self.b0:self.b1], sk_local, sv_local, lens_local, scale=scale,
                               out=self.o_s[0].view(self.nb, Hq, d), lse_out=self.l_s[0].view(self.nb, Hq))
                self.ev_suffix.record(self.side)
            else:
                ops.suffix(q[self.b0:self.b1], sk_local, sv_local, lens_local, scale=scale,
                           out=self.o_s[0].view(self.nb, Hq, d), lse_out=self.l_s[0].view(self.nb, Hq))
        # 3. the exchange (one collective)
        self._collective()
        if self.nb == 0:
            out = self.out[:0].view(0, Hq, d)
            return (out, self.lse[:0].view(0, Hq)) if return_lse else out
        if self.cuda:
            cur.wait_event(self.ev_suffix)
        # 5. one merge: N received prefix pieces (f16, read in place) + the suffix part (f32)
        rows = self.nb * Hq
        out, lse = ops.combine(self.recv_o, self.recv_l, out_dtype=self.out_dtype, out=self.out[:rows],
                               lse_out=self.lse[:rows], o_parts_f32=self.o_s[:, :rows], lse_parts_f32=self.l_s[:, :rows])
        if check_range and self.overflow is not None and bool(self.overflow):
            raise OverflowError("a prefix partial O exceeds the fp16 range (|V| > 65504): use exchange_dtype=float32")
        out = out.view(self.nb, Hq, d)
        return (out, lse.view(self.nb, Hq)) if return_lse else out


_PLANS = {}


def seqsplit_attention(q: torch.Tensor, pk_shard: torch.Tensor, pv_shard: torch.Tensor,
                       sk_local: torch.Tensor, sv_local: torch.Tensor, lens_local: torch.Tensor,
                       group: Optional[dist.ProcessGroup] = None, scale: Optional[float] = None,
                       exchange_dtype=torch.float16, out_dtype=None, ops=None, return_lse: bool = False,
                       exchange: str = "alltoall", check_range: bool = False):
    """Prefix sequence split across the ranks of `group` (see the module docstring).

    q: [B, Hq, d] replicated on every rank; pk/pv_shard: this rank's prefix tokens
    [P_r, Hkv, d]; sk/sv_local, lens_local: the suffixes of this rank's batch shard
    (`batch_shard(B, world, rank)`).  Returns this rank's output rows [nb, Hq, d].  The plan
    (buffers) is cached per shape, so repeated calls allocate nothing.
    """
    B, Hq, d = q.shape
    out_dtype = out_dtype or (torch.bfloat16 if q.dtype == torch.bfloat16 else torch.float32)
    key = (B, Hq, d, str(q.device), exchange_dtype, out_dtype, exchange, id(group), type(ops).__name__,
           dist.get_world_size(group), dist.get_rank(group))
    plan = _PLANS.get(key)
    if plan is None:
        plan = _PLANS[key] = SeqSplit(B, Hq, d, group=group, device=q.device, exchange_dtype=exchange_dtype,
                                      out_dtype=out_dtype, exchange=exchange, ops=ops)
    plan.ops = ops or plan.ops
    return plan(q, pk_shard, pv_shard, sk_local, sv_local, lens_local, scale=scale, return_lse=return_lse,
                check_range=check_range)


def release_plans():
    """Drop the cached sequence-split plans (their buffers)."""
    _PLANS.clear()
