"""Multi-GPU layer: one process per GPU, torch.distributed (NCCL) for the plumbing.

Two ways the shared-prefix decode attention shards:

* **KV-head sharding** (`head_shard`, `head_sharded_attention`): rank r owns KV heads
  [r*Hkv/N, (r+1)*Hkv/N) and their g*Hkv/N query heads, with their prefix and suffix
  K/V slices.  There is no collective: this is the tensor-parallel layout of the paper's
  end-to-end runs; the output stays head-sharded for the output projection.

* **Prefix sequence split** (`seqsplit_attention`), for a very long prefix with few KV
  heads (Yi-6B has 4 KV heads, so head sharding stops at 4 GPUs): rank r owns
  prefix tokens [r*P/N, (r+1)*P/N) for all heads and the batch shard
  [r*B/N, (r+1)*B/N) of the suffixes.  Each rank
    1. attends all B*g stacked queries to its prefix shard (tcgen05 prefix kernel),
    2. packs (O fp16, LSE fp32) of all rows (the combine kernel doing a 1-part combine with
       an f16 output); the rows of each destination rank's batch shard are contiguous,
    3. exchanges them all-to-all over NCCL (NVLink / NVSwitch): every rank receives only the
       N pieces of its own batch shard's rows -- 1/N of what an all-gather moves
       (`exchange="allgather"` keeps the all-gather of whole blocks for comparison),
    4. runs suffix attention for its batch shard,
    5. merges the N prefix pieces of its rows straight out of the received buffer
       (strided parts), then merges that with its suffix part -- both with the Eq. 5
       combine kernel, exactly as the single-GPU decomposition.
  fp16 (not bf16) is used for exchanged O: |O_r| <= max|V|, and fp16's 11-bit mantissa
  keeps the delivered bf16 output inside the parity gate.

The kernel calls go through an `ops` object (default: the CUDA library) so the
orchestration -- shard ranges, exchange layout, strides -- is exercised by world-size-2
gloo tests on CPU with reference ops.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous near-equal split of range(n) across `world` ranks."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


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

    def prefix(self, q, k, v, scale=None):
        return self._a.prefix_attn(q, k, v, scale=scale)

    def suffix(self, q, k, v, lens, scale=None, out=None, lse_out=None):
        return self._a.suffix_attn(q, k, v, lens, scale=scale, out=out, lse_out=lse_out)

    def combine(self, o_parts, lse_parts, out_dtype=torch.bfloat16, out=None, lse_out=None):
        return self._a.combine(o_parts, lse_parts, out_dtype=out_dtype, out=out, lse_out=lse_out)

    def attention(self, q, pk, pv, sk, sv, lens, scale=None):
        return self._a.hydragen_attention(q, pk, pv, sk, sv, lens, scale=scale)


def head_sharded_attention(q_local, pk_local, pv_local, sk_local, sv_local, lens, scale=None, ops=None):
    """Attention for this rank's KV-head shard (no communication)."""
    ops = ops or KernelOps()
    return ops.attention(q_local, pk_local, pv_local, sk_local, sv_local, lens, scale=scale)


def exchange_layout(B: int, Hq: int, d: int, exchange_dtype=torch.float16):
    """Byte layout of one rank's packed block: [O (B*Hq*d, exchange_dtype) | LSE (B*Hq, f32)]."""
    esz = torch.empty((), dtype=exchange_dtype).element_size()
    o_bytes = B * Hq * d * esz
    o_bytes = (o_bytes + 15) // 16 * 16  # keep the LSE region 16-B aligned
    return o_bytes, B * Hq * 4


def seqsplit_attention(q: torch.Tensor, pk_shard: torch.Tensor, pv_shard: torch.Tensor,
                       sk_local: torch.Tensor, sv_local: torch.Tensor, lens_local: torch.Tensor,
                       group: Optional[dist.ProcessGroup] = None, scale: Optional[float] = None,
                       exchange_dtype=torch.float16, out_dtype=None, ops=None, return_lse: bool = False,
                       exchange: str = "alltoall"):
    """Prefix sequence split across the ranks of `group` (see module docstring).

    q: [B, Hq, d] replicated on every rank; pk/pv_shard: this rank's prefix tokens
    [P_r, Hkv, d]; sk/sv_local, lens_local: the suffixes of this rank's batch shard
    (`shard_range(B, world, rank)`).  Returns the attention output of this rank's batch
    shard, [B_r, Hq, d].
    """
    ops = ops or KernelOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, Hq, d = q.shape
    b0, b1 = shard_range(B, world, rank)
    nb = b1 - b0
    dev = q.device
    out_dtype = out_dtype or (torch.bfloat16 if q.dtype == torch.bfloat16 else torch.float32)

    # 1-2. prefix pieces of all B*Hq rows over the local prefix shard, packed for the exchange
    o_p, l_p = ops.prefix(q, pk_shard, pv_shard, scale=scale)
    if exchange == "alltoall":
        # One slot of ceil(B/N) rows per destination rank; rank c's batch-shard rows are
        # packed at the start of slot c (pad rows are sent but never read).  Equal slots:
        # all_to_all_single without split sizes (the split-size form hangs process-group
        # teardown after CUDA-graph capture with this NCCL build).
        mb = -(-B // world)
        o_send = torch.empty(world * mb * Hq, d, dtype=exchange_dtype, device=dev)
        l_send = torch.empty(world * mb * Hq, dtype=torch.float32, device=dev)
        if B % world == 0:  # slots are exactly the shards: one pack for all rows
            ops.combine(o_p.view(1, B * Hq, d), l_p.view(1, B * Hq), out=o_send, lse_out=l_send)
        else:
            for c in range(world):
                c0, c1 = shard_range(B, world, c)
                if c1 > c0:
                    ops.combine(o_p[c0:c1].reshape(1, (c1 - c0) * Hq, d), l_p[c0:c1].reshape(1, (c1 - c0) * Hq),
                                out=o_send[c * mb * Hq:(c * mb + c1 - c0) * Hq],
                                lse_out=l_send[c * mb * Hq:(c * mb + c1 - c0) * Hq])
        o_all = torch.empty(world * mb * Hq, d, dtype=exchange_dtype, device=dev)
        l_all = torch.empty(world * mb * Hq, dtype=torch.float32, device=dev)
        dist.all_to_all_single(o_all, o_send, group=group)
        dist.all_to_all_single(l_all, l_send, group=group)
        return _finish(q, sk_local, sv_local, lens_local, o_all.view(world, mb * Hq, d)[:, : nb * Hq],
                       l_all.view(world, mb * Hq)[:, : nb * Hq], b0, b1, scale, out_dtype, ops, return_lse)
    o_bytes, l_bytes = exchange_layout(B, Hq, d, exchange_dtype)
    block = o_bytes + l_bytes
    send = torch.empty(block, dtype=torch.uint8, device=dev)
    o_send = send[: B * Hq * d * torch.empty((), dtype=exchange_dtype).element_size()].view(exchange_dtype)
    l_send = send[o_bytes:].view(torch.float32)
    ops.combine(o_p.view(1, B * Hq, d), l_p.view(1, B * Hq), out=o_send.view(B * Hq, d), lse_out=l_send)

    # 3. all-gather the packed blocks
    recv = torch.empty(world * block, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    blocks = recv.view(world, block)
    esz = torch.empty((), dtype=exchange_dtype).element_size()
    o_all = blocks[:, : B * Hq * d * esz].view(exchange_dtype).view(world, B, Hq, d)
    l_all = blocks[:, o_bytes:].view(torch.float32).view(world, B, Hq)
    return _finish(q, sk_local, sv_local, lens_local, o_all[:, b0:b1].reshape(world, nb * Hq, d),
                   l_all[:, b0:b1].reshape(world, nb * Hq), b0, b1, scale, out_dtype, ops, return_lse)


def _finish(q, sk_local, sv_local, lens_local, o_parts, l_parts, b0, b1, scale, out_dtype, ops, return_lse):
    """Steps 4-5: suffix of the batch shard, merge of the N exchanged prefix pieces of its
    rows (o_parts [N, rows, d], l_parts [N, rows], strided parts allowed), final merge."""
    B, Hq, d = q.shape
    nb = b1 - b0
    dev = q.device
    # 4. suffix of the local batch shard, written straight into part 1
    parts = torch.empty(2, nb * Hq, d, dtype=torch.float32, device=dev)
    lparts = torch.empty(2, nb * Hq, dtype=torch.float32, device=dev)
    if nb > 0:
        ops.suffix(q[b0:b1], sk_local, sv_local, lens_local, scale=scale, out=parts[1].view(nb, Hq, d),
                   lse_out=lparts[1].view(nb, Hq))
        # 5a. merge the world prefix pieces of these rows (strided parts of the exchanged buffer)
        ops.combine(o_parts, l_parts, out=parts[0], lse_out=lparts[0])
        # 5b. prefix (+) suffix
        out, lse = ops.combine(parts, lparts, out_dtype=out_dtype)
    else:
        out = torch.empty(0, d, dtype=out_dtype, device=dev)
        lse = torch.empty(0, dtype=torch.float32, device=dev)
    out = out.view(nb, Hq, d)
    return (out, lse.view(nb, Hq)) if return_lse else out
