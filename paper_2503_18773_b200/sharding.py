"""Single-box partitioning of the decode path.

One process per GPU, ``torch.distributed`` over NCCL for the plumbing.

* KV-head sharding (config C3): cells (b, h_kv) are independent, so rank p owns
  a contiguous range of KV heads for every batch row, plus the matching query
  heads ``h*n_group + g`` (attention.cpp:207-212).  No communication on the
  data path.
* Sequence split (config C5, 128K at batch 1): the packed blocks of every cell
  are divided into contiguous, block-aligned ranges; the residual window (and
  every append / flush) lives on the last rank.  Each rank computes the
  normalized partial output and log2-sum-exp of its range
  (``bdk_decode_partial``); one all-gather of the packed ``[o | lse]`` buffer
  exchanges them and every rank LSE-merges locally (``bdk_merge_partials``,
  the math of combine, attention.cpp:142-162).  Results are split-invariant
  within the reference's own tolerance (test_attention.cpp:312-340).
"""
from __future__ import annotations


def block_range(n_blocks: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block range of `rank`: the first n_blocks % world ranks get
    one extra block (the split rule of packed_attend, attention.cpp:116-130)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, rem = divmod(n_blocks, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def head_range(heads_kv: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous KV-head range of `rank` (KV-head sharding, config C3)."""
    if heads_kv % world:
        raise ValueError(f"heads_kv ({heads_kv}) must be divisible by the world size ({world})")
    per = heads_kv // world
    return rank * per, (rank + 1) * per


def query_head_range(heads_q: int, heads_kv: int, world: int, rank: int) -> tuple[int, int]:
    """Query heads served by the KV heads of `rank` (consecutive per KV head,
    config.cpp:43-49)."""
    lo, hi = head_range(heads_kv, world, rank)
    g = heads_q // heads_kv
    return lo * g, hi * g


class SeqSplitComm:
    """Exchange buffers of the sequence split.

    ``o`` [rows, d] and ``lse`` [rows] are views into one contiguous send
    buffer, so a partial decode writes straight into it and a single
    ``all_gather_into_tensor`` moves rows*(d+1) fp32 per rank."""

    def __init__(self, world: int, rows: int, d: int, device, group=None):
        import torch
        self.world, self.rows, self.d, self.group = world, rows, d, group
        self.part = rows * d + rows
        self.send = torch.zeros(self.part, dtype=torch.float32, device=device)
        # flat receive buffer (gloo's all_gather_into_tensor wants 1-D);
        # recv2d is the [world, part] view
        self.recv = torch.zeros(world * self.part, dtype=torch.float32, device=device)
        self.recv2d = self.recv.view(world, self.part)
        self.o = self.send[: rows * d].view(rows, d)
        self.lse = self.send[rows * d:]

    def exchange(self):
        """All-gather the packed partials; returns strided (o_parts, lse_parts)
        views [world, rows, d] / [world, rows] into the receive buffer."""
        import torch.distributed as dist
        if self.world > 1:
            dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        else:
            self.recv2d[0].copy_(self.send)
        o_parts = self.recv2d[:, : self.rows * self.d].unflatten(1, (self.rows, self.d))
        lse_parts = self.recv2d[:, self.rows * self.d:]
        return o_parts, lse_parts

    def merge(self, out):
        """exchange + on-device LSE merge into ``out`` [rows..., d]."""
        from . import bitkv
        o_parts, lse_parts = self.exchange()
        return bitkv.merge_partials(o_parts, lse_parts, out=out.view(self.rows, self.d))
