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
  ``PeerSeqSplit`` does the same exchange without NCCL: every rank's merge
  kernel reads the peers' partials straight out of their HBM over NVLink
  (bdk_peer_merge); ``SeqSplitComm`` is the NCCL all-gather version.
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


class PeerSeqSplit:
    """Sequence-split exchange over peer memory: one ``bdk_peer_merge`` launch
    per rank and step, no collective library on the data path.

    Every rank owns a buffer of two slots ``[2, rows*d + rows]`` (fp32 o then
    lse, the layout ``bdk_decode_partial`` writes) and a u32 step flag.  Step s
    (1, 2, ...) uses slot s % 2: ``next_slot()`` returns the (o, lse) views the
    rank's partial decode writes, then ``merge(out)`` publishes the step and
    merges every rank's slot into ``out``.  Across processes the buffers and
    flags are shared with CUDA IPC (torch's tensor reductions, exchanged once
    with ``all_gather_object``); peers on other GPUs are reached through the
    peer mapping the IPC open enables.  ``local_group`` builds the ranks of
    one process (e.g. one GPU, one stream per rank) for tests."""

    def __init__(self, world: int, rank: int, rows: int, d: int, device, group=None,
                 _shared=None, timeout_s: float = 2.0):
        import torch
        self.world, self.rank, self.rows, self.d = world, rank, rows, d
        self.part = rows * d + rows
        self.buf = torch.zeros((2, self.part), dtype=torch.float32, device=device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        self.timeout_ns = int(timeout_s * 1e9)
        self.step = 0
        self._keep = []
        if _shared is None:
            _shared = [(self.buf, self.flag)] if world == 1 else self._exchange(group)
        self._bind(_shared)

    def _exchange(self, group):
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        mine = (reduce_tensor(self.buf), reduce_tensor(self.flag))
        objs = [None] * self.world
        dist.all_gather_object(objs, mine, group=group)
        shared = []
        for p, (rb, rf) in enumerate(objs):
            if p == self.rank:
                shared.append((self.buf, self.flag))
            else:
                shared.append((rb[0](*rb[1]), rf[0](*rf[1])))
        return shared

    def _bind(self, shared):
        import ctypes as C
        self._keep = shared
        W = C.c_void_p * self.world
        self._parts = [W(*[b[slot].data_ptr() for b, _ in shared]) for slot in (0, 1)]
        self._flags = W(*[f.data_ptr() for _, f in shared])

    @classmethod
    def local_group(cls, world: int, rows: int, d: int, device) -> list["PeerSeqSplit"]:
        """All ranks of one process sharing plain device pointers."""
        ranks = [cls(1, 0, rows, d, device) for _ in range(world)]
        shared = [(r.buf, r.flag) for r in ranks]
        for i, r in enumerate(ranks):
            r.world, r.rank = world, i
            r._bind(shared)
        return ranks

    def next_slot(self):
        """(o [rows, d], lse [rows]) views this rank's partial of the next step
        is written into."""
        slot = self.buf[(self.step + 1) % 2]
        return slot[: self.rows * self.d].view(self.rows, self.d), slot[self.rows * self.d:]

    def merge(self, out, out_lse=None, stream=None) -> None:
        """Publish the next step and LSE-merge every rank's partial into out."""
        import ctypes as C
        from . import _lib as L
        from . import bitkv
        self.step += 1
        vp = C.c_void_p
        st = L.load().bdk_peer_merge(
            self._parts[self.step % 2], self._flags, self.world, self.rank, self.step, self.rows,
            self.d, vp(out.data_ptr()), vp(out_lse.data_ptr()) if out_lse is not None else None,
            vp(self.err.data_ptr()), self.timeout_ns,
            stream if stream is not None else bitkv._stream_ptr())
        bitkv._check(st)

    def check(self) -> None:
        """Raise if a merge timed out waiting for a peer (reads the device flag)."""
        from . import bitkv
        if int(self.err.item()):
            raise bitkv.CudaError("peer_merge: a peer did not publish its partial in time")
