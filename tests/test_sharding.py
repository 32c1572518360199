"""Host-side logic of the multi-GPU paths (paper_2503_18773_b200/sharding.py).

CPU only: the range planners, and the sequence-split exchange over a
world-size-2 ``gloo`` group.  Each rank computes the normalized partial output
and log2-sum-exp of its contiguous block range (numpy, test side), writes them
into the SeqSplitComm send views, all-gathers, and the LSE merge of the
gathered parts (combine, attention.cpp:142-162) must equal attention over the
whole context.  On the GPU the same exchange feeds bdk_merge_partials.
"""
import os
import socket

import numpy as np
import pytest

from paper_2503_18773_b200 import sharding


def test_block_range_partitions_contiguously():
    for n in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            spans = [sharding.block_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sharding.block_range(10, 2, 2)


def test_head_ranges():
    assert [sharding.head_range(32, 4, r) for r in range(4)] == [(0, 8), (8, 16), (16, 24),
                                                                (24, 32)]
    assert sharding.query_head_range(32, 8, 2, 1) == (16, 32)
    with pytest.raises(ValueError):
        sharding.head_range(8, 3, 0)


def _partial(q, k, v):
    """normalized o and log2-sum-exp of q over (k, v) in the exp2 domain."""
    s = (q @ k.T) / np.sqrt(q.shape[-1]) * np.log2(np.e)
    m = s.max(axis=1, keepdims=True)
    p = np.exp2(s - m)
    l_ = p.sum(axis=1, keepdims=True)
    return (p @ v) / l_, (m + np.log2(l_))[:, 0]


def _merge(o_parts, lse_parts):
    ms = lse_parts.max(axis=0)
    w = np.exp2(lse_parts - ms)
    return (o_parts * w[..., None]).sum(0) / w.sum(0)[..., None]


def _worker(rank, world, port, data, out_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v, n_r = data
        nblk = k.shape[0] // n_r
        lo, hi = sharding.block_range(nblk, world, rank)
        t_hi = hi * n_r if rank < world - 1 else k.shape[0]  # residual tail on the last rank
        comm = sharding.SeqSplitComm(world, q.shape[0], q.shape[1], "cpu")
        o, lse = _partial(q, k[lo * n_r:t_hi], v[lo * n_r:t_hi])
        comm.o.copy_(torch.from_numpy(o.astype(np.float32)))
        comm.lse.copy_(torch.from_numpy(lse.astype(np.float32)))
        o_parts, lse_parts = comm.exchange()
        merged = _merge(o_parts.numpy().astype(np.float64), lse_parts.numpy().astype(np.float64))
        out_q.put((rank, merged))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_seq_split_exchange_and_merge_over_gloo(world):
    import torch.multiprocessing as mp
    rng = np.random.default_rng(0)
    n_r, d, rows = 128, 128, 4
    length = 5 * n_r + 37
    q = rng.standard_normal((rows, d))
    k = rng.standard_normal((length, d))
    v = rng.standard_normal((length, d))
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (q, k, v, n_r), out_q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(out_q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full, _ = _partial(q, k, v)
    for r in range(world):
        np.testing.assert_allclose(results[r], full, atol=1e-5, rtol=0)


def _peer_worker(rank, world, port, data, out_q):
    """One process per rank on ONE GPU: the peer-memory exchange with its
    buffers and flags shared over CUDA IPC (the multi-GPU plumbing of
    PeerSeqSplit).  Partials are computed on the host (numpy) and copied into
    this rank's slot; bdk_peer_merge does the exchange + merge."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        q, k, v, n_r = data
        nblk = k.shape[0] // n_r
        lo, hi = sharding.block_range(nblk, world, rank)
        t_hi = hi * n_r if rank < world - 1 else k.shape[0]
        comm = sharding.PeerSeqSplit(world, rank, q.shape[0], q.shape[1], torch.device("cuda", 0),
                                     timeout_s=20.0)
        outs = []
        for step in range(2):
            o, lse = _partial(q * (step + 1), k[lo * n_r:t_hi], v[lo * n_r:t_hi])
            so, sl = comm.next_slot()
            so.copy_(torch.from_numpy(o.astype(np.float32)))
            sl.copy_(torch.from_numpy(lse.astype(np.float32)))
            out = torch.empty((q.shape[0], q.shape[1]), dtype=torch.float32, device="cuda")
            comm.merge(out)
            torch.cuda.synchronize()
            comm.check()
            outs.append(out.cpu().numpy().astype(np.float64))
        dist.barrier()  # peers keep their buffers mapped until everyone is done
        out_q.put((rank, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_merge_across_processes_over_cuda_ipc():
    import torch.multiprocessing as mp
    world = 2
    rng = np.random.default_rng(1)
    n_r, d, rows = 128, 128, 4
    length = 6 * n_r + 11
    q = rng.standard_normal((rows, d))
    k = rng.standard_normal((length, d))
    v = rng.standard_normal((length, d))
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, (q, k, v, n_r), out_q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(out_q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for step in range(2):
        full, _ = _partial(q * (step + 1), k, v)
        for r in range(world):
            np.testing.assert_allclose(results[r][step], full, atol=1e-5, rtol=0)
