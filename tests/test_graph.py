"""Graph-captured steady-state decode (Algorithm 2's loop).

A step is one launch -- append, attention, combine and the flush of a
residual window that fills (build_block + commit_block, kvcache.cpp:208-237,
committed after the step's attention as in attention.cpp:235-240) --
scheduled on the device from the device lengths.  So one captured graph of
n steps replays at any cache state: replays are bit-identical to the same
steps run eagerly, across >= 2 flushes, and the flushed blocks are
bit-exact against the CPU oracle (kvcache.cpp:170-251; flush timing pinned
by proj/tests/test_attention.cpp:401-421)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

D = 128
FAST_TOL = {"max_abs": 2e-3, "rel_l2": 1e-3}


def _setup(bits, warp_n, batch, hq, hkv, prefill, max_tokens, seed):
    from oracle import oracle as O
    from paper_2503_18773_b200 import bitkv as bk
    g = O.Gauss(seed)
    k = g.rounded(batch * hkv * prefill * D).reshape(batch, hkv, prefill, D)
    v = g.rounded(batch * hkv * prefill * D).reshape(batch, hkv, prefill, D)
    spec = bk.QuantSpec(bits, bk.QuantAxis.KChannel, 128)
    caches = []
    for _ in range(2):
        c = bk.KVCache(batch, hkv, D, warp_n, spec, max_tokens=max_tokens, precise=False)
        c.prefill_all(torch.from_numpy(k).cuda().half(), torch.from_numpy(v).cuda().half())
        caches.append(c)
    oc = O.OracleCache(batch, hkv, D, warp_n, bits, 0, 128, True, max_tokens=max_tokens)
    for b in range(batch):
        for h in range(hkv):
            oc.prefill(b, h, k[b, h], v[b, h])
    cfg = bk.AttentionConfig(batch=batch, heads_q=hq, heads_kv=hkv, head_dim=D,
                             tile_m=hq // hkv, tile_n=64, num_splits=4, warp_n=warp_n)
    return g, caches, oc, cfg


@pytest.mark.parametrize("bits,warp_n,prefill,n,launches", [(4, 4, 1000, 50, 4),
                                                            (2, 4, 250, 70, 4)])
def test_graph_replay_is_bit_identical_to_eager_across_flushes(bits, warp_n, prefill, n,
                                                               launches):
    from paper_2503_18773_b200 import bitkv as bk
    batch, hq, hkv = 2, 8, 2
    g, (eager, graphed), oc, cfg = _setup(bits, warp_n, batch, hq, hkv, prefill,
                                          prefill + n * launches + 64, seed=bits * 7)
    n_r = eager.n_r()
    flushes = sum(1 for s in range(1, n * launches + 1) if (prefill + s) % n_r == 0)
    assert flushes >= 2
    qs = torch.empty((n, batch, hq, D), dtype=torch.float16, device="cuda")
    ks = torch.empty((n, batch, hkv, D), dtype=torch.float16, device="cuda")
    vs = torch.empty_like(ks)
    outs = torch.empty((n, batch, hq, D), dtype=torch.float32, device="cuda")
    graph = bk.DecodeGraph(graphed, cfg, qs, ks, vs, outs)
    worst = {"max_abs": 0.0, "rel_l2": 0.0}
    for launch in range(launches):
        q = g.rounded(n * batch * hq * D).reshape(n, batch, hq, D)
        kn = g.rounded(n * batch * hkv * D).reshape(n, batch, hkv, D)
        vn = g.rounded(n * batch * hkv * D).reshape(n, batch, hkv, D)
        qs.copy_(torch.from_numpy(q))
        ks.copy_(torch.from_numpy(kn))
        vs.copy_(torch.from_numpy(vn))
        graph.launch()
        for i in range(n):
            ref_eager = bk.decode_step(eager, cfg, qs[i], ks[i], vs[i]).data
            torch.cuda.synchronize()
            assert torch.equal(outs[i], ref_eager), (launch, i)  # bit-identical
            ref = oc.decode_step(q[i], kn[i], vn[i])
            got = outs[i].cpu().numpy().astype(np.float64)
            d = got - ref
            worst["max_abs"] = max(worst["max_abs"], float(np.abs(d).max()))
            worst["rel_l2"] = max(worst["rel_l2"], float(np.linalg.norm(d) / np.linalg.norm(ref)))
    graph.close()
    assert worst["max_abs"] < FAST_TOL["max_abs"] and worst["rel_l2"] < FAST_TOL["rel_l2"], worst
    for b in range(batch):
        for h in range(hkv):
            assert graphed.packed_len(b, h) == eager.packed_len(b, h) == oc.packed_len(b, h)
            assert graphed.res_len(b, h) == eager.res_len(b, h) == oc.res_len(b, h)
            for i in range(oc.packed_len(b, h) // n_r):
                x, y, r = graphed.block(b, h, i), eager.block(b, h, i), oc.block(b, h, i)
                assert x == y
                assert np.array_equal(x.k_words, r[0]) and np.array_equal(x.v_words, r[1])
                assert np.array_equal(x.k_params, r[2]) and np.array_equal(x.v_params, r[3])
            rk, rv = graphed.residual_tile(b, h)
            ok_, ov_ = oc.residual(b, h)
            assert np.array_equal(rk, ok_) and np.array_equal(rv, ov_)


def test_graph_launch_checks_capacity_and_mode():
    from paper_2503_18773_b200 import bitkv as bk
    batch, hq, hkv, n = 1, 8, 2, 40
    _, (c, other), _, cfg = _setup(4, 4, batch, hq, hkv, 120, 256, seed=3)
    qs = torch.zeros((n, batch, hq, D), dtype=torch.float16, device="cuda")
    ks = torch.zeros((n, batch, hkv, D), dtype=torch.float16, device="cuda")
    outs = torch.empty((n, batch, hq, D), dtype=torch.float32, device="cuda")
    graph = bk.DecodeGraph(c, cfg, qs, ks, ks, outs)
    # max_tokens 256 -> 3 block slots (bdk_cache_create): flushes at tokens
    # 128, 256 and 384 fit, the one at 512 (launch 10: 480 -> 520) does not
    for _ in range(9):
        graph.launch()
    with pytest.raises(bk.CapacityError):
        graph.launch()
    torch.cuda.synchronize()
    assert c.packed_len(0, 0) == 384 and c.res_len(0, 0) == 96
    graph.close()
    other.set_precise(True)
    with pytest.raises(bk.Unsupported):
        bk.DecodeGraph(other, cfg, qs, ks, ks, outs)
