"""Span path (bdk_span.cu): decode_step for geometry outside the tensor-core
kernels' envelope, and the reference's attention internals (attend_tile,
partitioned_rowmax, residual_attend, packed_attend, combine;
attention.cpp:32-162), against the CPU oracle.

Tolerance: the reference's own 1e-5 max-abs (test_attention.cpp:54, :369,
:398) -- the span kernels keep the reference's summation order with unfused
fp32 arithmetic, so only expf differs."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

TOL = 1e-5

gpu = pytest.mark.gpu


def _bk():
    from paper_2503_18773_b200 import bitkv as bk
    return bk


def _naive(q, k, v):
    s = (q.astype(np.float64) @ k.astype(np.float64).T)
    s -= s.max(axis=1, keepdims=True)
    p = np.exp(s)
    return (p @ v.astype(np.float64)) / p.sum(axis=1, keepdims=True)


@gpu
@pytest.mark.parametrize("rows,len_,d,tile", [(1, 8, 32, 8), (4, 63, 32, 63), (3, 200, 16, 32),
                                             (8, 128, 128, 64), (2, 24, 8, 24)])
def test_attend_tile_matches_naive_softmax(rows, len_, d, tile):
    bk = _bk()
    g = O.Gauss(rows * 1000 + len_)
    q = g.rounded(rows * d).reshape(rows, d)
    k = g.rounded(len_ * d).reshape(len_, d)
    v = g.rounded(len_ * d).reshape(len_, d)
    st = bk.PartialOutput.init(rows, d)
    for t0 in range(0, len_, tile):
        n = min(tile, len_ - t0)
        bk.attend_tile(st, q, k[t0:t0 + n], v[t0:t0 + n], 1.0, warp_n=1)
    out = bk.combine([st])
    assert np.abs(out - _naive(q, k, v)).max() < TOL


@gpu
def test_partitioned_rowmax_is_exact_and_checks_partitions():
    bk = _bk()
    rng = np.random.default_rng(5)
    s = rng.standard_normal((7, 32)).astype(np.float32)
    for w in (1, 2, 4, 8, 32):
        assert np.array_equal(bk.partitioned_rowmax(s, w), s.max(axis=1))
    with pytest.raises(bk.ShapeError):
        bk.partitioned_rowmax(s, 5)


@gpu
def test_combine_is_lse_merge_and_order_invariant():
    bk = _bk()
    g = O.Gauss(37)
    rows, d, len_, tile = 2, 16, 96, 16
    q = g.rounded(rows * d).reshape(rows, d)
    k = g.rounded(len_ * d).reshape(len_, d)
    v = g.rounded(len_ * d).reshape(len_, d)
    parts = []
    for t0 in range(0, len_, 2 * tile):
        st = bk.PartialOutput.init(rows, d)
        for t in range(t0, t0 + 2 * tile, tile):
            bk.attend_tile(st, q, k[t:t + tile], v[t:t + tile], 0.25)
        parts.append(st)
    base = bk.combine(parts)
    assert np.abs(base - _naive(q * 0.25, k, v)).max() < TOL
    assert np.abs(bk.combine(parts[::-1]) - base).max() < 1e-6
    with pytest.raises(bk.EmptyInput):
        bk.combine([])


def _span_case(bits, axis, g, d, warp_n, hq, hkv, prefill, steps, tile_n, splits, seed):
    """decode steps through the device span path vs the oracle's decode_step"""
    bk = _bk()
    spec = bk.QuantSpec(bits, bk.QuantAxis(axis), g)
    gc = bk.KVCache(1, hkv, d, warp_n, spec, max_tokens=prefill + steps + 512)
    oc = O.OracleCache(1, hkv, d, warp_n, bits, axis, g, True, max_tokens=prefill + steps + 512)
    gauss = O.Gauss(seed)
    for h in range(hkv):
        k = gauss.rounded(prefill * d).reshape(prefill, d)
        v = gauss.rounded(prefill * d).reshape(prefill, d)
        oc.prefill(0, h, k, v)
        gc.prefill(0, h, k, v)
    cfg = bk.AttentionConfig(batch=1, heads_q=hq, heads_kv=hkv, head_dim=d, tile_m=hq // hkv,
                             tile_n=tile_n, num_splits=splits, warp_n=warp_n)
    worst = 0.0
    for _ in range(steps):
        q = gauss.rounded(hq * d).reshape(1, hq, d)
        kn = gauss.rounded(hkv * d).reshape(1, hkv, d)
        vn = gauss.rounded(hkv * d).reshape(1, hkv, d)
        ref = oc.decode_step(q, kn, vn, tile_n=tile_n, num_splits=splits)
        got = bk.decode_step(gc, cfg, q, kn, vn).data
        worst = max(worst, float(np.abs(got - ref).max()))
        for h in range(hkv):
            assert gc.packed_len(0, h) == oc.packed_len(0, h)
            assert gc.res_len(0, h) == oc.res_len(0, h)
    for h in range(hkv):
        for i in range(oc.packed_len(0, h) // oc.n_r):
            got, ref = gc.block(0, h, i), oc.block(0, h, i)
            assert np.array_equal(got.k_words, ref[0]) and np.array_equal(got.v_words, ref[1])
    return worst


@gpu
@pytest.mark.parametrize("bits,axis,g,d,warp_n,hq,hkv,prefill,steps,tile_n,splits", [
    (4, 0, 32, 64, 2, 4, 2, 300, 70, 32, 3),     # head_dim 64
    (2, 0, 16, 32, 2, 16, 1, 150, 40, 16, 2),    # n_group 16, 2-bit
    (8, 0, 16, 16, 1, 1, 1, 40, 20, 8, 4),       # 8-bit, N_r 16 (test_attention.cpp:401)
    (4, 1, 32, 96, 1, 6, 3, 100, 40, 8, 5),      # KToken keys, head_dim 96
    (16, 0, 64, 64, 4, 4, 2, 180, 36, 32, 2),    # fp16 passthrough (test_attention.cpp:350)
    (4, 0, 128, 128, 4, 64, 4, 600, 10, 64, 4),  # head_dim 128 with n_group 16
    # one requested split over ~300 tiles: decode_step raises the split count
    # (no CTA walks more than 4 tiles) -- the result stays within 1e-5
    (4, 0, 32, 64, 2, 4, 2, 5000, 3, 16, 1),
    # n_group 64, d 256, N_r 512: the K/V chunk stage and P.V sums do not fit
    # next to the score tile in shared memory, so the walk reads K/V from the
    # records and keeps the sums in global scratch (same order)
    (4, 0, 256, 256, 16, 64, 1, 600, 3, 128, 2),
])
def test_span_decode_matches_oracle(bits, axis, g, d, warp_n, hq, hkv, prefill, steps, tile_n,
                                    splits):
    worst = _span_case(bits, axis, g, d, warp_n, hq, hkv, prefill, steps, tile_n, splits,
                       seed=bits * 100 + d)
    assert worst < TOL, worst


@gpu
def test_residual_and_packed_attend_compose_to_decode():
    """residual_attend + packed_attend + combine over a cache equal naive
    attention on the cache's reconstruction (test_attention.cpp:285-348)"""
    bk = _bk()
    d, warp_n, bits, g = 32, 2, 4, 16
    spec = bk.QuantSpec(bits, bk.QuantAxis.KChannel, g)
    gc = bk.KVCache(1, 1, d, warp_n, spec)
    oc = O.OracleCache(1, 1, d, warp_n, bits, 0, g, True)
    gauss = O.Gauss(77)
    n = 3 * oc.n_r + 17
    k = gauss.rounded(n * d).reshape(n, d)
    v = gauss.rounded(n * d).reshape(n, d)
    gc.prefill(0, 0, k, v)
    oc.prefill(0, 0, k, v)
    kd, vd = oc.reconstruct(0, 0)
    q = gauss.rounded(2 * d).reshape(2, d)
    st = bk.PartialOutput.init(2, d)
    assert bk.residual_attend(gc, 0, 0, q, 1.0, st) is None
    for splits in (1, 2, 5, 64):
        parts = bk.packed_attend(gc, 0, 0, q, 16, splits, 1.0)
        assert len(parts) == min(splits, 3 * oc.n_r // 16)
        out = bk.combine([st] + parts)
        assert np.abs(out - _naive(q, kd, vd)).max() < TOL
    empty = bk.KVCache(1, 1, d, warp_n, spec)
    assert bk.packed_attend(empty, 0, 0, q, 16, 4, 1.0) == []
    with pytest.raises(bk.StateError):
        bk.residual_attend(empty, 0, 0, q, 1.0, bk.PartialOutput.init(2, d))
