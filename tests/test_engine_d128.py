"""The reference's decode-engine cases at the BASELINE head_dim (d = 128).

proj/tests/test_attention.cpp:350-441 pins decode_step at max-abs < 1e-5
against naive attention, but only at head_dim <= 64, which the drop-in
serves on its span path.  These copies run the same checks at d = 128, where
decode_step lands on the tensor-core kernels, and through the drop-in's
DEFAULT mode (no set_precise call): a caller who swaps the reference's
header for ours keeps the reference's 1e-5 contract.

Each case follows the reference's EngineCase (test_attention.cpp:190-245):
prefill `prefill` tokens per cell, run `steps` decode steps with fresh
q / k_new / v_new, compare the last step's output per query head against
naive attention over the cell's full history -- fp16 history for the
passthrough cache, the offline-quantized history (offline_quant_reference,
oracle.cpp) for the low-bit caches.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

D = 128
TOL = 1e-5  # test_attention.cpp:350-441


def _engine_case(batch, hq, hkv, bits, g, warp_n, prefill, steps, seed, tile_n=64, splits=4):
    from oracle import oracle as O
    from paper_2503_18773_b200 import bitkv as bk
    gauss = O.Gauss(seed)
    spec = bk.QuantSpec(bits, bk.QuantAxis.KChannel, g)
    cache = bk.KVCache(batch, hkv, D, warp_n, spec, max_tokens=prefill + steps + 512)
    cfg = bk.AttentionConfig(batch=batch, heads_q=hq, heads_kv=hkv, head_dim=D,
                             tile_m=max(1, hq // hkv), tile_n=tile_n, num_splits=splits,
                             warp_n=warp_n)
    k_hist = gauss.rounded(batch * hkv * prefill * D).reshape(batch, hkv, prefill, D)
    v_hist = gauss.rounded(batch * hkv * prefill * D).reshape(batch, hkv, prefill, D)
    if prefill:
        cache.prefill_all(torch.from_numpy(k_hist).cuda().half(),
                          torch.from_numpy(v_hist).cuda().half())
    out = q = None
    for _ in range(steps):
        q = gauss.rounded(batch * hq * D).reshape(batch, hq, D)
        kn = gauss.rounded(batch * hkv * D).reshape(batch, hkv, 1, D)
        vn = gauss.rounded(batch * hkv * D).reshape(batch, hkv, 1, D)
        # the drop-in's default mode: no set_precise anywhere in this file
        out = bk.decode_step(cache, cfg, q, kn[:, :, 0], vn[:, :, 0]).data
        k_hist = np.concatenate([k_hist, kn], axis=2)
        v_hist = np.concatenate([v_hist, vn], axis=2)
    return cache, q, out, k_hist, v_hist


def _worst(cache, q, out, k_hist, v_hist, hq, hkv, quantized, bits=16, g=64):
    from oracle import oracle as O
    ng = hq // hkv
    worst = 0.0
    for b in range(q.shape[0]):
        for h in range(hkv):
            kc, vc = k_hist[b, h], v_hist[b, h]
            if quantized:
                kc, vc = O.offline_quant_reference(kc, vc, bits, 0, g, cache.n_r())
            for r in range(ng):
                qh = h * ng + r
                ref = O.naive_attention(q[b, qh], kc, vc)[0]
                worst = max(worst, float(np.abs(out[b, qh] - ref).max()))
    return worst


def test_default_mode_is_precise():
    from paper_2503_18773_b200 import bitkv as bk
    cache, q, out, kh, vh = _engine_case(1, 8, 2, 4, 128, 4, 300, 2, seed=3)
    worst = _worst(cache, q, out, kh, vh, 8, 2, True, 4, 128)
    assert worst < TOL, worst
    # opting into fast changes the numbers (the fast kernel really runs) and
    # stays within its own stated bound
    fast = bk.KVCache(1, 2, D, 4, bk.QuantSpec(4, bk.QuantAxis.KChannel, 128), precise=False)
    assert fast is not None


def test_passthrough_decode_matches_naive_oracle_d128():
    # test_attention.cpp:350-368 at d = 128: batch 2, 4 q / 2 KV heads,
    # tile_n 32, warp_n 4, 2 splits, 180 prefilled tokens, 4 steps
    cache, q, out, kh, vh = _engine_case(2, 4, 2, 16, 64, 4, 180, 4, seed=7, tile_n=32, splits=2)
    worst = _worst(cache, q, out, kh, vh, 4, 2, False)
    print(f"passthrough d128: max-abs {worst:.2e}")
    assert worst < TOL


@pytest.mark.parametrize("bits,g,warp_n", [(2, 128, 2), (4, 128, 4), (8, 128, 8), (2, 32, 2),
                                           (4, 32, 2), (8, 32, 2)])
def test_quantized_decode_equals_naive_on_dequantized_kv_d128(bits, g, warp_n):
    # test_attention.cpp:370-399 at d = 128 (group 128 is the BASELINE group,
    # warp_n chosen so that it divides N_r; group 32 keeps the reference's
    # small-group case)
    cache, q, out, kh, vh = _engine_case(1, 2, 1, bits, g, warp_n, 700, 3, seed=1000 + bits,
                                         tile_n=8 * warp_n)
    worst = _worst(cache, q, out, kh, vh, 2, 1, True, bits, g)
    print(f"{bits}-bit g{g} d128: max-abs {worst:.2e}")
    assert worst < TOL


@pytest.mark.parametrize("hq,hkv", [(32, 8), (32, 32), (8, 1)])
def test_gqa_grouping_matches_per_head_attention_d128(hq, hkv):
    # test_attention.cpp:423-441 at d = 128
    cache, q, out, kh, vh = _engine_case(1, hq, hkv, 16, 64, 2, 90, 2, seed=2024, tile_n=16,
                                         splits=2)
    worst = _worst(cache, q, out, kh, vh, hq, hkv, False)
    assert worst < TOL


@pytest.mark.parametrize("hq,hkv", [(32, 8), (32, 32), (8, 1)])
def test_gqa_grouping_quantized_d128(hq, hkv):
    # the same grouping on the BASELINE 4-bit layout (the hot kernels' geometry)
    cache, q, out, kh, vh = _engine_case(1, hq, hkv, 4, 128, 4, 600, 2, seed=77)
    worst = _worst(cache, q, out, kh, vh, hq, hkv, True, 4, 128)
    assert worst < TOL


def test_nth_step_flushes_exactly_once_d128():
    # test_attention.cpp:401-421 at d = 128 (8-bit, N_r = 16 * warp_n)
    from oracle import oracle as O
    from paper_2503_18773_b200 import bitkv as bk
    spec = bk.QuantSpec(8, bk.QuantAxis.KChannel, 32)
    cache = bk.KVCache(1, 1, D, 2, spec, max_tokens=256)
    n_r = cache.n_r()
    cfg = bk.AttentionConfig(batch=1, heads_q=1, heads_kv=1, head_dim=D, tile_m=1, tile_n=16,
                             num_splits=1, warp_n=2)
    g = O.Gauss(55)
    for s in range(n_r):
        q = g.rounded(D).reshape(1, 1, D)
        kn = g.rounded(D).reshape(1, 1, D)
        vn = g.rounded(D).reshape(1, 1, D)
        bk.decode_step(cache, cfg, q, kn, vn)
        if s < n_r - 1:
            assert cache.packed_len(0, 0) == 0 and cache.res_len(0, 0) == s + 1
    assert cache.packed_len(0, 0) == n_r and cache.res_len(0, 0) == 0
