"""The reference's quant.hpp / layout.hpp API as the drop-in exposes it.

layout.hpp helpers are word-layout metadata (CPU tests against the
reference KATs in tests/golden/kat.json).  The quant.hpp functions run on
the device (bdk_quantize_tile & co.) and are checked against the same KATs
and against the oracle's group quantization (GPU tests)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2503_18773_b200 import bitkv as bk

KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kat.json")))


def test_orders_match_reference_kats():  # test_layout.cpp:13-26
    for bits, order in KAT["interleave_order"].items():
        if bits == "cite":
            continue
        assert bk.interleave_order(int(bits)) == order
        assert bk.identity_order(int(bits)) == list(range(16 // int(bits)))
    with pytest.raises(bk.UnsupportedBits):
        bk.interleave_order(3)


def test_pack_word_matches_reference_kats():  # test_layout.cpp:28-39 + random reference words
    for codes, bits, il, word in KAT["pack_word"]["cases"] + KAT["pack_word_random"]["cases"]:
        order = bk.interleave_order(bits) if il else bk.identity_order(bits)
        assert bk.pack_word(codes, bits, order) == word
        assert bk.unpack_word(word, bits, order) == list(codes)
    with pytest.raises(bk.CodeOverflow):
        bk.pack_word([16, 0, 0, 0], 4, bk.interleave_order(4))


def test_block_geometry_helpers():  # test_layout.cpp:70-83
    for bits, wn, n_r in KAT["residual_block_size"]["cases"]:
        assert bk.residual_block_size(bits, wn) == n_r
    assert bk.iteration_count(64, 4) == 2
    with pytest.raises(bk.ShapeError):
        bk.iteration_count(60, 4)


@pytest.mark.gpu
def test_group_params_and_quantize_kats_on_device():  # test_quant.cpp:27-69
    for x, bits, scale, zero in KAT["group_params"]["cases"]:
        gp = bk.compute_group_params(np.array(x, np.float32), bits)
        assert np.float32(gp.scale) == np.float32(scale) and np.float32(gp.zero) == np.float32(zero)
    r = KAT["quantize_rne"]
    codes = bk.quantize_group(np.array(r["group"], np.float32), r["scale"], r["zero"], r["bits"])
    assert codes.tolist() == r["codes"]
    vals = bk.dequantize_group(codes, r["scale"], r["zero"])
    ref = (codes.astype(np.float32) * np.float32(r["scale"])).astype(np.float32) + np.float32(r["zero"])
    assert np.array_equal(vals, ref.astype(np.float32))


@pytest.mark.gpu
@pytest.mark.parametrize("bits,axis,g", [(4, 0, 16), (2, 1, 8), (8, 0, 32), (4, 1, 128)])
def test_quantize_tile_round_trip_matches_oracle_groups(bits, axis, g):
    """quantize_tile (quant.cpp:47-93): params in push order and codes equal
    the oracle's per-group quantization; dequantize_tile rounds to binary16
    (quant.cpp:95-110)."""
    from oracle import oracle as O
    rows, d = 64, 128
    x = O.Gauss(bits * 7 + axis).rounded(rows * d).reshape(rows, d)
    x[3, :] = 0.0
    x[:, 5] = -0.0
    qt = bk.quantize_tile(x, bits, bk.QuantAxis(axis), g)
    groups = [(gr, c) for gr in range(rows // g) for c in range(d)] if axis == 0 else \
        [(t, gc) for t in range(rows) for gc in range(d // g)]
    for i, (a, b_) in enumerate(groups):
        grp = x[a * g:(a + 1) * g, b_] if axis == 0 else x[a, b_ * g:(b_ + 1) * g]
        s, z = O.group_params(grp, bits)
        assert qt.params.scale(i) == np.float32(s) and qt.params.zero(i) == np.float32(z)
        got = qt.codes[a * g:(a + 1) * g, b_] if axis == 0 else qt.codes[a, b_ * g:(b_ + 1) * g]
        assert np.array_equal(got, O.quantize_group(grp, s, z, bits))
    y = bk.dequantize_tile(qt.codes, qt.params, rows, d, bk.QuantAxis(axis), g)
    assert np.array_equal(y, y.astype(np.float16).astype(np.float32))
    with pytest.raises(bk.ShapeError):
        bk.quantize_tile(x[:, :100], bits, bk.QuantAxis(1), 64)


def test_pack_block_codes_round_trip_and_word_order():  # kvcache.cpp:79-112
    rng = np.random.default_rng(3)
    for bits in (2, 4, 8, 16):
        n_r, d = 8 * (16 // bits) * 2, 16
        codes = rng.integers(0, 1 << bits, (n_r, d), dtype=np.uint32).astype(np.uint16)
        order = bk.interleave_order(bits)
        words = bk.pack_block_codes(codes, n_r, d, bits, order)
        p = 16 // bits
        # word (c, g) packs tokens g*p .. g*p+p-1 of channel c (pack_word)
        assert words[3 * (n_r // p) + 1] == bk.pack_word(codes[p:2 * p, 3], bits, order)
        assert np.array_equal(bk.unpack_block_codes(words, n_r, d, bits, order), codes)
