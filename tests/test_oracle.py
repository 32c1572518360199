"""Pin the CPU oracle (oracle/bitkv_oracle.c) to the reference.  CPU only.

(a) against tests/golden/, generated from the UNMODIFIED reference engine by
    tests/golden/make_golden.py: the KATs of the reference's own doctest
    suites, run_bench output checksums (bench.cpp:80-210), per-geometry block
    hashes and decode_step outputs;
(b) against oracle/_ref (the reference compiled out-of-tree) directly on fresh
    seeded cases, when that library is present.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


KAT = load("kat.json")
BLOCKS = load("blocks.json")


# ------------------------------------------------------------------ KATs
def test_interleave_orders():  # test_layout.cpp:13-26
    for bits in (2, 4, 8, 16):
        assert O.perm(bits) == KAT["interleave_order"][str(bits)]
    assert O.perm(4, interleave=False) == [0, 1, 2, 3]
    with pytest.raises(O.OracleError):
        O.perm(3)


def test_pack_word_kats():  # test_layout.cpp:28-39 + random reference words
    for codes, bits, il, word in KAT["pack_word"]["cases"] + KAT["pack_word_random"]["cases"]:
        assert O.pack_word(codes, bits, bool(il)) == word
        assert O.unpack_word(word, bits, bool(il)) == codes
    with pytest.raises(O.OracleError) as e:  # test_layout.cpp:41-45
        O.pack_word([1, 2, 16, 4], 4)
    assert e.value.kind == "CodeOverflow"


@pytest.mark.parametrize("bits", [2, 4, 8, 16])
@pytest.mark.parametrize("il", [True, False])
def test_every_word_round_trips(bits, il):  # test_layout.cpp:56-68 (exhaustive)
    for w in range(0, 1 << 16, 7 if bits != 16 else 1):
        assert O.pack_word(O.unpack_word(w, bits, il), bits, il) == w


def test_residual_block_size():  # test_layout.cpp:70-83
    for bits, wn, n_r in KAT["residual_block_size"]["cases"]:
        assert O.residual_block_size(bits, wn) == n_r


def test_group_params_match_reference_bit_exact():  # quant.cpp:18-28
    for grp, bits, s, z in KAT["group_params"]["cases"]:
        gs, gz = O.group_params(np.array(grp, np.float32), bits)
        assert np.float32(gs).tobytes() == np.float32(s).tobytes(), (grp, bits)
        assert np.float32(gz).tobytes() == np.float32(z).tobytes(), (grp, bits)


def test_quantize_rounds_half_to_even():  # test_quant.cpp:62-69
    k = KAT["quantize_rne"]
    codes = O.quantize_group(np.array(k["group"], np.float32), k["scale"], k["zero"], k["bits"])
    assert codes.tolist() == k["codes"]


def test_fp16_kats():  # test_fp16.cpp:24-53
    for x, bits in KAT["fp16"]["to_bits"]:
        assert O.f32_to_f16_bits(x) == bits, x
    for bits, x in KAT["fp16"]["from_bits"]:
        assert O.f16_bits_to_f32(bits) == x


def test_fp16_narrowing_matches_numpy_rne_on_a_sweep():
    xs = np.random.default_rng(1).standard_normal(20000).astype(np.float32) * 3000
    xs = np.concatenate([xs, np.float32(2.0) ** np.arange(-30, 17, dtype=np.float32)])
    with np.errstate(over="ignore"):
        want = xs.astype(np.float16).view(np.uint16)
    got = np.array([O.f32_to_f16_bits(float(x)) for x in xs], np.uint16)
    assert np.array_equal(got, want)


# ------------------------------------------------- run_bench checksums
def _bench_checksum(c):
    """Restates run_bench's workload (bench.cpp:80-210) on the oracle."""
    g = O.Gauss(c["seed"])
    batch, hq, hkv, d = c["batch"], c["heads_q"], c["heads_kv"], c["head_dim"]
    oc = O.OracleCache(batch, hkv, d, c["warp_n"], c["bits"], c["k_axis"], c["group_size"],
                       bool(c["interleave"]), max_tokens=c["seq_len"] + c["steps"] + 1024)
    for b in range(batch):
        for h in range(hkv):
            k = g.rounded(c["seq_len"] * d).reshape(c["seq_len"], d)
            v = g.rounded(c["seq_len"] * d).reshape(c["seq_len"], d)
            oc.prefill(b, h, k, v)
    ck = 0xCBF29CE484222325
    for _ in range(c["steps"]):
        q = np.zeros((batch, hq, d), np.float32)
        kn = np.zeros((batch, hkv, d), np.float32)
        vn = np.zeros((batch, hkv, d), np.float32)
        for b in range(batch):
            q[b] = g.rounded(hq * d).reshape(hq, d)
            for h in range(hkv):
                kn[b, h] = g.rounded(d)
                vn[b, h] = g.rounded(d)
        out = oc.decode_step(q, kn, vn, tile_n=c["tile_n"], num_splits=c["num_splits"],
                             warp_n=c["warp_n"], threads=1)
        ck = O.fnv1a64(out, ck)
    return ck


@pytest.mark.parametrize("i", range(len(KAT["run_bench_checksums"]["cases"])))
def test_oracle_reproduces_reference_run_bench_checksum(i):
    c = KAT["run_bench_checksums"]["cases"][i]
    assert f"{_bench_checksum(c):016x}" == c["output_checksum"]


# ------------------------------------------------------ block fixtures
def _oracle_block_hashes(fx):
    oc = O.OracleCache(fx["batch"], fx["heads_kv"], fx["head_dim"], fx["warp_n"], fx["bits"],
                       fx["k_axis"], fx["group_size"], bool(fx["interleave"]),
                       max_tokens=fx["seq"] + 1024)
    g = O.Gauss(fx["seed"])
    for b in range(fx["batch"]):
        for h in range(fx["heads_kv"]):
            k = g.rounded(fx["seq"] * fx["head_dim"]).reshape(fx["seq"], -1)
            v = g.rounded(fx["seq"] * fx["head_dim"]).reshape(fx["seq"], -1)
            oc.prefill(b, h, k, v)
    out = []
    for cell in fx["cells"]:
        b, h = cell["b"], cell["h"]
        hs = hashlib.sha256()
        for i in range(oc.packed_len(b, h) // oc.n_r):
            for a in oc.block(b, h, i):
                hs.update(a.astype("<u2").tobytes())
        rk, rv = oc.residual(b, h)
        hr = hashlib.sha256()
        hr.update(rk.astype(np.float16).view(np.uint16).astype("<u2").tobytes())
        hr.update(rv.astype(np.float16).view(np.uint16).astype("<u2").tobytes())
        out.append((oc.packed_len(b, h), oc.res_len(b, h), hs.hexdigest(), hr.hexdigest()))
    return out


@pytest.mark.parametrize("fx", BLOCKS, ids=[f["name"] for f in BLOCKS])
def test_oracle_blocks_match_reference_golden(fx):
    got = _oracle_block_hashes(fx)
    for cell, (pl, rl, hb, hr) in zip(fx["cells"], got):
        assert (pl, rl) == (cell["packed_len"], cell["res_len"])
        assert hb == cell["blocks_sha256"], (fx["name"], cell["b"], cell["h"])
        assert hr == cell["residual_sha256"]


# ------------------------------------------------------ decode fixtures
@pytest.mark.parametrize("name", ["decode_4bit_gqa", "decode_2bit_wn4_flush", "decode_16bit"])
def test_oracle_decode_matches_reference_golden(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    batch, hq, hkv, seq, bits, wn, g, axis, steps, seed = z["meta"].tolist()
    oc = O.OracleCache(batch, hkv, 128, wn, bits, axis, g, True, max_tokens=seq + steps + 512)
    gauss = O.Gauss(seed)
    for b in range(batch):
        for h in range(hkv):
            k = gauss.rounded(seq * 128).reshape(seq, 128)
            v = gauss.rounded(seq * 128).reshape(seq, 128)
            oc.prefill(b, h, k, v)
    for s in range(steps):
        out = oc.decode_step(z["q"][s], z["k_new"][s], z["v_new"][s], tile_n=64, num_splits=4,
                             threads=2)
        assert np.array_equal(out, z["out"][s]), (name, s, np.abs(out - z["out"][s]).max())


# ------------------------------------------- live reference cross-checks
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("bits,wn,g,axis,il", [(4, 4, 128, 0, 1), (2, 2, 64, 0, 1),
                                               (8, 1, 16, 1, 0), (16, 2, 64, 0, 1),
                                               (2, 8, 128, 0, 0)])
def test_oracle_decode_equals_live_reference(bits, wn, g, axis, il):
    n_r = 8 * wn * (16 // bits)
    seq = 3 * n_r - 2  # residual 2 short of full: the 2nd step below flushes
    batch, hq, hkv = 2, 8, 2
    rc = O.RefCache(batch, hkv, 128, wn, bits, axis, g, bool(il))
    oc = O.OracleCache(batch, hkv, 128, wn, bits, axis, g, bool(il), max_tokens=seq + n_r * 3)
    gauss = O.Gauss(bits * 10 + wn)
    for b in range(batch):
        for h in range(hkv):
            k = gauss.rounded(seq * 128).reshape(seq, 128)
            v = gauss.rounded(seq * 128).reshape(seq, 128)
            rc.prefill(b, h, k, v)
            oc.prefill(b, h, k, v)
    for _ in range(4):  # crosses a flush
        q = gauss.rounded(batch * hq * 128).reshape(batch, hq, 128)
        kn = gauss.rounded(batch * hkv * 128).reshape(batch, hkv, 128)
        vn = gauss.rounded(batch * hkv * 128).reshape(batch, hkv, 128)
        assert np.array_equal(rc.decode_step(q, kn, vn), oc.decode_step(q, kn, vn, threads=1))
    for b in range(batch):
        for h in range(hkv):
            assert rc.packed_len(b, h) == oc.packed_len(b, h)
            for i in range(rc.packed_len(b, h) // rc.n_r):
                for x, y in zip(rc.block(b, h, i), oc.block(b, h, i)):
                    assert np.array_equal(x, y)


@needs_ref
def test_reference_verify_battery_passes():  # bench.cpp:602-613
    for bits in (2, 4, 8, 16):
        assert O.ref_run_verify(0, 1, bits) == 0


@needs_ref
def test_oracle_naive_attention_equals_reference():  # oracle.cpp:12-37
    g = O.Gauss(5)
    q = g.rounded(4 * 64).reshape(4, 64)
    k = g.rounded(300 * 64).reshape(300, 64)
    v = g.rounded(300 * 64).reshape(300, 64)
    assert np.array_equal(O.naive_attention(q, k, v), O.ref_naive_attention(q, k, v))


@needs_ref
@pytest.mark.parametrize("bits,wn", [(4, 4), (2, 4), (2, 2), (4, 8), (8, 8)])
def test_oracle_blocks_equal_live_reference_on_adversarial_data(bits, wn):
    """The oracle's quantize+pack equals the reference's on data built to hit
    exact .5 quotients, signed-zero extrema and constant groups (the inputs
    of test_gpu_parity.test_prefill_adversarial_bit_exact)."""
    from tests._cases import Case, adversarial_data
    c = Case(bits=bits, warp_n=wn, heads_kv=2, batch=1, prefill=4 * (8 * wn * (16 // bits)) + 5,
             seed=bits + wn)
    k, v = adversarial_data(c, c.seed)
    rc = O.RefCache(1, 2, 128, wn, bits, 0, 128, True)
    oc = O.OracleCache(1, 2, 128, wn, bits, 0, 128, True, max_tokens=c.prefill + 8)
    for h in range(2):
        rc.prefill(0, h, k[0, h], v[0, h])
        oc.prefill(0, h, k[0, h], v[0, h])
        for i in range(rc.packed_len(0, h) // rc.n_r):
            for x, y in zip(rc.block(0, h, i), oc.block(0, h, i)):
                assert np.array_equal(x, y)


@pytest.mark.parametrize("n,skip", [(0, 0), (1, 1), (7, 0), (4097, 1), (2_000_003, 0)])
def test_parallel_gauss_fill_is_the_same_stream(n, skip):
    """bench.py draws the run_bench stream (bench.cpp:18-35) with the
    Box-Muller transforms spread over threads: bit-identical to the
    sequential fill, including a pending spare and an odd length."""
    a, b = O.Gauss(11), O.Gauss(11)
    for _ in range(skip):
        a.next(), b.next()
    x, y = a.rounded(n), b.rounded(n, threads=6)
    assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert a.next() == b.next()
