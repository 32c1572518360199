"""BDKV v1 cache files (serialize.hpp:11-23, serialize.cpp:87-194) through the
C-ABI: the device cache dumps the reference's exact bytes, and loads them.

The byte-identity anchor is the golden BDKV dump of the UNMODIFIED reference
engine after prefill + decode steps (tests/golden/*.npz, make_golden.py); the
properties follow the reference's test_serialize.cpp (round trip, re-dump
byte identity, truncation / bad magic -> FormatError with an offset)."""
from __future__ import annotations

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

D = 128
GOLDEN = ["decode_4bit_gqa", "decode_2bit_wn4_flush", "decode_16bit"]


def _golden_cache(name):
    """Replay the fixture's prefill + decode steps on the device cache."""
    from oracle import oracle as O
    from paper_2503_18773_b200 import bitkv as bk
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", name + ".npz"))
    batch, hq, hkv, seq, bits, wn, g, axis, steps, seed = z["meta"].tolist()
    gauss = O.Gauss(seed)
    gc = bk.KVCache(batch, hkv, D, wn, bk.QuantSpec(bits, bk.QuantAxis(axis), g),
                    max_tokens=seq + steps + 512)
    for b in range(batch):
        for h in range(hkv):
            k = gauss.rounded(seq * D).reshape(seq, D)
            v = gauss.rounded(seq * D).reshape(seq, D)
            gc.prefill(b, h, k, v)
    cfg = bk.AttentionConfig(batch=batch, heads_q=hq, heads_kv=hkv, head_dim=D, warp_n=wn)
    for s in range(steps):
        bk.decode_step(gc, cfg, torch.from_numpy(z["q"][s]).cuda().half(),
                       torch.from_numpy(z["k_new"][s]).cuda().half(),
                       torch.from_numpy(z["v_new"][s]).cuda().half())
    torch.cuda.synchronize()
    return gc, z["bdkv"].tobytes()


@pytest.mark.parametrize("name", GOLDEN)
def test_dump_is_byte_identical_to_reference(name):
    from paper_2503_18773_b200 import bitkv as bk
    gc, ref = _golden_cache(name)
    got = bk.dump_cache(gc)
    assert len(got) == len(ref)
    assert got == ref


@pytest.mark.parametrize("name", GOLDEN)
def test_load_reference_dump_then_redump_is_identical(name, tmp_path):
    from paper_2503_18773_b200 import bitkv as bk
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", name + ".npz"))
    ref = z["bdkv"].tobytes()
    c = bk.load_cache(ref)
    assert bk.dump_cache(c) == ref
    p = tmp_path / "cache.bdkv"
    bk.dump_cache_file(c, str(p))
    assert p.read_bytes() == ref
    c2 = bk.load_cache_file(str(p), max_tokens=4096)
    assert bk.dump_cache(c2) == ref


def test_loaded_cache_decodes_like_the_original():
    """A loaded cache is a working cache: the next decode step matches the
    cache it was dumped from bit for bit (same kernels, same state)."""
    from oracle import oracle as O
    from paper_2503_18773_b200 import bitkv as bk
    gc, _ = _golden_cache("decode_4bit_gqa")
    lc = bk.load_cache(bk.dump_cache(gc), max_tokens=8192)
    for b in range(gc.batch()):
        for h in range(gc.heads_kv()):
            assert lc.packed_len(b, h) == gc.packed_len(b, h)
            assert lc.res_len(b, h) == gc.res_len(b, h)
    g = O.Gauss(5)
    q = torch.from_numpy(g.rounded(8 * D).reshape(1, 8, D)).cuda().half()
    kn = torch.from_numpy(g.rounded(2 * D).reshape(1, 2, D)).cuda().half()
    vn = torch.from_numpy(g.rounded(2 * D).reshape(1, 2, D)).cuda().half()
    cfg = bk.AttentionConfig(batch=1, heads_q=8, heads_kv=2, head_dim=D, warp_n=4)
    a = bk.decode_step(gc, cfg, q, kn, vn).data.cpu().numpy()
    b = bk.decode_step(lc, cfg, q, kn, vn).data.cpu().numpy()
    assert np.array_equal(a, b)


def test_truncated_and_bad_magic_raise_format_error():
    from paper_2503_18773_b200 import bitkv as bk
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "decode_2bit_wn4_flush.npz"))
    ref = z["bdkv"].tobytes()
    for cut in (0, 3, 9, len(ref) // 2, len(ref) - 1):  # test_serialize.cpp:84-91
        with pytest.raises(bk.FormatError):
            bk.load_cache(ref[:cut])
    bad = b"X" + ref[1:]  # test_serialize.cpp:93-104
    with pytest.raises(bk.FormatError) as e:
        bk.load_cache(bad)
    assert e.value.offset == 0
    badv = ref[:4] + bytes([2]) + ref[5:]
    with pytest.raises(bk.FormatError) as e:
        bk.load_cache(badv)
    assert e.value.offset == 4
