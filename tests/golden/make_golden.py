"""Generate tests/golden/ from the UNMODIFIED reference engine.

    make -C oracle all && python tests/golden/make_golden.py

Needs oracle/_ref/libbitkv_ref.so (the reference sources under
/root/reference/proj compiled out-of-tree by oracle/Makefile), so it runs in
the build container only; the fixtures it writes are small and committed, so
the GPU box (which has no /root/reference) checks against them.

Written files:
  kat.json     known-answer tests transcribed from the reference's own doctest
               suites (file:line cited per entry), each value re-computed by
               the reference library; plus run_bench output checksums of small
               seeded workloads (bench.cpp:80-210), which pin the GaussianSource
               stream (bench.cpp:18-35), prefill, decode_step and fnv1a64 in one
               number.
  blocks.json  sha256 of every packed block (k_words|v_words|k_params|v_params,
               little-endian u16, block order) + residual bits + lengths of the
               reference cache after prefill of GaussianSource(seed) data, per
               geometry (incl. the C1 prefill and the 32K x 8-head C4 flush).
  decode_*.npz reference decode_step outputs for seeded small workloads, plus
               the inputs (fp16-representable fp32) and the BDKV dump of the
               final cache (serialize.cpp:87-120).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

D = 128

# ---------------------------------------------------------------- geometries
# (name, batch, heads_kv, head_dim, seq, bits, warp_n, group, k_axis, interleave, seed)
BLOCK_CASES = [
    ("c1_prefill_4bit", 1, 8, 128, 4096, 4, 4, 128, 0, 1, 0),
    ("c4_flush_4bit_32k", 1, 8, 128, 32768, 4, 4, 128, 0, 1, 4),
    ("c4_flush_2bit_32k", 1, 8, 128, 32768, 2, 4, 128, 0, 1, 2),
    ("c2_geom_2bit_wn2", 2, 2, 128, 1000, 2, 2, 128, 0, 1, 21),
    ("8bit_wn2_g32", 1, 2, 128, 700, 8, 2, 32, 0, 1, 8),
    ("16bit_passthrough", 1, 2, 128, 300, 16, 4, 64, 0, 1, 16),
    ("4bit_ktoken_g32", 1, 2, 128, 640, 4, 2, 32, 1, 1, 41),
    ("2bit_ktoken_g64", 1, 2, 128, 1100, 2, 4, 64, 1, 1, 42),
    ("4bit_identity_perm", 1, 2, 128, 500, 4, 4, 128, 0, 0, 43),
    ("4bit_wn8", 1, 2, 128, 900, 4, 8, 128, 0, 1, 44),
    ("4bit_wn1_g32", 1, 2, 128, 333, 4, 1, 32, 0, 1, 45),
]

# run_bench workloads whose output checksum the oracle must reproduce
# (mode, seq, batch, hq, hkv, d, bits, g, axis, splits, steps, seed, tile_n, warp_n, interleave)
BENCH_CASES = [
    (0, 300, 1, 8, 2, 128, 4, 128, 0, 4, 3, 0, 64, 4, 1),
    (1, 520, 2, 8, 2, 128, 2, 128, 0, 3, 4, 1, 64, 4, 1),
    (0, 129, 1, 4, 4, 128, 8, 32, 0, 2, 3, 2, 32, 2, 1),
    (0, 90, 1, 4, 1, 128, 16, 64, 0, 4, 2, 3, 32, 4, 1),
    (0, 400, 1, 8, 2, 64, 4, 16, 1, 4, 3, 4, 64, 2, 0),
    (0, 257, 1, 2, 1, 8, 2, 8, 0, 1, 3, 5, 32, 1, 1),
]

# decode_step golden outputs: (name, batch, hq, hkv, seq, bits, warp_n, g, axis, steps, seed)
DECODE_CASES = [
    ("decode_4bit_gqa", 1, 8, 2, 700, 4, 4, 128, 0, 3, 11),
    ("decode_2bit_wn4_flush", 2, 8, 2, 250, 2, 4, 128, 0, 8, 12),
    ("decode_16bit", 1, 4, 1, 200, 16, 4, 64, 0, 2, 13),
]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).astype("<u2", copy=False).tobytes())
    return h.hexdigest()


def cell_data(gauss, seq, d):
    k = gauss.rounded(seq * d).reshape(seq, d)
    v = gauss.rounded(seq * d).reshape(seq, d)
    return k, v


def block_fixture(case):
    name, batch, hkv, d, seq, bits, wn, g, axis, il, seed = case
    rc = O.RefCache(batch, hkv, d, wn, bits, axis, g, bool(il))
    gauss = O.Gauss(seed)
    for b in range(batch):
        for h in range(hkv):
            k, v = cell_data(gauss, seq, d)
            rc.prefill(b, h, k, v)
    cells = []
    for b in range(batch):
        for h in range(hkv):
            blocks = [rc.block(b, h, i) for i in range(rc.packed_len(b, h) // rc.n_r)]
            h_all = hashlib.sha256()
            for blk in blocks:
                for a in blk:
                    h_all.update(np.ascontiguousarray(a).astype("<u2").tobytes())
            k_all, v_all = rc.reconstruct(b, h)
            res_k = k_all[rc.packed_len(b, h):]
            res_v = v_all[rc.packed_len(b, h):]
            cells.append({"b": b, "h": h, "packed_len": int(rc.packed_len(b, h)),
                          "res_len": int(rc.res_len(b, h)), "blocks_sha256": h_all.hexdigest(),
                          "residual_sha256": sha(res_k.astype(np.float16).view(np.uint16),
                                                 res_v.astype(np.float16).view(np.uint16))})
    return {"name": name, "batch": batch, "heads_kv": hkv, "head_dim": d, "seq": seq,
            "bits": bits, "warp_n": wn, "group_size": g, "k_axis": axis, "interleave": il,
            "seed": seed, "n_r": int(rc.n_r), "memory": list(map(int, rc.memory())),
            "cells": cells}


def step_inputs(gauss, batch, hq, hkv, d):
    """run_bench's per-step draw order (bench.cpp:144-155), fp16-rounded."""
    q = np.zeros((batch, hq, d), np.float32)
    kn = np.zeros((batch, hkv, d), np.float32)
    vn = np.zeros((batch, hkv, d), np.float32)
    for b in range(batch):
        q[b] = gauss.rounded(hq * d).reshape(hq, d)
        for h in range(hkv):
            kn[b, h] = gauss.rounded(d)
            vn[b, h] = gauss.rounded(d)
    return q, kn, vn


def decode_fixture(case):
    name, batch, hq, hkv, seq, bits, wn, g, axis, steps, seed = case
    rc = O.RefCache(batch, hkv, D, wn, bits, axis, g, True)
    gauss = O.Gauss(seed)
    for b in range(batch):
        for h in range(hkv):
            k, v = cell_data(gauss, seq, D)
            rc.prefill(b, h, k, v)
    qs, ks, vs, outs = [], [], [], []
    for _ in range(steps):
        q, kn, vn = step_inputs(gauss, batch, hq, hkv, D)
        outs.append(rc.decode_step(q, kn, vn, tile_n=64, num_splits=4))
        qs.append(q)
        ks.append(kn)
        vs.append(vn)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), q=np.stack(qs), k_new=np.stack(ks),
                        v_new=np.stack(vs), out=np.stack(outs),
                        bdkv=np.frombuffer(rc.dump(), np.uint8),
                        meta=np.array([batch, hq, hkv, seq, bits, wn, g, axis, steps, seed]))
    return name


def kats():
    R = O
    out = {"source": "/root/reference/proj tests, values recomputed by oracle/_ref"}
    out["interleave_order"] = {  # test_layout.cpp:13-26
        "cite": "test_layout.cpp:13-26",
        "2": [7, 5, 3, 1, 6, 4, 2, 0], "4": [3, 1, 2, 0], "8": [1, 0], "16": [0]}
    out["pack_word"] = {  # test_layout.cpp:28-39
        "cite": "test_layout.cpp:28-39",
        "cases": [[[1, 2, 3, 4], 4, 1, R.ref_pack_word([1, 2, 3, 4], 4)],
                  [[0, 0, 0, 0], 4, 1, R.ref_pack_word([0, 0, 0, 0], 4)],
                  [[3] * 8, 2, 1, R.ref_pack_word([3] * 8, 2)]]}
    assert out["pack_word"]["cases"][0][3] == 0x4231
    rng = np.random.default_rng(0)
    rand = []
    for bits in (2, 4, 8, 16):
        for il in (1, 0):
            for _ in range(64):
                codes = rng.integers(0, 1 << min(bits, 16), 16 // bits).tolist()
                rand.append([codes, bits, il, R.ref_pack_word(codes, bits, bool(il))])
    out["pack_word_random"] = {"cite": "layout.cpp:45-61 via oracle/_ref", "cases": rand}
    out["residual_block_size"] = {  # test_layout.cpp:70-83
        "cite": "test_layout.cpp:70-75",
        "cases": [[8, 1, 16], [4, 4, 128], [2, 4, 256], [16, 1, 8]]}
    gp = []  # test_quant.cpp:27-53
    for grp, bits in (([0, 1, 2, 3], 2), ([5, 5, 5, 5], 4), ([-1, 0, 2, 5], 4)):
        s, z = R.ref_group_params(grp, bits)
        gp.append([grp, bits, s, z])
    pool = [-100.0, -5.5, -1.0, -0.4, -0.1, -0.015625, 0.0, 0.0004, 0.25, 0.6, 1.0, 2.5, 7.75,
            33.0, 511.0, 1000.0, 64000.0]  # test_quant.cpp:105-130
    for bits in (2, 4, 8):
        for a in pool[::3]:
            for b in pool[1::4]:
                for c in pool[2::5]:
                    grp = [O.round_f16(a), O.round_f16(b), O.round_f16(c)]
                    s, z = R.ref_group_params(grp, bits)
                    gp.append([grp, bits, s, z])
    g2 = rng.standard_normal((200, 16)).astype(np.float32)
    for i, row in enumerate(g2):
        row = np.array([O.round_f16(x) for x in row], np.float32)
        s, z = R.ref_group_params(row, (2, 4, 8)[i % 3])
        gp.append([row.tolist(), (2, 4, 8)[i % 3], s, z])
    out["group_params"] = {"cite": "test_quant.cpp:27-53, :105-130; quant.cpp:18-28", "cases": gp}
    out["quantize_rne"] = {  # test_quant.cpp:62-69
        "cite": "test_quant.cpp:62-69", "group": [-1, 0, 2, 5], "scale": 0.4, "zero": -1.0,
        "bits": 4, "codes": [0, 2, 8, 15]}
    out["fp16"] = {  # test_fp16.cpp:24-53
        "cite": "test_fp16.cpp:24-53",
        "to_bits": [[0.0, 0], [-0.0, 0x8000], [65520.0, 0x7C00], [65519.996, 0x7BFF],
                    [1e30, 0x7C00], [-1e30, 0xFC00], [2.0 ** -26, 0], [1.5 * 2.0 ** -25, 1],
                    [1.0 + 2.0 ** -11, 0x3C00], [1.0 + 3 * 2.0 ** -11, 0x3C02]],
        "from_bits": [[0x3C00, 1.0], [0xC000, -2.0], [0x7BFF, 65504.0], [1, 2.0 ** -24],
                      [0x0400, 2.0 ** -14]]}
    bench = []
    for (mode, seq, batch, hq, hkv, d, bits, g, axis, splits, steps, seed, tile_n, wn,
         il) in BENCH_CASES:
        r = R.ref_run_bench(mode=mode, seq_len=seq, batch=batch, heads_q=hq, heads_kv=hkv,
                            head_dim=d, bits=bits, group_size=g, k_axis=axis, num_splits=splits,
                            steps=steps, seed=seed, tile_n=tile_n, warp_n=wn,
                            interleave=bool(il))
        bench.append({"mode": mode, "seq_len": seq, "batch": batch, "heads_q": hq,
                      "heads_kv": hkv, "head_dim": d, "bits": bits, "group_size": g,
                      "k_axis": axis, "num_splits": splits, "steps": steps, "seed": seed,
                      "tile_n": tile_n, "warp_n": wn, "interleave": il,
                      "output_checksum": f"{r['output_checksum']:016x}", "memory": r["memory"],
                      "n_r": r["n_r"]})
    out["run_bench_checksums"] = {"cite": "bench.cpp:80-210 (output_checksum :171)",
                                  "cases": bench}
    return out


def main():
    if not O.have_ref():
        O.build(ref=True)
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kats(), f, indent=1)
    blocks = [block_fixture(c) for c in BLOCK_CASES]
    with open(os.path.join(HERE, "blocks.json"), "w") as f:
        json.dump(blocks, f, indent=1)
    for c in DECODE_CASES:
        decode_fixture(c)
    print("golden written to", HERE)


if __name__ == "__main__":
    main()
