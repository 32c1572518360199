"""Helper process for tests/test_variants.py (not a test module).

python tests/variant_runner.py OUT.npz

Runs a fixed set of fast-mode decode sequences (prefill, then steps that cross
a residual flush, uneven cell lengths, GQA groupings) through the C-ABI under
whatever BDK_* kernel-variant knobs the environment sets, and saves every
step's output plus the oracle's (the CPU restatement of decode_step) for the
same inputs.  The parent compares variants bit for bit and against the oracle.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2503_18773_b200 import bitkv as bk  # noqa: E402

D = 128
# (tag, bits, batch, heads_q, heads_kv, cell lengths (None: uniform prefill), prefill, steps)
CASES = [
    ("b2_uniform_flush", 2, 2, 32, 8, None, 3 * 256 - 3, 6),
    ("b4_uniform_flush", 4, 2, 32, 8, None, 5 * 128 - 2, 5),
    ("b2_uneven", 2, 2, 16, 4, [5 * 256 + 3, 17, 0, 9 * 256, 255, 3 * 256 + 64, 1, 700], None, 3),
    ("b4_uneven", 4, 2, 16, 4, [5 * 128 + 3, 17, 0, 9 * 128, 127, 3 * 128 + 64, 1, 700], None, 3),
    ("b2_mha", 2, 3, 8, 8, None, 1000, 2),
    ("b4_gqa8", 4, 1, 64, 8, None, 2000, 2),
    ("b4_long", 4, 1, 32, 8, None, 32768 + 77, 2),
]


def run(tag, bits, batch, hq, hkv, lens, prefill, steps):
    g = O.Gauss(sum(map(ord, tag)) % 1000)
    cells = batch * hkv
    if lens is None:
        lens = [prefill] * cells
    mx = max(lens) + steps + 512
    oc = O.OracleCache(batch, hkv, D, 4, bits, 0, 128, True, max_tokens=mx)
    gc = bk.KVCache(batch, hkv, D, 4, bk.QuantSpec(bits, bk.QuantAxis.KChannel, 128), max_tokens=mx)
    gc.set_precise(False)
    for i, L in enumerate(lens):
        b, h = divmod(i, hkv)
        k = g.rounded(L * D).reshape(L, D)
        v = g.rounded(L * D).reshape(L, D)
        oc.prefill(b, h, k, v)
        gc.prefill(b, h, k, v)
    cfg = bk.AttentionConfig(batch=batch, heads_q=hq, heads_kv=hkv, head_dim=D, warp_n=4)
    got, ref = [], []
    for _ in range(steps):
        q = g.rounded(batch * hq * D).reshape(batch, hq, D)
        kn = g.rounded(batch * hkv * D).reshape(batch, hkv, D)
        vn = g.rounded(batch * hkv * D).reshape(batch, hkv, D)
        ref.append(oc.decode_step(q, kn, vn))
        out = bk.decode_step(gc, cfg, torch.from_numpy(q).cuda().half(),
                             torch.from_numpy(kn).cuda().half(), torch.from_numpy(vn).cuda().half())
        got.append(out.data.cpu().numpy())
    lens_after = [(gc.packed_len(b, h), gc.res_len(b, h)) for b in range(batch) for h in range(hkv)]
    lens_oc = [(oc.packed_len(b, h), oc.res_len(b, h)) for b in range(batch) for h in range(hkv)]
    return np.stack(got), np.stack(ref), np.array(lens_after), np.array(lens_oc)


def main(out):
    res = {}
    for c in CASES:
        got, ref, la, lo = run(*c)
        res[c[0] + "_got"] = got
        res[c[0] + "_ref"] = ref
        res[c[0] + "_len"] = la
        res[c[0] + "_len_ref"] = lo
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
