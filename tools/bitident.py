"""Dev: fast-mode decode outputs of the loaded library (BDK_LIB selects a build)
on fixed inputs, saved to argv[1] (.npy); with argv[2], compare bit for bit.
usage: BDK_LIB=a.so python tools/bitident.py out_a.npy
       python tools/bitident.py out_b.npy out_a.npy"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_18773_b200 import bitkv as bk  # noqa: E402

outs = []
for bits, hq, hkv, seq, b in ((4, 32, 8, 16384, 1), (2, 32, 8, 16384, 2), (4, 32, 32, 1024, 4)):
    g = torch.Generator().manual_seed(bits * 1000 + seq)
    d, wn = 128, 4
    cache = bk.KVCache(b, hkv, d, wn, bk.QuantSpec(bits, bk.QuantAxis.KChannel, 128), max_tokens=seq + 512)
    k = torch.randn(b, hkv, seq, d, generator=g).half().cuda()
    v = torch.randn(b, hkv, seq, d, generator=g).half().cuda()
    cache.prefill_all(k, v)
    cache.set_precise(False)
    cfg = bk.AttentionConfig(batch=b, heads_q=hq, heads_kv=hkv, head_dim=d, tile_m=hq // hkv,
                             tile_n=64, num_splits=4, warp_n=wn)
    for step in range(3):
        q = torch.randn(b, hq, d, generator=g).half().cuda()
        kn = torch.randn(b, hkv, d, generator=g).half().cuda()
        vn = torch.randn(b, hkv, d, generator=g).half().cuda()
        out = bk.decode_step(cache, cfg, q, kn, vn)
        outs.append(out.data.float().cpu().numpy().ravel())
res = np.concatenate(outs)
np.save(sys.argv[1], res)
if len(sys.argv) > 2:
    ref = np.load(sys.argv[2])
    same = np.array_equal(res.view(np.uint32), ref.view(np.uint32))
    print("bit-identical:", same, "max-abs diff:", float(np.abs(res - ref).max()))
else:
    print("saved", res.shape)
