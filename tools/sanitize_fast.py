"""Small fast-mode decode run for compute-sanitizer (dev tool): prefill,
then steps across a residual flush, eager and graph-replayed, uneven cells.

compute-sanitizer --tool memcheck python tools/sanitize_fast.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_18773_b200 import bitkv as bk  # noqa: E402

D = 128
for bits in (4, 2):
    batch, hq, hkv = 2, 8, 2
    n_r = 8 * 4 * (16 // bits)
    c = bk.KVCache(batch, hkv, D, 4, bk.QuantSpec(bits, bk.QuantAxis.KChannel, 128),
                   max_tokens=4 * n_r)
    c.set_precise(False)
    g = torch.Generator(device="cuda").manual_seed(bits)
    for b in range(batch):
        for h in range(hkv):
            L = n_r + 3 + 5 * (b * hkv + h)
            k = torch.randn(L, D, device="cuda", generator=g).half()
            c.prefill(b, h, k, k)
    cfg = bk.AttentionConfig(batch=batch, heads_q=hq, heads_kv=hkv, head_dim=D, warp_n=4)
    q = torch.randn(batch, hq, D, device="cuda").half()
    kn = torch.randn(batch, hkv, D, device="cuda").half()
    for _ in range(n_r + 2):  # every cell flushes once
        out = bk.decode_step(c, cfg, q, kn, kn).data
    qs = q.expand(4, -1, -1, -1).contiguous()
    ks = kn.expand(4, -1, -1, -1).contiguous()
    outs = torch.empty(4, batch, hq, D, device="cuda")
    gr = bk.DecodeGraph(c, cfg, qs, ks, ks, outs)
    gr.launch()
    gr.close()
    torch.cuda.synchronize()
    assert torch.isfinite(out).all() and torch.isfinite(outs).all()
print("sanitize_fast ok")
