"""Per-step isolated latency across a residual flush (dev tool).

python tools/flush_step.py [C5|C2|C3|C1]

Prefills the workload with res_len = N_r - 3, then times 6 decode steps one
by one (CUDA events, synchronized): step 3 fills the window, so its launch
also quantizes + packs it into a new block (the fused flush).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_18773_b200 import bitkv as bk  # noqa: E402

W = {"C1": (1, 32, 8, 4, 4096), "C2": (8, 32, 8, 2, 32768), "C3": (32, 32, 32, 4, 8192),
     "C5": (1, 32, 8, 4, 131072)}


def main(name):
    batch, hq, hkv, bits, seq = W[name]
    d = 128
    cache = bk.KVCache(batch, hkv, d, 4, bk.QuantSpec(bits, bk.QuantAxis.KChannel, 128),
                       max_tokens=seq + 1024)
    cache.set_precise(False)
    n_r = cache.n_r()
    L = seq - seq % n_r + n_r - 3
    g = torch.Generator(device="cuda").manual_seed(0)
    k = torch.randn(batch, hkv, L, d, device="cuda", generator=g).half()
    v = torch.randn(batch, hkv, L, d, device="cuda", generator=g).half()
    cache.prefill_all(k, v)
    del k, v
    cfg = bk.AttentionConfig(batch=batch, heads_q=hq, heads_kv=hkv, head_dim=d, warp_n=4)
    q = torch.randn(batch, hq, d, device="cuda").half()
    kn = torch.randn(batch, hkv, d, device="cuda").half()
    vn = torch.randn(batch, hkv, d, device="cuda").half()
    out = torch.empty(batch, hq, d, device="cuda")
    res = []
    for rep in range(3):
        times = []
        for s in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            bk.decode_step(cache, cfg, q, kn, vn, out)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3)
        res.append(times)
        # back to res_len = N_r - 3 for the next repetition
        while cache.res_len(0, 0) != n_r - 3:
            bk.decode_step(cache, cfg, q, kn, vn, out)
        torch.cuda.synchronize()
    for times in res:
        print(f"{name} N_r {n_r}: step us " + " ".join(f"{t:7.1f}" for t in times)
              + "   (step 3 flushes)", flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["C5", "C2"]:
        main(n)
