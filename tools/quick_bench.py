"""Quick device timing of the decode step for the BASELINE configs (dev tool).

python tools/quick_bench.py [C1|C2|C3|C5 ...] [--precise]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_18773_b200 import bitkv as bk  # noqa: E402

CONFIGS = {
    "C1": dict(batch=1, hq=32, hkv=8, bits=4, warp_n=4, seq=4096),
    "C2": dict(batch=8, hq=32, hkv=8, bits=2, warp_n=4, seq=32768),
    "C2w2": dict(batch=8, hq=32, hkv=8, bits=2, warp_n=2, seq=32768),
    "C3": dict(batch=32, hq=32, hkv=32, bits=4, warp_n=4, seq=8192),
    "C5": dict(batch=1, hq=32, hkv=8, bits=4, warp_n=4, seq=131072),
    "C5_32k": dict(batch=1, hq=32, hkv=8, bits=4, warp_n=4, seq=32768),
    "C5_b8_32k": dict(batch=8, hq=32, hkv=8, bits=4, warp_n=4, seq=32768),
}


def qbytes(cfg, n_r):
    d = 128
    plen = cfg["seq"] - cfg["seq"] % n_r
    cells = cfg["batch"] * cfg["hkv"]
    b = cells * (2 * plen * d * cfg["bits"] // 8 + 4 * d * plen // 128 + 4 * plen * d // 128)
    return b


def run(name, precise=False, iters=50):
    cfg = CONFIGS[name]
    d = 128
    spec = bk.QuantSpec(cfg["bits"], bk.QuantAxis.KChannel, 128)
    cache = bk.KVCache(cfg["batch"], cfg["hkv"], d, cfg["warp_n"], spec,
                       max_tokens=cfg["seq"] + 4096)
    cache.set_precise(precise)
    n_r = cache.n_r()
    g = torch.Generator(device="cuda").manual_seed(0)
    k = torch.randn(cfg["batch"], cfg["hkv"], cfg["seq"], d, device="cuda", generator=g).half()
    v = torch.randn(cfg["batch"], cfg["hkv"], cfg["seq"], d, device="cuda", generator=g).half()
    torch.cuda.synchronize()
    t0 = time.time()
    cache.prefill_all(k, v)
    torch.cuda.synchronize()
    tp = time.time() - t0
    # time prefill with events too
    del k, v
    att = bk.AttentionConfig(batch=cfg["batch"], heads_q=cfg["hq"], heads_kv=cfg["hkv"],
                             head_dim=d, warp_n=cfg["warp_n"])
    q = torch.randn(cfg["batch"], cfg["hq"], d, device="cuda").half()
    kn = torch.randn(cfg["batch"], cfg["hkv"], d, device="cuda").half()
    vn = torch.randn(cfg["batch"], cfg["hkv"], d, device="cuda").half()
    out = torch.empty(cfg["batch"], cfg["hq"], d, device="cuda")
    flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
    for _ in range(5):
        bk.decode_step(cache, att, q, kn, vn, out)
    torch.cuda.synchronize()
    times = []
    for _ in range(iters):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bk.decode_step(cache, att, q, kn, vn, out)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    times.sort()
    med = times[len(times) // 2]
    qb = qbytes(cfg, n_r)
    print(f"{name}{' precise' if precise else ''}: median {med:.1f} us  min {times[0]:.1f} us  "
          f"qbytes {qb/1e6:.1f} MB  -> {qb/med/1e3:.0f} GB/s  ({qb/med/1e3/6550:.2%} of 6550)"
          f"  prefill wall {tp*1e3:.1f} ms", flush=True)
    assert torch.isfinite(out).all()


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["C1", "C2", "C5", "C3"]
    for n in names:
        run(n, precise="--precise" in sys.argv)
