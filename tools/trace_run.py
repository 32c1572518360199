"""Collect BDK_TRACE stamps of n isolated fast-decode launches (dev tool).

python tools/trace_run.py C5 OUT.txt [n]
Then: python tools/trace_stats.py OUT.txt [launch]; python tools/trace_sm.py OUT.txt
"""
import os
import sys

name, out = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
os.environ["BDK_TRACE"] = out
if os.path.exists(out):
    os.remove(out)
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_18773_b200 import bitkv as bk  # noqa: E402

W = {"C1": (1, 32, 8, 4, 4096), "C2": (8, 32, 8, 2, 32768), "C3": (32, 32, 32, 4, 8192),
     "C5": (1, 32, 8, 4, 131072), "C2b4": (8, 32, 8, 4, 32768)}
batch, hq, hkv, bits, seq = W[name]
d = 128
cache = bk.KVCache(batch, hkv, d, 4, bk.QuantSpec(bits, bk.QuantAxis.KChannel, 128),
                   max_tokens=seq + 1024)
cache.set_precise(False)
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn(batch, hkv, seq, d, device="cuda", generator=g).half()
v = torch.randn(batch, hkv, seq, d, device="cuda", generator=g).half()
cache.prefill_all(k, v)
del k, v
cfg = bk.AttentionConfig(batch=batch, heads_q=hq, heads_kv=hkv, head_dim=d, warp_n=4)
q = torch.randn(batch, hq, d, device="cuda").half()
out_t = torch.empty(batch, hq, d, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
for _ in range(n):
    flush.zero_()
    bk.decode_partial(cache, cfg, q, None, None, out=out_t) if False else bk.decode_step(cache, cfg, q, torch.zeros(batch, hkv, d, device="cuda").half(), torch.zeros(batch, hkv, d, device="cuda").half(), out_t)
torch.cuda.synchronize()
print("traced", n, "launches ->", out)
