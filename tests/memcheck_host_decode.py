# dev check: host decode_step (fast kernel + PDL stage-in) vs the oracle, small enough for
# compute-sanitizer memcheck:  compute-sanitizer --tool memcheck python tests/memcheck_host_decode.py
import numpy as np, sys
sys.path.insert(0, '/root/repo')
from paper_2503_18773_b200 import bitkv as bk
from oracle import oracle as O
for bits, wn in ((4, 4), (2, 4)):
    d, hq, hkv, seq = 128, 8, 2, 700
    g = O.Gauss(3)
    c = bk.KVCache(1, hkv, d, wn, bk.QuantSpec(bits, bk.QuantAxis.KChannel, 128), max_tokens=2048)
    oc = O.OracleCache(1, hkv, d, wn, bits, 0, 128, True, max_tokens=2048)
    for h in range(hkv):
        k = g.rounded(seq * d).reshape(seq, d); v = g.rounded(seq * d).reshape(seq, d)
        c.prefill(0, h, k, v); oc.prefill(0, h, k, v)
    cfg = bk.AttentionConfig(batch=1, heads_q=hq, heads_kv=hkv, head_dim=d, tile_m=4, tile_n=64, num_splits=4, warp_n=wn)
    for s in range(70):
        q = g.rounded(hq * d).reshape(1, hq, d); kn = g.rounded(hkv * d).reshape(1, hkv, d); vn = g.rounded(hkv * d).reshape(1, hkv, d)
        got = bk.decode_step(c, cfg, q, kn, vn).data; ref = oc.decode_step(q, kn, vn)
        assert np.abs(got - ref).max() < 2e-3
print("memcheck script ok")
