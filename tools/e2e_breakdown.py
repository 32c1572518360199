"""Host decode call breakdown (dev tool): python decode_step vs the raw C-ABI call vs the
device step + sync vs CUDA events, for C5 and C2 shapes.

python tools/e2e_breakdown.py
"""
import time, numpy as np, torch, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2503_18773_b200 import bitkv as bk
import ctypes as C
for (b, hq, hkv, seq, bits) in [(1, 32, 8, 131072, 4), (8, 32, 8, 32768, 2)]:
    spec = bk.QuantSpec(bits, bk.QuantAxis.KChannel, 128)
    c = bk.KVCache(b, hkv, 128, 4, spec, max_tokens=seq + 4096)
    c.set_precise(False)
    k = torch.randn((b, hkv, seq, 128), device='cuda', dtype=torch.float16)
    c.prefill_all(k, k); torch.cuda.synchronize(); del k
    cfg = bk.AttentionConfig(batch=b, heads_q=hq, heads_kv=hkv, head_dim=128, warp_n=4)
    q = np.random.randn(b, hq, 128).astype(np.float16).astype(np.float32)
    kn = np.random.randn(b, hkv, 128).astype(np.float16).astype(np.float32)
    o = np.empty((b, hq, 128), np.float32)
    for _ in range(50): bk.decode_step(c, cfg, q, kn, kn, out=o)
    N = 300
    t = time.perf_counter()
    for _ in range(N): bk.decode_step(c, cfg, q, kn, kn, out=o)
    py = (time.perf_counter() - t) / N * 1e6
    L = bk._L.load(); cc = cfg._c()
    args = (c.handle(), C.byref(cc), q.ctypes.data, kn.ctypes.data, kn.ctypes.data, o.ctypes.data)
    t = time.perf_counter()
    for _ in range(N): L.bdk_decode_step_host(*args)
    raw = (time.perf_counter() - t) / N * 1e6
    qd = torch.from_numpy(q).cuda().half(); kd = torch.from_numpy(kn).cuda().half(); out = torch.empty((b, hq, 128), device='cuda')
    st = bk.DecodeStepper(c, cfg, qd, kd, kd, out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(N):
        st(); torch.cuda.synchronize()
    dev = (time.perf_counter() - t) / N * 1e6
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(50):
        e0.record(); st(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"b{b} {bits}-bit {seq}: python decode_step {py:.1f} us | raw C-ABI {raw:.1f} us | device step + sync {dev:.1f} us | events {np.median(ts):.1f} us")
