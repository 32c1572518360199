# dev probe: phase timing of the host decode path (not part of the repo)
import time, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
from paper_2503_18773_b200 import bitkv as bk
b, hq, hkv, seq, bits = 8, 32, 8, 32768, 2
spec = bk.QuantSpec(bits, bk.QuantAxis.KChannel, 128)
c = bk.KVCache(b, hkv, 128, 4, spec, max_tokens=seq + 1024)
k = torch.randn((b, hkv, seq, 128), device='cuda', dtype=torch.float16)
c.prefill_all(k, k); torch.cuda.synchronize()
cfg = bk.AttentionConfig(batch=b, heads_q=hq, heads_kv=hkv, head_dim=128, warp_n=4)
q = np.random.randn(b, hq, 128).astype(np.float16).astype(np.float32)
kn = np.random.randn(b, hkv, 128).astype(np.float16).astype(np.float32)
for _ in range(20): bk.decode_step(c, cfg, q, kn, kn)
N = 200
t = time.perf_counter()
for _ in range(N): bk.decode_step(c, cfg, q, kn, kn)
print("python decode_step us", (time.perf_counter() - t) / N * 1e6)
L = bk._L.load(); import ctypes as C
o = np.empty((b, hq, 128), np.float32); cc = cfg._c()
args = (c.handle(), C.byref(cc), q.ctypes.data, kn.ctypes.data, kn.ctypes.data, o.ctypes.data)
t = time.perf_counter()
for _ in range(N): L.bdk_decode_step_host(*args)
print("raw C-ABI call us", (time.perf_counter() - t) / N * 1e6)
qd = torch.from_numpy(q).cuda().half(); kd = torch.from_numpy(kn).cuda().half(); out = torch.empty((b, hq, 128), device='cuda')
st = bk.DecodeStepper(c, cfg, qd, kd, kd, out)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(N):
    st(); torch.cuda.synchronize()
print("device step + sync us", (time.perf_counter() - t) / N * 1e6)
t = time.perf_counter()
for _ in range(N): torch.cuda.synchronize()
print("empty sync us", (time.perf_counter() - t) / N * 1e6)
