# dev timing of the span path (decode_step for head_dim 64, outside the tensor-core envelope)
import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2503_18773_b200 import bitkv as bk
for d, seq in ((64, 8192), (64, 32768)):
    spec = bk.QuantSpec(4, bk.QuantAxis.KChannel, 64)
    c = bk.KVCache(1, 8, d, 4, spec, max_tokens=seq + 1024)
    k = torch.randn((1, 8, seq, d), device='cuda', dtype=torch.float16)
    c.prefill_all(k, k); torch.cuda.synchronize()
    cfg = bk.AttentionConfig(batch=1, heads_q=32, heads_kv=8, head_dim=d, tile_m=4, tile_n=64, num_splits=4, warp_n=4)
    q = torch.randn((1, 32, d), device='cuda', dtype=torch.float16); kn = torch.randn((1, 8, d), device='cuda', dtype=torch.float16)
    out = torch.empty((1, 32, d), device='cuda')
    for _ in range(3): bk.decode_step(c, cfg, q, kn, kn, out=out)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): bk.decode_step(c, cfg, q, kn, kn, out=out)
    torch.cuda.synchronize(); print(f"span path d={d} seq={seq}: {(time.perf_counter() - t) / 10 * 1e6:.0f} us/step")
