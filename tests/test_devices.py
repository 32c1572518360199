"""Device placement and boundary validation of the C-ABI.

Every C-ABI call runs on its cache's GPU and leaves the caller's current
device as it was (bdk_api.cu DevGuard); caller-provided outputs are checked
before any kernel writes them."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

D = 128


def _mk(device, precise=True):
    from paper_2503_18773_b200 import bitkv as bk
    spec = bk.QuantSpec(4, bk.QuantAxis.KChannel, 128)
    c = bk.KVCache(1, 2, D, 4, spec, max_tokens=1024, device=device, precise=precise)
    cfg = bk.AttentionConfig(batch=1, heads_q=8, heads_kv=2, head_dim=D, tile_m=4, tile_n=64,
                             num_splits=4, warp_n=4)
    g = torch.Generator(device=f"cuda:{device}").manual_seed(5)
    k = torch.randn((1, 2, 300, D), generator=g, device=f"cuda:{device}").half()
    v = torch.randn((1, 2, 300, D), generator=g, device=f"cuda:{device}").half()
    c.prefill_all(k, v)
    return c, cfg


@pytest.mark.parametrize("precise", [False, True])
def test_calls_keep_the_callers_device(precise):
    from paper_2503_18773_b200 import bitkv as bk
    torch.cuda.set_device(0)
    c, cfg = _mk(0, precise)
    q = np.random.default_rng(0).standard_normal((1, 8, D)).astype(np.float32)
    kn = np.random.default_rng(1).standard_normal((1, 2, D)).astype(np.float32)
    bk.decode_step(c, cfg, q, kn, kn)  # host API (staging allocation on first call)
    assert torch.cuda.current_device() == 0


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("precise", [False, True])
def test_caches_on_two_devices_decode_on_their_own_gpu(precise):
    """A cache on device 1 created after one on device 0: the first decode of
    the device-0 cache (workspace allocation included) runs on device 0."""
    from paper_2503_18773_b200 import bitkv as bk
    c0, cfg = _mk(0, precise)
    c1, _ = _mk(1, precise)
    torch.cuda.set_device(1)
    q = torch.randn((1, 8, D), device="cuda:0").half()
    kn = torch.randn((1, 2, D), device="cuda:0").half()
    out0 = bk.decode_step(c0, cfg, q, kn, kn).data
    torch.cuda.synchronize(0)
    assert out0.device.index == 0 and torch.isfinite(out0).all()
    assert torch.cuda.current_device() == 1
    q1, kn1 = q.to("cuda:1"), kn.to("cuda:1")
    out1 = bk.decode_step(c1, cfg, q1, kn1, kn1).data
    torch.cuda.synchronize(1)
    assert out1.device.index == 1 and torch.isfinite(out1).all()


def test_device_outputs_are_validated():
    from paper_2503_18773_b200 import bitkv as bk
    torch.cuda.set_device(0)
    c, cfg = _mk(0, precise=False)
    q = torch.randn((1, 8, D), device="cuda:0").half()
    kn = torch.randn((1, 2, D), device="cuda:0").half()
    for bad in (torch.empty((1, 8, D), device="cuda:0", dtype=torch.float16),
                torch.empty((1, 8, D - 1), device="cuda:0"),
                torch.empty((1, D, 8), device="cuda:0").transpose(1, 2),
                torch.empty((1, 8, D))):
        with pytest.raises(bk.ShapeError):
            bk.decode_step(c, cfg, q, kn, kn, out=bad)
        with pytest.raises(bk.ShapeError):
            bk.decode_partial(c, cfg, q, out=bad)
    with pytest.raises(bk.ShapeError):
        bk.decode_partial(c, cfg, q, lse=torch.empty((1, 9), device="cuda:0"))
    with pytest.raises(bk.ShapeError):  # host path: a mismatched out raises
        bk.decode_step(c, cfg, q.cpu().float().numpy(), kn.cpu().float().numpy(),
                       kn.cpu().float().numpy(), out=np.empty((1, 8, D), np.float64))
    # nothing was appended by the rejected calls
    assert c.res_len(0, 0) == 300 % c.n_r()
