"""B200-native (sm_100a) BitDecoding decode hot path: low-bit KV-cache decode
attention behind the C-ABI of include/bitdecode_b200.h.

    from paper_2503_18773_b200 import bitkv
    cache = bitkv.KVCache(1, 8, 128, 4, bitkv.QuantSpec(4, bitkv.QuantAxis.KChannel, 128))

See DESIGN.md for the data layout and kernels and INTEGRATION.md for the
reference-side bindings.
"""
from . import bitkv  # noqa: F401
from ._lib import LIB_PATH, load  # noqa: F401

__all__ = ["bitkv", "load", "LIB_PATH"]
