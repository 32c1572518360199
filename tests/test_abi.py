"""The C-ABI boundary: library loads and exports every declared symbol (CPU)."""
import ctypes
import os

import pytest

from paper_2503_18773_b200 import _lib


def test_header_declares_the_bound_symbols():
    declared = set(_lib.header_symbols())
    assert declared, "no BDK_API declarations found"
    assert declared == set(_lib.SIGNATURES), (declared ^ set(_lib.SIGNATURES))


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (python -m paper_2503_18773_b200.build)")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in _lib.header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_status_names_and_validation_without_a_gpu():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    from paper_2503_18773_b200 import bitkv
    L = _lib.load()
    assert L.bdk_status_name(5) == b"CapacityError"
    # validate_config is pure host logic (config.cpp:10-30); no device needed
    cfg = bitkv.AttentionConfig(batch=1, heads_q=32, heads_kv=8, head_dim=128, tile_m=4,
                                tile_n=64, num_splits=1, warp_n=4)
    assert bitkv.validate_config(cfg).n_group() == 4
    bad = bitkv.AttentionConfig(heads_q=32, heads_kv=5)
    with pytest.raises(bitkv.ConfigError):
        bitkv.validate_config(bad)
    bad = bitkv.AttentionConfig(tile_n=100, warp_n=4)
    with pytest.raises(bitkv.ConfigError):
        bitkv.validate_config(bad)
    bad = bitkv.AttentionConfig(head_dim=0)
    with pytest.raises(bitkv.ConfigError):
        bitkv.validate_config(bad)
