"""ctypes binding of the C-ABI in include/bitdecode_b200.h.

This is the stub a reference-side maintainer would add: one
``argtypes``/``restype`` declaration per exported symbol.  Loading fails
loudly when the in-tree library is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libbitdecode_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "bitdecode_b200.h")

u32, i32, u16, sz = C.c_uint32, C.c_int32, C.c_uint16, C.c_size_t
vp, fp, u16p = C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_uint16)


class CacheDesc(C.Structure):
    _fields_ = [("batch", u32), ("heads_kv", u32), ("head_dim", u32), ("warp_n", u32),
                ("num_bits", u32), ("k_axis", u32), ("group_size", u32), ("interleave", u32),
                ("max_tokens", u32), ("device", i32)]


class AttnConfig(C.Structure):
    _fields_ = [("batch", u32), ("heads_q", u32), ("heads_kv", u32), ("head_dim", u32),
                ("tile_m", u32), ("tile_n", u32), ("num_splits", u32), ("warp_n", u32),
                ("warp_m", u32)]


class CacheInfo(C.Structure):
    _fields_ = [("n_r", u32), ("pack_num", u32), ("words_per_block", u32), ("k_param_u16", u32),
                ("v_param_u16", u32), ("record_bytes", u32), ("max_blocks", u32),
                ("fast_path", u32)]


# symbol -> (restype, argtypes); mirrors include/bitdecode_b200.h one-to-one
SIGNATURES = {
    "bdk_last_error": (C.c_char_p, []),
    "bdk_status_name": (C.c_char_p, [C.c_int]),
    "bdk_validate_config": (C.c_int, [C.POINTER(AttnConfig)]),
    "bdk_cache_create": (C.c_int, [C.POINTER(CacheDesc), C.POINTER(vp)]),
    "bdk_cache_destroy": (C.c_int, [vp]),
    "bdk_cache_get_info": (C.c_int, [vp, C.POINTER(CacheInfo)]),
    "bdk_cache_lengths": (C.c_int, [vp, u32, u32, C.POINTER(u32), C.POINTER(u32)]),
    "bdk_prefill": (C.c_int, [vp, u32, u32, vp, vp, u32, vp]),
    "bdk_prefill_all": (C.c_int, [vp, vp, vp, u32, vp]),
    "bdk_cache_reset": (C.c_int, [vp, vp]),
    "bdk_quantize_tile": (C.c_int, [vp, u32, u32, u32, u32, u32, vp, vp, i32]),
    "bdk_dequantize_tile": (C.c_int, [vp, vp, u32, u32, u32, u32, vp, i32]),
    "bdk_compute_group_params": (C.c_int, [vp, u32, u32, fp, fp, i32]),
    "bdk_quantize_group": (C.c_int, [vp, u32, C.c_float, C.c_float, u32, vp, i32]),
    "bdk_dequantize_group": (C.c_int, [vp, u32, C.c_float, C.c_float, vp, i32]),
    "bdk_peer_merge": (C.c_int, [C.POINTER(vp), C.POINTER(vp), u32, u32, C.c_uint64, u32, u32, vp,
                                 vp, vp, C.c_uint64, vp]),
    "bdk_dump_cache": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(C.c_uint64)]),
    "bdk_load_cache": (C.c_int, [vp, C.c_uint64, u32, C.c_int32, C.POINTER(vp)]),
    "bdk_dump_cache_file": (C.c_int, [vp, C.c_char_p]),
    "bdk_load_cache_file": (C.c_int, [C.c_char_p, u32, C.c_int32, C.POINTER(vp)]),
    "bdk_prefill_host": (C.c_int, [vp, u32, u32, u16p, u16p, u32]),
    "bdk_append_token_host": (C.c_int, [vp, u32, u32, u16p, u16p]),
    "bdk_packed_tile_host": (C.c_int, [vp, u32, u32, u32, u32, u16p, u16p]),
    "bdk_append_token": (C.c_int, [vp, u32, u32, vp, vp, vp]),
    "bdk_flush_residual": (C.c_int, [vp, u32, u32, vp]),
    "bdk_decode_step": (C.c_int, [vp, C.POINTER(AttnConfig), vp, vp, vp, vp, vp]),
    "bdk_decode_step_host": (C.c_int, [vp, C.POINTER(AttnConfig), vp, vp, vp, vp]),
    "bdk_graph_create": (C.c_int, [vp, C.POINTER(AttnConfig), vp, vp, vp, vp, u32,
                                   C.POINTER(vp)]),
    "bdk_graph_launch": (C.c_int, [vp, vp]),
    "bdk_graph_destroy": (C.c_int, [vp]),
    "bdk_decode_partial": (C.c_int, [vp, C.POINTER(AttnConfig), vp, vp, vp, u32, u32, u32, vp,
                                     vp, vp]),
    "bdk_merge_partials": (C.c_int, [vp, vp, u32, u32, u32, C.c_uint64, C.c_uint64, vp, vp]),
    "bdk_attend_tile_host": (C.c_int, [vp, vp, vp, u32, u32, vp, vp, vp, u32, C.c_float, u32,
                                       i32]),
    "bdk_partitioned_rowmax_host": (C.c_int, [vp, u32, u32, u32, vp, i32]),
    "bdk_residual_attend_host": (C.c_int, [vp, u32, u32, vp, u32, C.c_float, vp, vp, vp]),
    "bdk_packed_attend_host": (C.c_int, [vp, u32, u32, vp, u32, u32, u32, C.c_float, vp, vp, vp,
                                         C.POINTER(u32)]),
    "bdk_combine_host": (C.c_int, [vp, vp, vp, u32, u32, u32, vp, i32]),
    "bdk_set_precise": (C.c_int, [vp, C.c_int]),
    "bdk_read_block": (C.c_int, [vp, u32, u32, u32, u16p, u16p, u16p, u16p]),
    "bdk_adopt_block": (C.c_int, [vp, u32, u32, u16p, u16p, u16p, u16p]),
    "bdk_build_block": (C.c_int, [vp, u32, u32, u16p, u16p, u16p, u16p]),
    "bdk_commit_block": (C.c_int, [vp, u32, u32, u16p, u16p, u16p, u16p]),
    "bdk_read_residual": (C.c_int, [vp, u32, u32, u16p, u16p]),
    "bdk_dequant_blocks": (C.c_int, [vp, u32, u32, u32, u32, vp, vp, vp]),
    "bdk_memory": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
    "bdk_corrupt_word": (C.c_int, [vp, u32, u32, u32, u32, u16]),
    "bdk_profile_begin": (C.c_int, [vp]),
    "bdk_profile_end": (C.c_int, [vp, fp, C.POINTER(u32)]),
    "bdk_launch_count": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
    "bdk_synchronize": (C.c_int, []),
}

_lib = None


def header_symbols() -> list[str]:
    """Every BDK_API function declared in include/bitdecode_b200.h."""
    import re
    src = open(HEADER).read()
    return re.findall(r"BDK_API\s+[\w\s\*]+?\b(bdk_\w+)\s*\(", src)


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    # BDK_LIB (dev A/B runs): another build of the same C-ABI
    path = os.environ.get("BDK_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2503_18773_b200.build` "
            "(nvcc, sm_100a).  There is no CPU fallback.")
    L = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        if path != LIB_PATH and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
