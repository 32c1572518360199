"""ctypes front end for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Two checkers live behind this module:

* ``Oracle`` -- oracle/liboracle.so, the C restatement (bitkv_oracle.c) of the
  reference engine's decode hot path; always buildable (gcc only).
* ``Reference`` -- oracle/_ref/libbitkv_ref.so, the UNMODIFIED reference engine
  (/root/reference/proj/src) compiled out-of-tree by oracle/Makefile plus the
  extern "C" shim ref_shim.cpp.  Only present where /root/reference existed at
  build time (the .so then travels to the GPU box with the repo snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module.  The product path (paper_2503_18773_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbitkv_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_sz = C.c_size_t

STATUS_NAMES = {0: "OK", 1: "ConfigError", 2: "ShapeError", 3: "UnsupportedBits",
                4: "CodeOverflow", 5: "CapacityError", 6: "StateError", 7: "FormatError",
                8: "EmptyInput", 99: "Error"}


class OracleError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}")
        self.status = status
        self.kind = STATUS_NAMES.get(status, str(status))


def build(ref: bool | None = None) -> None:
    """Compile the checkers (make -C oracle).  ref=None builds _ref iff the
    reference sources are present."""
    targets = ["oracle"]
    if ref or (ref is None and os.path.isdir("/root/reference/proj/src")):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def _check(st: int, where: str) -> None:
    if st != 0:
        raise OracleError(st, where)


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
class Oracle:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                build(ref=False)
            L = C.CDLL(ORACLE_SO)
            L.orc_f32_to_f16_bits.restype = C.c_uint16
            L.orc_f32_to_f16_bits.argtypes = [C.c_float]
            L.orc_f16_bits_to_f32.restype = C.c_float
            L.orc_f16_bits_to_f32.argtypes = [C.c_uint16]
            L.orc_perm.argtypes = [C.c_uint32, C.c_int, C.POINTER(C.c_uint8),
                                   C.POINTER(C.c_uint32)]
            L.orc_pack_word.argtypes = [_u16p, C.c_uint32, C.c_int, C.POINTER(C.c_uint16)]
            L.orc_unpack_word.argtypes = [C.c_uint16, C.c_uint32, C.c_int, _u16p]
            L.orc_residual_block_size.restype = _sz
            L.orc_residual_block_size.argtypes = [C.c_uint32, _sz]
            L.orc_group_params.argtypes = [_f32p, _sz, _sz, C.c_uint32, C.POINTER(C.c_float),
                                           C.POINTER(C.c_float)]
            L.orc_quantize_group.argtypes = [_f32p, _sz, _sz, C.c_float, C.c_float, C.c_uint32,
                                             _u16p, _sz]
            L.orc_make_block.argtypes = [_f32p, _f32p, _sz, _sz, C.c_uint32, C.c_uint32, _sz,
                                         C.c_int, _u16p, _u16p, _u16p, _u16p]
            L.orc_param_count.restype = _sz
            L.orc_param_count.argtypes = [_sz, _sz, C.c_uint32, C.c_uint32, _sz]
            L.orc_dequant_block.argtypes = [_u16p, _u16p, _u16p, _u16p, _sz, _sz, C.c_uint32,
                                            C.c_uint32, _sz, C.c_int, _f32p, _f32p]
            L.orc_cache_create.restype = C.c_void_p
            L.orc_cache_create.argtypes = [_sz, _sz, _sz, _sz, C.c_uint32, C.c_uint32, _sz,
                                           C.c_int, _sz, C.POINTER(C.c_int)]
            L.orc_cache_destroy.argtypes = [C.c_void_p]
            for f in ("orc_cache_packed_len", "orc_cache_res_len"):
                getattr(L, f).restype = _sz
                getattr(L, f).argtypes = [C.c_void_p, _sz, _sz]
            for f in ("orc_cache_n_r", "orc_cache_words_per_block", "orc_cache_k_param_count",
                      "orc_cache_v_param_count"):
                getattr(L, f).restype = _sz
                getattr(L, f).argtypes = [C.c_void_p]
            L.orc_cache_prefill.argtypes = [C.c_void_p, _sz, _sz, _f32p, _f32p, _sz]
            L.orc_cache_append.argtypes = [C.c_void_p, _sz, _sz, _f32p, _f32p]
            L.orc_cache_flush.argtypes = [C.c_void_p, _sz, _sz]
            L.orc_cache_block.restype = C.POINTER(C.c_uint16)
            L.orc_cache_block.argtypes = [C.c_void_p, _sz, _sz, _sz, C.c_int]
            L.orc_cache_residual.restype = C.POINTER(C.c_float)
            L.orc_cache_residual.argtypes = [C.c_void_p, _sz, _sz, C.c_int]
            L.orc_cache_reconstruct.argtypes = [C.c_void_p, _sz, _sz, _f32p, _f32p]
            L.orc_decode_step.argtypes = [C.c_void_p, _sz, _sz, _sz, _sz, _f32p, _f32p, _f32p,
                                          _f32p, C.c_int]
            L.orc_naive_attention.argtypes = [_f32p, _sz, _f32p, _f32p, _sz, _sz, _f32p]
            L.orc_offline_quant_reference.argtypes = [_f32p, _f32p, _sz, _sz, C.c_uint32,
                                                      C.c_uint32, _sz, _sz, _f32p, _f32p]
            L.orc_gauss_init.argtypes = [C.c_void_p, C.c_uint64]
            L.orc_gauss_next.restype = C.c_float
            L.orc_gauss_next.argtypes = [C.c_void_p]
            L.orc_gauss_fill_rounded.argtypes = [C.c_void_p, _f32p, _sz]
            L.orc_gauss_fill_f16.argtypes = [C.c_void_p, _u16p, _sz]
            L.orc_gauss_fill_rounded_par.argtypes = [C.c_void_p, _f32p, _sz, C.c_int]
            L.orc_fnv1a64.restype = C.c_uint64
            L.orc_fnv1a64.argtypes = [C.c_void_p, _sz, C.c_uint64]
            cls._lib = L
        return cls._lib


def lib():
    return Oracle.lib()


def f32_to_f16_bits(x: float) -> int:
    return lib().orc_f32_to_f16_bits(x)


def f16_bits_to_f32(h: int) -> float:
    return lib().orc_f16_bits_to_f32(h)


def round_f16(x: float) -> float:
    return f16_bits_to_f32(f32_to_f16_bits(x))


def perm(bits: int, interleave: bool = True) -> list[int]:
    order = (C.c_uint8 * 8)()
    p = C.c_uint32()
    _check(lib().orc_perm(bits, int(interleave), order, C.byref(p)), "perm")
    return list(order)[: p.value]


def pack_word(codes, bits: int, interleave: bool = True) -> int:
    w = C.c_uint16()
    _check(lib().orc_pack_word(np.ascontiguousarray(codes, np.uint16), bits, int(interleave),
                               C.byref(w)), "pack_word")
    return w.value


def unpack_word(word: int, bits: int, interleave: bool = True) -> list[int]:
    out = np.zeros(16 // bits, np.uint16)
    _check(lib().orc_unpack_word(word, bits, int(interleave), out), "unpack_word")
    return out.tolist()


def residual_block_size(bits: int, warp_n: int) -> int:
    return lib().orc_residual_block_size(bits, warp_n)


def group_params(x, bits: int):
    x = np.ascontiguousarray(x, np.float32)
    s, z = C.c_float(), C.c_float()
    lib().orc_group_params(x, 1, x.size, bits, C.byref(s), C.byref(z))
    return s.value, z.value


def quantize_group(x, scale: float, zero: float, bits: int):
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros(x.size, np.uint16)
    lib().orc_quantize_group(x, 1, x.size, scale, zero, bits, out, 1)
    return out


def param_count(n_r, d, bits, axis, g) -> int:
    return lib().orc_param_count(n_r, d, bits, axis, g)


def make_block(k, v, n_r, d, bits, k_axis=0, g=128, interleave=True):
    """kvcache.cpp:184-206: returns (k_words, v_words, k_params, v_params)."""
    k = np.ascontiguousarray(k, np.float32).reshape(-1)
    v = np.ascontiguousarray(v, np.float32).reshape(-1)
    wpb = d * n_r * bits // 16
    kw, vw = np.zeros(wpb, np.uint16), np.zeros(wpb, np.uint16)
    kp = np.zeros(max(1, param_count(n_r, d, bits, k_axis, g)), np.uint16)
    vp = np.zeros(max(1, param_count(n_r, d, bits, 1, g)), np.uint16)
    _check(lib().orc_make_block(k, v, n_r, d, bits, k_axis, g, int(interleave), kw, vw, kp, vp),
           "make_block")
    return kw, vw, kp[: param_count(n_r, d, bits, k_axis, g)], vp[: param_count(n_r, d, bits, 1, g)]


def dequant_block(kw, vw, kp, vp, n_r, d, bits, k_axis=0, g=128, interleave=True):
    ko = np.zeros(n_r * d, np.float32)
    vo = np.zeros(n_r * d, np.float32)
    kp = np.ascontiguousarray(kp if len(kp) else np.zeros(1), np.uint16)
    vp = np.ascontiguousarray(vp if len(vp) else np.zeros(1), np.uint16)
    lib().orc_dequant_block(np.ascontiguousarray(kw, np.uint16), np.ascontiguousarray(vw, np.uint16),
                            kp, vp, n_r, d, bits, k_axis, g, int(interleave), ko, vo)
    return ko.reshape(n_r, d), vo.reshape(n_r, d)


def naive_attention(q, k, v):
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    rows, d = q.reshape(-1, k.shape[-1]).shape
    out = np.zeros((rows, d), np.float32)
    lib().orc_naive_attention(q.reshape(-1), rows, k.reshape(-1), v.reshape(-1), k.size // d, d,
                              out.reshape(-1))
    return out


def offline_quant_reference(k, v, bits, k_axis, g, n_r):
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    length, d = k.shape
    ko, vo = np.zeros_like(k), np.zeros_like(v)
    lib().orc_offline_quant_reference(k.reshape(-1), v.reshape(-1), length, d, bits, k_axis, g,
                                      n_r, ko.reshape(-1), vo.reshape(-1))
    return ko, vo


class Gauss:
    """bench.cpp:18-35 GaussianSource (deterministic across platforms)."""

    def __init__(self, seed: int):
        self._buf = C.create_string_buffer(312 * 8 + 64)
        lib().orc_gauss_init(self._buf, seed)

    def next(self) -> float:
        return lib().orc_gauss_next(self._buf)

    def rounded(self, n: int, threads: int = 1) -> np.ndarray:
        """n fp16-rounded draws; threads > 1 spreads the Box-Muller
        transforms over host threads (the same stream, bit for bit)."""
        out = np.empty(n, np.float32)
        if threads > 1:
            lib().orc_gauss_fill_rounded_par(self._buf, out, n, threads)
        else:
            lib().orc_gauss_fill_rounded(self._buf, out, n)
        return out

    def f16(self, n: int) -> np.ndarray:
        out = np.empty(n, np.uint16)
        lib().orc_gauss_fill_f16(self._buf, out, n)
        return out


def fnv1a64(arr: np.ndarray, seed: int = 0xCBF29CE484222325) -> int:
    a = np.ascontiguousarray(arr)
    return lib().orc_fnv1a64(a.ctypes.data, a.nbytes, seed)


class OracleCache:
    """KVCache restated (kvcache.cpp) + decode_step (attention.cpp:164-242)."""

    def __init__(self, batch, heads_kv, d, warp_n, bits, k_axis=0, group_size=128,
                 interleave=True, max_tokens=1 << 16):
        st = C.c_int()
        self._h = lib().orc_cache_create(batch, heads_kv, d, warp_n, bits, k_axis, group_size,
                                         int(interleave), max_tokens, C.byref(st))
        _check(st.value, "KVCache")
        self.batch, self.heads_kv, self.d, self.warp_n = batch, heads_kv, d, warp_n
        self.bits, self.k_axis, self.g, self.interleave = bits, k_axis, group_size, interleave
        self.n_r = lib().orc_cache_n_r(self._h)
        self.wpb = lib().orc_cache_words_per_block(self._h)
        self.kpc = lib().orc_cache_k_param_count(self._h)
        self.vpc = lib().orc_cache_v_param_count(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:  # module globals may already be gone at interpreter exit
                lib().orc_cache_destroy(h)
            except Exception:
                pass
            self._h = None

    def packed_len(self, b, h):
        return lib().orc_cache_packed_len(self._h, b, h)

    def res_len(self, b, h):
        return lib().orc_cache_res_len(self._h, b, h)

    def prefill(self, b, h, k, v):
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        _check(lib().orc_cache_prefill(self._h, b, h, k.reshape(-1), v.reshape(-1),
                                       k.shape[0]), "prefill")

    def append_token(self, b, h, k_row, v_row):
        _check(lib().orc_cache_append(self._h, b, h, np.ascontiguousarray(k_row, np.float32),
                                      np.ascontiguousarray(v_row, np.float32)), "append_token")

    def flush_residual(self, b, h):
        _check(lib().orc_cache_flush(self._h, b, h), "flush_residual")

    def block(self, b, h, i):
        """(k_words, v_words, k_params, v_params) of packed block i."""
        n = [self.wpb, self.wpb, self.kpc, self.vpc]
        out = []
        for which in range(4):
            p = lib().orc_cache_block(self._h, b, h, i, which)
            if not p:
                raise IndexError(i)
            out.append(np.ctypeslib.as_array(p, (max(n[which], 1),))[: n[which]].copy())
        return tuple(out)

    def residual(self, b, h):
        r = self.res_len(b, h)
        ks = np.ctypeslib.as_array(lib().orc_cache_residual(self._h, b, h, 0), (self.n_r * self.d,))
        vs = np.ctypeslib.as_array(lib().orc_cache_residual(self._h, b, h, 1), (self.n_r * self.d,))
        return ks[: r * self.d].reshape(r, self.d).copy(), vs[: r * self.d].reshape(r, self.d).copy()

    def reconstruct(self, b, h):
        t = self.packed_len(b, h) + self.res_len(b, h)
        k = np.zeros((t, self.d), np.float32)
        v = np.zeros((t, self.d), np.float32)
        _check(lib().orc_cache_reconstruct(self._h, b, h, k.reshape(-1), v.reshape(-1)),
               "reconstruct")
        return k, v

    def decode_step(self, q, k_new, v_new, tile_n=64, num_splits=4, warp_n=None, threads=0):
        q = np.ascontiguousarray(q, np.float32)
        k_new = np.ascontiguousarray(k_new, np.float32)
        v_new = np.ascontiguousarray(v_new, np.float32)
        heads_q = q.shape[1]
        out = np.zeros(q.shape, np.float32)
        _check(lib().orc_decode_step(self._h, heads_q, tile_n, num_splits,
                                     warp_n or self.warp_n, q.reshape(-1), k_new.reshape(-1),
                                     v_new.reshape(-1), out.reshape(-1), threads), "decode_step")
        return out


# --------------------------------------------------------------------------
# the unmodified reference (oracle/_ref)
# --------------------------------------------------------------------------
class Reference:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not have_ref():
                raise FileNotFoundError(REF_SO + " (build with make -C oracle ref)")
            L = C.CDLL(REF_SO)
            L.ref_last_error.restype = C.c_char_p
            L.ref_pack_word.argtypes = [_u16p, C.c_uint32, C.c_int, C.POINTER(C.c_uint16)]
            L.ref_unpack_word.argtypes = [C.c_uint16, C.c_uint32, C.c_int, _u16p]
            L.ref_group_params.argtypes = [_f32p, _sz, C.c_uint32, C.POINTER(C.c_float),
                                           C.POINTER(C.c_float)]
            L.ref_cache_create.argtypes = [_sz, _sz, _sz, _sz, C.c_uint32, C.c_uint32, _sz,
                                           C.c_int, C.POINTER(C.c_void_p)]
            L.ref_cache_destroy.argtypes = [C.c_void_p]
            L.ref_cache_n_r.restype = _sz
            L.ref_cache_n_r.argtypes = [C.c_void_p]
            for f in ("ref_cache_packed_len", "ref_cache_res_len"):
                getattr(L, f).restype = _sz
                getattr(L, f).argtypes = [C.c_void_p, _sz, _sz]
            L.ref_cache_prefill.argtypes = [C.c_void_p, _sz, _sz, _f32p, _f32p, _sz]
            L.ref_cache_append.argtypes = [C.c_void_p, _sz, _sz, _f32p, _f32p]
            L.ref_cache_flush.argtypes = [C.c_void_p, _sz, _sz]
            L.ref_cache_block.argtypes = [C.c_void_p, _sz, _sz, _sz, C.c_int, _u16p, _sz,
                                          C.POINTER(_sz)]
            L.ref_cache_reconstruct.argtypes = [C.c_void_p, _sz, _sz, _f32p, _f32p]
            L.ref_cache_memory.argtypes = [C.c_void_p, C.POINTER(_sz)]
            L.ref_cache_dump.argtypes = [C.c_void_p, C.c_void_p, _sz, C.POINTER(_sz)]
            L.ref_cache_load.argtypes = [C.c_void_p, _sz, C.POINTER(C.c_void_p)]
            L.ref_decode_step.argtypes = [C.c_void_p, _sz, _sz, _sz, _sz, _f32p, _f32p, _f32p,
                                          _f32p]
            L.ref_naive_attention.argtypes = [_f32p, _sz, _f32p, _f32p, _sz, _sz, _f32p]
            L.ref_run_bench.argtypes = [C.c_int, _sz, _sz, _sz, _sz, _sz, C.c_uint32, _sz,
                                        C.c_uint32, _sz, _sz, C.c_uint64, _sz, _sz, C.c_int,
                                        C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), _sz]
            L.ref_run_verify.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32]
            cls._lib = L
        return cls._lib


def _rcheck(st, where):
    if st != 0:
        msg = Reference.lib().ref_last_error().decode(errors="replace")
        e = OracleError(st, where + ": " + msg)
        raise e


def ref_pack_word(codes, bits, interleave=True):
    w = C.c_uint16()
    _rcheck(Reference.lib().ref_pack_word(np.ascontiguousarray(codes, np.uint16), bits,
                                          int(interleave), C.byref(w)), "pack_word")
    return w.value


def ref_group_params(x, bits):
    x = np.ascontiguousarray(x, np.float32)
    s, z = C.c_float(), C.c_float()
    _rcheck(Reference.lib().ref_group_params(x, x.size, bits, C.byref(s), C.byref(z)),
            "group_params")
    return s.value, z.value


def ref_naive_attention(q, k, v):
    q = np.ascontiguousarray(q, np.float32)
    d = k.shape[-1]
    rows = q.size // d
    out = np.zeros((rows, d), np.float32)
    Reference.lib().ref_naive_attention(q.reshape(-1), rows,
                                        np.ascontiguousarray(k, np.float32).reshape(-1),
                                        np.ascontiguousarray(v, np.float32).reshape(-1),
                                        k.size // d, d, out.reshape(-1))
    return out


class RefCache:
    """Handle over the unmodified reference bitkv::KVCache."""

    def __init__(self, batch, heads_kv, d, warp_n, bits, k_axis=0, group_size=128,
                 interleave=True, _handle=None):
        L = Reference.lib()
        if _handle is None:
            h = C.c_void_p()
            _rcheck(L.ref_cache_create(batch, heads_kv, d, warp_n, bits, k_axis, group_size,
                                       int(interleave), C.byref(h)), "KVCache")
            _handle = h.value
        self._h = _handle
        self.batch, self.heads_kv, self.d, self.warp_n = batch, heads_kv, d, warp_n
        self.bits, self.k_axis, self.g = bits, k_axis, group_size
        self.n_r = L.ref_cache_n_r(self._h)

    @classmethod
    def load(cls, blob: bytes, **geom):
        h = C.c_void_p()
        buf = C.create_string_buffer(blob, len(blob))
        _rcheck(Reference.lib().ref_cache_load(buf, len(blob), C.byref(h)), "load_cache")
        return cls(_handle=h.value, **geom)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and Reference._lib is not None:
            Reference._lib.ref_cache_destroy(h)
            self._h = None

    def packed_len(self, b, h):
        return Reference.lib().ref_cache_packed_len(self._h, b, h)

    def res_len(self, b, h):
        return Reference.lib().ref_cache_res_len(self._h, b, h)

    def prefill(self, b, h, k, v):
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        _rcheck(Reference.lib().ref_cache_prefill(self._h, b, h, k.reshape(-1), v.reshape(-1),
                                                  k.shape[0]), "prefill")

    def append_token(self, b, h, k_row, v_row):
        _rcheck(Reference.lib().ref_cache_append(self._h, b, h,
                                                 np.ascontiguousarray(k_row, np.float32),
                                                 np.ascontiguousarray(v_row, np.float32)),
                "append_token")

    def flush_residual(self, b, h):
        _rcheck(Reference.lib().ref_cache_flush(self._h, b, h), "flush_residual")

    def block(self, b, h, i):
        out = []
        for which in range(4):
            cap = 1 << 20
            buf = np.zeros(cap, np.uint16)
            n = _sz()
            _rcheck(Reference.lib().ref_cache_block(self._h, b, h, i, which, buf, cap,
                                                    C.byref(n)), "block")
            out.append(buf[: n.value].copy())
        return tuple(out)

    def reconstruct(self, b, h):
        t = self.packed_len(b, h) + self.res_len(b, h)
        k = np.zeros((t, self.d), np.float32)
        v = np.zeros((t, self.d), np.float32)
        _rcheck(Reference.lib().ref_cache_reconstruct(self._h, b, h, k.reshape(-1),
                                                      v.reshape(-1)), "reconstruct")
        return k, v

    def memory(self):
        out = (_sz * 4)()
        _rcheck(Reference.lib().ref_cache_memory(self._h, out), "memory")
        return tuple(out)

    def dump(self) -> bytes:
        n = _sz()
        Reference.lib().ref_cache_dump(self._h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value)
        _rcheck(Reference.lib().ref_cache_dump(self._h, buf, n.value, C.byref(n)), "dump")
        return buf.raw[: n.value]

    def decode_step(self, q, k_new, v_new, tile_n=64, num_splits=4, warp_n=None):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(q.shape, np.float32)
        _rcheck(Reference.lib().ref_decode_step(
            self._h, q.shape[1], tile_n, num_splits, warp_n or self.warp_n, q.reshape(-1),
            np.ascontiguousarray(k_new, np.float32).reshape(-1),
            np.ascontiguousarray(v_new, np.float32).reshape(-1), out.reshape(-1)),
            "decode_step")
        return out


def ref_run_bench(*, mode=0, seq_len=4096, batch=1, heads_q=32, heads_kv=8, head_dim=128,
                  bits=4, group_size=128, k_axis=0, num_splits=4, steps=4, seed=0, tile_n=64,
                  warp_n=4, interleave=True, verify=False) -> dict:
    """The reference's own run_bench (bench.cpp:80-210)."""
    out = (C.c_double * 11)()
    orc = (C.c_double * 3)()
    step_ms = (C.c_double * max(1, steps))()
    _rcheck(Reference.lib().ref_run_bench(mode, seq_len, batch, heads_q, heads_kv, head_dim, bits,
                                          group_size, k_axis, num_splits, steps, seed, tile_n,
                                          warp_n, int(interleave), int(verify), out, orc,
                                          step_ms, steps),
            "run_bench")
    ck = np.array([out[5]], np.float64).view(np.uint64)[0]
    return {"prefill_seconds": out[0], "mean_ms": out[1], "p50_ms": out[2], "p99_ms": out[3],
            "tokens_per_second": out[4], "output_checksum": int(ck),
            "memory": [int(out[6]), int(out[7]), int(out[8]), int(out[9])], "n_r": int(out[10]),
            "oracle": list(orc), "step_ms": list(step_ms)[:steps]}


def ref_run_verify(seed_begin=0, seed_end=2, bits=4) -> int:
    return Reference.lib().ref_run_verify(seed_begin, seed_end, bits)
