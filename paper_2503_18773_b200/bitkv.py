"""Host-side mirror of the reference ``bitkv::`` API over the sm_100a C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/bitkv (cited per symbol) so tests read like the
reference's doctest suites.  The cache lives in HBM; every numeric step
(quantize+pack, dequant, attention, combine) runs in the CUDA kernels behind
include/bitdecode_b200.h.  Host-side code only converts layouts, checks the
reference preconditions and moves bytes.

Tensor arguments accept either CUDA ``torch.float16`` tensors (used in place,
stream-ordered on the current torch stream) or host arrays of
binary16-representable fp32 values (the reference Tensor contract,
tensor.hpp:16-46), which are uploaded.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib as _L

try:
    import torch
except ImportError:  # pragma: no cover - torch is the device-memory plumbing
    torch = None


# --------------------------------------------------------------- errors.hpp
class Error(RuntimeError):
    """bitkv::Error (errors.hpp:9-12)."""


class ConfigError(Error):
    pass


class ShapeError(Error):
    pass


class UnsupportedBits(Error):
    pass


class CodeOverflow(Error):
    pass


class CapacityError(Error):
    pass


class StateError(Error):
    pass


class FormatError(Error):
    """bitkv::FormatError (errors.hpp); ``offset`` is the byte offset."""

    @property
    def offset(self) -> int | None:
        import re
        m = re.search(r"byte offset (\d+)", str(self))
        return int(m.group(1)) if m else None


class EmptyInput(Error):
    pass


class CudaError(Error):
    pass


class Unsupported(Error):
    pass


_STATUS = {1: ConfigError, 2: ShapeError, 3: UnsupportedBits, 4: CodeOverflow, 5: CapacityError,
           6: StateError, 7: FormatError, 8: EmptyInput, 20: CudaError, 21: Unsupported,
           22: Error}


def _check(status: int) -> None:
    if status != 0:
        msg = _L.load().bdk_last_error().decode(errors="replace")
        raise _STATUS.get(status, Error)(msg)


# ----------------------------------------------------------------- quant.hpp
class QuantAxis(enum.IntEnum):
    """quant.hpp:12-15"""
    KChannel = 0
    KToken = 1


@dataclass
class QuantSpec:
    """quant.hpp:19-25"""
    num_bits: int = 4
    k_axis: QuantAxis = QuantAxis.KChannel
    group_size: int = 64

    def passthrough(self) -> bool:
        return self.num_bits == 16


class CacheBackend(enum.IntEnum):
    """kvcache.hpp:100 (the paged backend is host bookkeeping)."""
    Contiguous = 0
    Paged = 1


# ---------------------------------------------------------------- config.hpp
@dataclass
class AttentionConfig:
    """config.hpp:13-25"""
    batch: int = 1
    heads_q: int = 32
    heads_kv: int = 8
    head_dim: int = 128
    tile_m: int = 1
    tile_n: int = 64
    num_splits: int = 1
    warp_n: int = 4
    warp_m: int = 1

    def n_group(self) -> int:
        return self.heads_q // self.heads_kv

    def __setattr__(self, name, value):
        # the fields are plain and mutable: a change drops the cached C struct
        self.__dict__.pop("_c_cache", None)
        object.__setattr__(self, name, value)

    def _c(self) -> _L.AttnConfig:
        return self._c_ref()[0]

    def _c_ref(self):
        """(C struct, reusable byref of it, its address, q / k_new element
        counts, q / kv shapes), built on first use after a field change."""
        cached = self.__dict__.get("_c_cache")
        if cached is None:
            key = (self.batch, self.heads_q, self.heads_kv, self.head_dim, self.tile_m,
                   self.tile_n, self.num_splits, self.warp_n, self.warp_m)
            st = _L.AttnConfig(*key)
            sq = (self.batch, self.heads_q, self.head_dim)
            skv = (self.batch, self.heads_kv, self.head_dim)
            cached = (st, C.byref(st), C.addressof(st), math.prod(sq), math.prod(skv), sq, skv)
            self.__dict__["_c_cache"] = cached
        return cached


def validate_config(cfg: AttentionConfig) -> AttentionConfig:
    """validate_config (config.hpp:29, config.cpp:10-30)."""
    c = cfg._c()
    _check(_L.load().bdk_validate_config(C.byref(c)))
    return cfg


def residual_block_size(num_bits: int, warp_n: int) -> int:
    """layout.cpp:74-77: N_r = 8 * W_n * (16 / B)."""
    if num_bits not in (2, 4, 8, 16):
        raise UnsupportedBits(f"num_bits must be one of 2, 4, 8, 16; got {num_bits}")
    return 8 * warp_n * (16 // num_bits)


# --------------------------------------------------------------- kvcache.hpp
# ----------------------------------------------------------- quant.hpp API
@dataclass
class GroupParams:
    """quant.hpp:45-48"""
    scale: float
    zero: float


@dataclass
class QuantParams:
    """quant.hpp:30-43: (scale, zero) binary16 bit pairs, grid rows x cols."""
    rows: int
    cols: int
    data: np.ndarray  # uint16 [2 * rows * cols]

    def group_count(self) -> int:
        return self.rows * self.cols

    def scale(self, g: int) -> float:
        return float(self.data[2 * g:2 * g + 1].view(np.float16)[0])

    def zero(self, g: int) -> float:
        return float(self.data[2 * g + 1:2 * g + 2].view(np.float16)[0])


@dataclass
class QuantizedTile:
    """quant.hpp:62-65: row-major [rows, d] codes + params."""
    codes: np.ndarray  # uint16 [rows, d]
    params: QuantParams


def compute_group_params(group, num_bits: int, device: int = 0) -> GroupParams:
    """compute_group_params (quant.cpp:18-28), on the device."""
    x = np.ascontiguousarray(group, np.float32).ravel()
    s, z = C.c_float(), C.c_float()
    _check(_L.load().bdk_compute_group_params(x.ctypes.data, x.size, num_bits, C.byref(s),
                                              C.byref(z), device))
    return GroupParams(s.value, z.value)


def quantize_group(group, scale: float, zero: float, num_bits: int, device: int = 0) -> np.ndarray:
    """quantize_group (quant.cpp:30-38), on the device -> uint16 codes."""
    x = np.ascontiguousarray(group, np.float32).ravel()
    codes = np.zeros(x.size, np.uint16)
    _check(_L.load().bdk_quantize_group(x.ctypes.data, x.size, scale, zero, num_bits,
                                        codes.ctypes.data, device))
    return codes


def dequantize_group(codes, scale: float, zero: float, device: int = 0) -> np.ndarray:
    """dequantize_group (quant.cpp:40-44): code * scale + zero in fp32."""
    c = np.ascontiguousarray(codes, np.uint16).ravel()
    out = np.zeros(c.size, np.float32)
    _check(_L.load().bdk_dequantize_group(c.ctypes.data, c.size, scale, zero, out.ctypes.data,
                                          device))
    return out


def quantize_tile(tile, num_bits: int, axis: QuantAxis, group_size: int,
                  device: int = 0) -> QuantizedTile:
    """quantize_tile (quant.cpp:47-93) of a row-major [rows, d] tile."""
    x = np.ascontiguousarray(tile, np.float32)
    rows, d = x.shape
    codes = np.zeros((rows, d), np.uint16)
    groups = rows * d // group_size if group_size else 0
    prm = np.zeros(2 * max(groups, 1), np.uint16)
    _check(_L.load().bdk_quantize_tile(x.ctypes.data, rows, d, num_bits, int(axis), group_size,
                                       codes.ctypes.data, prm.ctypes.data, device))
    pr, pc = ((rows // group_size, d) if QuantAxis(axis) == QuantAxis.KChannel
              else (rows, d // group_size))
    return QuantizedTile(codes, QuantParams(pr, pc, prm[:2 * groups]))


def dequantize_tile(codes, params: QuantParams, rows: int, d: int, axis: QuantAxis,
                    group_size: int, device: int = 0) -> np.ndarray:
    """dequantize_tile (quant.cpp:95-110): values rounded to binary16."""
    c = np.ascontiguousarray(codes, np.uint16)
    if c.size != rows * d:
        raise ShapeError("dequantize_tile: codes do not cover the tile")
    prm = np.ascontiguousarray(params.data, np.uint16)
    out = np.zeros((rows, d), np.float32)
    _check(_L.load().bdk_dequantize_tile(c.ctypes.data, prm.ctypes.data, rows, d, int(axis),
                                         group_size, out.ctypes.data, device))
    return out


# ---------------------------------------------------------- layout.hpp API
# The word layout is metadata (which field holds which token), not
# arithmetic: these mirror layout.cpp:21-86 for callers of the reference API.
def interleave_order(num_bits: int) -> list[int]:
    """interleave_order (layout.cpp:21-34): odd indices descending, then even."""
    p = _pack_num(num_bits)
    return [i for i in range(p - 1, -1, -1) if i % 2] + [i for i in range(p - 1, -1, -1)
                                                        if i % 2 == 0]


def identity_order(num_bits: int) -> list[int]:
    """identity_order (layout.cpp:36-43)."""
    return list(range(_pack_num(num_bits)))


def _pack_num(num_bits: int) -> int:
    if num_bits not in (2, 4, 8, 16):
        raise UnsupportedBits(f"num_bits must be one of 2, 4, 8, 16, got {num_bits}")
    return 16 // num_bits


def pack_word(codes, num_bits: int, order: list[int]) -> int:
    """pack_word (layout.cpp:45-61): field k (from the MSB) holds codes[order[k]];
    CodeOverflow if a code needs more than num_bits bits."""
    p = _pack_num(num_bits)
    w = 0
    for k in range(p):
        c = int(codes[order[k]])
        if c >> num_bits:
            raise CodeOverflow(f"code {c} does not fit in {num_bits} bits")
        w |= c << (16 - (k + 1) * num_bits)
    return w


def unpack_word(word: int, num_bits: int, order: list[int]) -> list[int]:
    """unpack_word (layout.cpp:63-72)."""
    p = _pack_num(num_bits)
    out = [0] * p
    for k in range(p):
        out[order[k]] = (word >> (16 - (k + 1) * num_bits)) & ((1 << num_bits) - 1)
    return out


def pack_block_codes(codes, n_r: int, d: int, num_bits: int, order: list[int]) -> np.ndarray:
    """pack_block_codes (kvcache.cpp:79-95): row-major [n_r, d] codes ->
    channel-major words, pack_num consecutive tokens per word."""
    p = _pack_num(num_bits)
    c = np.asarray(codes, np.uint32).reshape(n_r, d)
    if n_r % p:
        raise ShapeError("pack_block_codes: N_r not pack-aligned")
    if num_bits < 16 and (c >> num_bits).any():
        raise CodeOverflow(f"a code does not fit in {num_bits} bits")
    g = c.reshape(n_r // p, p, d)  # [word group, token in word, channel]
    w = np.zeros((n_r // p, d), np.uint32)
    for k in range(p):
        w |= g[:, order[k], :] << (16 - (k + 1) * num_bits)
    return w.T.reshape(-1).astype(np.uint16)  # [d][n_r / p]


def unpack_block_codes(words, n_r: int, d: int, num_bits: int, order: list[int]) -> np.ndarray:
    """unpack_block_codes (kvcache.cpp:97-112)."""
    p = _pack_num(num_bits)
    w = np.asarray(words, np.uint32).reshape(d, n_r // p).T  # [word group, channel]
    mask = (1 << num_bits) - 1 if num_bits < 16 else 0xFFFF
    out = np.zeros((n_r // p, p, d), np.uint16)
    for k in range(p):
        out[:, order[k], :] = (w >> (16 - (k + 1) * num_bits)) & mask
    return out.reshape(n_r, d)


def iteration_count(tile_n: int, warp_n: int) -> int:
    """iteration_count (layout.cpp:79-86): T_n / (W_n * 8)."""
    if warp_n == 0 or tile_n % (warp_n * 8):
        raise ShapeError(f"tile_n ({tile_n}) must be a multiple of warp_n * 8")
    return tile_n // (warp_n * 8)


@dataclass
class PackedBlock:
    """kvcache.hpp:17-26 (u16 arrays in the reference layout)."""
    k_words: np.ndarray
    v_words: np.ndarray
    k_params: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint16))
    v_params: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint16))

    def __eq__(self, other) -> bool:
        return all(np.array_equal(getattr(self, f), getattr(other, f))
                   for f in ("k_words", "v_words", "k_params", "v_params"))


@dataclass
class Memory:
    """KVCache::Memory (kvcache.hpp:165-171)."""
    k_packed_payload_bytes: int
    v_packed_payload_bytes: int
    params_bytes: int
    residual_bytes: int


def _u16p(a: np.ndarray):
    return a.ctypes.data_as(_L.u16p) if a is not None and a.size else None


def _stream_ptr():
    if torch is not None and torch.cuda.is_available():
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return None


def _as_f16_cuda(x, shape=None, device=0):
    """torch CUDA fp16 contiguous view of x (kept alive by the caller)."""
    if torch is None:
        raise Error("torch is required for device memory plumbing")
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.to(f"cuda:{device}")
        if t.dtype != torch.float16:
            t = t.to(torch.float16)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(f"cuda:{device}").half()
    t = t.contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        if t.numel() != math.prod(shape):
            raise ShapeError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
        t = t.reshape(shape)
    return t


class KVCache:
    """bitkv::KVCache (kvcache.hpp:103-189) with the packed segment and the
    residual window resident in HBM.  ``max_tokens`` sizes the per-cell arena
    (the reference grows host vectors instead)."""

    def __init__(self, batch: int, heads_kv: int, head_dim: int, warp_n: int,
                 spec: QuantSpec | None = None, backend: CacheBackend = CacheBackend.Contiguous,
                 page_size: int = 16, max_pages: int = 0, interleave: bool = True, *,
                 max_tokens: int = 1 << 16, device: int = 0, precise: bool = True):
        spec = spec or QuantSpec()
        self._h = None
        if backend == CacheBackend.Paged:
            n_r = residual_block_size(spec.num_bits, warp_n)
            if page_size == 0 or n_r % page_size:
                raise ConfigError(f"page_size ({page_size}) must divide N_r ({n_r})")
        desc = _L.CacheDesc(batch, heads_kv, head_dim, warp_n, spec.num_bits, int(spec.k_axis),
                            spec.group_size, 1 if interleave else 0, max_tokens, device)
        h = C.c_void_p()
        _check(_L.load().bdk_cache_create(C.byref(desc), C.byref(h)))
        self._h = h
        self._batch, self._heads_kv, self._d, self._warp_n = batch, heads_kv, head_dim, warp_n
        self._spec, self._interleave, self._device = spec, bool(interleave), device
        self._backend, self._page_size = backend, page_size
        info = _L.CacheInfo()
        _check(_L.load().bdk_cache_get_info(self._h, C.byref(info)))
        self.info = info
        if not precise:
            self.set_precise(False)

    @classmethod
    def _adopt(cls, handle, header: bytes, device: int) -> "KVCache":
        """Wrap a cache the C-ABI created (load_cache); geometry from the
        BDKV header (serialize.hpp:11-20)."""
        import struct
        flags = header[5]
        bits, axis, g, n_r, d, batch, heads = struct.unpack_from("<7I", header, 6)
        self = cls.__new__(cls)
        self._h = handle
        self._batch, self._heads_kv, self._d = batch, heads, d
        self._warp_n = n_r // (8 * (16 // bits))
        self._spec = QuantSpec(bits, QuantAxis(axis), g)
        self._interleave, self._device = bool(flags & 1), device
        self._backend, self._page_size = CacheBackend.Contiguous, 16
        info = _L.CacheInfo()
        _check(_L.load().bdk_cache_get_info(self._h, C.byref(info)))
        self.info = info
        return self

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                _L.load().bdk_cache_destroy(self._h)
            except Exception:
                pass
            self._h = None

    # accessors (kvcache.hpp:111-121)
    def batch(self) -> int:
        return self._batch

    def heads_kv(self) -> int:
        return self._heads_kv

    def head_dim(self) -> int:
        return self._d

    def warp_n(self) -> int:
        return self._warp_n

    def n_r(self) -> int:
        return self.info.n_r

    def spec(self) -> QuantSpec:
        return self._spec

    def backend(self) -> CacheBackend:
        return self._backend

    def interleaved(self) -> bool:
        return self._interleave

    def handle(self):
        return self._h

    # state machine (kvcache.hpp:123-143)
    def prefill(self, b: int, h: int, k, v, length: int | None = None) -> None:
        """KVCache::prefill (kvcache.cpp:155-168); k, v: [len, d]."""
        k = _as_f16_cuda(k, device=self._device).reshape(-1, self._d)
        v = _as_f16_cuda(v, device=self._device).reshape(-1, self._d)
        n = k.shape[0] if length is None else length
        _check(_L.load().bdk_prefill(self._h, b, h, C.c_void_p(k.data_ptr()),
                                     C.c_void_p(v.data_ptr()), n, _stream_ptr()))
        self._keep = (k, v)

    def prefill_all(self, k, v) -> None:
        """All cells at once; k, v: [batch, heads_kv, len, d] (CUDA fp16)."""
        k = _as_f16_cuda(k, device=self._device)
        v = _as_f16_cuda(v, device=self._device)
        _check(_L.load().bdk_prefill_all(self._h, C.c_void_p(k.data_ptr()),
                                         C.c_void_p(v.data_ptr()), k.shape[-2], _stream_ptr()))
        self._keep = (k, v)

    def reset(self) -> None:
        """Empty every cell (a fresh KVCache of the same geometry, kvcache.cpp:114-148),
        keeping the device arena; stream-ordered."""
        _check(_L.load().bdk_cache_reset(self._h, _stream_ptr()))

    def append_token(self, b: int, h: int, k_row, v_row) -> None:
        """KVCache::append_token (kvcache.cpp:170-182)."""
        k = _as_f16_cuda(k_row, (self._d,), self._device)
        v = _as_f16_cuda(v_row, (self._d,), self._device)
        _check(_L.load().bdk_append_token(self._h, b, h, C.c_void_p(k.data_ptr()),
                                          C.c_void_p(v.data_ptr()), _stream_ptr()))
        self._keep = (k, v)

    def flush_residual(self, b: int, h: int) -> None:
        """KVCache::flush_residual (kvcache.cpp:245-251)."""
        _check(_L.load().bdk_flush_residual(self._h, b, h, _stream_ptr()))

    def adopt_block(self, b: int, h: int, block: PackedBlock) -> None:
        """KVCache::adopt_block (kvcache.cpp:239-243)."""
        kw = np.ascontiguousarray(block.k_words, np.uint16)
        vw = np.ascontiguousarray(block.v_words, np.uint16)
        kp = np.ascontiguousarray(block.k_params, np.uint16)
        vpp = np.ascontiguousarray(block.v_params, np.uint16)
        _check(_L.load().bdk_adopt_block(self._h, b, h, _u16p(kw), _u16p(vw), _u16p(kp),
                                         _u16p(vpp)))

    def build_block(self, b: int, h: int) -> PackedBlock:
        """KVCache::build_block (kvcache.cpp:208-219): the full residual
        quantized + packed on the device, not committed."""
        kw = np.zeros(self.info.words_per_block, np.uint16)
        vw = np.zeros(self.info.words_per_block, np.uint16)
        kp = np.zeros(self.info.k_param_u16, np.uint16)
        vpp = np.zeros(self.info.v_param_u16, np.uint16)
        _check(_L.load().bdk_build_block(self._h, b, h, _u16p(kw), _u16p(vw), _u16p(kp),
                                         _u16p(vpp)))
        return PackedBlock(kw, vw, kp, vpp)

    def commit_block(self, b: int, h: int, block: PackedBlock) -> None:
        """KVCache::commit_block (kvcache.cpp:231-237): append the block and
        clear the (full) residual."""
        kw = np.ascontiguousarray(block.k_words, np.uint16)
        vw = np.ascontiguousarray(block.v_words, np.uint16)
        kp = np.ascontiguousarray(block.k_params, np.uint16)
        vpp = np.ascontiguousarray(block.v_params, np.uint16)
        _check(_L.load().bdk_commit_block(self._h, b, h, _u16p(kw), _u16p(vw), _u16p(kp),
                                          _u16p(vpp)))

    def _lengths(self, b, h):
        p, r = C.c_uint32(), C.c_uint32()
        _check(_L.load().bdk_cache_lengths(self._h, b, h, C.byref(p), C.byref(r)))
        return p.value, r.value

    def packed_len(self, b: int, h: int) -> int:
        return self._lengths(b, h)[0]

    def res_len(self, b: int, h: int) -> int:
        return self._lengths(b, h)[1]

    def total_len(self, b: int, h: int) -> int:
        p, r = self._lengths(b, h)
        return p + r

    # readback (kvcache.hpp:145-160)
    def block(self, b: int, h: int, i: int) -> PackedBlock:
        kw = np.zeros(self.info.words_per_block, np.uint16)
        vw = np.zeros(self.info.words_per_block, np.uint16)
        kp = np.zeros(self.info.k_param_u16, np.uint16)
        vpp = np.zeros(self.info.v_param_u16, np.uint16)
        _check(_L.load().bdk_read_block(self._h, b, h, i, _u16p(kw), _u16p(vw), _u16p(kp),
                                        _u16p(vpp)))
        return PackedBlock(kw, vw, kp, vpp)

    def packed(self, b: int, h: int) -> list[PackedBlock]:
        """KVCache::packed(b, h).blocks (kvcache.hpp:148)."""
        return [self.block(b, h, i) for i in range(self.packed_len(b, h) // self.n_r())]

    def residual_tile(self, b: int, h: int):
        """KVCache::residual_tile (kvcache.cpp:253-261) -> fp32 [res_len, d] x2."""
        r = self.res_len(b, h)
        k = np.zeros(r * self._d, np.uint16)
        v = np.zeros(r * self._d, np.uint16)
        _check(_L.load().bdk_read_residual(self._h, b, h, _u16p(k), _u16p(v)))
        return (k.view(np.float16).astype(np.float32).reshape(r, self._d),
                v.view(np.float16).astype(np.float32).reshape(r, self._d))

    def packed_tile(self, b: int, h: int, t0: int, length: int):
        """KVCache::packed_tile (kvcache.cpp:263-312), dequantized on device."""
        n_r = self.n_r()
        if t0 + length > self.packed_len(b, h):
            raise ShapeError("packed_tile: range past packed segment")
        if length == 0:
            z = np.zeros((0, self._d), np.float32)
            return z, z.copy()
        blk0, blk1 = t0 // n_r, (t0 + length + n_r - 1) // n_r
        nb = blk1 - blk0
        kd = torch.empty((nb * n_r, self._d), dtype=torch.float16, device=f"cuda:{self._device}")
        vd = torch.empty_like(kd)
        _check(_L.load().bdk_dequant_blocks(self._h, b, h, blk0, nb, C.c_void_p(kd.data_ptr()),
                                            C.c_void_p(vd.data_ptr()), _stream_ptr()))
        off = t0 - blk0 * n_r
        return (kd[off:off + length].float().cpu().numpy(),
                vd[off:off + length].float().cpu().numpy())

    def reconstruct(self, b: int, h: int):
        """KVCache::reconstruct (kvcache.cpp:314-324)."""
        plen = self.packed_len(b, h)
        pk, pv = self.packed_tile(b, h, 0, plen)
        rk, rv = self.residual_tile(b, h)
        return np.concatenate([pk, rk]), np.concatenate([pv, rv])

    def corrupt_word(self, b: int, h: int, block: int, word: int, value: int) -> None:
        """KVCache::corrupt_word (kvcache.cpp:326-328)."""
        _check(_L.load().bdk_corrupt_word(self._h, b, h, block, word, value))

    def memory(self) -> Memory:
        """KVCache::memory (kvcache.cpp:330-345)."""
        out = (C.c_uint64 * 4)()
        _check(_L.load().bdk_memory(self._h, out))
        return Memory(*[int(x) for x in out])

    def profile_begin(self) -> None:
        """Start CUDA-event timing of the attention kernel (bdk_profile_begin)."""
        _check(_L.load().bdk_profile_begin(self._h))

    def profile_end(self) -> tuple[float, int]:
        """(summed attention-kernel ms, launches) since profile_begin."""
        ms, n = C.c_float(), C.c_uint32()
        _check(_L.load().bdk_profile_end(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def launch_count(self) -> int:
        """sm_100a kernels launched for this cache so far (bdk_launch_count)."""
        n = C.c_uint64()
        _check(_L.load().bdk_launch_count(self._h, C.byref(n)))
        return n.value

    def set_precise(self, precise: bool) -> None:
        """Decode numerics.  True (the default of every cache): bit-faithful
        dequant + P_hi + P_lo split PV, the reference's 1e-5 contract
        (test_attention.cpp:350-441).  False: the fast throughput kernel
        (folded scales, fp16 P; an explicit opt-in), SURVEY.md F4."""
        _check(_L.load().bdk_set_precise(self._h, 1 if precise else 0))


# ------------------------------------------------------------ attention.hpp
@dataclass
class AttnOutput:
    """attention.hpp:73-84: fp32 [batch, heads, d]."""
    batch: int
    heads: int
    d: int
    data: object  # torch CUDA tensor (device path) or numpy array (host path)

    def row(self, b: int, h: int):
        return self.data[b, h]


# ------------------------------------------------------------- serialize.hpp
def dump_cache(cache: KVCache) -> bytes:
    """dump_cache (serialize.hpp:19, serialize.cpp:87-122): BDKV v1 bytes."""
    n = C.c_uint64()
    L = _L.load()
    _check(L.bdk_dump_cache(cache.handle(), None, 0, C.byref(n)))
    buf = (C.c_uint8 * n.value)()
    _check(L.bdk_dump_cache(cache.handle(), buf, n.value, C.byref(n)))
    return bytes(buf)


def load_cache(data: bytes, *, max_tokens: int = 0, device: int = 0) -> KVCache:
    """load_cache (serialize.hpp:20, serialize.cpp:124-194); always a
    contiguous backend.  The arena holds max(max_tokens, longest cell + N_r)."""
    data = bytes(data)
    h = C.c_void_p()
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
    _check(_L.load().bdk_load_cache(buf, len(data), max_tokens, device, C.byref(h)))
    return KVCache._adopt(h, data[:34], device)


def dump_cache_file(cache: KVCache, path: str) -> None:
    """dump_cache_file (serialize.hpp:22)."""
    _check(_L.load().bdk_dump_cache_file(cache.handle(), str(path).encode()))


def load_cache_file(path: str, *, max_tokens: int = 0, device: int = 0) -> KVCache:
    """load_cache_file (serialize.hpp:23)."""
    h = C.c_void_p()
    _check(_L.load().bdk_load_cache_file(str(path).encode(), max_tokens, device, C.byref(h)))
    with open(path, "rb") as f:
        header = f.read(34)
    return KVCache._adopt(h, header, device)


_PYHOST = None


def _pyhost():
    """(step, address of bdk_decode_step_host) of the CPython fast path
    (csrc/bdk_pyhost.c, built in-tree next to the library), or False."""
    global _PYHOST
    if _PYHOST is None:
        _PYHOST = False
        try:
            import importlib.util
            import os
            from . import build as _B
            path = _B.pyhost_path()
            if os.path.exists(path):
                spec = importlib.util.spec_from_file_location("_bdk_pyhost", path)
                mod = importlib.util.module_from_spec(spec)
                spec.loader.exec_module(mod)
                fn = C.cast(_L.load().bdk_decode_step_host, C.c_void_p).value
                _PYHOST = (mod.step, fn)
        except Exception:
            _PYHOST = False
    return _PYHOST


def _addr(a: np.ndarray) -> int:
    """Data address of a C-contiguous array (the cheap way for writable
    buffers; ``ndarray.ctypes`` builds an object per access)."""
    try:
        return C.addressof(C.c_byte.from_buffer(a))
    except (TypeError, ValueError):
        return a.ctypes.data


def decode_step(cache: KVCache, cfg: AttentionConfig, q, k_new, v_new, out=None) -> AttnOutput:
    """decode_step (attention.hpp:87-88, attention.cpp:164-242).

    CUDA fp16 tensors in -> CUDA fp32 ``out`` (stream-ordered, no sync).
    Host arrays in -> numpy out via the host C-ABI entry (H2D/D2H inside);
    ``out`` may then be a C-contiguous float32 numpy array of q's shape to
    reuse across steps."""
    c, c_ref, c_addr, nq, nkv, shape_q, shape_kv = cfg._c_ref()
    if type(q) is np.ndarray and type(k_new) is np.ndarray and type(v_new) is np.ndarray \
            and type(out) is np.ndarray and q.shape == shape_q and k_new.shape == shape_kv \
            and v_new.shape == shape_kv and out.shape == shape_q:
        # the steady host loop: float32 C-contiguous arrays straight into the
        # C-ABI through the buffer protocol (csrc/bdk_pyhost.c); anything else
        # (other dtypes / layouts) takes the general path below
        ph = _pyhost()
        if ph:
            st = ph[0](ph[1], cache._h.value, c_addr, q, k_new, v_new, out, nq, nkv)
            if st != -1000:
                _check(st)
                return AttnOutput(cfg.batch, cfg.heads_q, cfg.head_dim, out)
    if type(q) is np.ndarray or not (torch is not None and isinstance(q, torch.Tensor) and q.is_cuda):
        qh = np.ascontiguousarray(q, np.float32)
        kh = np.ascontiguousarray(k_new, np.float32)
        vh = np.ascontiguousarray(v_new, np.float32)
        if qh.shape != shape_q or kh.shape != shape_kv or vh.shape != shape_kv:
            validate_config(cfg)
            raise ShapeError("decode_step: q must be [batch, heads_q, d], k_new/v_new "
                             "[batch, heads_kv, d]")
        if out is None:
            o = np.empty(shape_q, np.float32)
        elif isinstance(out, np.ndarray) and out.shape == shape_q and out.dtype == np.float32 \
                and out.flags.c_contiguous and out.flags.writeable:
            o = out
        else:
            raise ShapeError(f"decode_step: out must be a writable C-contiguous float32 array "
                             f"of shape {shape_q}")
        _check(_L.load().bdk_decode_step_host(cache.handle(), c_ref, _addr(qh), _addr(kh),
                                              _addr(vh), _addr(o)))
        return AttnOutput(cfg.batch, cfg.heads_q, cfg.head_dim, o)
    if tuple(q.shape) != shape_q or tuple(k_new.shape) != shape_kv or \
            tuple(v_new.shape) != shape_kv:
        validate_config(cfg)
        raise ShapeError("decode_step: q must be [batch, heads_q, d], k_new/v_new "
                         "[batch, heads_kv, d]")
    qd, kd, vd = (_as_f16_cuda(x, device=cache._device) for x in (q, k_new, v_new))
    if out is None:
        out = torch.empty(shape_q, dtype=torch.float32, device=qd.device)
    else:
        _check_f32_out(out, shape_q, cache, "out")
    _check(_L.load().bdk_decode_step(cache.handle(), C.byref(c), C.c_void_p(qd.data_ptr()),
                                     C.c_void_p(kd.data_ptr()), C.c_void_p(vd.data_ptr()),
                                     C.c_void_p(out.data_ptr()), _stream_ptr()))
    return AttnOutput(cfg.batch, cfg.heads_q, cfg.head_dim, out)


def _check_f32_out(t, shape, cache: KVCache, name: str) -> None:
    """A caller-provided device output must be a contiguous fp32 CUDA tensor
    of the exact shape on the cache's GPU (the kernels write it blindly)."""
    ok = (torch is not None and isinstance(t, torch.Tensor) and t.is_cuda
          and t.dtype == torch.float32 and t.is_contiguous() and tuple(t.shape) == tuple(shape)
          and t.device.index == cache._device)
    if not ok:
        raise ShapeError(f"{name} must be a contiguous float32 CUDA tensor of shape "
                         f"{tuple(shape)} on cuda:{cache._device}")


class DecodeStepper:
    """Pointer-bound ``decode_step`` for steady-state loops: the C-ABI call
    with arguments prepared once (q/k_new/v_new/out are CUDA tensors whose
    storage stays fixed; refill them in place between steps).  Same kernels
    and semantics as :func:`decode_step`."""

    def __init__(self, cache: KVCache, cfg: AttentionConfig, q, k_new, v_new, out):
        for t in (q, k_new, v_new):
            if not (t.is_cuda and t.dtype == torch.float16 and t.is_contiguous()):
                raise ShapeError("DecodeStepper needs contiguous CUDA fp16 q/k_new/v_new")
        if not (out.is_cuda and out.dtype == torch.float32 and out.is_contiguous()):
            raise ShapeError("DecodeStepper needs a contiguous CUDA fp32 out")
        self._cfg = cfg._c()
        self._fn = _L.load().bdk_decode_step
        self._args = (cache.handle(), C.byref(self._cfg), C.c_void_p(q.data_ptr()),
                      C.c_void_p(k_new.data_ptr()), C.c_void_p(v_new.data_ptr()),
                      C.c_void_p(out.data_ptr()))
        self._keep = (cache, q, k_new, v_new, out)

    def __call__(self, stream=None) -> None:
        st = self._fn(*self._args, stream if stream is not None else _stream_ptr())
        if st:
            _check(st)

    def prebind(self, qs, ks, vs, stream=None) -> None:
        """Pointer arguments for a preloaded input sequence (qs[i], ks[i],
        vs[i] stay alive in the caller), for :meth:`step_pre`."""
        self._pre = [(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()))
                     for q, k, v in zip(qs, ks, vs)]
        self._pre_stream = stream if stream is not None else _stream_ptr()

    def step_pre(self, i: int) -> None:
        """The decode step on the i-th prebound inputs: one C-ABI call."""
        a, p = self._args, self._pre[i]
        st = self._fn(a[0], a[1], p[0], p[1], p[2], a[5], self._pre_stream)
        if st:
            _check(st)

    def step(self, q, k_new, v_new, stream=None) -> None:
        """Same call on other (contiguous CUDA fp16, same-shape) input
        tensors, e.g. one preloaded slice per step; writes the bound out."""
        a = self._args
        st = self._fn(a[0], a[1], C.c_void_p(q.data_ptr()), C.c_void_p(k_new.data_ptr()),
                      C.c_void_p(v_new.data_ptr()), a[5],
                      stream if stream is not None else _stream_ptr())
        if st:
            _check(st)


class DecodeGraph:
    """A CUDA graph of ``n`` consecutive decode steps (bdk_graph_create): the
    steady-state loop of Algorithm 2 -- append, attention, combine and the
    flush of any residual that fills, one kernel per step -- captured once
    and replayed at any cache state.  ``qs`` [n, batch, heads_q, d],
    ``ks``/``vs`` [n, batch, heads_kv, d] (contiguous CUDA fp16, refill them
    in place between launches) and ``outs`` [n, batch, heads_q, d] (fp32).
    Fast mode only.  Replays are bit-identical to the same steps run with
    :func:`decode_step`."""

    def __init__(self, cache: KVCache, cfg: AttentionConfig, qs, ks, vs, outs):
        n = qs.shape[0]
        shape_q = (n, cfg.batch, cfg.heads_q, cfg.head_dim)
        shape_kv = (n, cfg.batch, cfg.heads_kv, cfg.head_dim)
        for t, shp in ((qs, shape_q), (ks, shape_kv), (vs, shape_kv)):
            if not (t.is_cuda and t.dtype == torch.float16 and t.is_contiguous()
                    and tuple(t.shape) == shp and t.device.index == cache._device):
                raise ShapeError(f"DecodeGraph inputs must be contiguous CUDA fp16 {shp}")
        _check_f32_out(outs, shape_q, cache, "outs")
        self._cfg = cfg._c()
        h = C.c_void_p()
        _check(_L.load().bdk_graph_create(cache.handle(), C.byref(self._cfg),
                                          C.c_void_p(qs.data_ptr()), C.c_void_p(ks.data_ptr()),
                                          C.c_void_p(vs.data_ptr()), C.c_void_p(outs.data_ptr()),
                                          n, C.byref(h)))
        self._h = h
        self.n_steps = n
        self._keep = (cache, qs, ks, vs, outs)

    def launch(self, stream=None) -> None:
        """Run the n steps (stream-ordered, no sync)."""
        _check(_L.load().bdk_graph_launch(self._h, stream if stream is not None
                                          else _stream_ptr()))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _L.load().bdk_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decode_partial(cache: KVCache, cfg: AttentionConfig, q, k_new=None, v_new=None,
                   blk_begin: int = 0, blk_end: int = 1 << 30, out=None, lse=None,
                   include_residual: bool = True):
    """Sequence-split partial (see bdk_decode_partial): returns the normalized
    partial output [batch, heads_q, d] and its log2-sum-exp [batch, heads_q].
    k_new/v_new None: attend only (no append, no commit)."""
    c = cfg._c()
    dev = cache._device
    qd = _as_f16_cuda(q, (cfg.batch, cfg.heads_q, cfg.head_dim), dev)
    shape_kv = (cfg.batch, cfg.heads_kv, cfg.head_dim)
    kd = _as_f16_cuda(k_new, shape_kv, dev) if k_new is not None else None
    vd = _as_f16_cuda(v_new, shape_kv, dev) if v_new is not None else None
    if out is None:
        o = torch.empty((cfg.batch, cfg.heads_q, cfg.head_dim), dtype=torch.float32,
                        device=qd.device)
    else:
        _check_f32_out(out, (cfg.batch, cfg.heads_q, cfg.head_dim), cache, "out")
        o = out
    if lse is None:
        lse = torch.empty((cfg.batch, cfg.heads_q), dtype=torch.float32, device=qd.device)
    else:
        _check_f32_out(lse, (cfg.batch, cfg.heads_q), cache, "lse")
    _check(_L.load().bdk_decode_partial(
        cache.handle(), C.byref(c), C.c_void_p(qd.data_ptr()),
        C.c_void_p(kd.data_ptr()) if kd is not None else None,
        C.c_void_p(vd.data_ptr()) if vd is not None else None, blk_begin,
        min(blk_end, (1 << 32) - 1), 0 if include_residual else 1, C.c_void_p(o.data_ptr()),
        C.c_void_p(lse.data_ptr()), _stream_ptr()))
    return o, lse


# ------------------------------------------------- attention internals
# The reference's decode decomposition (attention.hpp:17-70), on the device
# (bdk_span.cu); numpy fp32 in and out, synchronous.

@dataclass
class PartialOutput:
    """PartialOutput (attention.hpp:17-26): unnormalized o [rows, d], running
    max m [rows] (-inf initially) and exp-sum l [rows] (0 initially)."""
    o: np.ndarray
    m: np.ndarray
    l: np.ndarray

    @property
    def rows(self) -> int:
        return self.o.shape[0]

    @property
    def d(self) -> int:
        return self.o.shape[1]

    @staticmethod
    def init(rows: int, d: int) -> "PartialOutput":
        return PartialOutput(np.zeros((rows, d), np.float32), np.full(rows, -np.inf, np.float32),
                             np.zeros(rows, np.float32))


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(x, np.float32)


def partitioned_rowmax(s, warp_n: int, device: int = 0) -> np.ndarray:
    """partitioned_rowmax (attention.cpp:32-50) of s [rows, cols]."""
    x = _f32(s)
    rows, cols = x.shape
    out = np.zeros(rows, np.float32)
    _check(_L.load().bdk_partitioned_rowmax_host(x.ctypes.data, rows, cols, warp_n,
                                                 out.ctypes.data, device))
    return out


def attend_tile(state: PartialOutput, q, k, v, scale: float, warp_n: int = 1,
                device: int = 0) -> None:
    """attend_tile (attention.cpp:52-90): one online-softmax step over the
    tokens of k/v [tile_n, d]; updates state in place."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    if k.shape != v.shape or k.shape[1] != state.d or q.shape != (state.rows, state.d):
        raise ShapeError("attend_tile: q [rows, d], k/v [tile_n, d] must match the state")
    _check(_L.load().bdk_attend_tile_host(state.o.ctypes.data, state.m.ctypes.data,
                                          state.l.ctypes.data, state.rows, state.d,
                                          q.ctypes.data, k.ctypes.data, v.ctypes.data,
                                          k.shape[0], scale, warp_n, device))


def residual_attend(cache: "KVCache", b: int, h: int, q, scale: float,
                    state: PartialOutput, warp_n: int = 1):
    """residual_attend (attention.cpp:92-105): attention over the residual of
    cell (b, h) into state; returns the PackedBlock of a full residual (for
    the caller to commit) or None."""
    q = _f32(q)
    if q.shape != (state.rows, state.d):
        raise ShapeError("residual_attend: state rows != q rows")
    _check(_L.load().bdk_residual_attend_host(cache.handle(), b, h, q.ctypes.data, q.shape[0],
                                              scale, state.o.ctypes.data, state.m.ctypes.data,
                                              state.l.ctypes.data))
    return cache.build_block(b, h) if cache.res_len(b, h) == cache.n_r() else None


def packed_attend(cache: "KVCache", b: int, h: int, q, tile_n: int, num_splits: int,
                  scale: float, warp_n: int = 1) -> list:
    """packed_attend (attention.cpp:107-140): one PartialOutput per non-empty
    split of the packed segment of cell (b, h)."""
    q = _f32(q)
    rows, d = q.shape
    cap = max(1, num_splits)
    o = np.zeros((cap, rows, d), np.float32)
    m = np.zeros((cap, rows), np.float32)
    l = np.zeros((cap, rows), np.float32)
    n = C.c_uint32(0)
    _check(_L.load().bdk_packed_attend_host(cache.handle(), b, h, q.ctypes.data, rows, tile_n,
                                            num_splits, scale, o.ctypes.data, m.ctypes.data,
                                            l.ctypes.data, C.byref(n)))
    return [PartialOutput(o[i].copy(), m[i].copy(), l[i].copy()) for i in range(n.value)]


def combine(partials, device: int = 0) -> np.ndarray:
    """combine (attention.cpp:142-162): O = sum o_i w_i / sum l_i w_i with
    w_i = e^(m_i - max m) -> [rows, d]."""
    if len(partials) == 0:
        raise EmptyInput("combine: no partial outputs")
    rows, d = partials[0].o.shape
    if any(p.o.shape != (rows, d) for p in partials):
        raise ShapeError("combine: partial shapes differ")
    o = _f32(np.stack([p.o for p in partials]))
    m = _f32(np.stack([p.m for p in partials]))
    l = _f32(np.stack([p.l for p in partials]))
    out = np.zeros((rows, d), np.float32)
    _check(_L.load().bdk_combine_host(o.ctypes.data, m.ctypes.data, l.ctypes.data, len(partials),
                                      rows, d, out.ctypes.data, device))
    return out


def merge_partials(o_parts, lse_parts, out=None):
    """combine (attention.cpp:142-162) of normalized partials:
    o_parts [n, rows..., d], lse_parts [n, rows...] (CUDA fp32; the part
    dimension may be strided, e.g. views into one all-gathered buffer)."""
    n = o_parts.shape[0]
    d = o_parts.shape[-1]
    rows = lse_parts[0].numel()
    if o_parts.dtype != torch.float32 or lse_parts.dtype != torch.float32:
        raise ShapeError("merge_partials needs fp32 partials")
    if not (o_parts[0].is_contiguous() and lse_parts[0].is_contiguous()):
        o_parts, lse_parts = o_parts.contiguous(), lse_parts.contiguous()
    if out is None:
        out = torch.empty(o_parts.shape[1:], dtype=torch.float32, device=o_parts.device)
    _check(_L.load().bdk_merge_partials(C.c_void_p(o_parts.data_ptr()),
                                        C.c_void_p(lse_parts.data_ptr()), n, rows, d,
                                        o_parts.stride(0), lse_parts.stride(0),
                                        C.c_void_p(out.data_ptr()), _stream_ptr()))
    return out


def synchronize() -> None:
    _check(_L.load().bdk_synchronize())
