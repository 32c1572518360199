"""Shared seeded workloads for the parity tests.

Inputs come from the oracle's GaussianSource restatement (bench.cpp:18-35,
pinned to the reference by tests/golden), so the CUDA path and the CPU
oracle see identical binary16 bytes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle import oracle as O

D = 128


@dataclass
class Case:
    bits: int = 4
    warp_n: int = 4
    group_size: int = 128
    k_axis: int = 0
    heads_q: int = 32
    heads_kv: int = 8
    batch: int = 1
    prefill: int = 4096
    steps: int = 2
    seed: int = 0
    interleave: bool = True
    precise: bool = False

    @property
    def n_r(self) -> int:
        return 8 * self.warp_n * (16 // self.bits)


def prefill_data(c: Case, gauss: O.Gauss):
    n = c.batch * c.heads_kv * c.prefill * D
    k = gauss.rounded(n).reshape(c.batch, c.heads_kv, c.prefill, D)
    v = gauss.rounded(n).reshape(c.batch, c.heads_kv, c.prefill, D)
    return k, v


def adversarial_data(c: Case, seed: int):
    """binary16 data that stresses the exactness rules of quantize_tile
    (quant.cpp:18-93): a coarse grid (exact .5 quotients -> the ties-to-even
    path), zeros of both signs as group extrema (the first-zero sign rule),
    constant groups (scale clamped to kMinScale), and a large-magnitude
    channel."""
    rng = np.random.default_rng(seed)
    shape = (c.batch, c.heads_kv, c.prefill, D)
    grid = np.array([-2.0, -1.5, -1.0, -0.5, -0.0, 0.0, 0.5, 1.0, 1.5, 2.0], np.float32)
    k = grid[rng.integers(0, grid.size, shape)]
    v = grid[rng.integers(0, grid.size, shape)]
    k[..., 3] = 0.0                       # a channel of +0
    k[..., 5] = -0.0                      # a channel of -0
    k[..., 7] = 7.25                      # a constant channel
    k[..., 9] = rng.normal(0, 300, shape[:-1]).astype(np.float16).astype(np.float32)
    # a large offset with a small spread (|z/s| ~ 1e4): the fast quantizer's
    # FMA form needs its widest tie margin here
    k[..., 11] = 1000.0 + 0.5 * rng.integers(0, 4, shape[:-1])
    v[:, :, ::17, :] = -0.0               # all-zero tokens
    v[:, :, 1::19, :] = 3.0               # constant tokens
    v[:, :, 2::23, :] = 500.0 + 0.25 * rng.integers(0, 5, v[:, :, 2::23, :].shape)
    return k.astype(np.float16).astype(np.float32), v.astype(np.float16).astype(np.float32)


def step_data(c: Case, gauss: O.Gauss):
    q = gauss.rounded(c.batch * c.heads_q * D).reshape(c.batch, c.heads_q, D)
    kn = gauss.rounded(c.batch * c.heads_kv * D).reshape(c.batch, c.heads_kv, D)
    vn = gauss.rounded(c.batch * c.heads_kv * D).reshape(c.batch, c.heads_kv, D)
    return q, kn, vn


def oracle_cache(c: Case, k, v) -> O.OracleCache:
    oc = O.OracleCache(c.batch, c.heads_kv, D, c.warp_n, c.bits, c.k_axis, c.group_size,
                       c.interleave, max_tokens=c.prefill + c.steps + 2 * c.n_r)
    for b in range(c.batch):
        for h in range(c.heads_kv):
            oc.prefill(b, h, k[b, h], v[b, h])
    return oc


def errors(out: np.ndarray, ref: np.ndarray) -> dict:
    a = out.astype(np.float64).ravel()
    r = ref.astype(np.float64).ravel()
    diff = a - r
    nr = np.linalg.norm(r)
    return {"max_abs": float(np.abs(diff).max()) if diff.size else 0.0,
            "rel_l2": float(np.linalg.norm(diff) / nr) if nr > 0 else float(np.linalg.norm(diff))}
