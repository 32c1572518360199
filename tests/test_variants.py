"""Kernel variants of the fast decode against each other and the oracle.

The split-consumer kernel (QK / PV warp pairs, bdk_decode_split.cuh) must give
results bit-identical to the fused kernel without column packing (same
extraction, same MMA order, same online softmax), and both must meet the
fast-mode tolerance against the CPU oracle across residual flushes, uneven
cell lengths and GQA groupings.  Variants are process-wide knobs (BDK_SPLIT,
BDK_COLPACK), so each runs in its own process (tests/variant_runner.py).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAST_TOL = {"max_abs": 2e-3, "rel_l2": 1e-3}


def _run(tmp_path, name, **env):
    out = str(tmp_path / f"{name}.npz")
    e = dict(os.environ, **{k: str(v) for k, v in env.items()})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "variant_runner.py"), out],
                       env=e, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    return dict(np.load(out))


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    t = tmp_path_factory.mktemp("variants")
    return {"split": _run(t, "split", BDK_SPLIT=1),
            "fused_cp1": _run(t, "fused_cp1", BDK_SPLIT=0, BDK_COLPACK=0),
            "default": _run(t, "default")}


def test_split_is_bit_identical_to_fused_without_column_packing(runs):
    a, b = runs["split"], runs["fused_cp1"]
    for k in a:
        if k.endswith("_got"):
            assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("name", ["split", "fused_cp1", "default"])
def test_variant_meets_fast_tolerance_and_lengths(runs, name):
    r = runs[name]
    for k in r:
        if not k.endswith("_got"):
            continue
        tag = k[:-4]
        got, ref = r[k].astype(np.float64), r[tag + "_ref"].astype(np.float64)
        d = got - ref
        max_abs = float(np.abs(d).max())
        rel = float(np.linalg.norm(d) / np.linalg.norm(ref))
        assert max_abs < FAST_TOL["max_abs"] and rel < FAST_TOL["rel_l2"], (name, tag, max_abs, rel)
        assert np.array_equal(r[tag + "_len"], r[tag + "_len_ref"]), (name, tag)
