"""Build the reference's own unit-test sources against the B200 drop-in.

    python tests/cpp/ref_suite/build.py

Each /root/reference/proj/tests/<name>.cpp in SUITES is compiled unchanged:
- its `#include "bitkv/*.hpp"` resolves to the shims here, which include
  include/bitkv_b200.hpp;
- `<doctest.h>` resolves to the minimal stand-in here;
- `bitkv/oracle.hpp` is the reference's test oracle, served by oracle/.
Binaries go to paper_2503_18773_b200/lib/ref_suite/ (git-ignored; they travel
to the GPU box with the tree).  Needs /root/reference (only in the build
container); tests/test_ref_suite.py runs whatever was built.

Not built: test_bench.cpp drives the reference's CPU benchmark harness
(run_bench, CaseDriver, CSV output), a caller outside the hot path.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(HERE)))
REF_TESTS = "/root/reference/proj/tests"
OUT = os.path.join(ROOT, "paper_2503_18773_b200", "lib", "ref_suite")
LIBDIR = os.path.join(ROOT, "paper_2503_18773_b200", "lib")
ORACLE = os.path.join(ROOT, "oracle")
SUITES = ["test_fp16", "test_layout", "test_quant", "test_config", "test_kvcache", "test_attention",
          "test_serialize", "test_oracle"]


REF_INC = "/root/reference/proj/include"
REF_OUT = os.path.join(ORACLE, "_ref", "ref_suite")
OUTCOMES = os.path.join(ROOT, "tests", "golden", "ref_suite_outcomes.json")


def _compile(cmds: list[list[str]]) -> None:
    procs = [subprocess.Popen(c) for c in cmds]
    if any(p.wait() != 0 for p in procs):
        raise RuntimeError("ref-suite build failed")


def build() -> list[str]:
    """The suites against the drop-in (include/bitkv_b200.hpp over the C-ABI)."""
    if not os.path.isdir(REF_TESTS):
        return []
    os.makedirs(OUT, exist_ok=True)
    cmds, outs = [], []
    for name in SUITES:
        exe = os.path.join(OUT, name)
        cmds.append(["g++", "-std=c++20", "-O1", "-w", "-I", HERE, "-I",
                     os.path.join(ROOT, "include"), "-I", ORACLE,
                     os.path.join(REF_TESTS, name + ".cpp"), "-o", exe, "-L", LIBDIR,
                     "-lbitdecode_b200", "-L", ORACLE, "-loracle",
                     "-Wl,-rpath,$ORIGIN/..:$ORIGIN/../../../oracle"])
        outs.append(exe)
    _compile(cmds)
    return outs


def build_reference() -> list[str]:
    """The same suites against the UNMODIFIED reference engine (oracle/_ref,
    CPU): the reference's own headers come first on the include path, so only
    <doctest.h> resolves to the stand-in here.  Their per-case outcomes are
    the expectation the drop-in's runs are held to."""
    lib = os.path.join(ORACLE, "_ref", "libbitkv_ref.so")
    if not (os.path.isdir(REF_TESTS) and os.path.exists(lib)):
        return []
    os.makedirs(REF_OUT, exist_ok=True)
    cmds, outs = [], []
    for name in SUITES:
        exe = os.path.join(REF_OUT, name)
        cmds.append(["g++", "-std=c++20", "-O1", "-w", "-I", REF_INC, "-I", HERE,
                     os.path.join(REF_TESTS, name + ".cpp"), "-o", exe, lib,
                     "-Wl,-rpath,$ORIGIN/.."])
        outs.append(exe)
    _compile(cmds)
    return outs


def parse_cases(stdout: str) -> dict[str, bool]:
    """`[PASS] name` / `[FAIL] name` lines of the stand-in runner."""
    out = {}
    for line in stdout.splitlines():
        if line.startswith("[PASS] ") or line.startswith("[FAIL] "):
            out[line[7:].strip()] = line.startswith("[PASS]")
    return out


def run_suite(exe: str, timeout: int = 600) -> tuple[int, dict[str, bool], str]:
    r = subprocess.run([exe], capture_output=True, text=True, timeout=timeout)
    return r.returncode, parse_cases(r.stdout), r.stdout + r.stderr


def reference_outcomes() -> dict[str, dict[str, bool]]:
    res = {}
    for exe in build_reference():
        _, cases, _ = run_suite(exe)
        res[os.path.basename(exe)] = cases
    return res


if __name__ == "__main__":
    import json
    print("\n".join(build()) or "reference tests absent: nothing built", file=sys.stderr)
    if "--outcomes" in sys.argv:
        oc = reference_outcomes()
        with open(OUTCOMES, "w") as f:
            json.dump(oc, f, indent=1, sort_keys=True)
            f.write("\n")
        print(f"wrote {OUTCOMES}", file=sys.stderr)
