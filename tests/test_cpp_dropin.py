"""The C++ drop-in (include/bitkv_b200.hpp): builds against the library here
(CPU), runs tests/cpp/test_dropin.cpp on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2503_18773_b200", "lib")
ORACLE = os.path.join(ROOT, "oracle")
EXE = os.path.join(LIBDIR, "test_dropin")


def build_exe() -> str:
    from paper_2503_18773_b200 import build as B
    from oracle import oracle as O
    if not os.path.exists(B.LIB):
        pytest.skip("library not built")
    if not os.path.exists(O.ORACLE_SO):
        O.build(ref=False)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           "-I", ORACLE, SRC, "-o", EXE, "-L", LIBDIR, "-lbitdecode_b200", "-L", ORACLE,
           "-loracle", f"-Wl,-rpath,{LIBDIR}:{ORACLE}"]
    subprocess.run(cmd, check=True)
    return EXE


def test_cpp_dropin_compiles_and_links():
    assert os.path.exists(build_exe())


@pytest.mark.gpu
def test_cpp_dropin_runs_against_oracle():
    exe = build_exe()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
