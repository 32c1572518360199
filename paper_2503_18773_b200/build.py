"""Build the in-tree sm_100a shared library (nvcc, no torch JIT cache).

    python -m paper_2503_18773_b200.build

produces paper_2503_18773_b200/lib/libbitdecode_b200.so (git-ignored; it
travels to the GPU box with the repo snapshot).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libbitdecode_b200.so")
SOURCES = ["bdk_kernels.cu", "bdk_decode_fast.cu", "bdk_span.cu", "bdk_api.cu"]
HEADERS = ["bdk_common.cuh", "bdk_frag.cuh", "bdk_qpack.cuh", "bdk_qpack_fast.cuh", "bdk_launch.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-diag-suppress", "177", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-cudart", "static"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "bitdecode_b200.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        build_pyhost()
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(LIBDIR, src.replace(".cu", ".o"))
        extra = ["-Xcompiler", "-fopenmp"] if src == "bdk_api.cu" else []  # host-side threads
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fopenmp", "-o", LIB, *objs]
    subprocess.run(cmd, check=True)
    build_pyhost(force=True)
    return LIB


PYHOST_SRC = os.path.join(CSRC, "bdk_pyhost.c")


def pyhost_path() -> str:
    import sysconfig
    return os.path.join(LIBDIR, "_bdk_pyhost" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def build_pyhost(force: bool = False) -> str | None:
    """The CPython fast path of the host decode call (csrc/bdk_pyhost.c);
    None when no C compiler / Python headers (bitkv then keeps to ctypes)."""
    import sysconfig
    out = pyhost_path()
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(PYHOST_SRC):
        return out
    inc = sysconfig.get_paths().get("include")
    if not inc or not os.path.exists(os.path.join(inc, "Python.h")):
        return None
    os.makedirs(LIBDIR, exist_ok=True)
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-I", inc, PYHOST_SRC, "-o", out]
    return out if subprocess.run(cmd).returncode == 0 else None


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
