"""Build libbtask.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1304_0878_b200.build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libbtask.so")
SOURCES = ["scheduler.cu", "runtime.cpp", "builder.cpp", "comm.cpp"]
HEADERS = ["device_abi.h", "builder.hpp", "pool.hpp", "comm.hpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                 # no FFMA contraction: bit-exact AXPY (R14)
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-O2,-fno-fast-math,-Wall,-pthread",
    "-Xptxas", "-warn-spills",
    "--cudart", "static",
    "-shared",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "btask.h"),
                                                               os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    target = out or LIB
    if not (force or out or _stale()):
        return LIB
    tmp = target + f".{os.getpid()}.tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
