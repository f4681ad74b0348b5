"""Build the in-tree CUDA library ``libtokensim.so`` for sm_100a with nvcc.

    python -m paper_2503_08415_b200.build [--force]

Flags: ``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false``
(no FMA contraction anywhere: the fp64 cost model and det_log must round exactly
as SURVEY c.2/c.5 write them) and ``-ffp-contract=off`` for the host side.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in ("workload.cu", "sim.cu", "metrics.cu", "host.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("ts_internal.cuh", "dev_common.cuh")] + \
    [os.path.join(ROOT, "include", "tokensim.h")]
LIB = os.path.join(PKG, "libtokensim.so")

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo", "--fmad=false",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-warn-spills",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", tmp, *SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
