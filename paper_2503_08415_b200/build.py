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
SOURCES = [os.path.join(CSRC, f) for f in ("sim_full.cu", "sim_full_h.cu", "sim_node.cu", "sim_pair.cu", "sim_base.cu", "sim_base_c.cu", "sim_base_n.cu", "workload.cu",
                                           "metrics.cu", "host.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("ts_internal.cuh", "dev_common.cuh", "sim_core.cuh", "sim_pd.cuh",
                                           "sim_pdn.cuh")] + [os.path.join(ROOT, "include", "tokensim.h")]
LIB = os.path.join(PKG, "libtokensim.so")

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo", "--fmad=false",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-warn-spills",
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


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: list | None = None) -> str:
    """Compile every translation unit to an object in parallel, then link the shared library.

    ``out``/``defines`` build an A/B variant elsewhere (e.g. ``-DTS_PROFILE=0``); the default
    in-tree library is the product."""
    lib = out or LIB
    if out is None and not force and not stale():
        return LIB
    import concurrent.futures as cf
    import tempfile
    with tempfile.TemporaryDirectory(prefix="tokensim_build_") as td:
        objs = [os.path.join(td, os.path.basename(s) + ".o") for s in SOURCES]
        cmds = [[nvcc(), *NVCC_FLAGS, *(defines or []), "-I", os.path.join(ROOT, "include"), "-c", "-o", o, s]
                for s, o in zip(SOURCES, objs)]
        if verbose:
            for c in cmds:
                print(" ".join(c), file=sys.stderr)
        with cf.ThreadPoolExecutor(len(cmds)) as ex:
            for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
                f.result()
        tmp = lib + f".tmp{os.getpid()}"
        subprocess.check_call([nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs])
        os.replace(tmp, lib)
    return lib


PROF_LIB = os.path.join(PKG, "libtokensim_prof.so")


def build_profiling() -> str:
    """The observability build (-DTS_PROFILE=1: per-path/phase cycle counters); tools only."""
    if os.path.exists(PROF_LIB) and not any(os.path.getmtime(p) > os.path.getmtime(PROF_LIB)
                                            for p in SOURCES + HEADERS):
        return PROF_LIB
    return build(out=PROF_LIB, defines=["-DTS_PROFILE=1"])


if __name__ == "__main__":
    args = sys.argv[1:]
    o = args[args.index("--out") + 1] if "--out" in args else None
    print(build(force="--force" in args, verbose=True, out=o, defines=[a for a in args if a.startswith("-D")]))
