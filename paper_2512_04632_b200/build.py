"""Build libturbons.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python paper_2512_04632_b200/build.py [--force]     (or __graft_entry__.build())
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libturbons.so")
SOURCES = ["api.cu", "umma_gemm.cu", "simt.cu", "muon.cu", "cluster_ns.cu", "cluster_tc.cu"]
HEADERS = ["ptx.cuh", "jobs.h", "kernels.h", "precond_rows.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared",
    "-I", os.path.join(ROOT, "include"),
]
# Measurement build (never the default): TNS_MEASURE=1 compiles in the clock64 epilogue
# counters / timeline read through nsx_epilogue_counters under TNS_DBG bits 8 and 16.
if os.environ.get("TNS_MEASURE"):
    FLAGS += ["-DTNS_MEASURE=1"]
# A/B builds: extra -D flags (e.g. TNS_EXTRA_FLAGS=-DTNS_NO_DIAG); never set in production
FLAGS += os.environ.get("TNS_EXTRA_FLAGS", "").split()


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "turbo_ns.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + ".tmp"
    cmd = [NVCC, *FLAGS, "-o", tmp, *[os.path.join(CSRC, f) for f in SOURCES]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
