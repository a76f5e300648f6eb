"""Build libposet.so (sm_100a CUDA + host C++) in-tree.

    python paper_2211_13706_b200/build.py

nvcc cross-compiles for sm_100a without a GPU.  The .so lands next to this
file so that gpurun ships it with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libposet.so")
SOURCES = ["api.cu", "kernels.cu", "moebius_ring.cu", "moebius_csr.cu", "moebius_ringws.cu", "moebius_ringdf.cu", "setup.cpp"]
HEADERS = ["internal.h", "kernels.cuh", "ptx.cuh", os.path.join("..", "..", "include", "poset.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return SO
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O2",
           "-o", SO] + [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
