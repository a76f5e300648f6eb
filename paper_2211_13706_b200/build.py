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
SOURCES = ["api.cu", "kernels.cu", "moebius_ring.cu", "moebius_csr.cu", "moebius_ringws.cu", "moebius_ringdf.cu", "gather_pi.cu", "gather_delta.cu", "setup.cpp"]
HEADERS = ["internal.h", "kernels.cuh", "ptx.cuh", os.path.join("..", "..", "include", "poset.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile each source to an object in parallel (the template-heavy
    schedules dominate), then link the shared library."""
    if not force and not _stale():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2"]
    jobs = []
    for f in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(f)[0] + ".o")
        jobs.append((obj, [NVCC, *flags, "-c", "-o", obj, os.path.join(CSRC, f)]))

    def run(job):
        if verbose:
            print(" ".join(job[1]), file=sys.stderr)
        subprocess.check_call(job[1])
        return job[0]

    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(run, jobs))
    link = [NVCC, *ARCH, "-shared", "-o", SO] + objs
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.check_call(link)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
