"""Tiny instances for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every Möbius schedule that applies, the dense and sparse zeta
gathers, the scan and the split phases, on C1 (n=1000), the paper's 12-node
example and a Boolean lattice 2^8.  numpy buffers only (the library stages
them), so the only kernels in the process are libposet.so's.

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_13706_b200 as pz  # noqa: E402
import workloads as W  # noqa: E402

NAMES = {pz.MOEB_LEVEL: "LEVEL", pz.MOEB_GRID: "GRID", pz.MOEB_WARP: "WARP", pz.MOEB_RING: "RING",
         pz.MOEB_CSR: "CSR", pz.MOEB_RINGWS: "RINGWS", pz.MOEB_RINGDF: "RINGDF", pz.MOEB_RINGCL: "RINGCL"}
only = set(sys.argv[1].split(",")) if len(sys.argv) > 1 else None


def schedules(P):
    i = P.info()
    out = [pz.MOEB_LEVEL, pz.MOEB_GRID, pz.MOEB_WARP]
    if i["dist_bytes"]:
        out.append(pz.MOEB_RING)
    if i["csr_bytes"]:
        out.append(pz.MOEB_CSR)
    if i["ringws"]:
        out.append(pz.MOEB_RINGWS)
    if i["ringdf"] & 1:
        out.append(pz.MOEB_RINGDF)
    if i["ringdf"] & 2:
        out.append(pz.MOEB_RINGCL)
    return out


cases = [("example12", 12, *W.paper_example_edges()),
         ("C1", 1000, *W.window_dag(1000, 3, 50, 0)),
         ("C5w_3k", 3000, *W.window_dag(3000, 2, 64, 0, forced=True)),
         ("bool8", 256, *W.boolean_lattice(8))]
bad = 0
for name, n, src, dst in cases:
    P = pz.Poset(n, src, dst)
    for B in (1, 32):
        f = W.int_values(n, B, -1000, 1000, seed=B)
        g = P.zeta(f)
        for s in schedules(P):
            if only and NAMES[s] not in only:
                continue
            P.set_option("moebius_kernel", s)
            back = P.moebius(g)
            ok = bool((back == f).all())
            bad += not ok
            print(f"{name} B={B} {NAMES[s]}: {'ok' if ok else 'MISMATCH'}", flush=True)
        P.set_option("moebius_kernel", 0)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
