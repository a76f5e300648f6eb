"""Seeded synthetic inputs: DAG edge lists and poset-function values.

This module is shared by BOTH sides of the parity contract (the CPU oracle in
``oracle/`` and the CUDA path in ``paper_2211_13706_b200/``).  It therefore
holds NONE of the method's arithmetic -- no closure, no chains, no niv, no
transform -- only random draws.  Everything is a pure function of its seed.

Conventions (§2.1, "x ⪯ y iff there is a path from y to x"):
an edge ``(src[e], dst[e])`` means ``dst[e] ⪯ src[e]``.  Every generator below
emits edges ``i -> j`` with ``j < i``, i.e. vertex ids increase bottom-up, so
id order is a (bottom-up) topological order.  The library does NOT rely on
that; it is only what makes the workloads chain-local.

Configs (BASELINE.json ``configs`` + SURVEY.md §8(d)):

=====  ======================================================================
C1     window DAG n=1000, node i -> min(i,3) distinct j in [max(0,i-50), i)
C2     Boolean lattice 2^16, S -> S\\{b} (cover edges)
C3     window DAG n=1M, 2 distinct j in [max(0,i-1000), i)      (literal)
C3w    C3 width-bounded: i>=1000 -> {i-1000} + 1 distinct j in [i-999,i-1]
C4     layered 4096 x 256, 3 distinct nodes of previous layer  (literal)
C4w    C4 width-bounded: {pi_L(r)} + 2 distinct others of previous layer
C5     window DAG n=16M, 2 distinct j in [max(0,i-64), i)       (literal)
C5w    C5 width-bounded: i>=64 -> {i-64} + 1 distinct j in [i-63, i-1]
ER     Erdos-Renyi DAG (paper §5), p = delta/(n-1)  (NEXT row N4)
=====  ======================================================================

The literal C3/C4/C5 have width Theta(n); the ``w`` variants are
the width-bounded readings recorded in DESIGN.md.  All draws use numpy's
PCG64 ``default_rng(seed)``; edge draws are vectorised (one batch of uniforms
per config), so they differ from SURVEY Appendix A's per-node loop while
following the same distributions.
"""
from __future__ import annotations

import dataclasses
import hashlib

import numpy as np

__all__ = [
    "window_dag", "layered_dag", "boolean_lattice", "erdos_renyi",
    "paper_example_edges", "chain_dag", "antichain_dag",
    "int_values", "normal_values", "Workload", "CONFIGS", "make_workload",
    "sha256_arrays",
]


def _distinct_draws(rng, m: np.ndarray, d: int) -> np.ndarray:
    """For each row i draw ``d`` distinct integers uniform in [0, m[i]).

    Rows with m[i] < d are the caller's business (masked out).  Sequential
    sampling without replacement: draw u_t uniform in [0, m-t) and shift it
    past the already-drawn values (in sorted order) -- exact uniformity.
    Returns an (len(m), d) int64 array.
    """
    m = np.asarray(m, dtype=np.int64)
    u = rng.random((m.shape[0], d))
    out = np.empty((m.shape[0], d), dtype=np.int64)
    for t in range(d):
        span = np.maximum(m - t, 1)
        v = np.minimum((u[:, t] * span).astype(np.int64), span - 1)
        if t:
            prev = np.sort(out[:, :t], axis=1)
            for c in range(t):
                v = v + (v >= prev[:, c])
        out[:, t] = v
    return out


def window_dag(n: int, d: int, W: int, seed: int = 0, forced: bool = False):
    """Random window DAG (BASELINE.json configs[0], [2], [4]).

    Node i gets ``min(d, i - lo)`` distinct out-edges to uniform j in
    ``[lo, i)``, ``lo = max(0, i - W)``.  ``forced=True`` is the width-bounded
    reading (SURVEY §8(d) C3'/C5'): for i >= W the edges are ``{i - W}`` plus
    ``d - 1`` distinct uniform j in ``[i - W + 1, i - 1]``.
    Returns ``(src, dst)`` int64 arrays, edges grouped by src ascending.
    """
    rng = np.random.default_rng(seed)
    i = np.arange(1, n, dtype=np.int64)
    lo = np.maximum(0, i - W)
    m = i - lo
    srcs, dsts = [], []
    small = m <= d                      # take every option
    if small.any():
        ii = i[small]
        cnt = m[small]
        s = np.repeat(ii, cnt)
        starts = np.repeat(lo[small], cnt)
        offs = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        srcs.append(s)
        dsts.append(starts + offs)
    big = ~small
    if forced:
        fz = big & (i >= W)
        big = big & ~fz
        if fz.any():
            ii = i[fz]
            srcs.append(ii)
            dsts.append(ii - W)
            if d > 1:
                r = _distinct_draws(rng, np.full(ii.shape[0], W - 1), d - 1)
                srcs.append(np.repeat(ii, d - 1))
                dsts.append((ii[:, None] - W + 1 + r).reshape(-1))
    if big.any():
        ii = i[big]
        r = _distinct_draws(rng, m[big], d)
        srcs.append(np.repeat(ii, d))
        dsts.append((lo[big][:, None] + r).reshape(-1))
    src = np.concatenate(srcs) if srcs else np.zeros(0, np.int64)
    dst = np.concatenate(dsts) if dsts else np.zeros(0, np.int64)
    order = np.argsort(src, kind="stable")
    return src[order], dst[order]


def layered_dag(layers: int, width: int, d: int = 3, seed: int = 0,
                forced: bool = False):
    """Layered DAG (BASELINE.json configs[3]); node id = layer*width + r.

    Each node of layer L >= 1 gets ``d`` distinct edges to uniform nodes of
    layer L-1.  ``forced=True`` (SURVEY §8(d) C4'): node r of layer L gets
    ``{pi_L(r)}`` plus ``d - 1`` distinct others, pi_L a uniform permutation.
    """
    rng = np.random.default_rng(seed)
    L = layers - 1
    if L <= 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    ids = (np.arange(1, layers, dtype=np.int64)[:, None] * width
           + np.arange(width, dtype=np.int64)[None, :]).reshape(-1)
    prev_base = np.repeat(np.arange(0, layers - 1, dtype=np.int64) * width, width)
    if forced:
        perm = rng.permuted(np.tile(np.arange(width, dtype=np.int64), (L, 1)), axis=1).reshape(-1)
        r = _distinct_draws(rng, np.full(ids.shape[0], width - 1), d - 1)
        others = (perm[:, None] + 1 + r) % width
        tgt = np.concatenate([perm[:, None], others], axis=1)
    else:
        tgt = _distinct_draws(rng, np.full(ids.shape[0], width), d)
    src = np.repeat(ids, d)
    dst = (prev_base[:, None] + tgt).reshape(-1)
    return src, dst


def boolean_lattice(bits: int):
    """Boolean lattice 2^bits as its cover graph: S -> S\\{b} for b in S
    (BASELINE.json configs[1]; PAPER.md P:L26 powerset lattice)."""
    n = 1 << bits
    S = np.arange(n, dtype=np.int64)
    srcs, dsts = [], []
    for b in range(bits):
        has = (S >> b) & 1 == 1
        srcs.append(S[has])
        dsts.append(S[has] ^ (1 << b))
    src = np.concatenate(srcs)
    dst = np.concatenate(dsts)
    order = np.argsort(src, kind="stable")
    return src[order], dst[order]


def erdos_renyi(n: int, delta: float, seed: int = 0):
    """Erdos-Renyi DAG (§5): every pair {i, j}, j < i,
    is an edge i -> j independently with p = delta / (n - 1), so the
    expected total degree 2|E|/n is delta (reading G10 in DESIGN.md).
    Sampled by drawing the Binomial edge count and then distinct pairs."""
    rng = np.random.default_rng(seed)
    if n < 2 or delta <= 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    p = min(1.0, delta / (n - 1))
    total = n * (n - 1) // 2
    cnt = int(rng.binomial(total, p))
    picked = np.unique(rng.integers(0, total, size=int(cnt * 1.05) + 16, dtype=np.int64))
    while picked.shape[0] < cnt:
        extra = rng.integers(0, total, size=cnt - picked.shape[0] + 16, dtype=np.int64)
        picked = np.unique(np.concatenate([picked, extra]))
    picked = rng.permutation(picked)[:cnt]
    # pair index t -> (i, j) with 0 <= j < i:  t = i*(i-1)/2 + j
    i = ((1 + np.sqrt(1 + 8 * picked.astype(np.float64))) // 2).astype(np.int64)
    i = np.where(i * (i - 1) // 2 > picked, i - 1, i)
    i = np.where((i + 1) * i // 2 <= picked, i + 1, i)
    j = picked - i * (i - 1) // 2
    order = np.lexsort((j, i))
    return i[order], j[order]


def paper_example_edges():
    """The 12-node example of PAPER.md §2.2 (adjacency matrix A, P:L160-178;
    edge list verbatim at SPEC.md S:L50).  Paper vertex v -> id v-1 and the
    paper's edge (u, v) (v covered by u) -> src=u-1, dst=v-1."""
    pe = [(1, 3), (1, 4), (1, 6), (2, 4), (2, 5), (3, 7), (3, 8), (4, 7), (4, 9),
          (5, 10), (6, 8), (6, 9), (7, 10), (8, 11), (9, 12), (10, 11), (10, 12)]
    src = np.array([u - 1 for u, _ in pe], dtype=np.int64)
    dst = np.array([v - 1 for _, v in pe], dtype=np.int64)
    return src, dst


def chain_dag(n: int):
    """Total order 0 < 1 < ... < n-1 as a path (i -> i-1)."""
    i = np.arange(1, n, dtype=np.int64)
    return i, i - 1


def antichain_dag(n: int):
    """n pairwise incomparable elements (no edges)."""
    return np.zeros(0, np.int64), np.zeros(0, np.int64)


def int_values(n: int, B: int, lo: int, hi: int, seed: int = 1) -> np.ndarray:
    """int64 function values uniform in [lo, hi], shape (n, B), row-major."""
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi + 1, size=(n, B), dtype=np.int64)


def normal_values(n: int, B: int, seed: int = 1) -> np.ndarray:
    """fp64 N(0,1) function values, shape (n, B), row-major."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, B))


@dataclasses.dataclass
class Workload:
    name: str
    n: int
    src: np.ndarray
    dst: np.ndarray
    batch: int
    dtype: str            # "i64" | "f64"
    value_range: tuple | None
    desc: str

    def values(self, seed: int = 1, batch: int | None = None) -> np.ndarray:
        B = self.batch if batch is None else batch
        if self.dtype == "i64":
            lo, hi = self.value_range
            return int_values(self.n, B, lo, hi, seed)
        return normal_values(self.n, B, seed)


# name -> (builder(scale) -> (n, src, dst), batch, dtype, range, description)
def _c1(scale):
    n = max(2, int(1000 * scale))
    return (n,) + window_dag(n, 3, 50, 0)


def _c2(scale):
    bits = 16 if scale >= 1 else max(2, int(round(16 + np.log2(scale))))
    return (1 << bits,) + boolean_lattice(bits)


def _win(n0, W, forced):
    def b(scale):
        n = max(2, int(n0 * scale))
        return (n,) + window_dag(n, 2, W, 0, forced)
    return b


def _lay(forced):
    def b(scale):
        L = max(2, int(4096 * scale))
        return (L * 256,) + layered_dag(L, 256, 3, 0, forced)
    return b


def _er(n0, delta):
    def b(scale):
        n = max(2, int(n0 * scale))
        return (n,) + erdos_renyi(n, delta, 0)
    return b


CONFIGS = {
    "C1": (_c1, 1, "i64", (-100, 100), "random DAG n=1000, min(i,3) edges into [i-50,i)"),
    "C2": (_c2, 1, "f64", None, "Boolean lattice 2^16"),
    "C3": (_win(1_000_000, 1000, False), 1, "f64", None, "window DAG n=1M W=1000 (literal)"),
    "C3w": (_win(1_000_000, 1000, True), 1, "f64", None, "window DAG n=1M W=1000 width-bounded"),
    "C4": (_lay(False), 64, "i64", (-1000, 1000), "layered 4096x256 (literal)"),
    "C4w": (_lay(True), 64, "i64", (-1000, 1000), "layered 4096x256 width-bounded"),
    "C5": (_win(16_000_000, 64, False), 32, "f64", None, "window DAG n=16M W=64 (literal)"),
    "C5w": (_win(16_000_000, 64, True), 32, "f64", None, "window DAG n=16M W=64 width-bounded"),
    # literal C4 through the sparse rows (N1): one function (B=64 would be
    # 64 x the gathers of a 3.1e10-entry table)
    "C4lit1": (_lay(False), 1, "i64", (-1000, 1000), "layered 4096x256 (literal, sparse rows), B=1"),
    # the paper's own workload (§5): Erdos-Renyi DAGs,
    # average degree 4 and 6, n = 9M (its largest size); one fp64 function
    "ER4": (_er(9_000_000, 4), 1, "f64", None, "Erdos-Renyi DAG n=9M, delta=4 (paper §5)"),
    "ER6": (_er(9_000_000, 6), 1, "f64", None, "Erdos-Renyi DAG n=9M, delta=6 (paper §5)"),
}


def make_workload(name: str, scale: float = 1.0, dtype: str | None = None,
                  batch: int | None = None) -> Workload:
    """Build config ``name`` at ``scale`` (n multiplied by scale; C2 halves
    the bit count per factor 2).  ``dtype``/``batch`` override the config's
    (e.g. int64 round-trip parity on C5w, reading G8)."""
    builder, B, dt, rng_, desc = CONFIGS[name]
    n, src, dst = builder(scale)
    dt = dtype or dt
    if dt == "i64" and rng_ is None:
        rng_ = (-1000, 1000)
    return Workload(name, n, src, dst, batch or B, dt, rng_, desc)


def sha256_arrays(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(memoryview(a).cast("B"))
    return h.hexdigest()
