"""Oracle O1: brute-force definitions (TEST INFRASTRUCTURE ONLY, see
``oracle/__init__.py``).

Everything is in USER vertex ids: an edge (src, dst) means dst ⪯ src
(PAPER.md P:L86-88).  int64 arithmetic is Z/2^64 (uint64 wraparound, reading
G14 in DESIGN.md); fp64 uses numpy float64.
"""
from __future__ import annotations

import itertools

import numpy as np


class CycleError(ValueError):
    pass


class SelfLoopError(ValueError):
    pass


def children_lists(n, src, dst):
    ch = [set() for _ in range(n)]
    for u, v in zip(np.asarray(src).tolist(), np.asarray(dst).tolist()):
        if u == v:
            raise SelfLoopError(f"self loop at {u}")
        ch[u].add(v)
    return [sorted(c) for c in ch]


def bottom_up_order(n, ch):
    """A topological order in which every vertex comes after all of its
    children (Kahn on out-degrees); raises CycleError."""
    outdeg = [len(c) for c in ch]
    parents = [[] for _ in range(n)]
    for u in range(n):
        for v in ch[u]:
            parents[v].append(u)
    order = [v for v in range(n) if outdeg[v] == 0]
    h = 0
    while h < len(order):
        v = order[h]
        h += 1
        for u in parents[v]:
            outdeg[u] -= 1
            if outdeg[u] == 0:
                order.append(u)
    if len(order) != n:
        raise CycleError("graph has a directed cycle")
    return order


def downsets(n, src, dst):
    """↓x = {y : y ⪯ x} for every x as Python-int bitsets (bit y set),
    by ↓x = {x} ∪ ⋃_{c child of x} ↓c in bottom-up order (P:L88 closure)."""
    ch = children_lists(n, src, dst)
    order = bottom_up_order(n, ch)
    down = [0] * n
    for x in order:
        s = 1 << x
        for c in ch[x]:
            s |= down[c]
        down[x] = s
    return down


def zeta_matrix(n, src, dst) -> np.ndarray:
    """Z[x, y] = 1 iff y ⪯ x (Cor. 1), as a dense uint8 matrix."""
    down = downsets(n, src, dst)
    Z = np.zeros((n, n), dtype=np.uint8)
    for x in range(n):
        b = down[x]
        ys = [y for y in range(n) if (b >> y) & 1] if n <= 64 else _bits(b, n)
        Z[x, ys] = 1
    return Z


def _bits(b: int, n: int):
    by = b.to_bytes((n + 7) // 8, "little")
    arr = np.unpackbits(np.frombuffer(by, dtype=np.uint8), bitorder="little")[:n]
    return np.nonzero(arr)[0]


def zeta(n, src, dst, f: np.ndarray) -> np.ndarray:
    """g(x) = Σ_{y ⪯ x} f(y)  (Eq. inv-formula) by direct sums."""
    Z = zeta_matrix(n, src, dst)
    f = np.asarray(f)
    if f.dtype == np.int64:
        fu = f.view(np.uint64)
        g = np.zeros_like(fu)
        for x in range(n):
            g[x] = fu[Z[x] == 1].sum(axis=0, dtype=np.uint64)
        return g.view(np.int64)
    return Z.astype(np.float64) @ f


def zeta_abs(n, src, dst, f: np.ndarray) -> np.ndarray:
    """Σ_{y ⪯ x} |f(y)| -- the scale of the fp64 tolerance (north star)."""
    return zeta(n, src, dst, np.abs(np.asarray(f, dtype=np.float64)))


def moebius(n, src, dst, g: np.ndarray) -> np.ndarray:
    """f = Z^{-1} g by back-substitution: in bottom-up order,
    f(x) = g(x) - Σ_{y ≺ x} f(y)."""
    ch = children_lists(n, src, dst)
    order = bottom_up_order(n, ch)
    Z = zeta_matrix(n, src, dst)
    g = np.asarray(g)
    integer = g.dtype == np.int64
    gv = g.view(np.uint64) if integer else g.astype(np.float64)
    f = np.zeros_like(gv)
    for x in order:
        below = Z[x] == 1
        below[x] = False
        if integer:
            f[x] = gv[x] - f[below].sum(axis=0, dtype=np.uint64)
        else:
            f[x] = gv[x] - f[below].sum(axis=0)
    return f.view(np.int64) if integer else f


def mobius_function(n, src, dst):
    """μ(x, y) by the recursion of Thm. 1, exact Python ints:
    μ(x,x) = 1, μ(x,y) = -Σ_{x ⪯ z ≺ y} μ(x,z), 0 if x ⋠ y.
    Returns the paper's M with M[y][x] = μ(x, y) (Cor. 1: M = [μ(y,x)]_{x,y}
    indexed so that f = M g)."""
    Z = zeta_matrix(n, src, dst)
    ch = children_lists(n, src, dst)
    order = bottom_up_order(n, ch)
    rank = {v: i for i, v in enumerate(order)}
    mu = {}
    for x in range(n):
        # all y with x ⪯ y, in bottom-up order so z ≺ y comes first
        ups = sorted([y for y in range(n) if Z[y, x]], key=lambda v: rank[v])
        for y in ups:
            if y == x:
                mu[(x, y)] = 1
            else:
                mu[(x, y)] = -sum(mu[(x, z)] for z in ups if Z[y, z] and z != y)
    M = [[0] * n for _ in range(n)]
    for (x, y), v in mu.items():
        M[y][x] = v
    return M


def yates_zeta(bits: int, f: np.ndarray) -> np.ndarray:
    """Boolean-lattice zeta g(S) = Σ_{T ⊆ S} f(T) by Yates' O(n log n)
    subset-sum transform: for each bit b, for S ∋ b: g[S] += g[S\\b]."""
    g = np.array(f, copy=True)
    integer = g.dtype == np.int64
    if integer:
        g = g.view(np.uint64)
    n = 1 << bits
    S = np.arange(n)
    for b in range(bits):
        has = (S >> b) & 1 == 1
        g[S[has]] = g[S[has]] + g[S[has] ^ (1 << b)]
    return g.view(np.int64) if integer else g


def yates_moebius(bits: int, g: np.ndarray) -> np.ndarray:
    """Inverse of ``yates_zeta``: for each bit b, for S ∋ b: f[S] -= f[S\\b]."""
    f = np.array(g, copy=True)
    integer = f.dtype == np.int64
    if integer:
        f = f.view(np.uint64)
    n = 1 << bits
    S = np.arange(n)
    for b in range(bits):
        has = (S >> b) & 1 == 1
        f[S[has]] = f[S[has]] - f[S[has] ^ (1 << b)]
    return f.view(np.int64) if integer else f


def width_bruteforce(n, src, dst) -> int:
    """Largest antichain by exhaustive search (Dilworth, Thm. 2);
    n <= 24."""
    if n > 24:
        raise ValueError("width_bruteforce: n too large")
    Z = zeta_matrix(n, src, dst)
    comp = [0] * n
    for x in range(n):
        for y in range(n):
            if x != y and (Z[x, y] or Z[y, x]):
                comp[x] |= 1 << y
    best = 0

    def rec(cand: int, size: int):
        nonlocal best
        if size + bin(cand).count("1") <= best:
            return
        if cand == 0:
            best = max(best, size)
            return
        v = (cand & -cand).bit_length() - 1
        rec(cand & ~(1 << v) & ~comp[v], size + 1)
        rec(cand & ~(1 << v), size)

    rec((1 << n) - 1, 0)
    return best


def longest_chain(n, src, dst) -> int:
    """ℓ = number of elements of a longest chain (Thm. 5 Mirsky),
    by DP over a bottom-up order."""
    ch = children_lists(n, src, dst)
    order = bottom_up_order(n, ch)
    h = [0] * n
    for x in order:
        h[x] = 1 + max((h[c] for c in ch[x]), default=0)
    return max(h, default=0)


def max_matching_bruteforce(n, src, dst) -> int:
    """Size of a maximum matching of the split graph G' (Alg. 1)
    by exhaustive search over edge subsets (tiny graphs only)."""
    edges = sorted(set(zip(np.asarray(src).tolist(), np.asarray(dst).tolist())))
    if len(edges) > 20:
        raise ValueError("max_matching_bruteforce: too many edges")
    best = 0
    for r in range(len(edges), 0, -1):
        for sub in itertools.combinations(edges, r):
            ls = {a for a, _ in sub}
            rs = {b for _, b in sub}
            if len(ls) == r and len(rs) == r:
                return r
    return best
