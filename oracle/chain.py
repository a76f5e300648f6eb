"""Oracle O2 wrapper: the paper's sequential chain algorithm in plain C
(``oracle/chain_oracle.c``).  TEST INFRASTRUCTURE ONLY (see
``oracle/__init__.py``).  Builds ``oracle/_chain_oracle.so`` with gcc on
first use (``__graft_entry__.build()`` also builds it)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "chain_oracle.c")
_SO = os.path.join(_HERE, "_chain_oracle.so")
_lib = None

ERRORS = {-1: "cycle", -2: "self loop", -3: "invalid input", -4: "out of memory",
          -5: "not a chain", -6: "not a partition"}


def build(force: bool = False) -> str:
    """gcc -O2; with -fopenmp for the parallel CPU baseline (oracle_*_omp)
    when the compiler supports it, else single-threaded."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        base = ["gcc", "-O2", "-std=gnu99", "-shared", "-fPIC", _SRC, "-o", _SO]
        try:
            subprocess.check_call(base + ["-fopenmp"], stderr=subprocess.DEVNULL)
        except subprocess.CalledProcessError:
            subprocess.check_call(base)
    return _SO


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.oracle_build.argtypes = [i64, i64, P, P, i64, P, P, ctypes.POINTER(ctypes.c_void_p)]
        lib.oracle_build.restype = ctypes.c_int
        lib.oracle_free.argtypes = [P]
        lib.oracle_info.argtypes = [P, P]
        lib.oracle_export_chains.argtypes = [P, P, P, P, P]
        lib.oracle_export_niv.argtypes = [P, P]
        lib.oracle_threads.restype = ctypes.c_int
        for fn in (lib.oracle_zeta, lib.oracle_moebius, lib.oracle_zeta_omp, lib.oracle_moebius_omp):
            fn.argtypes = [P, P, P, i64, ctypes.c_int]
            fn.restype = ctypes.c_int
        lib.oracle_zeta_sampled.argtypes = [P, P, i64, ctypes.c_int, i64, P, P, P]
        lib.oracle_zeta_sampled.restype = ctypes.c_int
        lib.oracle_zeta_sampled_edges.argtypes = [i64, i64, P, P, P, i64, ctypes.c_int, i64, P, P, P]
        lib.oracle_zeta_sampled_edges.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class ChainOracle:
    """O2 for one poset.  ``chains`` (optional): list of user-id lists, each
    listed top-down, injected instead of running Alg. 1."""

    def __init__(self, n, src, dst, chains=None):
        lib = _load()
        self._lib = lib
        src = np.ascontiguousarray(src, dtype=np.int64)
        dst = np.ascontiguousarray(dst, dtype=np.int64)
        h = ctypes.c_void_p()
        if chains is not None:
            ptr = np.zeros(len(chains) + 1, dtype=np.int64)
            ptr[1:] = np.cumsum([len(c) for c in chains])
            el = np.ascontiguousarray(np.concatenate([np.asarray(c, np.int64) for c in chains])
                                      if chains else np.zeros(0, np.int64))
            rc = lib.oracle_build(n, src.shape[0], _ptr(src), _ptr(dst), len(chains),
                                  _ptr(ptr), _ptr(el), ctypes.byref(h))
        else:
            rc = lib.oracle_build(n, src.shape[0], _ptr(src), _ptr(dst), 0, None, None,
                                  ctypes.byref(h))
        if rc:
            raise ValueError(f"oracle_build: {ERRORS.get(rc, rc)}")
        self._h = h
        info = np.zeros(6, dtype=np.int64)
        lib.oracle_info(h, _ptr(info))
        self.n, self.m, self.k, self.q, self.ell, self.nnz = (int(v) for v in info)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.oracle_free(h)
            self._h = None

    def chains(self):
        """(chain id 0-based, next user id, Alg. 6 level 1-based, paper index) per user vertex."""
        n = self.n
        c, nx, lv, pp = (np.zeros(n, dtype=np.int64) for _ in range(4))
        self._lib.oracle_export_chains(self._h, _ptr(c), _ptr(nx), _ptr(lv), _ptr(pp))
        return c, nx, lv, pp

    def niv_dense(self):
        """out[u, j] = user id of niv_{j}(u) (chain j 0-based) or -1 (∞)."""
        out = np.zeros((self.n, self.k), dtype=np.int64)
        self._lib.oracle_export_niv(self._h, _ptr(out))
        return out

    @staticmethod
    def _dt(a):
        if a.dtype == np.int64:
            return 0
        if a.dtype == np.float64:
            return 1
        raise TypeError(a.dtype)

    def zeta(self, f):
        f = np.ascontiguousarray(f)
        f2 = f.reshape(self.n, -1)
        g = np.empty_like(f2)
        rc = self._lib.oracle_zeta(self._h, _ptr(f2), _ptr(g), f2.shape[1], self._dt(f2))
        if rc:
            raise MemoryError("oracle_zeta")
        return g.reshape(f.shape)

    def moebius(self, g):
        g = np.ascontiguousarray(g)
        g2 = g.reshape(self.n, -1)
        f = np.empty_like(g2)
        rc = self._lib.oracle_moebius(self._h, _ptr(g2), _ptr(f), g2.shape[1], self._dt(g2))
        if rc:
            raise MemoryError("oracle_moebius")
        return f.reshape(g.shape)

    def _run(self, fn, x):
        x = np.ascontiguousarray(x)
        x2 = x.reshape(self.n, -1)
        y = np.empty_like(x2)
        if fn(self._h, _ptr(x2), _ptr(y), x2.shape[1], self._dt(x2)):
            raise MemoryError(fn.__name__)
        return y.reshape(x.shape)

    def zeta_omp(self, f):
        """Alg. 3 with chains / rows in parallel (OpenMP, all threads)."""
        return self._run(self._lib.oracle_zeta_omp, f)

    def moebius_omp(self, g):
        """Alg. 4 scheduled by Alg. 5 (antichains in order, elements of an
        antichain in parallel)."""
        return self._run(self._lib.oracle_moebius_omp, g)

    def zeta_sampled(self, f, xs):
        """Brute-force g(x) = Σ_{y ⪯ x} f(y) for the user vertices ``xs`` only
        (DFS of ↓x); for fp64 also returns Σ_{y ⪯ x}|f(y)|."""
        f = np.ascontiguousarray(f).reshape(self.n, -1)
        xs = np.ascontiguousarray(xs, dtype=np.int64)
        B = f.shape[1]
        g = np.empty((xs.shape[0], B), dtype=f.dtype)
        ab = np.empty((xs.shape[0], B), dtype=np.float64) if f.dtype == np.float64 else None
        rc = self._lib.oracle_zeta_sampled(self._h, _ptr(f), B, self._dt(f), xs.shape[0],
                                           _ptr(xs), _ptr(g), _ptr(ab) if ab is not None else None)
        if rc:
            raise MemoryError("oracle_zeta_sampled")
        return g, ab


def threads() -> int:
    """OpenMP threads the parallel oracle uses (1 without OpenMP)."""
    return int(_load().oracle_threads())


def zeta_sampled_edges(n, src, dst, f, xs):
    """Brute-force g(x) = Σ_{y ⪯ x} f(y) for user vertices ``xs`` straight
    from the edge list (DFS of ↓x; no chains, no niv).  For fp64 also
    returns Σ_{y ⪯ x}|f(y)| (the tolerance scale)."""
    lib = _load()
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    f = np.ascontiguousarray(f).reshape(n, -1)
    xs = np.ascontiguousarray(xs, dtype=np.int64)
    B = f.shape[1]
    dt = 0 if f.dtype == np.int64 else 1
    g = np.empty((xs.shape[0], B), dtype=f.dtype)
    ab = np.empty((xs.shape[0], B), dtype=np.float64) if dt == 1 else None
    rc = lib.oracle_zeta_sampled_edges(n, src.shape[0], _ptr(src), _ptr(dst), _ptr(f), B, dt,
                                       xs.shape[0], _ptr(xs), _ptr(g),
                                       _ptr(ab) if ab is not None else None)
    if rc:
        raise MemoryError("oracle_zeta_sampled_edges")
    return g, ab
