"""B200-native chain-decomposition zeta / Moebius transforms on posets
(arXiv 2211.13706).

Thin Python binding over the C-ABI of ``libposet.so`` (``include/poset.h``):
argument marshalling only -- every step of the transforms runs in the
library's sm_100a kernels.  PyTorch supplies device memory and streams; numpy
arrays (host memory) are accepted too and are staged by the library itself.

There is no CPU fallback: if ``libposet.so`` is missing or fails to load,
importing the binding raises ``ImportError`` (build it with
``python paper_2211_13706_b200/build.py``).

    import torch, paper_2211_13706_b200 as pz
    P = pz.Poset(n, src, dst)               # one-time setup (host + kernel ii)
    g = P.zeta(f)                           # f: [n][B] int64 / float64 tensor
    f2 = P.moebius(g)
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

__all__ = ["Poset", "PosetError", "analyze", "lib", "MOEB_AUTO", "MOEB_LEVEL", "MOEB_GRID", "MOEB_WARP",
           "MOEB_RING", "MOEB_CSR", "MOEB_RINGWS", "MOEB_RINGDF",
           "MOEB_RINGCL", "MOEB_RINGCW", "LIB_PATH"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libposet.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2211_13706_b200/build.py` "
                      "(there is no CPU fallback)")
try:
    lib = ctypes.CDLL(LIB_PATH)
except OSError as e:   # pragma: no cover
    raise ImportError(f"cannot load {LIB_PATH}: {e} (there is no CPU fallback)") from e

MOEB_AUTO, MOEB_LEVEL, MOEB_GRID, MOEB_WARP, MOEB_RING, MOEB_CSR, MOEB_RINGWS, MOEB_RINGDF, MOEB_RINGCL, \
    MOEB_RINGCW = (0, 1, 2, 3, 4, 5, 6, 7, 8, 9)
_I64, _F64 = 0, 1
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64


class PosetInfo(ctypes.Structure):
    _fields_ = [("n", _i64), ("m", _i64), ("k", _i64), ("q", _i64), ("ell", _i64), ("nnz", _i64),
                ("table_bytes", _i64), ("max_level_width", _i64),
                ("t_ingest", ctypes.c_double), ("t_levels", ctypes.c_double),
                ("t_match", ctypes.c_double), ("t_chains", ctypes.c_double),
                ("t_upload", ctypes.c_double), ("t_mtable", ctypes.c_double),
                ("device", ctypes.c_int32), ("moebius_kernel", ctypes.c_int32),
                ("reach", _i64), ("dist_bytes", _i64), ("t_dist", ctypes.c_double),
                ("csr_bytes", _i64), ("zeta_sparse", _i64), ("ringws", _i64), ("ringdf", _i64),
                ("rdf_bytes", _i64), ("ring_bytes", _i64), ("rws_bytes", _i64),
                ("depth_u", _i64), ("t_depth", ctypes.c_double), ("gather_bytes", _i64),
                ("gather_entries", _i64), ("gather_resets", _i64),
                ("moebius_sms", _i64), ("num_sms", _i64)]


def _sig(name, args, res=ctypes.c_int):
    fn = getattr(lib, name)
    fn.argtypes = args
    fn.restype = res
    return fn


_sig("poset_setup", [_i64, _i64, _vp, _vp, ctypes.c_int, ctypes.POINTER(_vp)])
_sig("poset_setup_ex", [_i64, _i64, _vp, _vp, ctypes.c_int, ctypes.c_uint32, ctypes.POINTER(_vp)])
_sig("poset_setup_chains", [_i64, _i64, _vp, _vp, _i64, _vp, _vp, ctypes.c_int, ctypes.POINTER(_vp)])
_sig("poset_zeta", [_vp, _vp, _vp, _i64, ctypes.c_int, _vp])
_sig("poset_moebius", [_vp, _vp, _vp, _i64, ctypes.c_int, _vp])
_sig("poset_scan_slots", [_vp, _vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp])
_sig("poset_scan_carry", [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp])
_sig("poset_gather_rows", [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp])
_sig("poset_rank_to_user", [_vp, _vp, _vp, _i64, ctypes.c_int, _vp])
_sig("poset_combine_tails", [_vp, _vp, _i64, _i64, _vp, _i64, ctypes.c_int, _vp])
_sig("poset_query", [_vp, ctypes.POINTER(PosetInfo)])
_sig("poset_analyze", [_i64, _i64, _vp, _vp, ctypes.POINTER(PosetInfo), _vp, _vp, _vp])
_sig("poset_set_option", [_vp, ctypes.c_char_p, _i64])
_sig("poset_profile_read", [_vp, _vp, _vp, _vp])
_sig("poset_export_chains", [_vp, _vp, _vp, _vp, _vp])
_sig("poset_export_mtable", [_vp, _vp])
_sig("poset_debug_read", [_vp, _vp])
_sig("poset_destroy", [_vp], None)
_sig("poset_strerror", [ctypes.c_int], ctypes.c_char_p)
_sig("poset_last_error", [], ctypes.c_char_p)
_sig("poset_shard_rows", [_vp, _i64, _i64, ctypes.c_uint32])
_sig("poset_abi_version", [], ctypes.c_int)
_sig("poset_sync", [_vp, _vp])
_sig("poset_nvls_create", [ctypes.POINTER(ctypes.c_int), ctypes.c_int, _i64, ctypes.POINTER(_vp)])
_sig("poset_nvls_ptrs", [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_i64)])
_sig("poset_nvls_destroy", [_vp], None)
_sig("poset_scan_slots_mc", [_vp, _vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp])
ABI_VERSION = 2   # poset_info layout (PosetInfo) this binding marshals
if lib.poset_abi_version() != ABI_VERSION:
    raise ImportError(f"libposet.so ABI {lib.poset_abi_version()} != binding ABI {ABI_VERSION}: rebuild "
                      "(python -c 'import __graft_entry__ as g; g.build()')")

STATUS = {0: "OK", 1: "EINVAL", 2: "ESELFLOOP", 3: "ECYCLE", 4: "ENOTCHAIN", 5: "ENOTPARTITION",
          6: "ETOOBIG", 7: "ENOMEM", 8: "ECUDA"}


class PosetError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.code = STATUS.get(status, str(status))


def _check(rc: int):
    if rc != 0:
        raise PosetError(rc, lib.poset_last_error().decode(errors="replace"))


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def _torch():
    import torch
    return torch


def _dtype_code(x) -> int:
    if isinstance(x, np.ndarray):
        if x.dtype == np.int64:
            return _I64
        if x.dtype == np.float64:
            return _F64
        raise TypeError(f"unsupported dtype {x.dtype} (int64 or float64)")
    torch = _torch()
    if x.dtype == torch.int64:
        return _I64
    if x.dtype == torch.float64:
        return _F64
    raise TypeError(f"unsupported dtype {x.dtype} (int64 or float64)")


def _ptr(x):
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return _vp(x.ctypes.data)
    if not x.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return _vp(x.data_ptr())


def _stream_ptr(stream, x):
    if stream is not None:
        return _vp(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    if not isinstance(x, np.ndarray) and x.is_cuda:
        return _vp(_torch().cuda.current_stream(x.device).cuda_stream)
    return _vp(0)


def analyze(n: int, src, dst, want_chains: bool = False):
    """Host-only setup analysis (``poset_analyze``): no GPU needed.  Returns
    the info dict, plus (chain, pos, level) numpy arrays if ``want_chains``."""
    src = np.ascontiguousarray(np.asarray(src, dtype=np.int64))
    dst = np.ascontiguousarray(np.asarray(dst, dtype=np.int64))
    out = PosetInfo()
    arrs = [np.zeros(n, dtype=np.int64) for _ in range(3)] if want_chains else None
    ptrs = [_np_ptr(a) for a in arrs] if arrs else [None, None, None]
    _check(lib.poset_analyze(n, src.shape[0], _np_ptr(src), _np_ptr(dst), ctypes.byref(out), *ptrs))
    info = {name: getattr(out, name) for name, _ in PosetInfo._fields_}
    return (info, *arrs) if want_chains else info


class Poset:
    """One poset, set up once (``poset_setup``), transformed many times.

    ``src``/``dst``: int64 edge arrays, edge e meaning ``dst[e] ⪯ src[e]``.
    ``chains``: optional injected chain decomposition (list of user-id lists,
    each top-down) -- ``poset_setup_chains``.  ``sparse``: build only the
    sparse rows, straight from the DAG (``POSET_SETUP_SPARSE``); the library
    also does this on its own when the dense table does not fit.
    """

    def __init__(self, n: int, src, dst, device: int = 0, chains=None, sparse: bool = False):
        src = np.ascontiguousarray(np.asarray(src, dtype=np.int64))
        dst = np.ascontiguousarray(np.asarray(dst, dtype=np.int64))
        if src.shape != dst.shape:
            raise ValueError("src and dst must have the same length")
        h = _vp()
        if chains is None:
            rc = lib.poset_setup_ex(n, src.shape[0], _np_ptr(src), _np_ptr(dst), device, 1 if sparse else 0,
                                    ctypes.byref(h))
        else:
            ptr = np.zeros(len(chains) + 1, dtype=np.int64)
            ptr[1:] = np.cumsum([len(c) for c in chains])
            el = np.ascontiguousarray(np.concatenate([np.asarray(c, np.int64) for c in chains])
                                      if len(chains) else np.zeros(0, np.int64))
            rc = lib.poset_setup_chains(n, src.shape[0], _np_ptr(src), _np_ptr(dst), len(chains),
                                        _np_ptr(ptr), _np_ptr(el), device, ctypes.byref(h))
        _check(rc)
        self._h = h
        self.n = int(n)
        self.device = device
        inf = self.info()
        self.k = inf["k"]
        self.ell = inf["ell"]

    def close(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.poset_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    # ---------------------------------------------------------------- info --
    def info(self) -> dict:
        out = PosetInfo()
        _check(lib.poset_query(self._h, ctypes.byref(out)))
        return {name: getattr(out, name) for name, _ in PosetInfo._fields_}

    def set_option(self, key: str, value: int):
        _check(lib.poset_set_option(self._h, key.encode(), int(value)))

    PHASES = ("scan", "gather", "moebius_solve", "chain_diff", "h2d", "d2h", "perm")

    def profile_read(self):
        """{phase: (ms summed, calls)} since the last read + kernel launches."""
        ms = np.zeros(8, dtype=np.float64)
        calls = np.zeros(8, dtype=np.int64)
        launches = ctypes.c_int64(0)
        _check(lib.poset_profile_read(self._h, _np_ptr(ms), _np_ptr(calls), ctypes.byref(launches)))
        return {p: (float(ms[i]), int(calls[i])) for i, p in enumerate(self.PHASES)}, launches.value

    def export_chains(self):
        """(chain, pos, level, rank) per user vertex, numpy int64."""
        c, p, l, r = (np.zeros(self.n, dtype=np.int64) for _ in range(4))
        _check(lib.poset_export_chains(self._h, _np_ptr(c), _np_ptr(p), _np_ptr(l), _np_ptr(r)))
        return c, p, l, r

    def debug_read(self):
        """Tuning hook (poset_debug_read): clock64 phase sums of the last
        instrumented RING call."""
        out = np.zeros(8, dtype=np.int64)
        _check(lib.poset_debug_read(self._h, _np_ptr(out)))
        return out

    def export_mtable(self) -> np.ndarray:
        """m(x, j) as an [n][k] int32 array (bottom-up position, -1 = ∞)."""
        out = np.zeros((self.n, self.k), dtype=np.int32)
        _check(lib.poset_export_mtable(self._h, _np_ptr(out)))
        return out

    # ---------------------------------------------------------- transforms --
    def _run(self, fn, x, out, stream):
        if x.ndim == 1:
            x2 = x.reshape(-1, 1)
        else:
            x2 = x
        if x2.shape[0] != self.n:
            raise ValueError(f"expected {self.n} rows, got {x2.shape[0]}")
        batch = x2.shape[1]
        if out is None:
            if isinstance(x, np.ndarray):
                out = np.empty_like(x)
            else:
                out = _torch().empty_like(x)
        if tuple(out.shape) != tuple(x.shape):
            raise ValueError("output shape mismatch")
        dt = _dtype_code(x)
        if _dtype_code(out) != dt:
            raise TypeError("input and output dtypes differ")
        for t in (x, out):
            if not isinstance(t, np.ndarray) and t.is_cuda and t.device.index != self.device:
                raise ValueError(f"tensor on {t.device}, poset on cuda:{self.device}")
        sp = _stream_ptr(stream, x)
        _check(fn(self._h, _ptr(x), _ptr(out), batch, dt, sp))
        if isinstance(out, np.ndarray) or not out.is_cuda:
            # a host result is complete only once the staging copy has landed
            _check(lib.poset_sync(self._h, sp))
        return out

    def zeta(self, f, out=None, stream=None):
        """g = Z f (Eq. inv-formula; Alg. 3).  f: [n] or [n][B]."""
        return self._run(lib.poset_zeta, f, out, stream)

    def moebius(self, g, out=None, stream=None):
        """f = Z^{-1} g (Cor. 1 P:L143-151; Alg. 4).  g: [n] or [n][B]."""
        return self._run(lib.poset_moebius, g, out, stream)

    # ------------------------------------------------ split phases (dist) --
    def scan_slots(self, f, F, tail, lo, hi, stream=None):
        B = f.shape[1] if f.ndim == 2 else 1
        _check(lib.poset_scan_slots(self._h, _ptr(f), _ptr(F), _ptr(tail), lo, hi, B,
                                    _dtype_code(f), _stream_ptr(stream, f)))

    def scan_slots_mc(self, f, F_mc: int, tail, lo, hi, stream=None):
        """scan_slots with every F row stored through the NVLS multicast
        address ``F_mc`` (an ``NvlsBuffer.mc``): the all-gather of F fused
        into the scan epilogue (poset_scan_slots_mc)."""
        B = f.shape[1] if f.ndim == 2 else 1
        _check(lib.poset_scan_slots_mc(self._h, _ptr(f), _vp(int(F_mc)), _ptr(tail), lo, hi, B,
                                       _dtype_code(f), _stream_ptr(stream, f)))

    def scan_carry(self, F, carry, lo, hi, stream=None):
        B = F.shape[1] if F.ndim == 2 else 1
        _check(lib.poset_scan_carry(self._h, _ptr(F), _ptr(carry), lo, hi, B, _dtype_code(F),
                                    _stream_ptr(stream, F)))

    def gather_rows(self, F, g_rank, lo, hi, stream=None):
        B = F.shape[1] if F.ndim == 2 else 1
        _check(lib.poset_gather_rows(self._h, _ptr(F), _ptr(g_rank), lo, hi, B, _dtype_code(F),
                                     _stream_ptr(stream, F)))

    def shard_rows(self, lo, hi, drop_moebius=False):
        """Keep only the index rows [lo, hi) on this handle (poset_shard_rows)."""
        _check(lib.poset_shard_rows(self._h, int(lo), int(hi), 1 if drop_moebius else 0))

    def combine_tails(self, tails_all, world, rank, carry, stream=None):
        B = carry.shape[-1]
        _check(lib.poset_combine_tails(self._h, _ptr(tails_all), world, rank, _ptr(carry), B,
                                       _dtype_code(carry), _stream_ptr(stream, carry)))

    def rank_to_user(self, g_rank, g_user, stream=None):
        B = g_rank.shape[1] if g_rank.ndim == 2 else 1
        _check(lib.poset_rank_to_user(self._h, _ptr(g_rank), _ptr(g_user), B,
                                      _dtype_code(g_rank), _stream_ptr(stream, g_rank)))


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "strides": None, "version": 3}


class NvlsBuffer:
    """One buffer per listed device bound to an NVLS multicast object
    (poset_nvls_create): a store through ``mc`` lands on every device's
    buffer.  ``tensor(i, shape, dtype)`` views device i's buffer."""

    def __init__(self, devices, nbytes: int):
        devs = (ctypes.c_int * len(devices))(*devices)
        h = _vp()
        _check(lib.poset_nvls_create(devs, len(devices), int(nbytes), ctypes.byref(h)))
        self._h = h
        self.devices = list(devices)
        mc = _vp()
        uc = (_vp * len(devices))()
        nb = _i64()
        _check(lib.poset_nvls_ptrs(h, ctypes.byref(mc), uc, ctypes.byref(nb)))
        self.mc = int(mc.value)
        self.uc = [int(u) for u in uc]
        self.nbytes = int(nb.value)

    def tensor(self, i: int, shape, dtype):
        torch = _torch()
        item = torch.empty((), dtype=dtype).element_size()
        if math.prod(shape) * item > self.nbytes:
            raise ValueError("view larger than the buffer")
        typestr = {torch.float64: "<f8", torch.int64: "<i8"}[dtype]
        return torch.as_tensor(_CudaArray(self.uc[i], shape, typestr), device=f"cuda:{self.devices[i]}")

    def close(self):
        if getattr(self, "_h", None):
            lib.poset_nvls_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
