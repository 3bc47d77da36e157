"""ctypes loader for the C oracle (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py)."""
from __future__ import annotations

import ctypes
import os
import subprocess

from . import mapa_oracle as mo

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (called by __graft_entry__.build())."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               "-o", _LIB, _SRC])
    return _LIB


class OracleResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("k", ctypes.c_int32),
                ("device_mask", ctypes.c_uint32), ("mapping", ctypes.c_int8 * 8),
                ("m", ctypes.c_int32), ("used", (ctypes.c_int32 * 2) * 28),
                ("x", ctypes.c_int32), ("y", ctypes.c_int32), ("z", ctypes.c_int32),
                ("agg_bw", ctypes.c_int32), ("preserved_bw", ctypes.c_int32),
                ("pad", ctypes.c_int32),
                ("pred_effbw", ctypes.c_double), ("score", ctypes.c_double),
                ("raw", ctypes.c_uint64), ("distinct", ctypes.c_uint64)]


class OracleResultDeep(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("k", ctypes.c_int32),
                ("device_mask", ctypes.c_uint64), ("mapping", ctypes.c_int8 * 16),
                ("m", ctypes.c_int32), ("used", (ctypes.c_int32 * 2) * 120),
                ("x", ctypes.c_int32), ("y", ctypes.c_int32), ("z", ctypes.c_int32),
                ("agg_bw", ctypes.c_int32), ("preserved_bw", ctypes.c_int32),
                ("pad", ctypes.c_int32),
                ("pred_effbw", ctypes.c_double), ("score", ctypes.c_double),
                ("raw", ctypes.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_allocate.restype = ctypes.c_int
        _lib.oracle_allocate.argtypes = [
            ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.c_uint32, ctypes.c_int,
            ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(OracleResult)]
        _lib.oracle_allocate_deep.restype = ctypes.c_int
        _lib.oracle_allocate_deep.argtypes = [
            ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.c_uint64, ctypes.c_int,
            ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(OracleResultDeep)]
        _lib.oracle_eq2.restype = ctypes.c_double
        _lib.oracle_eq2.argtypes = [ctypes.c_int] * 3
    return _lib


def allocate(topo: mo.Topology, busy: int, k: int, pedges, selector: int, sensitive: bool,
             nthreads: int | None = None, a_lo: int = -1, a_hi: int = -1, b_lo: int = -1,
             b_hi: int = -1) -> dict:
    """Same result dict as mapa_oracle.allocate (without the exact Fraction)."""
    n = topo.n
    w = (ctypes.c_int32 * (n * n))(*[topo.w[u][v] for u in range(n) for v in range(n)])
    flat = [c for e in pedges for c in e]
    pe = (ctypes.c_int32 * max(1, len(flat)))(*flat)
    r = OracleResult()
    nt = nthreads or os.cpu_count() or 1
    rc = lib().oracle_allocate(n, w, busy, k, len(pedges), pe, selector, int(bool(sensitive)),
                               nt, a_lo, a_hi, b_lo, b_hi, ctypes.byref(r))
    if rc != 0:
        raise ValueError(f"oracle_allocate rc={rc}")
    if r.status == 1:
        return dict(status="no_capacity", raw=int(r.raw), distinct=int(r.distinct))
    devs = tuple(d for d in range(n) if (r.device_mask >> d) & 1)
    return dict(status="ok", devices=devs, mapping=tuple(r.mapping[i] for i in range(k)),
                used_edges=[(r.used[i][0], r.used[i][1]) for i in range(len(pedges))],
                x=r.x, y=r.y, z=r.z, agg_bw=r.agg_bw, preserved_bw=r.preserved_bw,
                pred_effbw=r.pred_effbw, raw=int(r.raw), distinct=int(r.distinct))


def allocate_deep(topo: mo.Topology, busy: int, k: int, pedges, selector: int, sensitive: bool,
                  nthreads: int | None = None, max_subsets: int = 4096, sub_lo: int = -1,
                  sub_hi: int = -1) -> dict:
    """Deep oracle (k <= 16): same decision fields as allocate(); 'distinct'
    is not counted (None).  [sub_lo, sub_hi): lex indices of the k-subsets
    scored (negative = unrestricted)."""
    n = topo.n
    w = (ctypes.c_int32 * (n * n))(*[topo.w[u][v] for u in range(n) for v in range(n)])
    flat = [c for e in pedges for c in e]
    pe = (ctypes.c_int32 * max(1, len(flat)))(*flat)
    r = OracleResultDeep()
    nt = nthreads or os.cpu_count() or 1
    rc = lib().oracle_allocate_deep(n, w, busy, k, len(pedges), pe, selector, int(bool(sensitive)), nt,
                                    max_subsets, sub_lo, sub_hi, ctypes.byref(r))
    if rc != 0:
        raise ValueError(f"oracle_allocate_deep rc={rc}")
    if r.status == 1:
        return dict(status="no_capacity", raw=int(r.raw), distinct=None)
    devs = tuple(d for d in range(n) if (r.device_mask >> d) & 1)
    return dict(status="ok", devices=devs, mapping=tuple(r.mapping[i] for i in range(k)),
                used_edges=[(r.used[i][0], r.used[i][1]) for i in range(len(pedges))],
                x=r.x, y=r.y, z=r.z, agg_bw=r.agg_bw, preserved_bw=r.preserved_bw,
                pred_effbw=r.pred_effbw, raw=int(r.raw), distinct=None)


def eq2(x: int, y: int, z: int) -> float:
    return lib().oracle_eq2(x, y, z)
