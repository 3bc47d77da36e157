"""Thin Python binding of libmapa.so (include/mapa.h) — argument marshalling only.

Every step of the hot path (enumerate, score, argmax) runs in the sm_100a
kernels of ``csrc/esa.cu``; the host pieces (topology encode, pattern compile,
key decode) are C++ in ``csrc/mapa_host.cpp``.  There is no Python or CPU
fallback: if ``libmapa.so`` is missing the import fails loudly.  PyTorch is
used only for device memory, streams and ``torch.distributed`` (see
``dist.py``).

Names follow the C-ABI (``mapa_allocate`` -> ``allocate`` etc.).  Device ids
are 0-based (the paper's 1-based id - 1).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmapa.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the MAPA hot path has no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

OK, NO_CAPACITY = 0, 1
E_INVALID_ARG, E_PARSE, E_ALREADY_BUSY, E_NOT_BUSY, E_ID_RANGE = -1, -2, -3, -4, -5
E_UNSUPPORTED, E_CUDA, E_DISCONNECTED, E_INTERNAL = -6, -7, -8, -10
SEL_GREEDY, SEL_PRESERVE, SEL_BASELINE, SEL_TOPO = 0, 1, 2, 3
POLICIES = {"baseline": 0, "topo": 1, "greedy": 2, "preserve": 3}
F_COMMIT, F_RAW, F_ALLOW_DISCONNECTED, F_PRUNE, F_DEEP, F_ZEROED = 1, 2, 4, 8, 16, 32
MAX_K = 16
SHAPES = {"ring": 0, "tree": 1, "ringtree": 2, "full": 3, "edgeless": 4}


class MapaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"mapa status {status}: {msg}")
        self.status = status


class Decision(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("k", ctypes.c_int32), ("device_mask", ctypes.c_uint64),
                ("mapping", ctypes.c_int8 * 16), ("m", ctypes.c_int32), ("used", (ctypes.c_int32 * 2) * 120),
                ("x", ctypes.c_int32), ("y", ctypes.c_int32), ("z", ctypes.c_int32),
                ("agg_bw", ctypes.c_int32), ("preserved_bw", ctypes.c_int32), ("score", ctypes.c_int32),
                ("pred_effbw", ctypes.c_double), ("raw_embeddings", ctypes.c_uint64),
                ("distinct_matches", ctypes.c_uint64), ("leaves_scored", ctypes.c_uint64),
                ("key", ctypes.c_uint64), ("ecode", ctypes.c_uint64 * 2)]


class Query(ctypes.Structure):
    _fields_ = [("busy", ctypes.c_uint32), ("pattern", ctypes.c_uint32), ("selector", ctypes.c_int32),
                ("sensitive", ctypes.c_int32)]


class Record(ctypes.Structure):
    _fields_ = [("key", ctypes.c_uint64), ("leaves", ctypes.c_uint64), ("ctr", ctypes.c_uint32),
                ("status", ctypes.c_uint32), ("reserved", ctypes.c_uint64)]


class WideRecord(ctypes.Structure):
    """mapa_wide_record (deep path): 256-bit key (score, set, ecode_hi, ecode_lo)."""
    _fields_ = [("score", ctypes.c_uint64), ("set", ctypes.c_uint64), ("ecode_hi", ctypes.c_uint64),
                ("ecode_lo", ctypes.c_uint64), ("leaves", ctypes.c_uint64), ("ctr", ctypes.c_uint32),
                ("lock", ctypes.c_uint32), ("status", ctypes.c_uint32), ("pad", ctypes.c_uint32),
                ("reserved", ctypes.c_uint64)]


class PatternInfo(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("m", ctypes.c_int32), ("aut_order", ctypes.c_int32),
                ("back", ctypes.c_uint16 * 16), ("lex_src", ctypes.c_uint16 * 16),
                ("edges", (ctypes.c_int32 * 2) * 120), ("aut_order64", ctypes.c_uint64)]


class Job(ctypes.Structure):
    _fields_ = [("pattern", ctypes.c_int32), ("sensitive", ctypes.c_int32), ("duration", ctypes.c_double),
                ("arrival", ctypes.c_double)]


class JobLog(ctypes.Structure):
    _fields_ = [("job", ctypes.c_int32), ("k", ctypes.c_int32), ("device_mask", ctypes.c_uint32),
                ("x", ctypes.c_int32), ("y", ctypes.c_int32), ("z", ctypes.c_int32), ("agg_bw", ctypes.c_int32),
                ("preserved_bw", ctypes.c_int32), ("pred_effbw", ctypes.c_double), ("arrival", ctypes.c_double),
                ("start", ctypes.c_double), ("end", ctypes.c_double), ("wait", ctypes.c_double)]


class TraceOp(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("job", ctypes.c_int32)]


assert ctypes.sizeof(Query) == 16 and ctypes.sizeof(Record) == 32 and ctypes.sizeof(WideRecord) == 64

_vp = ctypes.c_void_p
_S = ctypes.c_int32
_SIGS = {
    "mapa_load_topology": (_S, [ctypes.c_char_p, ctypes.c_int32, ctypes.POINTER(_vp)]),
    "mapa_free_topology": (None, [_vp]),
    "mapa_topology_info": (_S, [_vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint64)]),
    "mapa_claim": (_S, [_vp, ctypes.c_uint64]),
    "mapa_release": (_S, [_vp, ctypes.c_uint64]),
    "mapa_set_busy": (_S, [_vp, ctypes.c_uint64]),
    "mapa_load_pattern": (_S, [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.c_uint32,
                               ctypes.POINTER(_vp)]),
    "mapa_make_pattern": (_S, [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_vp)]),
    "mapa_free_pattern": (None, [_vp]),
    "mapa_get_pattern_info": (_S, [_vp, ctypes.POINTER(PatternInfo)]),
    "mapa_pred_effbw": (ctypes.c_double, [ctypes.c_int32] * 3),
    "mapa_effbw_rank_table": (_S, [ctypes.c_int32, ctypes.POINTER(ctypes.c_uint16)]),
    "mapa_allocate": (_S, [_vp, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, _vp,
                           ctypes.POINTER(Decision)]),
    "mapa_allocate_many": (_S, [_vp, ctypes.POINTER(_vp), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                ctypes.POINTER(ctypes.c_int32), ctypes.c_uint32, _vp, ctypes.POINTER(Decision)]),
    "mapa_launch_query": (_S, [_vp, _vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp, ctypes.c_uint32,
                               ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, _vp]),
    "mapa_reduce_records": (_S, [ctypes.POINTER(Record), ctypes.c_int32, ctypes.POINTER(Record)]),
    "mapa_launch_queries": (_S, [_vp, ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(Query),
                                 _vp, _vp, ctypes.c_uint32, ctypes.c_int32, _vp]),
    "mapa_launch_query_wide": (_S, [_vp, _vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp, ctypes.c_uint32,
                                    ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, _vp]),
    "mapa_reduce_wide_records": (_S, [ctypes.POINTER(WideRecord), ctypes.c_int32, ctypes.POINTER(WideRecord)]),
    "mapa_decode_wide": (_S, [_vp, _vp, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32,
                              ctypes.POINTER(WideRecord), ctypes.POINTER(Decision)]),
    "mapa_decode": (_S, [_vp, _vp, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32,
                         ctypes.POINTER(Record), ctypes.POINTER(Decision)]),
    "mapa_allocate_batch": (_S, [_vp, ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int64, _vp, _vp, _vp,
                                 ctypes.c_uint32, _vp]),
    "mapa_trace_replay": (_S, [_vp, ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp,
                               ctypes.c_int32, _vp, _vp, ctypes.c_uint32, _vp]),
    "mapa_decode_trace": (_S, [_vp, ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(TraceOp),
                               ctypes.c_int32, ctypes.POINTER(Query), ctypes.POINTER(ctypes.c_uint64), ctypes.c_uint32,
                               ctypes.POINTER(Decision)]),
    "mapa_shard_queries": (_S, [_vp, ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(Query),
                                ctypes.c_uint32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                ctypes.POINTER(ctypes.c_double)]),
    "mapa_fifo_schedule": (_S, [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(TraceOp), ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double)]),
    "mapa_simulate": (_S, [_vp, ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(Job),
                           ctypes.c_int32, ctypes.c_uint32, _vp, ctypes.POINTER(JobLog)]),
    "mapa_quantiles": (_S, [ctypes.POINTER(ctypes.c_double), ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]),
    "mapa_pred_effbw_theta": (ctypes.c_double, [ctypes.POINTER(ctypes.c_double)] + [ctypes.c_int32] * 3),
    "mapa_fit_effbw": (_S, [ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double),
                            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "mapa_pattern_set_effbw_model": (_S, [_vp, ctypes.POINTER(ctypes.c_double)]),
    "mapa_last_error": (ctypes.c_char_p, []),
    "mapa_version": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTS = tuple(_SIGS)


def _check(st: int, allow_no_capacity: bool = False) -> int:
    if st == OK or (allow_no_capacity and st == NO_CAPACITY):
        return st
    raise MapaError(st, _lib.mapa_last_error().decode())


def last_error() -> str:
    return _lib.mapa_last_error().decode()


def version() -> str:
    return _lib.mapa_version().decode()


def pred_effbw(x: int, y: int, z: int) -> float:
    """Eq. 2 with Table 4 theta."""
    return _lib.mapa_pred_effbw(x, y, z)


def pred_effbw_theta(theta, x: int, y: int, z: int) -> float:
    th = (ctypes.c_double * 14)(*theta)
    return _lib.mapa_pred_effbw_theta(th, x, y, z)


def fit_effbw(samples):
    """mapa_fit_effbw: samples [(x, y, z, bw)] -> (theta[14], {rel_err, rmse, mae, cond})."""
    n = len(samples)
    cen = (ctypes.c_int32 * max(1, 3 * n))(*[c for s in samples for c in s[:3]])
    bw = (ctypes.c_double * max(1, n))(*[s[3] for s in samples])
    th = (ctypes.c_double * 14)()
    dg = (ctypes.c_double * 4)()
    _check(_lib.mapa_fit_effbw(n, cen, bw, th, dg))
    return list(th), dict(rel_err=dg[0], rmse=dg[1], mae=dg[2], cond=dg[3])


def effbw_rank_table(m: int) -> list[int]:
    buf = (ctypes.c_uint16 * ((m + 1) * (m + 1)))()
    _check(_lib.mapa_effbw_rank_table(m, buf))
    return list(buf)


_torch = None


def _stream_ptr(stream) -> int | None:
    """cudaStream_t of `stream`, or of torch's current stream when None
    (without a CUDA-capable torch: the legacy default stream)."""
    global _torch
    if stream is None:
        if _torch is None:
            try:
                import torch
                _torch = torch if torch.cuda.is_available() else False
            except Exception:  # pragma: no cover
                _torch = False
        if _torch:
            raw = getattr(_torch._C, "_cuda_getCurrentRawStream", None)
            if raw is not None:  # the raw cudaStream_t without building a Stream object
                return raw(_torch._C._cuda_getDevice())
            return _torch.cuda.current_stream().cuda_stream
        return None
    return getattr(stream, "cuda_stream", stream)


class Topology:
    """mapa_topology handle (hardware graph + busy mask, §3.2 / §3.6)."""

    def __init__(self, builtin: str | None = None, text: str | None = None):
        h = _vp()
        if text is not None:
            _check(_lib.mapa_load_topology(text.encode(), 1, ctypes.byref(h)))
        else:
            _check(_lib.mapa_load_topology(builtin.encode(), 0, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.mapa_free_topology(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    @property
    def handle(self):
        return self._h

    def info(self):
        n, w, busy = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_uint64()
        _check(_lib.mapa_topology_info(self._h, ctypes.byref(n), ctypes.byref(w), None, ctypes.byref(busy)))
        bw = (ctypes.c_int32 * (n.value * n.value))()
        _check(_lib.mapa_topology_info(self._h, None, None, bw, None))
        mat = [[bw[u * n.value + v] for v in range(n.value)] for u in range(n.value)]
        return dict(n=n.value, width=w.value, busy=busy.value, bw=mat)

    @property
    def n(self) -> int:
        return self.info()["n"]

    @property
    def width(self) -> int:
        return self.info()["width"]

    @property
    def busy(self) -> int:
        return self.info()["busy"]

    def claim(self, mask: int):
        _check(_lib.mapa_claim(self._h, mask))

    def release(self, mask: int):
        _check(_lib.mapa_release(self._h, mask))

    def set_busy(self, mask: int):
        _check(_lib.mapa_set_busy(self._h, mask))


class Pattern:
    """mapa_pattern handle (application graph, §3.1 / Fig. 4)."""

    def __init__(self, k: int, edges=None, shape: str | None = None, allow_disconnected: bool = False):
        h = _vp()
        if shape is not None:
            _check(_lib.mapa_make_pattern(SHAPES[shape], k, ctypes.byref(h)))
        else:
            edges = list(edges or [])
            flat = (ctypes.c_int32 * max(1, 2 * len(edges)))(*[c for e in edges for c in e])
            _check(_lib.mapa_load_pattern(k, len(edges), flat,
                                          F_ALLOW_DISCONNECTED if allow_disconnected else 0, ctypes.byref(h)))
        self._h = h

    @classmethod
    def make(cls, shape: str, k: int) -> "Pattern":
        return cls(k, shape=shape)

    def set_effbw_model(self, theta):
        """mapa_pattern_set_effbw_model: Eq. 2 coefficients for this pattern."""
        th = (ctypes.c_double * 14)(*theta)
        _check(_lib.mapa_pattern_set_effbw_model(self._h, th))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.mapa_free_pattern(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        pi = PatternInfo()
        _check(_lib.mapa_get_pattern_info(self._h, ctypes.byref(pi)))
        return dict(k=pi.k, m=pi.m, aut=int(pi.aut_order64), back=list(pi.back)[:pi.k],
                    lex_src=list(pi.lex_src)[:pi.k], edges=[(pi.edges[i][0], pi.edges[i][1]) for i in range(pi.m)])


def decision_dict(d: Decision) -> dict:
    if d.status == NO_CAPACITY:
        return dict(status="no_capacity", raw=0, distinct=0, leaves=0, key=0)
    devs = []
    m = d.device_mask
    while m:
        low = m & -m
        devs.append(low.bit_length() - 1)
        m ^= low
    k, used = d.k, d.used
    return dict(status="ok", devices=tuple(devs), mapping=tuple(d.mapping[:k]),
                used_edges=[(used[i][0], used[i][1]) for i in range(d.m)],
                x=d.x, y=d.y, z=d.z, agg_bw=d.agg_bw, preserved_bw=d.preserved_bw,
                pred_effbw=d.pred_effbw, score=d.score, raw=int(d.raw_embeddings),
                distinct=int(d.distinct_matches), leaves=int(d.leaves_scored), key=int(d.key),
                ecode=(int(d.ecode[0]) << 64) | int(d.ecode[1]))


def _flags(raw: bool, prune: bool = False, deep: bool = False) -> int:
    return (F_RAW if raw else 0) | (F_PRUNE if prune else 0) | (F_DEEP if deep else 0)


_tls = __import__("threading").local()


def _decision_buf() -> Decision:
    """Per-thread reusable output struct (mapa_allocate overwrites it whole)."""
    d = getattr(_tls, "decision", None)
    if d is None:
        d = _tls.decision = Decision()
    return d


def allocate(topo: Topology, pat: Pattern, selector: int, sensitive: bool = False, raw: bool = False,
             commit: bool = False, stream=None, prune: bool = False, deep: bool = False) -> dict:
    """mapa_allocate: one allocation end to end from host buffers (H2D query,
    kernel, D2H record, host decode).  prune = MAPA_F_PRUNE (branch and bound,
    same decision, fewer leaves scored); deep = MAPA_F_DEEP (the wide-key
    kernel even when the narrow one fits; patterns with k > 8 always take it)."""
    d = _decision_buf()
    flags = _flags(raw, prune, deep) | (F_COMMIT if commit else 0)
    _check(_lib.mapa_allocate(topo.handle, pat.handle, selector, int(bool(sensitive)), flags,
                              _stream_ptr(stream), ctypes.byref(d)), allow_no_capacity=True)
    return decision_dict(d)


def allocate_many(topo: Topology, queries, raw: bool = False, stream=None, prune: bool = False,
                  deep: bool = False) -> list[dict]:
    """mapa_allocate_many: independent allocations [(pattern, selector,
    sensitive)] on the topology's current state in one call (one graph: one
    H2D copy, parallel launches, one D2H copy, host decode); never commits."""
    n = len(queries)
    arr = (_vp * n)(*[q[0].handle for q in queries])
    sel = (ctypes.c_int32 * n)(*[q[1] for q in queries])
    sen = (ctypes.c_int32 * n)(*[int(bool(q[2])) for q in queries])
    out = (Decision * n)()
    _check(_lib.mapa_allocate_many(topo.handle, arr, n, sel, sen, _flags(raw, prune, deep), _stream_ptr(stream), out))
    return [decision_dict(out[i]) for i in range(n)]


def launch_query(topo: Topology, pat: Pattern, selector: int, sensitive: bool, d_query_ptr: int,
                 d_record_ptr: int, raw: bool = False, rank: int = 0, world: int = 1,
                 busy_hint: int = (1 << 64) - 1, stream=None, prune: bool = False, zeroed: bool = False):
    """mapa_launch_query: device-resident launch (asynchronous); zeroed =
    MAPA_F_ZEROED (the caller already zeroed the record on `stream`)."""
    _check(_lib.mapa_launch_query(topo.handle, pat.handle, selector, int(bool(sensitive)), d_query_ptr,
                                  d_record_ptr, _flags(raw, prune) | (F_ZEROED if zeroed else 0), rank, world,
                                  busy_hint, _stream_ptr(stream)))


def launch_query_wide(topo: Topology, pat: Pattern, selector: int, sensitive: bool, d_query_ptr: int,
                      d_record_ptr: int, busy: int, raw: bool = False, rank: int = 0, world: int = 1, stream=None,
                      prune: bool = False):
    """mapa_launch_query_wide: deep-path device-resident launch (asynchronous);
    d_query_ptr -> mapa_query64; busy must equal its busy mask (it sizes the
    suffix tables)."""
    _check(_lib.mapa_launch_query_wide(topo.handle, pat.handle, selector, int(bool(sensitive)), d_query_ptr,
                                       d_record_ptr, _flags(raw, prune), rank, world, busy, _stream_ptr(stream)))


def reduce_wide_records(records) -> WideRecord:
    arr = (WideRecord * len(records))(*records)
    out = WideRecord()
    _check(_lib.mapa_reduce_wide_records(arr, len(records), ctypes.byref(out)))
    return out


def decode_wide(topo: Topology, pat: Pattern, busy: int, selector: int, sensitive: bool, record: WideRecord,
                raw: bool = False, prune: bool = False) -> dict:
    d = Decision()
    _check(_lib.mapa_decode_wide(topo.handle, pat.handle, busy, selector, int(bool(sensitive)), _flags(raw, prune),
                                 ctypes.byref(record), ctypes.byref(d)), allow_no_capacity=True)
    return decision_dict(d)


def launch_queries(topo: Topology, pats, rows, d_queries_ptr: int, d_records_ptr: int, raw: bool = False,
                   nstreams: int = 8, stream=None):
    """mapa_launch_queries: independent full-GPU single-query launches for
    rows [(busy, pattern index, selector, sensitive)] over `nstreams`
    internal streams, ordered like one launch on `stream` (asynchronous)."""
    arr = (_vp * len(pats))(*[p.handle for p in pats])
    hq = (Query * max(1, len(rows)))(*[Query(b & 0xFFFFFFFF, pi, sel, int(bool(sens))) for b, pi, sel, sens in rows])
    _check(_lib.mapa_launch_queries(topo.handle, arr, len(pats), len(rows), hq, d_queries_ptr, d_records_ptr,
                                    F_RAW if raw else 0, nstreams, _stream_ptr(stream)))


def record_from_bytes(b: bytes) -> Record:
    return Record.from_buffer_copy(b)


def reduce_records(records) -> Record:
    arr = (Record * len(records))(*records)
    out = Record()
    _check(_lib.mapa_reduce_records(arr, len(records), ctypes.byref(out)))
    return out


def decode(topo: Topology, pat: Pattern, busy: int, selector: int, sensitive: bool, record: Record,
           raw: bool = False, prune: bool = False) -> dict:
    d = Decision()
    _check(_lib.mapa_decode(topo.handle, pat.handle, busy, selector, int(bool(sensitive)),
                            _flags(raw, prune), ctypes.byref(record), ctypes.byref(d)), allow_no_capacity=True)
    return decision_dict(d)


def allocate_batch(topo: Topology, pats, nq: int, d_queries_ptr: int, d_results_ptr: int, d_scratch_ptr: int,
                   raw: bool = False, stream=None):
    arr = (_vp * len(pats))(*[p.handle for p in pats])
    _check(_lib.mapa_allocate_batch(topo.handle, arr, len(pats), nq, d_queries_ptr, d_results_ptr,
                                    d_scratch_ptr, F_RAW if raw else 0, _stream_ptr(stream)))


def shard_queries(topo: Topology, pats, rows, world: int, raw: bool = False):
    """mapa_shard_queries: LPT deal of batch queries rows [(busy, pattern
    index, selector, sensitive)] over `world` ranks -> (owner per query, load
    per rank in leaves)."""
    arr = (_vp * len(pats))(*[p.handle for p in pats])
    hq = (Query * max(1, len(rows)))(*[Query(b & 0xFFFFFFFF, pi, sel, int(bool(sens))) for b, pi, sel, sens in rows])
    own = (ctypes.c_int32 * max(1, len(rows)))()
    ld = (ctypes.c_double * world)()
    _check(_lib.mapa_shard_queries(topo.handle, arr, len(pats), len(rows), hq, F_RAW if raw else 0, world, own, ld))
    return list(own)[:len(rows)], list(ld)


def trace_replay(topo: Topology, pats, ntraces: int, nops: int, d_ops_ptr: int, njobs: int, d_jobs_ptr: int,
                 d_keys_ptr: int, raw: bool = False, stream=None):
    arr = (_vp * len(pats))(*[p.handle for p in pats])
    _check(_lib.mapa_trace_replay(topo.handle, arr, len(pats), ntraces, nops, d_ops_ptr, njobs, d_jobs_ptr,
                                  d_keys_ptr, F_RAW if raw else 0, _stream_ptr(stream)))


def decode_trace(topo: Topology, pats, ops, jobs, keys, raw: bool = False) -> list[dict]:
    """mapa_decode_trace: one replayed trace's keys -> full decisions (job
    order).  ops [(op, job)], jobs [(pattern index, selector, sensitive)],
    keys = the trace's njobs keys (ints)."""
    arr = (_vp * len(pats))(*[p.handle for p in pats])
    o = (TraceOp * max(1, len(ops)))(*[TraceOp(a, b) for a, b in ops])
    q = (Query * max(1, len(jobs)))(*[Query(0, pi, sel, int(bool(sens))) for pi, sel, sens in jobs])
    ky = (ctypes.c_uint64 * max(1, len(keys)))(*[k & ((1 << 64) - 1) for k in keys])
    out = (Decision * max(1, len(jobs)))()
    _check(_lib.mapa_decode_trace(topo.handle, arr, len(pats), len(ops), o, len(jobs), q, ky, F_RAW if raw else 0,
                                  out))
    return [decision_dict(out[i]) for i in range(len(jobs))]


# ------------------------------------------------------------------ simulator

def fifo_schedule(n_devices: int, ks, durations, arrivals=None):
    """mapa_fifo_schedule: strict-FIFO (op, job) order and start / end times."""
    n = len(ks)
    K = (ctypes.c_int32 * max(1, n))(*ks)
    Dd = (ctypes.c_double * max(1, n))(*durations)
    Aa = (ctypes.c_double * max(1, n))(*(arrivals if arrivals is not None else [0.0] * n))
    ops = (TraceOp * max(1, 2 * n))()
    st = (ctypes.c_double * max(1, n))()
    en = (ctypes.c_double * max(1, n))()
    _check(_lib.mapa_fifo_schedule(n_devices, n, K, Dd, Aa, ops, st, en))
    return [(ops[i].op, ops[i].job) for i in range(2 * n)], list(st)[:n], list(en)[:n]


def simulate(topo: Topology, pats, jobs, policy: str, raw: bool = False, stream=None):
    """mapa_simulate (SPEC run_simulation): jobs = [(pattern_index, sensitive,
    duration[, arrival])]; returns one log dict per job (job order)."""
    arr = (_vp * len(pats))(*[p.handle for p in pats])
    js = (Job * max(1, len(jobs)))(*[Job(j[0], int(bool(j[1])), float(j[2]), float(j[3]) if len(j) > 3 else 0.0)
                                     for j in jobs])
    out = (JobLog * max(1, len(jobs)))()
    _check(_lib.mapa_simulate(topo.handle, arr, len(pats), len(jobs), js, POLICIES[policy],
                              F_RAW if raw else 0, _stream_ptr(stream), out))
    res = []
    for i in range(len(jobs)):
        L = out[i]
        res.append(dict(job=L.job, k=L.k, devices=tuple(d for d in range(32) if (L.device_mask >> d) & 1),
                        x=L.x, y=L.y, z=L.z, agg_bw=L.agg_bw, preserved_bw=L.preserved_bw,
                        pred_effbw=L.pred_effbw, arrival=L.arrival, start=L.start, end=L.end, wait=L.wait))
    return res


def quantiles(values):
    """mapa_quantiles: (min, p25, p50, p75, max), linear interpolation (type 7)."""
    v = (ctypes.c_double * max(1, len(values)))(*values)
    out = (ctypes.c_double * 5)()
    _check(_lib.mapa_quantiles(v, len(values), out))
    return tuple(out)


def summarize(records, group_by=None):
    """SPEC summarize_log: per group the five quantiles of
    pred_effbw and of wait, the makespan and the job count."""
    groups = {}
    for r in records:
        groups.setdefault(r[group_by] if group_by else "all", []).append(r)
    return {g: dict(pred_effbw=quantiles([r["pred_effbw"] for r in rs]), wait=quantiles([r["wait"] for r in rs]),
                    makespan=max(r["end"] for r in rs), jobs=len(rs)) for g, rs in groups.items()}
