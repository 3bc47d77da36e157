"""torch plumbing around the C-ABI: device buffers, streams, torch.distributed.

PyTorch supplies device memory (tensors whose data_ptr() go to the C-ABI),
the CUDA stream, and the process group.  Nothing here computes any part of
the method.

Multi-GPU: one process per GPU.  A single large query is
sharded by work item (item i goes to rank i % world); every rank produces a
32-byte record {key, leaves}; the records are exchanged with ONE
all_gather over NCCL (NVLink/NVSwitch) and combined by max(key) / sum(leaves)
(mapa_reduce_records); every rank decodes the same key, so no broadcast is
needed and the decision is identical for any world size.
Batches shard queries with no data-path collective ("weak" scaling).
"""
from __future__ import annotations

import struct

import torch
import torch.distributed as dist

from . import (Pattern, Record, Topology, WideRecord, decode, decode_wide, launch_query, launch_queries, launch_query_wide,
               allocate_batch, reduce_records, reduce_wide_records, shard_queries, trace_replay, SEL_PRESERVE)

U32 = 0xFFFFFFFF


def _i32(v: int) -> int:
    v &= U32
    return v - (1 << 32) if v >= (1 << 31) else v


def query_tensor(busy: int, pattern: int = 0, selector: int = 0, sensitive: bool = False, device="cuda"):
    """One mapa_query (16 B) as an int32[4] tensor."""
    return torch.tensor([_i32(busy), pattern, selector, int(bool(sensitive))], dtype=torch.int32, device=device)


def queries_tensor(queries, device="cuda"):
    """[(busy, pattern, selector, sensitive), ...] -> int32[nq, 4]."""
    rows = [[_i32(b), p, s, int(bool(t))] for b, p, s, t in queries]
    return torch.tensor(rows, dtype=torch.int32, device=device).reshape(-1, 4)


def records_from_tensor(t: torch.Tensor):
    """int64[..., 4] (32 B rows) -> list[Record]."""
    raw = t.detach().cpu().contiguous().numpy().tobytes()
    return [Record.from_buffer_copy(raw[i:i + 32]) for i in range(0, len(raw), 32)]


def record_tensor(rec: Record, device="cpu"):
    return torch.tensor(list(struct.unpack("<4q", bytes(rec))), dtype=torch.int64, device=device)


def run_query(topo: Topology, pat: Pattern, selector: int, sensitive: bool, busy: int, raw: bool = False,
              rank: int = 0, world: int = 1, stream=None, prune: bool = False):
    """Launch one (shard of a) query on the current device; returns the record
    tensor (int64[4], device) without synchronising."""
    q = query_tensor(busy, 0, selector, sensitive)
    rec = torch.empty(4, dtype=torch.int64, device="cuda")
    launch_query(topo, pat, selector, sensitive, q.data_ptr(), rec.data_ptr(), raw=raw, rank=rank, world=world,
                 busy_hint=busy, stream=stream, prune=prune)
    return rec, q


def run_queries(topo: Topology, pats, rows, raw: bool = False, nstreams: int = 8, stream=None):
    """Independent single-query launches (the full GPU per query) through ONE
    mapa_launch_queries call: the library spreads them over `nstreams`
    internal streams so small queries' launch / drain overlap, ordered like a
    single launch on `stream`.  rows: [(busy, pattern index, selector,
    sensitive)].  Returns int64[nq, 4] records (device) without synchronising."""
    cur = stream or torch.cuda.current_stream()
    q = queries_tensor(rows, device=cur.device)
    recs = torch.empty((max(1, len(rows)), 4), dtype=torch.int64, device=cur.device)
    launch_queries(topo, pats, rows, q.data_ptr(), recs.data_ptr(), raw=raw, nstreams=nstreams, stream=cur)
    return recs[:len(rows)]


def gather_records(rec: torch.Tensor, width: int, group=None) -> torch.Tensor:
    """The one collective of a sharded allocation: all_gather every rank's
    record (`width` int64 words: 4 narrow, 8 deep) -> int64[world, width].
    NCCL: device tensors, all_gather_into_tensor (NVLink / NVSwitch); gloo (the
    CPU tests of the multi-rank path): host tensors."""
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world, width), dtype=torch.int64, device=rec.device)
        dist.all_gather_into_tensor(out, rec.reshape(width), group=group)
        return out
    parts = [torch.empty(width, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, rec.reshape(width).cpu(), group=group)
    return torch.stack(parts)


def combine_records(rec: torch.Tensor, group=None) -> Record:
    """all_gather the per-rank 32-B records (one collective) and combine them
    by max(key), sum(leaves) on the host."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return records_from_tensor(rec)[0]
    return reduce_records(records_from_tensor(gather_records(rec, 4, group)))


def allocate_sharded(topo: Topology, pat: Pattern, selector: int, sensitive: bool, busy: int, raw: bool = False,
                     group=None, prune: bool = False) -> dict:
    """Sharded single allocation over the process group (one rank per GPU)."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rec, _q = run_query(topo, pat, selector, sensitive, busy, raw=raw, rank=rank, world=world, prune=prune)
    r = combine_records(rec, group)
    return decode(topo, pat, busy, selector, sensitive, r, raw=raw, prune=prune)


def wide_records_from_tensor(t: torch.Tensor):
    """int64[..., 8] (64 B rows) -> list[WideRecord]."""
    raw = t.detach().cpu().contiguous().numpy().tobytes()
    return [WideRecord.from_buffer_copy(raw[i:i + 64]) for i in range(0, len(raw), 64)]


def wide_record_tensor(rec: WideRecord, device="cpu"):
    return torch.tensor(list(struct.unpack("<8q", bytes(rec))), dtype=torch.int64, device=device)


def _i64(v: int) -> int:
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def query64_tensor(busy: int, selector: int = 0, sensitive: bool = False, device="cuda"):
    """One mapa_query64 (16 B: u64 busy, i32 selector, i32 sensitive) as int64[2]."""
    return torch.tensor([_i64(busy), _i64(selector | (int(bool(sensitive)) << 32))], dtype=torch.int64,
                        device=device)


def run_query_wide(topo: Topology, pat: Pattern, selector: int, sensitive: bool, busy: int, raw: bool = False,
                   rank: int = 0, world: int = 1, stream=None, prune: bool = False):
    """Deep path: launch one (shard of a) query; returns the 64-B record tensor
    (int64[8], device) without synchronising."""
    q = query64_tensor(busy, selector, sensitive)
    rec = torch.empty(8, dtype=torch.int64, device="cuda")
    launch_query_wide(topo, pat, selector, sensitive, q.data_ptr(), rec.data_ptr(), busy, raw=raw, rank=rank,
                      world=world, stream=stream, prune=prune)
    return rec, q


def combine_wide_records(rec: torch.Tensor, group=None) -> WideRecord:
    """all_gather the per-rank 64-B deep records (one collective), combine by
    the lexicographic max of the 256-bit key and the sum of leaves."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return wide_records_from_tensor(rec)[0]
    return reduce_wide_records(wide_records_from_tensor(gather_records(rec, 8, group)))


def allocate_sharded_wide(topo: Topology, pat: Pattern, selector: int, sensitive: bool, busy: int,
                          raw: bool = False, group=None, prune: bool = False) -> dict:
    """Deep-path sharded single allocation over the process group (prune =
    MAPA_F_PRUNE: each rank's branch and bound, same combined decision)."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rec, _q = run_query_wide(topo, pat, selector, sensitive, busy, raw=raw, rank=rank, world=world, prune=prune)
    r = combine_wide_records(rec, group)
    return decode_wide(topo, pat, busy, selector, sensitive, r, raw=raw, prune=prune)


def shard_rows(topo: Topology, pats, rows, raw: bool = False, group=None):
    """This rank's share of a multi-GPU batch: the library's LPT deal
    (mapa_shard_queries, identical on every rank) -> (indices, rows) owned by
    this rank.  No collective: each rank runs its own queries."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    owner, _ = shard_queries(topo, pats, rows, world, raw=raw)
    idx = [i for i, o in enumerate(owner) if o == rank]
    return idx, [rows[i] for i in idx]


def run_batch(topo: Topology, pats, queries, raw: bool = False, stream=None):
    """queries: int32[nq,4] device tensor -> int64[nq,4] device records."""
    nq = queries.shape[0]
    res = torch.empty((max(nq, 1), 4), dtype=torch.int64, device=queries.device)
    scratch = torch.empty(64 + (nq + 1) // 2, dtype=torch.int64, device=queries.device)  # >= 512 + 4 nq bytes
    allocate_batch(topo, pats, nq, queries.data_ptr(), res.data_ptr(), scratch.data_ptr(), raw=raw, stream=stream)
    return res[:nq]


def run_trace(topo: Topology, pats, ops, jobs, raw: bool = False, stream=None):
    """ops: int32[ntraces, nops, 2] device; jobs: int32[ntraces, njobs, 4] device
    -> int64[ntraces, njobs] keys (device)."""
    ntr, nops = ops.shape[0], ops.shape[1]
    njobs = jobs.shape[1]
    keys = torch.empty((ntr, njobs), dtype=torch.int64, device=ops.device)
    trace_replay(topo, pats, ntr, nops, ops.data_ptr(), njobs, jobs.data_ptr(), keys.data_ptr(), raw=raw,
                 stream=stream)
    return keys


def is_sensitive_selector(selector: int, sensitive: bool) -> bool:
    return selector == SEL_PRESERVE and bool(sensitive)
