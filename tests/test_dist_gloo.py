"""Multi-rank path on CPU (gloo, world_size 2): each rank holds the record of
its shard of the enumeration, the records are exchanged with one all_gather
(paper_2110_03214_b200.dist.combine_records, the same call the NCCL path
uses), combined (mapa_reduce_records) and decoded (mapa_decode); every rank
must obtain the unsharded oracle decision.  Shard records are built from the
oracle restricted to the rank's subsets (units S[0] in a contiguous range),
encoded with the key definition of include/mapa.h."""
import os
import socket

import pytest
import torch.multiprocessing as tmp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, cases, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from oracle import coracle as co
    from oracle import mapa_oracle as mo
    from tests.keyutil import encode_key, selector_score
    import paper_2110_03214_b200 as mp
    from paper_2110_03214_b200 import dist as md

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    results = []
    for name, busy, shape, k, sel, sens in cases:
        o = mo.builtin(name)
        kk, e = mo.make_pattern(shape, k)
        nf = o.n - bin(busy).count("1")
        units = nf - k + 1
        half = (units + 1) // 2
        lo, hi = (0, half) if rank == 0 else (half, units)
        part = co.allocate(o, busy, kk, e, sel, sens, nthreads=2, a_lo=lo, a_hi=hi)
        t = mp.Topology(name)
        tab = mp.effbw_rank_table(len(e))
        if part["status"] == "ok":
            key = encode_key(part, selector_score(part, sel, sens, tab, len(e)), t.width, k)
        else:
            key = 0
        rec = md.record_tensor(mp.Record(key=key, leaves=part["distinct"]))
        comb = md.combine_records(rec)
        got = mp.decode(t, mp.Pattern.make(shape, k), busy, sel, sens, comb)
        results.append(got)
    out_q.put((rank, results))
    dist.barrier()
    dist.destroy_process_group()


CASES = [("dgx1v", 0, "ring", 3, 0, False), ("dgx1v", 0b00010010, "tree", 4, 1, True),
         ("cubemesh16", 0x0F0F, "full", 4, 1, False), ("summit", 0, "ring", 2, 1, True),
         ("dgx1p", 0b10000001, "ringtree", 5, 0, False), ("torus2d16", 0xF00F, "ring", 4, 1, False)]


def test_two_rank_combine_matches_unsharded_oracle():
    from oracle import coracle as co
    from oracle import mapa_oracle as mo

    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, CASES, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (name, busy, shape, k, sel, sens) in enumerate(CASES):
        o = mo.builtin(name)
        kk, e = mo.make_pattern(shape, k)
        exp = co.allocate(o, busy, kk, e, sel, sens)
        for r in range(WORLD):
            g = got[r][i]
            for f in ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "distinct"):
                assert g[f] == exp[f], (name, r, f, g[f], exp[f])


def _worker_wide(rank, port, cases, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import math as _m

    import torch.distributed as dist

    from oracle import coracle as co
    from oracle import mapa_oracle as mo
    from tests.keyutil import encode_wide_key, selector_score
    import paper_2110_03214_b200 as mp
    from paper_2110_03214_b200 import dist as md

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    results = []
    for name, busy, shape, k, sel, sens in cases:
        o = mo.builtin(name)
        kk, e = mo.make_pattern(shape, k)
        nf = o.n - bin(busy).count("1")
        nsub = _m.comb(nf, k)
        half = (nsub + 1) // 2
        lo, hi = (0, half) if rank == 0 else (half, nsub)
        part = co.allocate_deep(o, busy, kk, e, sel, sens, nthreads=2, sub_lo=lo, sub_hi=hi)
        t = mp.Topology(name)
        tab = mp.effbw_rank_table(len(e))
        if part["status"] == "ok":
            sc, st, eh, el = encode_wide_key(part, selector_score(part, sel, sens, tab, len(e)), k)
        else:
            sc = st = eh = el = 0
        rec = md.wide_record_tensor(mp.WideRecord(score=sc, set=st, ecode_hi=eh, ecode_lo=el, leaves=part["raw"]))
        comb = md.combine_wide_records(rec)
        got = mp.decode_wide(t, mp.Pattern.make(shape, k), busy, sel, sens, comb, raw=True)
        results.append(got)
    out_q.put((rank, results))
    dist.barrier()
    dist.destroy_process_group()


WIDE_CASES = [("cubemesh16", 0b0110000000100100, "ring", 10, 0, False),          # 11 free: 11 x 10!
              ("torus2d16", 0b1000010000010010, "tree", 9, 1, True),            # 11 free: C(11,9) x 9!
              ("cubemesh16", 0b0001000100010001, "ringtree", 9, 1, False),      # 12 free
              ("dgx1v", 0b00100000, "full", 5, 0, False)]


def test_two_rank_wide_combine_matches_unsharded_deep_oracle():
    """Deep path (256-bit keys): the same exchange with 64-B wide records
    (dist.combine_wide_records -> mapa_reduce_wide_records -> mapa_decode_wide)."""
    from oracle import coracle as co
    from oracle import mapa_oracle as mo

    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_wide, args=(r, port, WIDE_CASES, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=400) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (name, busy, shape, k, sel, sens) in enumerate(WIDE_CASES):
        o = mo.builtin(name)
        kk, e = mo.make_pattern(shape, k)
        exp = co.allocate_deep(o, busy, kk, e, sel, sens)
        for r in range(WORLD):
            g = got[r][i]
            for f in ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "raw"):
                assert g[f] == exp[f], (name, r, f, g[f], exp[f])


def _worker_shard(rank, port, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import workloads as W
    import paper_2110_03214_b200 as mp
    from paper_2110_03214_b200 import dist as md

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    t = mp.Topology(text=W.het32_text())
    shapes = [(s, k) for s in ("ring", "tree", "full") for k in range(2, 6)]
    pats = [mp.Pattern.make(s, k) for s, k in shapes]
    pid = {sk: i for i, sk in enumerate(shapes)}
    rows = [(q["busy"], pid[(q["shape"], q["k"])], q["selector"], q["sensitive"])
            for q in W.c5_queries(32, count=3000, seed=11)]
    idx, mine = md.shard_rows(t, pats, rows, raw=True)
    assert mine == [rows[i] for i in idx]
    out_q.put((rank, idx))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_batch_lpt_deal_partitions_the_queries():
    """Multi-GPU batches: every rank calls dist.shard_rows (the
    library's LPT deal, no collective) on the same rows; the two ranks' query
    sets are disjoint, cover the batch, and their work differs by at most the
    largest query."""
    import math

    import workloads as W

    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_shard, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = set(got[0]), set(got[1])
    assert not a & b and a | b == set(range(3000))
    qs = W.c5_queries(32, count=3000, seed=11)
    work = [math.perm(32 - bin(x["busy"]).count("1"), x["k"]) for x in qs]
    assert abs(sum(work[i] for i in a) - sum(work[i] for i in b)) <= max(work)
