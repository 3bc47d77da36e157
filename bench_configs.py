"""Secondary bench modes (`bench.py --config c1|c2|c3|c5`): measurements of the
SURVEY.md §8(d) configs other than the headline C4.  Same timing rules as
bench.py (warm-up, CUDA events on the launching stream, max over ranks);
multi-rank runs are replicas / query shards with no data-path collective.

  c1  dgx1v ring-3 all free: end-to-end latency of mapa_allocate (median of
      per-call wall time) and device throughput of 1e5 identical batched queries
  c2  dgx1p + summit 1000-job FIFO traces replayed on the device, R replicas
      (one CTA each) per (topology, policy)
  c3  cubemesh16 {ring,tree,full} x k in {4,6,8} random-busy queries, one
      single-query launch each (the full GPU per query)
  c5  1e5 random queries per topology (cubemesh16, het32) in one batch launch
All modes score every injective embedding (RAW mode)."""
from __future__ import annotations

import math
import statistics
import time

import workloads as W

SHAPE_K = [(s, k) for s in ("ring", "tree", "full") for k in range(2, 6)]


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _timed(torch, stream, fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        a, b = _events(torch)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot  # ms


def _base(cfg, world, steps, warmup):
    return {"config_id": cfg, "n_gpus": world, "steps": steps, "warmup": warmup, "higher_is_better": True,
            "dtype": "int32", "data": "synthetic"}


def run_config(args, mp, md, torch, dev, stream, rank, world, max_over_ranks):
    steps, warmup = args.steps, max(args.warmup, 3)
    if args.config == "c1":
        topo = mp.Topology("dgx1v")
        pat = mp.Pattern.make("ring", 3)
        lat = {}
        for sel, sens, name in ((0, False, "greedy"), (1, True, "sensitive"), (1, False, "insensitive")):
            for _ in range(20):
                mp.allocate(topo, pat, sel, sens, raw=True)
            ts = []
            for _ in range(500):
                t0 = time.perf_counter()
                d = mp.allocate(topo, pat, sel, sens, raw=True)
                ts.append(time.perf_counter() - t0)
            assert d["devices"] == (0, 2, 3) and d["raw"] == 336
            lat[name] = statistics.median(ts) * 1e6
        B = 100_000
        rows = [(0, 0, [0, 1, 1][i % 3], [0, 1, 0][i % 3]) for i in range(B)]
        q = md.queries_tensor(rows, device=dev)
        pats = [pat]
        ms = _timed(torch, stream, lambda: md.run_batch(topo, pats, q, raw=True, stream=stream), steps, warmup)
        ms = max_over_ranks(ms)
        allocs = B * steps * world / (ms / 1e3)
        line = _base("c1", world, steps, warmup)
        line.update(metric="allocations/sec (C1: dgx1v ring-3, all free)", value=allocs, unit="allocations/s",
                    embeddings_per_s=allocs * 336, batch=B, e2e_latency_us_median=lat,
                    config={"workload": "C1 dgx1v ring-3 all free; 1e5 identical queries per batch launch "
                                        "(selectors rotate); latency = one mapa_allocate call"})
        return line

    if args.config == "c2":
        R = 296
        res = {}
        total_allocs = total_emb = 0
        total_ms = 0.0
        for tname in ("dgx1p", "summit"):
            n = 8 if tname == "dgx1p" else 6
            topo = mp.Topology(tname)
            pats = [mp.Pattern.make(s, k) for s, k in SHAPE_K]
            pid = {sk: i for i, sk in enumerate(SHAPE_K)}
            for policy in ("preserve", "greedy"):
                ops_all, jobs_all, emb = [], [], 0
                for r in range(R):
                    seed = 2110 + 1000 * rank + r
                    jobs = W.c2_jobs(seed, 1000)
                    ops = W.fifo_ops(jobs, n)
                    free = n
                    for o, j in ops:  # embeddings scored per ALLOC = P(|F|, k) (count only)
                        if o == W.OP_ALLOC:
                            emb += math.perm(free, jobs[j]["k"])
                            free -= jobs[j]["k"]
                        else:
                            free += jobs[j]["k"]
                    ops_all.append([[o, j] for o, j in ops])
                    jobs_all.append([[0, pid[(j["shape"], j["k"])], 1 if policy == "preserve" else 0,
                                      j["sensitive"] if policy == "preserve" else 0] for j in jobs])
                dops = torch.tensor(ops_all, dtype=torch.int32, device=dev)
                djobs = torch.tensor(jobs_all, dtype=torch.int32, device=dev)
                ms = _timed(torch, stream, lambda: md.run_trace(topo, pats, dops, djobs, raw=True, stream=stream),
                            max(1, steps // 10), warmup)
                per = ms / max(1, steps // 10)
                res[f"{tname}/{policy}"] = {"ms_per_launch": per, "allocations_per_s": R * 1000 / (per / 1e3)}
                total_allocs += R * 1000
                total_emb += emb
                total_ms += per
        total_ms = max_over_ranks(total_ms)
        line = _base("c2", world, max(1, steps // 10), warmup)
        line.update(metric="allocations/sec (C2: 1000-job FIFO traces replayed on device)",
                    value=total_allocs * world / (total_ms / 1e3), unit="allocations/s",
                    embeddings_per_s=total_emb * world / (total_ms / 1e3), per_case=res, replicas_per_case=R,
                    scaling="weak",
                    config={"workload": "C2 dgx1p + summit, 1000 jobs (k U{2..5}, shape U{ring,tree,full}), "
                                        f"{R} replica traces per (topology, policy), one CTA per trace"})
        return line

    if args.config == "c3":
        per_case = 50
        qs = W.c3_queries(per_case=per_case)
        qs = qs[rank::world]
        topo = mp.Topology("cubemesh16")
        pats = {(s, k): mp.Pattern.make(s, k) for s in ("ring", "tree", "full") for k in (4, 6, 8)}
        qt = md.queries_tensor([(q["busy"], 0, q["selector"], q["sensitive"]) for q in qs], device=dev)
        recs = torch.empty((len(qs), 4), dtype=torch.int64, device=dev)
        emb = sum(math.perm(16 - bin(q["busy"]).count("1"), q["k"]) for q in qs
                  if q["k"] <= 16 - bin(q["busy"]).count("1"))

        def run():
            for i, q in enumerate(qs):
                mp.launch_query(topo, pats[(q["shape"], q["k"])], q["selector"], q["sensitive"],
                                qt[i].data_ptr(), recs[i].data_ptr(), raw=True, busy_hint=q["busy"], stream=stream)

        ms = _timed(torch, stream, run, max(1, steps // 10), warmup)
        ms = max_over_ranks(ms / max(1, steps // 10))
        line = _base("c3", world, max(1, steps // 10), warmup)
        line.update(metric="embeddings/sec (C3: cubemesh16, k in {4,6,8}, random busy)", value=emb * world / (ms / 1e3),
                    unit="embeddings/s", allocations_per_s=len(qs) * world / (ms / 1e3), queries=len(qs) * world,
                    scaling="weak",
                    config={"workload": f"C3 cubemesh16 {{ring,tree,full}} x k {{4,6,8}}, {per_case} queries per case, "
                                        "one single-query launch each"})
        return line

    if args.config == "c5":
        res = {}
        tot_emb = tot_q = 0
        tot_ms = 0.0
        for tname in ("cubemesh16", "het32"):
            n = 16 if tname == "cubemesh16" else 32
            topo = mp.Topology(tname) if tname == "cubemesh16" else mp.Topology(text=W.het32_text())
            qs = W.c5_queries(n, count=100_000)[rank::world]
            pats = [mp.Pattern.make(s, k) for s, k in SHAPE_K]
            pid = {sk: i for i, sk in enumerate(SHAPE_K)}
            qt = md.queries_tensor([(q["busy"], pid[(q["shape"], q["k"])], q["selector"], q["sensitive"])
                                    for q in qs], device=dev)
            emb = sum(math.perm(n - bin(q["busy"]).count("1"), q["k"]) for q in qs)
            ms = _timed(torch, stream, lambda: md.run_batch(topo, pats, qt, raw=True, stream=stream),
                        max(1, steps // 10), warmup) / max(1, steps // 10)
            res[tname] = {"ms_per_batch": ms, "queries": len(qs), "embeddings": emb,
                          "embeddings_per_s": emb / (ms / 1e3), "allocations_per_s": len(qs) / (ms / 1e3)}
            tot_emb += emb
            tot_q += len(qs)
            tot_ms += ms
        tot_ms = max_over_ranks(tot_ms)
        line = _base("c5", world, max(1, steps // 10), warmup)
        line.update(metric="embeddings/sec (C5: 1e5 batched random queries per topology)",
                    value=tot_emb * world / (tot_ms / 1e3), unit="embeddings/s",
                    allocations_per_s=tot_q * world / (tot_ms / 1e3), per_topology=res, scaling="weak",
                    config={"workload": "C5 cubemesh16 + het32, 1e5 queries each (k U{2..5}, shape U{ring,tree,full}, "
                                        "busy U{0..N-k}, selector U{3}), one batch launch per topology, queries "
                                        "sharded across ranks"})
        return line
    return None
