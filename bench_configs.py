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


def _peak_gops():
    """148 SMs x the measured issue rate (lane-instructions per SM per clock,
    profiles/r02_int_peaks.json: IADD3 + IMAD 1:1) x the measured max SM clock."""
    import json
    import os
    root = os.path.dirname(os.path.abspath(__file__))
    lanes, mhz = 128.0, 1965.0
    try:
        d = json.load(open(os.path.join(root, "profiles", "r02_int_peaks.json")))
        lanes = {r["op"]: r["lane_ops_per_sm_per_clk"] for r in d["results"]}["IADD3+IMAD (1:1)"]
    except Exception:
        pass
    try:
        mhz = json.load(open(os.path.join(root, "MEASURED_PEAKS.json"))).get("sm_max_mhz") or mhz
    except Exception:
        pass
    return 148 * lanes * mhz * 1e6 / 1e9


def _traffic(cfg):
    """DRAM bytes per launch of the config's dominant kernel from one ncu
    --set full capture (profiles/ncu_summary.json "config_traffic"), or None."""
    import json
    import os
    try:
        d = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_summary.json")))
        return d.get("config_traffic", {}).get(cfg)
    except Exception:
        return None


PEAK_GOPS = _peak_gops()               # int32 issue roofline
OPS_MIX = (2 + 3 + 2) / 3              # ops/embedding, selectors U{Greedy, Sensitive, Insensitive}


def _roof(emb_per_s, kernel, note="", cfg=None):
    ach = OPS_MIX * emb_per_s / 1e9
    return {"bound": "alu", "kernel": kernel, "achieved": ach, "peak": PEAK_GOPS, "unit": "Gop/s",
            "frac": ach / PEAK_GOPS, "traffic": _traffic(cfg), "ops_per_embedding": OPS_MIX, "note": note}


def _cpu(fn, what):
    """Time the CPU oracle (oracle/, all host threads) on a bounded sample."""
    import os
    t0 = time.perf_counter()
    n_emb, n_alloc = fn()
    dt = time.perf_counter() - t0
    return {"value": n_emb / dt, "unit": "embeddings/s", "allocations_per_s": n_alloc / dt,
            "cores": os.cpu_count(), "kind": "oracle", "sample": what}


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
        if rank == 0:
            from oracle import coracle as co
            from oracle import mapa_oracle as mo
            o = mo.builtin("dgx1v")
            kk, ee = mo.make_pattern("ring", 3)

            def c1_cpu():
                for i in range(600):
                    co.allocate(o, 0, kk, ee, [0, 1, 1][i % 3], [0, 1, 0][i % 3], nthreads=1)
                return 600 * 336, 600
            line["cpu_baseline"] = _cpu(c1_cpu, "600 C1 allocations, C oracle, 1 thread each")
        line["roofline"] = _roof(allocs * 336, "esa_batch<8> (C1 queries)", cfg="c1")
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
        if rank == 0:
            from oracle import coracle as co
            from oracle import mapa_oracle as mo

            def c2_cpu():
                jobs = W.c2_jobs(2110, 1000)
                ops = W.fifo_ops(jobs, 8)
                patd = {(s_, k_): mo.make_pattern(s_, k_) for s_, k_ in SHAPE_K}
                emb, free = 0, 8
                for o_, j in ops:
                    if o_ == W.OP_ALLOC:
                        emb += math.perm(free, jobs[j]["k"])
                        free -= jobs[j]["k"]
                    else:
                        free += jobs[j]["k"]
                mo.replay_trace(mo.builtin("dgx1p"), jobs, ops, patd, "preserve",
                                allocate_fn=lambda t_, b_, k_, e_, s_, x_: co.allocate(t_, b_, k_, e_, s_, x_, nthreads=1))
                return emb, 1000
            line["cpu_baseline"] = _cpu(c2_cpu, "one dgx1p Preserve 1000-job trace replayed by the C oracle")
        line["roofline"] = _roof(total_emb * world / (total_ms / 1e3), "esa_trace<8> / esa_trace<8> (summit)",
                                 "dependent ALLOC/RELEASE chain per CTA: latency-bound, not issue-bound", cfg="c2")
        line.update(metric="allocations/sec (C2: 1000-job FIFO traces replayed on device)",
                    value=total_allocs * world / (total_ms / 1e3), unit="allocations/s",
                    embeddings_per_s=total_emb * world / (total_ms / 1e3), per_case=res, replicas_per_case=R,
                    scaling="weak",
                    config={"workload": "C2 dgx1p + summit, 1000 jobs (k U{2..5}, shape U{ring,tree,full}), "
                                        f"{R} replica traces per (topology, policy), one CTA per trace"})
        return line

    if args.config == "c3":
        per_case = 1000  # 1000 queries per (shape, k)
        allq = W.c3_queries(per_case=per_case)
        topo = mp.Topology("cubemesh16")
        keys = [(s, k) for s in ("ring", "tree", "full") for k in (4, 6, 8)]
        pats = [mp.Pattern.make(s, k) for s, k in keys]
        allrows = [(q["busy"], keys.index((q["shape"], q["k"])), q["selector"], q["sensitive"]) for q in allq]
        idx, rows = md.shard_rows(topo, pats, allrows, raw=True)  # LPT deal over the ranks (no collective)
        qs = [allq[i] for i in idx]
        emb_all = sum(math.perm(16 - bin(q["busy"]).count("1"), q["k"]) for q in allq
                      if q["k"] <= 16 - bin(q["busy"]).count("1"))

        def run():  # md.run_queries: big queries one full-GPU launch each over 8 streams, small ones one batch
            md.run_queries(topo, pats, rows, raw=True, nstreams=8, stream=stream)

        ms = _timed(torch, stream, run, max(1, steps // 10), warmup)
        ms = max_over_ranks(ms / max(1, steps // 10))
        line = _base("c3", world, max(1, steps // 10), warmup)
        if rank == 0:
            from oracle import coracle as co
            from oracle import mapa_oracle as mo
            o = mo.builtin("cubemesh16")
            sample = [q for q in qs if q["k"] <= 6][:24]

            def c3_cpu():
                emb_ = 0
                for q in sample:
                    kk, ee = mo.make_pattern(q["shape"], q["k"])
                    r = co.allocate(o, q["busy"], kk, ee, q["selector"], q["sensitive"])
                    emb_ += r["raw"]
                return emb_, len(sample)
            line["cpu_baseline"] = _cpu(c3_cpu, f"{len(sample)} C3 queries with k <= 6, C oracle, all host threads")
        line["roofline"] = _roof(emb_all / (ms / 1e3), "esa_single<16,K,*> (C3 queries)", cfg="c3")
        line.update(metric="embeddings/sec (C3: cubemesh16, k in {4,6,8}, random busy)", value=emb_all / (ms / 1e3),
                    unit="embeddings/s", allocations_per_s=len(allq) / (ms / 1e3), queries=len(allq),
                    scaling="strong" if world > 1 else "weak",
                    config={"workload": f"C3 cubemesh16 {{ring,tree,full}} x k {{4,6,8}}, {per_case} queries per case "
                                        f"({len(allq)}), LPT-dealt over {world} rank(s); per rank mapa_launch_queries: "
                                        "queries under 2^22 leaves in one batch launch, the rest one full-GPU launch "
                                        "each, over 8 CUDA streams"})
        return line

    if args.config == "c5":
        res = {}
        tot_emb = tot_q = 0
        tot_ms = 0.0
        for tname in ("cubemesh16", "het32"):
            n = 16 if tname == "cubemesh16" else 32
            topo = mp.Topology(tname) if tname == "cubemesh16" else mp.Topology(text=W.het32_text())
            allq = W.c5_queries(n, count=100_000)
            pats = [mp.Pattern.make(s, k) for s, k in SHAPE_K]
            pid = {sk: i for i, sk in enumerate(SHAPE_K)}
            rows = [(q["busy"], pid[(q["shape"], q["k"])], q["selector"], q["sensitive"]) for q in allq]
            # the library's LPT deal (mapa_shard_queries): heaviest queries first, each to the
            # least-loaded rank; no data-path collective
            idx, myrows = md.shard_rows(topo, pats, rows, raw=True)
            qs = [allq[i] for i in idx]
            qt = md.queries_tensor(myrows, device=dev)
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
        if rank == 0:
            from oracle import coracle as co
            from oracle import mapa_oracle as mo
            o32 = mo.parse_topology(W.het32_text())
            sample = W.c5_queries(32, count=100_000)[:40]

            def c5_cpu():
                emb_ = 0
                for q in sample:
                    kk, ee = mo.make_pattern(q["shape"], q["k"])
                    r = co.allocate(o32, q["busy"], kk, ee, q["selector"], q["sensitive"])
                    emb_ += r["raw"]
                return emb_, len(sample)
            line["cpu_baseline"] = _cpu(c5_cpu, "first 40 het32 C5 queries, C oracle, all host threads")
        line["roofline"] = _roof(tot_emb * world / (tot_ms / 1e3), "esa_batch<32> + esa_batch<16>", cfg="c5")
        line.update(metric="embeddings/sec (C5: 1e5 batched random queries per topology)",
                    value=tot_emb * world / (tot_ms / 1e3), unit="embeddings/s",
                    allocations_per_s=tot_q * world / (tot_ms / 1e3), per_topology=res, scaling="weak",
                    config={"workload": "C5 cubemesh16 + het32, 1e5 queries each (k U{2..5}, shape U{ring,tree,full}, "
                                        "busy U{0..N-k}, selector U{3}), one batch launch per topology, queries "
                                        "sharded across ranks"})
        return line

    if args.config == "deep":
        topo = mp.Topology("cubemesh16")
        busy = 0
        sels = ((0, False, "greedy"), (1, True, "preserve_sensitive"), (1, False, "preserve_insensitive"))
        k = 10
        pat = mp.Pattern.make("ring", k)
        per = math.perm(16, k)  # 29,059,430,400 embeddings per allocation
        q = md.query64_tensor(busy, device=dev)
        recs = torch.zeros((3, 8), dtype=torch.int64, device=dev)
        kms = {}
        nsteps = max(3, steps // 5)
        for i, (sel, sens, name) in enumerate(sels):
            def fn(i=i, sel=sel, sens=sens):
                mp.launch_query_wide(topo, pat, sel, sens, q.data_ptr(), recs[i].data_ptr(), busy, raw=True,
                                     rank=rank, world=world, stream=stream)
            kms[name] = max_over_ranks(_timed(torch, stream, fn, nsteps, warmup) / nsteps)
        torch.cuda.synchronize()
        if world == 1:
            for i, (sel, sens, name) in enumerate(sels):
                d = mp.decode_wide(topo, pat, busy, sel, sens, md.wide_records_from_tensor(recs[i])[0], raw=True)
                assert d["raw"] == per, d
        tot = sum(kms.values())
        line = _base("deep", world, nsteps, warmup)
        canon = {}
        if rank == 0 and world == 1:
            for kk in (12, 14):
                p2 = mp.Pattern.make("ring", kk)
                a, b = _events(torch)
                a.record(stream)
                d = mp.allocate(topo, p2, 0, False)
                b.record(stream)
                b.synchronize()
                ms = a.elapsed_time(b)
                canon[f"ring{kk}_greedy"] = {"ms": ms, "distinct": d["distinct"], "raw": d["raw"],
                                             "distinct_per_s": d["distinct"] / (ms / 1e3),
                                             "devices": list(d["devices"])}
            from oracle import coracle as co
            from oracle import mapa_oracle as mo
            o = mo.builtin("cubemesh16")
            kk_, ee = mo.make_pattern("ring", k)

            def deep_cpu():
                r = co.allocate_deep(o, 0b11111 << 11, kk_, ee, 0, False)  # 11 free devices
                return r["raw"], 1
            line["cpu_baseline"] = _cpu(deep_cpu, "ring-10 greedy on 11 free cubemesh16 devices (11!/1! = 39,916,800 "
                                                  "embeddings), deep C oracle, all host threads")
        pruned = {}
        if rank == 0 and world == 1:
            # the paper's overhead study (fig:preserve_policy_overhead): milliseconds per
            # allocation for 9+ GPU jobs on 16-GPU graphs; Greedy with MAPA_F_PRUNE (exact), end to end
            # (Preserve-insensitive: set search over the full-k pattern + cached lex-smallest labelling;
            # Preserve-sensitive: Eq. 2 rank bound tables + the set bound on score ties)
            for tname in ("cubemesh16", "torus2d16"):
                tt = mp.Topology(tname)
                for shape, kk in (("ring", 9), ("ring", 12), ("ring", 14), ("ring", 16), ("tree", 12), ("tree", 14)):
                    p2 = mp.Pattern.make(shape, kk)
                    for sel, sens, sname in ((0, False, "greedy"), (1, False, "preserve_insensitive"),
                                             (1, True, "preserve_sensitive")):
                        if sens and kk == 16:
                            continue  # k = N all free: the set is forced, ties fall to the edge code (~5 s)
                        mp.allocate(tt, p2, sel, sens, prune=True)
                        ts = []
                        for _ in range(5 if not sens else 3):
                            t0 = time.perf_counter()
                            d = mp.allocate(tt, p2, sel, sens, prune=True)
                            ts.append((time.perf_counter() - t0) * 1e3)
                        pruned[f"{tname}_{shape}{kk}_{sname}"] = {
                            "ms_median": statistics.median(ts), "leaves_scored": d["leaves"],
                            "distinct": d["distinct"], "agg_bw": d["agg_bw"], "preserved_bw": d["preserved_bw"],
                            "pred_effbw": d["pred_effbw"]}
        emb_s = 3 * per / (tot / 1e3)
        ach = 2 * emb_s / 1e9
        line["roofline"] = {"bound": "alu", "kernel": "esa_deep<NT,SEL> (ring-10 RAW)",
                            "achieved": ach, "peak": PEAK_GOPS, "unit": "Gop/s", "frac": ach / PEAK_GOPS,
                            "traffic": _traffic("deep"), "ops_per_embedding": 2,
                            "note": "same algorithmic count as the narrow kernel (complete the score from the "
                                    "shared prefix partial + compare)"}
        line.update(metric="embeddings/sec (deep path: cubemesh16 ring-10 all free, RAW)", value=emb_s,
                    unit="embeddings/s", allocations_per_s=3 / (tot / 1e3), kernel_ms=kms, scaling="strong",
                    canonical=canon,
                    pruned_latency={"mode": "MAPA_F_PRUNE branch and bound (exact; all free)", "allocations": pruned},
                    config={"workload": "cubemesh16 x ring-10 (k > 8: 256-bit-key deep kernel), all free, RAW, "
                                        "1 allocation per selector per step, sharded by work item"})
        return line
    return None
