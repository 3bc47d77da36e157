#!/usr/bin/env python
"""MAPA hot-path benchmark (BASELINE.json metric: candidate embeddings scored /s
and allocations /s at 1/2/4/8 B200).

Workload (config C4): het32 (32-vertex heterogeneous-link
topology), 6-vertex all-to-all pattern (m = 15), all devices free, RAW mode:
every one of the P(32,6) = 652,458,240 injective embeddings is scored.  One
step = one allocation per selector (Greedy / Preserve-sensitive /
Preserve-insensitive): 3 x 652,458,240 = 1,957,374,720 embeddings.  With N
GPUs (torchrun, one process per GPU) each query is sharded by work chunk
(global chunk q*N + r -> rank r) and the per-rank 32-B records are combined
with one all_gather over NCCL: the total work per step is fixed ("strong"
scaling).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints ONE JSON line on rank 0.  `value` = embeddings/s from device (CUDA
event) time, inputs resident in HBM, max over ranks; `e2e` = the same metric
through mapa_allocate (N=1: host buffers, H2D query + D2H record + host
decode) or the sharded public API (N>1).  `--impl reference` times the CPU
oracle (oracle/, the task's reference arm) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "candidate embeddings scored/sec and allocations/sec at 1/2/4/8 B200"
K_PAT, M_PAT = 6, 15
RAW_PER_QUERY = math.perm(32, K_PAT)                    # 652,458,240
SELECTORS = ((0, False, "greedy"), (1, True, "preserve_sensitive"), (1, False, "preserve_insensitive"))
# Algorithmic integer work per scored embedding: with
# the enumeration tree sharing every partial sum of an embedding's prefix, what
# remains per embedding is to complete its score from two shared partials (1
# add) and compare it (1 max); Eq. 2 also reads the rank table (+1).  The
# kernel fuses add+max (VIADDMNMX), so these counts are reachable.  SURVEY
# 8(d)'s unamortised figure (~2m = 30-43 ops: every edge weight re-read) is
# reported beside it as "ops_unamortised" for context.
ALG_OPS = {"greedy": 2, "preserve_sensitive": 3, "preserve_insensitive": 2}
ALG_OPS_UNAMORTISED = {"greedy": 2 * M_PAT, "preserve_sensitive": 2 * M_PAT + 2,
                       "preserve_insensitive": 2 * (K_PAT * (K_PAT - 1) // 2 + K_PAT) + 1}
# Reference-arm / cpu_baseline sample: the C4 subsets whose smallest device is
# device 0 and second smallest >= device 8 (30,602,880 embeddings).
SAMPLE = dict(a_lo=0, a_hi=1, b_lo=8, b_hi=-1)
SAMPLE_DESC = ("C4 het32 full-6 greedy, embeddings of the 6-subsets with min device 0 and second device >= 8 "
               "(30,602,880 of 652,458,240 = 4.7%), plain brute force with per-subset dedup")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def int_peaks():
    """The integer issue / pipe microbenchmark (scripts/int_ubench.cu, run on a
    B200 of this pool): lane-ops per SM per clock of each instruction class."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02_int_peaks.json")))
        return {r["op"]: r["lane_ops_per_sm_per_clk"] for r in d["results"]}
    except Exception:
        return {}


def issue_lanes_per_sm_clk() -> float:
    """Issue roofline in lane-instructions per SM per clock: MEASURED with an
    independent IADD3 (ALU pipe) + IMAD (FMA pipe) 1:1 mix, 128.06 (one
    warp-instruction per SMSP per clock; each pipe alone 64,
    profiles/r02_int_peaks.json).  Fallback: the nominal 128 (B300_MICROARCH)."""
    return int_peaks().get("IADD3+IMAD (1:1)", 128.0)


def alu_peak_gops(clock_mhz: float) -> float:
    """Integer issue roofline: 148 SMs x the measured lane-instructions per SM
    per clock (issue_lanes_per_sm_clk) at the measured max SM clock."""
    return 148 * issue_lanes_per_sm_clk() * clock_mhz * 1e6 / 1e9


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self, which):
        setattr(self, which, time.time())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        rows = [s for t, s in self.samples if self.t0 and self.t1 and self.t0 <= t <= self.t1 + 0.05]
        if len(rows) < 3:
            rows = [s for _, s in self.samples]
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model() -> str:
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_oracle_sample(nthreads=None):
    """Oracle (oracle/oracle.c) on the bounded sample, all host threads (or nthreads)."""
    from oracle import coracle as co
    from oracle import mapa_oracle as mo
    t = mo.parse_topology(W.het32_text())
    k, e = mo.make_pattern("full", K_PAT)
    nthreads = nthreads or os.cpu_count() or 1
    t0 = time.perf_counter()
    r = co.allocate(t, 0, k, e, 0, False, nthreads=nthreads, **SAMPLE)
    dt = time.perf_counter() - t0
    units = 31 - 8  # (S[0], S[1]) work units in the sample bound the usable threads
    return r["raw"], dt, min(nthreads, units)


def run_reference(args):
    """Reference arm = the CPU oracle as it stands (task tier framing)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_oracle_sample()
    tot_raw, tot_t, cores = 0, 0.0, 1
    for _ in range(args.steps):
        raw, dt, cores = cpu_oracle_sample()
        tot_raw += raw
        tot_t += dt
    v = tot_raw / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "embeddings/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": "C4 het32 full-6 all-free raw (bounded sample per step)",
                                            "sample": SAMPLE_DESC},
            "cpu_baseline": {"value": v, "unit": "embeddings/s", "cores": cores, "kind": "oracle",
                             "sample": SAMPLE_DESC},
            "e2e": {"value": v, "unit": "embeddings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mapa", choices=["mapa", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prune", action="store_true", help="skip the MAPA_F_PRUNE side measurement")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--streams", type=int, default=0,
                    help="C4: streams for the three selector launches of a step (default 1 at N=1, 3 at N>1)")
    ap.add_argument("--config", default="c4", choices=["c4", "c1", "c2", "c3", "c5", "deep"],
                    help="c4 = the headline workload (default); c1/c2/c3/c5 measure the other SURVEY 8(d) configs; "
                         "deep = the k > 8 path (SURVEY 8(f) NEXT 1)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "mapa" and not args.no_cpu_baseline:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2110_03214_b200 as mp
    from paper_2110_03214_b200 import dist as md

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    # MAPA_BENCH_BACKEND=gloo lets several ranks share one GPU (tests of this
    # script's multi-rank logic); production runs use NCCL over NVLink.
    backend = os.environ.get("MAPA_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    def all_gather_dev(out, inp):
        if backend == "nccl":
            dist.all_gather_into_tensor(out, inp)
        else:
            parts = [torch.empty_like(inp, device="cpu") for _ in range(world)]
            dist.all_gather(parts, inp.cpu())
            out.copy_(torch.cat(parts).view_as(out))

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if args.config != "c4":
        from bench_configs import run_config
        sampler = ClockSampler(local)
        if rank == 0:
            sampler.start()
        sampler.mark("t0")
        line = run_config(args, mp, md, torch, dev, stream, rank, world, max_over_ranks)
        sampler.mark("t1")
        sampler.stop()
        if line is not None and rank == 0:
            line["clocks"] = dict(sampler.summary(), window="the whole config run (GPU legs and CPU baseline)")
        if rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    topo = mp.Topology(text=W.het32_text())
    pat = mp.Pattern.make("full", K_PAT)
    busy = 0
    qbuf = md.query_tensor(busy, 0, 0, False, device=dev)          # resident input (16 B)
    recs = torch.zeros((len(SELECTORS), 4), dtype=torch.int64, device=dev)
    gath = torch.zeros((world, len(SELECTORS), 4), dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    kev = {name: [] for _, _, name in SELECTORS}
    # One memset zeroes the three records (MAPA_F_ZEROED launches: no memset node
    # per launch).  With N > 1 ranks each rank's three shards are small, so the
    # three launches go to three streams and their prologues / tails overlap;
    # at N = 1 they stay on one stream, so the per-kernel CUDA events of the
    # timed region give each kernel's own duration (the roofline's input).
    nstreams = args.streams or (len(SELECTORS) if world > 1 else 1)
    lstreams = [stream] if nstreams == 1 else [torch.cuda.Stream(device=dev) for _ in range(nstreams)]

    def step(timed):
        recs.zero_()
        if nstreams > 1:
            fork = torch.cuda.Event()
            fork.record(stream)
        for i, (sel, sens, name) in enumerate(SELECTORS):
            ls = lstreams[i % nstreams]
            if nstreams > 1:
                ls.wait_event(fork)
            if timed:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(ls)
            mp.launch_query(topo, pat, sel, sens, qbuf.data_ptr(), recs[i].data_ptr(), raw=True, rank=rank,
                            world=world, busy_hint=busy, stream=ls, zeroed=True)
            if timed:
                b.record(ls)
                kev[name].append((a, b))
        if nstreams > 1:
            for ls in lstreams:
                j = torch.cuda.Event()
                j.record(ls)
                stream.wait_event(j)
        if world > 1:
            all_gather_dev(gath.view(world, -1), recs.view(-1))

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    # correctness guard on the timed configuration: combined records decode consistently
    rlist = md.records_from_tensor(gath if world > 1 else recs.unsqueeze(0))
    for i, (sel, sens, name) in enumerate(SELECTORS):
        rr = [rlist[r * len(SELECTORS) + i] for r in range(world)]
        d = mp.decode(topo, pat, busy, sel, sens, mp.reduce_records(rr), raw=True)
        assert d["raw"] == RAW_PER_QUERY, d

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
        time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.mark("t0")
    steps_ev = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step(True)
        b.record(stream)
        steps_ev.append((a, b))
        flush.zero_()  # L2 flush between timed steps, outside the step events
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.mark("t1")
    dev_ms = sum(a.elapsed_time(b) for a, b in steps_ev)
    kern_ms = {n: sum(a.elapsed_time(b) for a, b in v) / len(v) for n, v in kev.items()}
    dev_ms = max_over_ranks(dev_ms)

    # ---- MAPA_F_PRUNE (branch and bound): same decisions,
    # fewer embeddings scored; reported beside the headline, never as it
    prune_ms = {n: [] for _, _, n in SELECTORS}
    prune_leaves = {}
    if not args.no_prune:
        precs = torch.zeros((len(SELECTORS), 4), dtype=torch.int64, device=dev)
        for it in range(args.warmup + args.steps):
            for i, (sel, sens, name) in enumerate(SELECTORS):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                mp.launch_query(topo, pat, sel, sens, qbuf.data_ptr(), precs[i].data_ptr(), raw=True, rank=rank,
                                world=world, busy_hint=busy, stream=stream, prune=True)
                b.record(stream)
                if it >= args.warmup:
                    prune_ms[name].append((a, b))
            flush.zero_()
        torch.cuda.synchronize()
        prl = md.records_from_tensor(precs)
        for i, (sel, sens, name) in enumerate(SELECTORS):
            prune_leaves[name] = int(prl[i].leaves)  # rank 0's shard when world > 1
            if world == 1:  # same decision as the exhaustive launch
                dp = mp.decode(topo, pat, busy, sel, sens, prl[i], raw=True, prune=True)
                de = mp.decode(topo, pat, busy, sel, sens, rlist[i], raw=True)
                assert dp["key"] == de["key"], (name, dp["key"], de["key"])
    prune_kms = {n: (max_over_ranks(sum(a.elapsed_time(b) for a, b in v) / len(v)) if v else None)
                 for n, v in prune_ms.items()}

    sampler.stop()  # the nvidia-smi poller competes for host cores; clocks are sampled above
    # ---- e2e through the public API (host buffers, copies inside the region)
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 50))
    many = [(pat, sel, sens) for sel, sens, _name in SELECTORS]
    for _ in range(args.warmup):  # untimed: first call allocates the staging buffers and captures the graph
        if world == 1:
            mp.allocate_many(topo, many, raw=True)
        else:
            for sel, sens, _name in SELECTORS:
                md.allocate_sharded(topo, pat, sel, sens, busy, raw=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        if world == 1:
            # mapa_allocate_many: one H2D copy of the three queries (+ zero records), the three
            # launches as parallel graph branches, one D2H copy of the records, host decode
            ds = mp.allocate_many(topo, many, raw=True)
            assert ds[0]["raw"] == RAW_PER_QUERY
        else:
            for sel, sens, _name in SELECTORS:
                d = md.allocate_sharded(topo, pat, sel, sens, busy, raw=True)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - w0
    e2e_s = max_over_ranks(e2e_s)

    if rank == 0:
        emb_step = RAW_PER_QUERY * len(SELECTORS)
        value = emb_step * args.steps / (dev_ms / 1e3)
        allocs = len(SELECTORS) * args.steps / (dev_ms / 1e3)
        pk = peaks()
        clk = sampler.summary()
        max_mhz = pk.get("sm_max_mhz") or 1965.0
        peak = alu_peak_gops(max_mhz)
        # dominant kernel = the selector kernel with the largest share of the step
        dom = max(kern_ms, key=kern_ms.get)
        leaves_per_launch = RAW_PER_QUERY / world
        achieved = ALG_OPS[dom] * leaves_per_launch / (kern_ms[dom] / 1e3) / 1e9
        traffic, lipe, swpe = None, None, None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
            traffic = prof.get("dram_bytes_per_launch", {}).get(dom)
            lipe = prof.get("lane_instr_per_embedding", {}).get(dom)
            swpe = prof.get("smem_wavefronts_per_embedding", {}).get(dom)
        except Exception:
            pass
        # issue_frac: the kernel's executed lane-instructions per embedding (ncu,
        # profiles/ncu_summary.json) x embeddings/s / the measured issue peak
        emb_s = leaves_per_launch / (kern_ms[dom] / 1e3)
        issue_frac = lipe * emb_s / (peak * 1e9) if lipe else None
        # lsu_frac: shared-memory data-pipe wavefronts per embedding (ncu) x embeddings/s
        # / (148 SMs x 1 wavefront per SM per clock x the max SM clock) -- the Eq. 2
        # kernel's gathers make this its binding resource
        lsu_frac = swpe * emb_s / (148 * max_mhz * 1e6) if swpe else None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            raw, dt, cores = cpu_oracle_sample()
            raw1, dt1, _ = cpu_oracle_sample(1)
            cpu = {"value": raw / dt, "unit": "embeddings/s", "cores": cores, "kind": "oracle",
                   "sample": SAMPLE_DESC, "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
                   "value_1thread": raw1 / dt1, "seconds": dt, "seconds_1thread": dt1}
        line = {
            "metric": METRIC, "value": value, "unit": "embeddings/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": "C4: het32 (32-vertex heterogeneous-link) x full-6 (all-to-all, m=15), all free, "
                                   "RAW mode, 1 allocation per selector per step",
                       "embeddings_per_step": emb_step, "allocations_per_step": len(SELECTORS),
                       "parallelism": f"shard-by-work-item x{world} + 1 NCCL all_gather/step" if world > 1
                       else "1 GPU", "launch_streams": nstreams,
                       "l2": "flushed between steps (256 MiB memset outside step events)"},
            "allocations_per_s": allocs,
            "kernel_ms": kern_ms,
            "roofline": {"bound": "alu", "kernel": f"esa_single<32,6,{'SENS' if dom == 'preserve_sensitive' else 'LIN'}> ({dom})",
                         "achieved": achieved, "peak": peak, "unit": "Gop/s", "frac": achieved / peak,
                         "traffic": traffic,
                         "ops_per_embedding": ALG_OPS[dom], "ops_unamortised": ALG_OPS_UNAMORTISED[dom],
                         "frac_unamortised": ALG_OPS_UNAMORTISED[dom] * emb_s / (peak * 1e9),
                         "lane_instr_per_embedding": lipe, "issue_frac": issue_frac,
                         "smem_wavefronts_per_embedding": swpe, "lsu_frac": lsu_frac,
                         "note": f"frac = {ALG_OPS[dom]} algorithmic int ops per embedding (complete the score from two "
                                 f"shared partials + compare; DESIGN.md Roofline) x embeddings/s / peak; peak = 148 SM x "
                                 f"{issue_lanes_per_sm_clk():.2f} lane-ops/SM/clk (measured issue rate, "
                                 f"profiles/r02_int_peaks.json) x {max_mhz:.0f} MHz (measured max SM clock); issue_frac = "
                                 f"ncu lane-instructions per embedding (profiles/ncu_summary.json) x embeddings/s / peak; "
                                 f"lsu_frac = ncu shared-memory wavefronts per embedding x embeddings/s / (148 SM x 1 "
                                 f"wavefront/SM/clk x the max SM clock) -- the Eq. 2 gathers' binding pipe; "
                                 f"frac_unamortised = SURVEY 8(d)'s per-embedding count (every weight re-read) over the "
                                 f"same peak, > 1 because the enumeration tree shares prefix work"},
            "cpu_baseline": cpu,
            "e2e": {"value": emb_step * e2e_steps / e2e_s, "unit": "embeddings/s",
                    # N=1: mapa_allocate_many -- one H2D staging copy of 128 B per query (16-B query +
                    # a zero record image) and one D2H copy of the 64-B record slots; N>1: per
                    # allocation the query tensor + the all_gather'd records
                    "api": "mapa_allocate_many (3 queries per call)" if world == 1 else "dist.allocate_sharded",
                    "h2d_bytes_per_step": (128 if world == 1 else 16) * len(SELECTORS),
                    "d2h_bytes_per_step": (64 if world == 1 else 32 * world) * len(SELECTORS),
                    "allocations_per_s": len(SELECTORS) * e2e_steps / e2e_s},
            "gpu_launches": len(SELECTORS) * args.steps,
            "clocks": clk,
        }
        if not args.no_prune:
            tot = sum(prune_kms.values())
            line["pruned"] = {
                "mode": "MAPA_F_PRUNE branch-and-bound (exact: same decisions, asserted against the exhaustive run)",
                "kernel_ms": prune_kms, "allocations_per_s": len(SELECTORS) / (tot / 1e3),
                "embeddings_searched_per_s": emb_step / (tot / 1e3),
                "leaves_scored": prune_leaves,
                "scored_fraction": {n: v / RAW_PER_QUERY for n, v in prune_leaves.items()},
                "note": "not the headline: skipped embeddings are not scored (SURVEY §8(f) NEXT 3)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
