"""Writes the full-size C3 / C5 parity sets (SURVEY.md §8(d) "Full parity
sets") by calling ONLY oracle/ (the plain C brute force, oracle/oracle.c) on
the seeded workloads of workloads/ -- nothing here touches the CUDA path.

Parts (one compressed .npz per part, plus tests/golden/c3c5_manifest.json):
  c5_cubemesh16   C5, 1e5 queries (workloads.c5_queries(16, 100_000))
  c5_het32        C5, 1e5 queries (workloads.c5_queries(32, 100_000)), ~1.2e11 perms
  c3_k46          C3, cubemesh16, {ring,tree,full} x k in {4,6}, 1000 queries per case
  c3_k8           C3, cubemesh16, {ring,tree,full} x k = 8, the first 200 queries
                  of each shape's 1000 (workloads.c3_queries(per_case=1000))

Per query: the query (shape, k, busy, selector, sensitive) as generated, and
the oracle's decision: status (0 ok / 1 no capacity), device mask, mapping
(lex-first permutation of the winning orbit, -1 padded), used edges (sorted
(lo, hi) pairs coded lo*64+hi, 0xFFFF padded), census x/y/z, AggBW (Eq. 1),
PreservedBW (Eq. 3), predicted EffBW (Eq. 2, double), raw = #injective maps,
distinct = #(device set, used-edge set) matches, both counted by the oracle.

Run:  nice python tests/golden/make_golden_c3c5.py [part ...] [--jobs J]
(c5_het32 is about 40 core-minutes, c3_k8 a few core-hours; parts are
independent and each file is written when its part finishes)."""
import argparse
import hashlib
import json
import math
import multiprocessing as mpc
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import coracle as co  # noqa: E402
from oracle import mapa_oracle as mo  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
SHAPES = ("ring", "tree", "full")
MAXK, MAXM = 8, 28

REC = np.dtype([("shape", "u1"), ("k", "u1"), ("busy", "<u4"), ("selector", "u1"), ("sensitive", "u1"),
                ("status", "u1"), ("mask", "<u4"), ("mapping", "i1", (MAXK,)), ("used", "<u2", (MAXM,)),
                ("x", "<i4"), ("y", "<i4"), ("z", "<i4"), ("agg", "<i4"), ("pres", "<i4"),
                ("eff", "<f8"), ("raw", "<u8"), ("distinct", "<u8")])


def part_queries(part):
    """(topology name, topology text or None, list of query dicts) of a part."""
    if part == "c5_cubemesh16":
        return "cubemesh16", None, W.c5_queries(16, count=100_000)
    if part == "c5_het32":
        return "het32", W.het32_text(), W.c5_queries(32, count=100_000)
    qs = W.c3_queries(per_case=1000)
    if part == "c3_k46":
        return "cubemesh16", None, [q for q in qs if q["k"] in (4, 6)]
    if part == "c3_k8":
        out = []
        for s in SHAPES:
            out += [q for q in qs if q["k"] == 8 and q["shape"] == s][:200]
        return "cubemesh16", None, out
    raise ValueError(part)


_topo = None


def _init(name, text):
    global _topo
    _topo = mo.builtin(name) if text is None else mo.parse_topology(text)


def _solve(args):
    i, q = args
    k, e = mo.make_pattern(q["shape"], q["k"])
    d = co.allocate(_topo, q["busy"], k, e, q["selector"], q["sensitive"], nthreads=1)
    return i, d


def _work(n, q):
    nf = n - bin(q["busy"]).count("1")
    return math.perm(nf, q["k"]) if q["k"] <= nf else 0


def run_part(part, jobs):
    name, text, qs = part_queries(part)
    n = 32 if name == "het32" else 16
    rec = np.zeros(len(qs), dtype=REC)
    for i, q in enumerate(qs):
        r = rec[i]
        r["shape"], r["k"], r["busy"] = SHAPES.index(q["shape"]), q["k"], q["busy"]
        r["selector"], r["sensitive"] = q["selector"], q["sensitive"]
    order = sorted(range(len(qs)), key=lambda i: -_work(n, qs[i]))  # LPT: biggest queries first
    t0 = time.time()
    done = 0
    with mpc.get_context("fork").Pool(jobs, initializer=_init, initargs=(name, text)) as pool:
        chunk = 1 if part == "c3_k8" else 16
        for i, d in pool.imap_unordered(_solve, [(i, qs[i]) for i in order], chunksize=chunk):
            r = rec[i]
            r["raw"], r["distinct"] = d["raw"], d["distinct"]
            r["mapping"][:] = -1
            r["used"][:] = 0xFFFF
            if d["status"] != "ok":
                r["status"] = 1
            else:
                r["status"] = 0
                r["mask"] = sum(1 << v for v in d["devices"])
                r["mapping"][:len(d["mapping"])] = d["mapping"]
                r["used"][:len(d["used_edges"])] = [a * 64 + b for a, b in d["used_edges"]]
                r["x"], r["y"], r["z"] = d["x"], d["y"], d["z"]
                r["agg"], r["pres"], r["eff"] = d["agg_bw"], d["preserved_bw"], d["pred_effbw"]
            done += 1
            if done % max(1, len(qs) // 20) == 0:
                print(f"{part}: {done}/{len(qs)} {time.time() - t0:.0f}s", flush=True)
    path = os.path.join(GOLD, f"{part}.npz")
    np.savez_compressed(path, rec=rec)
    sha = hashlib.sha256(open(path, "rb").read()).hexdigest()
    man_path = os.path.join(GOLD, "c3c5_manifest.json")
    man = json.load(open(man_path)) if os.path.exists(man_path) else {
        "_doc": "Full-size C3/C5 parity sets written by tests/golden/make_golden_c3c5.py from oracle/ only "
                "(oracle/oracle.c, one thread per query). Device ids 0-based; see the script for the fields.",
        "parts": {}}
    man["parts"][part] = {"file": f"{part}.npz", "sha256": sha, "topology": name, "queries": len(qs),
                          "raw_total": int(rec["raw"].sum()), "oracle_seconds": round(time.time() - t0, 1),
                          "jobs": jobs}
    with open(man_path, "w") as f:
        json.dump(man, f, indent=1, sort_keys=True)
    print(f"{part}: wrote {path} ({len(qs)} queries, {time.time() - t0:.0f}s)", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("parts", nargs="*", default=["c5_cubemesh16", "c3_k46", "c5_het32", "c3_k8"])
    ap.add_argument("--jobs", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    co.build()
    for p in a.parts:
        run_part(p, a.jobs)


if __name__ == "__main__":
    main()
