"""Writes tests/golden/deep_k12_13.json -- deep-path parity goldens for
non-clique patterns with k = 12 and 13 (the paper's
overhead study reaches "9 GPUs and above" on 16-GPU graphs) --
by calling ONLY oracle/ (the deep C brute force, oracle_allocate_deep: every
permutation of every k-subset, lexicographic, strict '>' with the used-edge
tie-break).

Cases: {cubemesh16, torus2d16} x {ring, tree, ringtree} x k = 12 with exactly
12 and 13 free devices, and {cubemesh16, torus2d16} x {ring, ringtree} x
k = 13 with 13 free; the busy devices are drawn by the seeded generator
(workloads.stream), the selector rotates Greedy / Preserve-sensitive /
Preserve-insensitive.  12! = 4.8e8 and 13! = 6.2e9 permutations per case.

Run:  python tests/golden/make_golden_deep.py [--jobs J]   (~10 min on 16 cores)"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import coracle as co  # noqa: E402
from oracle import mapa_oracle as mo  # noqa: E402

SELS = [(0, False), (1, True), (1, False)]


def cases():
    out = []
    i = 0
    for k, shapes, frees in ((12, ("ring", "tree", "ringtree"), (12, 13)), (13, ("ring", "ringtree"), (13,))):
        for name in ("cubemesh16", "torus2d16"):
            for shape in shapes:
                for nfree in frees:
                    r = W.stream(W.MASTER_SEED ^ 0xDEE9, i)
                    devs = list(range(16))
                    busy = 0
                    for _ in range(16 - nfree):  # seeded busy devices
                        d = devs.pop(r.below(len(devs)))
                        busy |= 1 << d
                    sel, sens = SELS[i % 3]
                    out.append(dict(topology=name, shape=shape, k=k, busy=busy, selector=sel, sensitive=int(sens)))
                    i += 1
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    co.build()
    res = []
    for c in cases():
        t0 = time.time()
        kk, e = mo.make_pattern(c["shape"], c["k"])
        d = co.allocate_deep(mo.builtin(c["topology"]), c["busy"], kk, e, c["selector"], bool(c["sensitive"]),
                             nthreads=a.jobs, max_subsets=64)
        d = {f: (list(v) if isinstance(v, tuple) else v) for f, v in d.items()}
        d.update(c)
        d["oracle_seconds"] = round(time.time() - t0, 1)
        print(c, d.get("devices"), d.get("raw"), d["oracle_seconds"], flush=True)
        res.append(d)
    doc = {"_doc": "Deep-path goldens (k = 12, 13, non-clique) written by tests/golden/make_golden_deep.py from "
                   "oracle/ only (oracle_allocate_deep). Device ids 0-based; busy = bit mask.", "cases": res}
    with open(os.path.join(ROOT, "tests", "golden", "deep_k12_13.json"), "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
