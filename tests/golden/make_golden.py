"""Writes tests/golden/c4_expected.json by calling ONLY oracle/ (the C brute
force) on the C4 workload: het32 and rand32(2110), full-6
(m=15), all free, selectors GREEDY / PRESERVE-sensitive / PRESERVE-insensitive.
Run:  python tests/golden/make_golden.py   (minutes on a few cores)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import coracle as co  # noqa: E402
from oracle import mapa_oracle as mo  # noqa: E402

SELS = {"greedy": (0, 0), "sensitive": (1, 1), "insensitive": (1, 0)}


def main():
    out = {"_doc": "C4 expected decisions written by tests/golden/make_golden.py from oracle/ only "
                   "(plain brute force, oracle/oracle.c). Device ids 0-based.", "cases": []}
    topos = {"het32": W.het32_text(), "rand32_2110": W.rand_text(32, W.MASTER_SEED)}
    k, e = mo.make_pattern("full", 6)
    for tname, text in topos.items():
        t = mo.parse_topology(text)
        for sname, (sel, sens) in SELS.items():
            t0 = time.time()
            d = co.allocate(t, 0, k, e, sel, sens)
            d["topology"] = tname
            d["selector"] = sname
            d["shape"] = "full"
            d["k"] = 6
            d["busy"] = 0
            d["oracle_seconds"] = round(time.time() - t0, 1)
            print(tname, sname, d["devices"], d["agg_bw"], d["pred_effbw"], d["oracle_seconds"], flush=True)
            out["cases"].append(d)
    with open(os.path.join(ROOT, "tests", "golden", "c4_expected.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
