"""Loader of the full-size C3 / C5 parity sets (tests/golden/*.npz written by
tests/golden/make_golden_c3c5.py from oracle/ only).  Test infrastructure."""
import hashlib
import json
import os

import numpy as np

import workloads as W

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SHAPES = ("ring", "tree", "full")


def manifest():
    return json.load(open(os.path.join(GOLD, "c3c5_manifest.json")))


def have(part: str) -> bool:
    return os.path.exists(os.path.join(GOLD, f"{part}.npz")) and part in manifest()["parts"]


def load(part: str):
    """(records, query dicts regenerated from workloads/) -- asserts that the
    stored queries are the generator's and the file is the manifest's."""
    path = os.path.join(GOLD, f"{part}.npz")
    man = manifest()["parts"][part]
    assert hashlib.sha256(open(path, "rb").read()).hexdigest() == man["sha256"], part
    rec = np.load(path)["rec"]
    if part == "c5_cubemesh16":
        qs = W.c5_queries(16, count=100_000)
    elif part == "c5_het32":
        qs = W.c5_queries(32, count=100_000)
    else:
        allq = W.c3_queries(per_case=1000)
        if part == "c3_k46":
            qs = [q for q in allq if q["k"] in (4, 6)]
        else:
            qs = []
            for s in SHAPES:
                qs += [q for q in allq if q["k"] == 8 and q["shape"] == s][:200]
    assert len(qs) == len(rec) == man["queries"], part
    for i in (0, len(qs) // 2, len(qs) - 1):
        q, r = qs[i], rec[i]
        assert (SHAPES[r["shape"]], int(r["k"]), int(r["busy"]), int(r["selector"]), int(r["sensitive"])) == \
            (q["shape"], q["k"], q["busy"], q["selector"], q["sensitive"]), (part, i)
    sh = np.array([SHAPES.index(q["shape"]) for q in qs])
    assert (sh == rec["shape"]).all() and (np.array([q["busy"] for q in qs], dtype=np.uint64) ==
                                           rec["busy"].astype(np.uint64)).all(), part
    return rec, qs


def expected(r) -> dict:
    """One golden record as the decision dict of the binding (oracle fields)."""
    if r["status"] != 0:
        return dict(status="no_capacity", raw=int(r["raw"]), distinct=int(r["distinct"]))
    k = int(r["k"])
    m = int((r["used"] != 0xFFFF).sum())
    mask = int(r["mask"])
    return dict(status="ok", devices=tuple(d for d in range(32) if (mask >> d) & 1),
                mapping=tuple(int(v) for v in r["mapping"][:k]),
                used_edges=[(int(c) >> 6, int(c) & 63) for c in r["used"][:m]],
                x=int(r["x"]), y=int(r["y"]), z=int(r["z"]), agg_bw=int(r["agg"]), preserved_bw=int(r["pres"]),
                pred_effbw=float(r["eff"]), raw=int(r["raw"]), distinct=int(r["distinct"]))
