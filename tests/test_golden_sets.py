"""CPU checks of the full-size C3 / C5 parity sets (tests/golden/*.npz): the
files hold exactly the generator's queries, their counts are the closed forms
(raw = P(|F|,k), distinct = raw / |Aut(P)| -- orbit theorem, pinned in
test_oracle_pins.py), every decision is a set of free devices, and a sample
of records re-computed by the oracle here equals the stored ones."""
import math
import random

import pytest

from oracle import coracle as co
from oracle import mapa_oracle as mo
from tests import goldenutil as G

PARTS = ("c5_cubemesh16", "c5_het32", "c3_k46", "c3_k8")


def _topo(part):
    import workloads as W
    return mo.parse_topology(W.het32_text()) if part == "c5_het32" else mo.builtin("cubemesh16")


@pytest.mark.parametrize("part", PARTS)
def test_golden_set_counts_and_validity(part):
    if not G.have(part):
        pytest.skip(f"{part} not generated yet")
    rec, qs = G.load(part)
    n = 32 if part == "c5_het32" else 16
    aut = {}
    for q, r in zip(qs, rec):
        k = q["k"]
        nf = n - bin(q["busy"]).count("1")
        key = (q["shape"], k)
        if key not in aut:
            kk, e = mo.make_pattern(q["shape"], k)
            aut[key] = mo.automorphism_count(kk, e)
        raw = math.perm(nf, k) if k <= nf else 0
        assert int(r["raw"]) == raw and int(r["distinct"]) == raw // aut[key], (part, q)
        if k > nf:
            assert r["status"] == 1
            continue
        assert r["status"] == 0
        mask = int(r["mask"])
        assert bin(mask).count("1") == k and mask & q["busy"] == 0, (part, q)
        assert sorted(int(v) for v in r["mapping"][:k]) == [d for d in range(n) if (mask >> d) & 1]
        assert int(r["x"]) + int(r["y"]) + int(r["z"]) == len(mo.make_pattern(q["shape"], k)[1])


@pytest.mark.parametrize("part", PARTS)
def test_golden_set_sample_recomputed(part):
    if not G.have(part):
        pytest.skip(f"{part} not generated yet")
    rec, qs = G.load(part)
    t = _topo(part)
    rng = random.Random(11)
    n = 32 if part == "c5_het32" else 16
    cheap = [i for i, q in enumerate(qs) if math.perm(n - bin(q["busy"]).count("1"), q["k"]) < 2e5]
    for i in rng.sample(cheap, min(40, len(cheap))):
        q = qs[i]
        k, e = mo.make_pattern(q["shape"], q["k"])
        d = co.allocate(t, q["busy"], k, e, q["selector"], q["sensitive"], nthreads=1)
        exp = G.expected(rec[i])
        assert d["status"] == exp["status"]
        for f in ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "raw", "distinct"):
            if d["status"] == "ok" or f in ("raw", "distinct"):
                assert (list(d[f]) if f == "used_edges" else d[f]) == (list(exp[f]) if f == "used_edges" else exp[f]), \
                    (part, i, f)
