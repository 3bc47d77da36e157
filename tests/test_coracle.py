"""The C oracle (used for sizes Python cannot finish) must equal the pinned
Python oracle on every small instance.  CPU only."""
import itertools
import json
import os
import random
from fractions import Fraction

import pytest

import workloads as W
from oracle import coracle as co
from oracle import mapa_oracle as mo

FIELDS = ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "raw", "distinct")


def _same(p, c):
    assert p["status"] == c["status"]
    if p["status"] != "ok":
        return
    for f in FIELDS:
        assert p[f] == c[f], (f, p[f], c[f])
    assert abs(p["pred_effbw"] - c["pred_effbw"]) <= 1e-9 * max(1.0, abs(p["pred_effbw"]))


@pytest.mark.parametrize("topo", ["dgx1v", "dgx1p", "summit", "rand8"])
def test_c_vs_python_small(topo):
    t = mo.parse_topology(W.rand_text(8, 99)) if topo == "rand8" else mo.builtin(topo)
    rng = random.Random(sum(map(ord, topo)))
    for trial in range(40):
        busy = rng.randrange(0, 1 << t.n)
        shape = rng.choice(["ring", "tree", "ringtree", "full"])
        k = rng.randint(2 if shape == "ring" else 1, 5)
        kk, e = mo.make_pattern(shape, k)
        sel = rng.choice([(0, 0), (1, 1), (1, 0), (2, 0)])
        _same(mo.allocate(t, busy, kk, e, *sel), co.allocate(t, busy, kk, e, *sel, nthreads=1 + trial % 3))


def test_c_eq2_matches_exact():
    for x, y, z in itertools.product(range(6), repeat=3):
        assert abs(co.eq2(x, y, z) - float(mo.eq2_exact(x, y, z))) < 1e-9


def test_c_thread_count_invariance():
    t = mo.builtin("cubemesh16")
    kk, e = mo.make_pattern("ring", 4)
    busy = 0b1010_0110_0000_0001
    r1 = co.allocate(t, busy, kk, e, 1, 0, nthreads=1)
    r7 = co.allocate(t, busy, kk, e, 1, 0, nthreads=7)
    assert r1 == r7


def test_c_sample_range_partitions_raw():
    # bounded samples (a_lo, a_hi) over S[0] partition the full enumeration
    t = mo.builtin("dgx1v")
    kk, e = mo.make_pattern("tree", 4)
    full = co.allocate(t, 0, kk, e, 0, 0)
    parts = [co.allocate(t, 0, kk, e, 0, 0, a_lo=a, a_hi=a + 1) for a in range(0, 5)]
    assert sum(p["raw"] for p in parts) == full["raw"]
    assert sum(p["distinct"] for p in parts) == full["distinct"]
