"""Pins of the deep C oracle (oracle_allocate_deep, k <= 16) — CPU only.

The deep oracle restates the definition of oracle_allocate without the
per-subset table (tie-break SPEC S:349/Alg. 1 first-wins
P:691/P:698).  It is pinned to things other than itself:
  * the narrow C oracle (itself pinned in test_oracle_pins.py) on every
    selector for k <= 8, including tie-heavy instances;
  * the Python itertools oracle (mapa_oracle.allocate) at k = 9;
  * closed forms: raw = P(|F|, k) for k up to 12;
  * special cases: a uniform topology and the Baseline selector reduce to the
    lowest free ids."""
import math
import random

import pytest

from oracle import coracle as co
from oracle import mapa_oracle as mo

FIELDS = ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "raw")
SELS = [(0, False), (1, True), (1, False), (2, False)]


def _same(a, b, ctx):
    assert a["status"] == b["status"], ctx
    if a["status"] != "ok":
        return
    for f in FIELDS:
        assert a[f] == b[f], (ctx, f, a[f], b[f])
    assert abs(a["pred_effbw"] - b["pred_effbw"]) <= 1e-9 * max(1.0, abs(a["pred_effbw"]))


@pytest.mark.parametrize("name", ["dgx1v", "dgx1p", "summit", "cubemesh16"])
def test_deep_oracle_equals_narrow_oracle(name):
    o = mo.builtin(name)
    rng = random.Random(77 + len(name))
    for trial in range(40):
        shape = rng.choice(["ring", "tree", "ringtree", "full"])
        k = rng.randint(2, min(6, o.n))
        busy = rng.randrange(0, 1 << o.n)
        if o.n > 8:
            busy |= (1 << 8) - 1  # keep at most 8 free devices
        sel, sens = rng.choice(SELS)
        kk, e = mo.make_pattern(shape, k)
        a = co.allocate(o, busy, kk, e, sel, sens, nthreads=4)
        b = co.allocate_deep(o, busy, kk, e, sel, sens, nthreads=4)
        _same(a, b, (name, shape, k, busy, sel, sens))


def test_deep_oracle_equals_python_oracle_k9():
    """k = 9 on cubemesh16 with 9 free devices: the itertools oracle (dedup by
    edge list, exact Eq. 2) and the deep C oracle agree on every field."""
    o = mo.builtin("cubemesh16")
    busy = sum(1 << d for d in (1, 3, 4, 8, 10, 12, 14))  # 9 free
    for shape, sel, sens in (("ring", 0, False), ("tree", 1, True), ("ring", 1, False)):
        kk, e = mo.make_pattern(shape, 9)
        a = mo.allocate(o, busy, kk, e, sel, sens)
        b = co.allocate_deep(o, busy, kk, e, sel, sens, nthreads=8)
        _same(a, b, (shape, sel, sens))


@pytest.mark.parametrize("k,nfree", [(9, 10), (10, 10), (11, 11)])
def test_deep_oracle_raw_closed_form(k, nfree):
    o = mo.builtin("torus2d16")
    busy = ((1 << 16) - 1) & ~((1 << nfree) - 1)
    kk, e = mo.make_pattern("ring", k)
    r = co.allocate_deep(o, busy, kk, e, 0, False, nthreads=8)
    assert r["raw"] == math.perm(nfree, k)
    assert set(r["devices"]) <= set(range(nfree))


def test_deep_oracle_uniform_topology_lowest_ids():
    """All pairs one class: every score ties, the lex-smallest device tuple
    wins (P:777 Baseline reduction), for every selector."""
    text = "name uni\ndevices 12\n" + "".join(
        f"link {a} {b} nv2x1\n" for a in range(1, 13) for b in range(a + 1, 13))
    o = mo.parse_topology(text)
    busy = 0b000000100101  # devices 0, 2, 5 busy -> 9 free
    kk, e = mo.make_pattern("ringtree", 9)
    for sel, sens in SELS:
        r = co.allocate_deep(o, busy, kk, e, sel, sens, nthreads=8)
        assert r["devices"] == (1, 3, 4, 6, 7, 8, 9, 10, 11)
        assert r["y"] == len(e)


def test_deep_oracle_no_capacity():
    o = mo.builtin("dgx1v")
    kk, e = mo.make_pattern("ring", 9)
    assert co.allocate_deep(o, 0, kk, e, 0, False)["status"] == "no_capacity"
