"""Pins of the stored goldens and of the C oracle at N = 32 against values
fixed independently of the oracle's own code (CPU only).

* tests/golden/c4_expected.json (written by the oracle) against SURVEY §8(c)'s
  independently derived C4 values and against a subset brute force with a
  different enumeration (numpy over all C(32,6) device sets: for a clique
  every set is one orbit, so the set search IS the match search -- orbit
  theorem) that scores Eq. 3 through the edge-partition identity
   instead of the oracle's direct double loop over surviving pairs.
* oracle/oracle.c (every N = 32 golden rests on it) against the Python oracle
  on het32 / rand32 instances with at most 8 free devices.
* mapa_oracle.replay_trace against SPEC's worked selections
  and a release that restores the fresh answer (§3.6)."""
import itertools
import json
import math
import os
import random

import numpy as np
import pytest

import workloads as W
from oracle import coracle as co
from oracle import mapa_oracle as mo

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# SURVEY §8(c) "Selection, C4 expected" (het32, full-6, all free), 1-based ids
SURVEY_C4 = {
    "greedy": dict(devices=(1, 2, 3, 4, 5, 6), census=(5, 4, 6), agg_bw=422, preserved_bw=5322),
    "insensitive": dict(devices=(1, 2, 3, 4, 5, 6), census=(5, 4, 6), agg_bw=422, preserved_bw=5322),
    "sensitive": dict(devices=(1, 2, 9, 10, 17, 18), census=(0, 7, 8), agg_bw=251, pred_effbw=709.351385),
}


def _cases():
    return json.load(open(os.path.join(GOLD, "c4_expected.json")))["cases"]


def _weights(topo):
    return np.array([[0 if u == v else topo.bw(u, v) for v in range(topo.n)] for u in range(topo.n)], dtype=np.int64)


def _set_brute_force(topo, k=6):
    """All k-subsets in lex order; per set: AggBW of the clique (= induced
    total), census, PreservedBW by the identity T_F - sum inc_F + inside."""
    w = _weights(topo)
    sets = np.array(list(itertools.combinations(range(topo.n), k)), dtype=np.int64)
    pw = np.stack([w[sets[:, a], sets[:, b]] for a, b in itertools.combinations(range(k), 2)], axis=1)
    agg = pw.sum(axis=1)
    x = (pw == 50).sum(axis=1)
    y = ((pw == 25) | (pw == 20)).sum(axis=1)
    z = (pw == 12).sum(axis=1)
    inc = w.sum(axis=1)                       # all devices free
    T = int(w.sum()) // 2
    pres = T - inc[sets].sum(axis=1) + agg
    return sets, agg, x, y, z, pres


def test_c4_golden_equals_survey_values():
    """The oracle-written C4 golden must carry SURVEY §8(c)'s independently
    derived het32 answers (a wrong golden writer, or an oracle that drifted,
    fails here)."""
    got = {c["selector"]: c for c in _cases() if c["topology"] == "het32"}
    assert set(got) == set(SURVEY_C4)
    for sel, exp in SURVEY_C4.items():
        c = got[sel]
        assert tuple(d + 1 for d in c["devices"]) == exp["devices"], sel
        assert (c["x"], c["y"], c["z"]) == exp["census"], sel
        assert c["agg_bw"] == exp["agg_bw"], sel
        if "preserved_bw" in exp:
            assert c["preserved_bw"] == exp["preserved_bw"], sel
        if "pred_effbw" in exp:
            assert abs(c["pred_effbw"] - exp["pred_effbw"]) < 1e-6, sel
        assert c["raw"] == math.perm(32, 6) == 652_458_240
        assert c["distinct"] == math.comb(32, 6) == 906_192


@pytest.mark.parametrize("topo_name", ["het32", "rand32_2110"])
def test_c4_golden_equals_set_brute_force(topo_name):
    """Every field of the C4 golden (het32 and rand32) re-derived by the numpy
    set search: argmax with the first (lex-smallest) set on ties, the clique's
    mapping = the sorted set (lex-first permutation) and used edges = all
    pairs."""
    text = W.het32_text() if topo_name == "het32" else W.rand_text(32, W.MASTER_SEED)
    topo = mo.parse_topology(text)
    sets, agg, x, y, z, pres = _set_brute_force(topo)
    cens = sorted(set(zip(x.tolist(), y.tolist(), z.tolist())))
    effx = {c: mo.eq2_exact(*c) for c in cens}   # exact rationals (A9)
    eff_rank = {c: i for i, c in enumerate(sorted(cens, key=lambda c: effx[c]))}
    sens_key = np.array([eff_rank[c] for c in zip(x.tolist(), y.tolist(), z.tolist())])
    score = {"greedy": agg, "insensitive": pres, "sensitive": sens_key}
    for c in _cases():
        if c["topology"] != topo_name:
            continue
        i = int(np.argmax(score[c["selector"]]))   # first maximum = lex-smallest set
        S = tuple(int(d) for d in sets[i])
        assert tuple(c["devices"]) == S and tuple(c["mapping"]) == S, (topo_name, c["selector"])
        assert [tuple(e) for e in c["used_edges"]] == list(itertools.combinations(S, 2))
        assert (c["x"], c["y"], c["z"]) == (int(x[i]), int(y[i]), int(z[i]))
        assert c["agg_bw"] == int(agg[i]) and c["preserved_bw"] == int(pres[i])
        assert abs(c["pred_effbw"] - float(effx[(int(x[i]), int(y[i]), int(z[i]))])) < 1e-9


@pytest.mark.parametrize("topo_name", ["het32", "rand32"])
def test_c_oracle_equals_python_oracle_n32(topo_name):
    """oracle.c at N = 32 (the width of every C4 / C5-het32 golden) equals the
    pinned Python oracle on instances with <= 8 free devices, k <= 5."""
    text = W.het32_text() if topo_name == "het32" else W.rand_text(32, W.MASTER_SEED)
    t = mo.parse_topology(text)
    rng = random.Random(32 + len(topo_name))
    for trial in range(16):
        free = rng.sample(range(32), rng.randint(4, 8))
        busy = ((1 << 32) - 1) & ~sum(1 << d for d in free)
        shape = rng.choice(["ring", "tree", "ringtree", "full"])
        k = rng.randint(2, min(5, len(free)))
        kk, e = mo.make_pattern(shape, k)
        for sel in ((0, 0), (1, 1), (1, 0)):
            p = mo.allocate(t, busy, kk, e, *sel)
            c = co.allocate(t, busy, kk, e, *sel, nthreads=2)
            assert p["status"] == c["status"] == "ok"
            for f in ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "raw",
                      "distinct"):
                assert p[f] == c[f], (topo_name, trial, sel, f, p[f], c[f])
            assert abs(p["pred_effbw"] - c["pred_effbw"]) <= 1e-9 * max(1.0, abs(p["pred_effbw"]))


def test_replay_trace_spec_sequence():
    """replay_trace on dgx1v: job 0 (ring-4, Greedy) takes a 4-set of maximal
    ring AggBW (brute force over all 4-sets and ring labellings below); with
    {1,2,3,4} busy, job 1 (ring-3) gets {5,7,8} at 125; releasing both
    and allocating job 2 (ring-3) gives the fresh answer {1,3,4} at 125."""
    o = mo.builtin("dgx1v")
    jobs = [dict(shape="ring", k=4, sensitive=0), dict(shape="ring", k=3, sensitive=0),
            dict(shape="ring", k=3, sensitive=0)]
    ops = [(0, 0), (0, 1), (1, 0), (1, 1), (0, 2), (1, 2)]
    pats = {("ring", 4): mo.make_pattern("ring", 4), ("ring", 3): mo.make_pattern("ring", 3)}
    out = mo.replay_trace(o, jobs, ops, pats, "greedy")
    w = _weights(o)
    best4 = max(sum(int(w[p[i], p[(i + 1) % 4]]) for i in range(4)) for p in itertools.permutations(range(8), 4))
    assert out[0]["agg_bw"] == best4
    first = next(S for S in itertools.combinations(range(8), 4)  # lex-smallest 4-set reaching it
                 if max(sum(int(w[p[i], p[(i + 1) % 4]]) for i in range(4)) for p in itertools.permutations(S)) == best4)
    assert out[0]["devices"] == first
    assert tuple(d + 1 for d in out[1]["devices"]) == (5, 7, 8) and out[1]["agg_bw"] == 125
    assert tuple(d + 1 for d in out[2]["devices"]) == (1, 3, 4) and out[2]["agg_bw"] == 125
