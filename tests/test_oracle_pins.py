"""Pins the CPU oracle to values fixed by the paper / SPEC / mathematics
(not to itself).  CPU only.

Each test names the plausible oracle mistake it would catch."""
import itertools
import json
import math
import os
import random
from fractions import Fraction

import pytest

import workloads as W
from oracle import mapa_oracle as mo

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))
DGX = mo.builtin("dgx1v")


def m1(ids):  # 1-based ids -> 0-based mask
    return sum(1 << (i - 1) for i in ids)


def test_table1_and_theta_digits():
    for name, bw in GOLD["table1_bw"].items():
        if name != "cite":
            assert mo.LINK_BW[name] == bw
    assert [str(t) for t in mo.THETA] == [str(Fraction(s)) for s in GOLD["table4_theta"]["theta"]]


def test_link_classes_p261():
    # catches a mis-wired dgx1v (wrong edge class on a paper-named pair)
    for a, b, bw in GOLD["link_classes_dgx1v"]["pairs"]:
        assert DGX.bw(a - 1, b - 1) == bw
        assert DGX.bw(b - 1, a - 1) == bw


def test_triangles_p294():
    # catches a wrong Eq. 1 sum or census classification
    for c in GOLD["triangles_dgx1v"]["cases"]:
        S = [d - 1 for d in c["devices"]]
        E = mo.used_edges(S, mo.make_pattern("ring", 3)[1])
        assert mo.aggregated_bw(DGX, E) == c["agg_bw"]
        assert list(mo.link_census(DGX, E)) == c["census"]
        assert mo.induced_total_bandwidth(DGX, S) == c["agg_bw"]


def test_dgx1v_structure_s94_s103():
    assert mo.induced_total_bandwidth(DGX, range(8)) == GOLD["totals_dgx1v"]["total"]
    for v in range(8):
        others = [DGX.bw(v, u) for u in range(8) if u != v]
        assert others.count(50) == 2 and others.count(25) == 2 and others.count(12) == 3
    for u, v in itertools.combinations(range(8), 2):  # symmetric, classes in Table 1
        assert DGX.bw(u, v) == DGX.bw(v, u) in (50, 25, 20, 12)


def test_eq2_paper_printed_values():
    # catches a sign / coefficient / feature error in the terms active at these censuses
    for c in GOLD["eq2_printed"]["cases"]:
        assert abs(mo.eq2(*c["census"]) - c["value"]) <= c["tol"], c


def test_eq2_spec_values_exact():
    for c in GOLD["eq2_spec"]["cases"]:
        assert mo.eq2_exact(*c["census"]) == Fraction(c["exact"])


def test_eq2_feature_closed_forms():
    """Independent pins of every feature: Eq. 2 is linear in theta, so with
    theta = e_i the model must return feature i (P:616 feature list: linear,
    inverse-linear, pairwise, inverse-pairwise, triplet, inverse-triplet).
    Evaluated at censuses where each feature has a distinct known value."""
    feats = [
        lambda x, y, z: x, lambda x, y, z: y, lambda x, y, z: z,
        lambda x, y, z: Fraction(1, x + 1), lambda x, y, z: Fraction(1, y + 1), lambda x, y, z: Fraction(1, z + 1),
        lambda x, y, z: x * y, lambda x, y, z: y * z, lambda x, y, z: z * x,
        lambda x, y, z: Fraction(1, x * y + 1), lambda x, y, z: Fraction(1, y * z + 1),
        lambda x, y, z: Fraction(1, z * x + 1),
        lambda x, y, z: x * y * z, lambda x, y, z: Fraction(1, x * y * z + 1)]
    for i in range(14):
        th = [Fraction(0)] * 14
        th[i] = Fraction(1)
        for (x, y, z) in [(2, 3, 5), (1, 4, 7), (0, 2, 9)]:
            assert mo.eq2_exact(x, y, z, theta=th) == feats[i](x, y, z), i


def test_eq2_negative_values_kept():
    # SPEC S:303 design decision (raw negative outputs are used for ranking);
    # SPEC's example value is wrong: (0,0,1) is +10.0855, (1,0,5) < 0
    assert mo.eq2_exact(0, 0, 1) == Fraction("10.0855")
    assert mo.eq2(1, 0, 5) < 0


def test_preserved_s283_and_identity():
    for c in GOLD["preserved_dgx1v"]["cases"]:
        assert mo.preserved_bw(DGX, range(8), [d - 1 for d in c["devices"]]) == c["value"]
    # edge-partition identity (acceptance #9): exhaustive, |S| <= 4
    for k in range(0, 5):
        for S in itertools.combinations(range(8), k):
            touch = sum(DGX.bw(u, v) for u, v in itertools.combinations(range(8), 2) if u in S or v in S)
            assert mo.preserved_bw(DGX, range(8), S) + touch == 744


def test_preserved_respects_busy():
    # catches Eq. 3 computed over the whole G instead of the AVAILABLE graph (§3.6)
    free = [0, 1, 2, 5, 6]
    S = [1, 5]
    assert mo.preserved_bw(DGX, free, S) == DGX.bw(0, 2) + DGX.bw(0, 6) + DGX.bw(2, 6)


def test_match_counts_spec_and_closed_forms():
    for c in GOLD["match_counts"]["cases"]:
        k, e = mo.make_pattern(c["shape"], c["k"])
        busy = m1(range(c["free"] + 1, 9))
        ms, raw = mo.find_matches(DGX, busy, k, e)
        assert len(ms) == c["distinct"]
        assert raw == math.perm(c["free"], k)
    # raw = P(|F|,k) for every pattern; edgeless distinct = n!/(n-k)!
    for n_free in range(1, 7):
        busy = m1(range(n_free + 1, 9))
        for k in range(1, n_free + 1):
            ke, ee = mo.make_pattern("edgeless", k)
            ms, raw = mo.find_matches(DGX, busy, ke, ee)
            assert raw == math.perm(n_free, k)
            assert len(ms) == math.comb(n_free, k)  # (S, E=empty): one per set (A2, A12)
            kf, ef = mo.make_pattern("full", k)
            assert len(mo.find_matches(DGX, busy, kf, ef)[0]) == math.comb(n_free, k)
            if k >= 3:
                kr, er = mo.make_pattern("ring", k)
                assert len(mo.find_matches(DGX, busy, kr, er)[0]) == math.perm(n_free, k) // (2 * k)


def test_automorphism_counts_textbook():
    # ring-k: dihedral group 2k; full-k: k!; full binary tree of 7 vertices: 2^3
    for k in range(3, 8):
        assert mo.automorphism_count(*mo.make_pattern("ring", k)) == 2 * k
    for k in range(1, 7):
        assert mo.automorphism_count(*mo.make_pattern("full", k)) == math.factorial(k)
    assert mo.automorphism_count(*mo.make_pattern("tree", 7)) == 8
    assert mo.automorphism_count(*mo.make_pattern("ring", 2)) == 2


def test_orbit_theorem_distinct_equals_raw_over_aut():
    # distinct (S,E) matches = P(|F|,k)/|Aut| (SURVEY §8(c) orbit theorem)
    rng = random.Random(7)
    for shape in ("ring", "tree", "ringtree", "full"):
        for k in range(2, 6):
            busy = rng.randrange(0, 256) & ~0x0F  # keep >= 4 free
            kk, e = mo.make_pattern(shape, k)
            ms, raw = mo.find_matches(DGX, busy, kk, e)
            aut = mo.automorphism_count(kk, e)
            assert raw % aut == 0 and len(ms) == raw // aut


def test_patterns_spec_s146():
    assert mo.make_pattern("ring", 3)[1] == [(0, 1), (0, 2), (1, 2)]
    assert len(mo.make_pattern("ring", 5)[1]) == 5
    assert mo.make_pattern("tree", 5)[1] == [(0, 1), (0, 2), (1, 3), (1, 4)]
    assert mo.make_pattern("ring", 2)[1] == [(0, 1)]
    for n in range(2, 9):
        assert len(mo.make_pattern("full", n)[1]) == n * (n - 1) // 2
        assert len(mo.make_pattern("tree", n)[1]) == n - 1
    with pytest.raises(ValueError):
        mo.make_pattern("ring", 1)


SELS = {"greedy": (mo.GREEDY, False), "sensitive": (mo.PRESERVE, True),
        "insensitive": (mo.PRESERVE, False), "baseline": (mo.BASELINE, False)}


def test_selections_spec_examples():
    for c in GOLD["selections_dgx1v"]["cases"]:
        k, e = mo.make_pattern(c["shape"], c["k"])
        sel, sens = SELS[c["selector"]]
        d = mo.allocate(DGX, m1(c["busy"]), k, e, sel, sens)
        if c.get("no_capacity"):
            assert d["status"] == "no_capacity"
            continue
        assert [x + 1 for x in d["devices"]] == c["devices"], c
        for f in ("agg_bw", "preserved_bw"):
            if f in c:
                assert d[f] == c[f]
        if "pred_effbw" in c:
            assert abs(d["pred_effbw"] - c["pred_effbw"]) < 1e-9


def test_c1_expected_answer():
    """C1: dgx1v ring-3 all free: {1,3,4} under all three
    selectors, census (2,1,0), agg 125, pres 311 = 744 - 3*186 + 125."""
    k, e = mo.make_pattern("ring", 3)
    for sel, sens in SELS.values():
        if sel == mo.BASELINE:
            continue
        d = mo.allocate(DGX, 0, k, e, sel, sens)
        assert [x + 1 for x in d["devices"]] == [1, 3, 4]
        assert (d["x"], d["y"], d["z"]) == (2, 1, 0)
        assert d["agg_bw"] == 125 and d["preserved_bw"] == 744 - 3 * 186 + 125
        assert d["raw"] == 336 and d["distinct"] == 56


def test_ring4_edge_tiebreak():
    g = GOLD["ring4_edge_tiebreak"]
    d = mo.allocate(DGX, 0, *mo.make_pattern("ring", 4), mo.PRESERVE, False)
    assert [x + 1 for x in d["devices"]] == g["devices"]
    assert [x + 1 for x in d["mapping"]] == g["mapping"]
    assert [d["x"], d["y"], d["z"]] == g["census"]
    assert d["agg_bw"] == g["agg_bw"] and d["preserved_bw"] == g["preserved_bw"]


def test_baseline_and_uniform_reduce_to_lowest_ids():
    # P:777 Baseline = lowest free ids; on a uniform topology every score ties
    uni = mo.Topology("uni", 7, {})
    rng = random.Random(3)
    for _ in range(20):
        busy = rng.randrange(0, 128)
        free = mo.free_devices(uni, busy)
        for shape in ("ring", "tree", "full"):
            for k in range(2, min(5, len(free)) + 1):
                kk, e = mo.make_pattern(shape, k)
                for sel, sens in SELS.values():
                    d = mo.allocate(uni, busy, kk, e, sel, sens)
                    assert list(d["devices"]) == free[:k]


def test_optimality_against_exhaustive_max():
    """Policy argmax oracles (SPEC acceptance #5): the chosen score equals the
    max over ALL injective placements scored without dedup (a different
    enumeration: itertools.permutations over F directly)."""
    rng = random.Random(11)
    for _ in range(25):
        busy = rng.randrange(0, 256)
        F = mo.free_devices(DGX, busy)
        shape = rng.choice(["ring", "tree", "full"])
        k = rng.randint(2, 5)
        if k > len(F):
            continue
        kk, e = mo.make_pattern(shape, k)
        best_agg = best_pres = best_eff = None
        for pi in itertools.permutations(F, k):
            E = mo.used_edges(pi, e)
            a = mo.aggregated_bw(DGX, E)
            pr = mo.preserved_bw(DGX, F, pi)
            ef = mo.eq2_exact(*mo.link_census(DGX, E))
            best_agg = a if best_agg is None else max(best_agg, a)
            best_pres = pr if best_pres is None else max(best_pres, pr)
            best_eff = ef if best_eff is None else max(best_eff, ef)
        assert mo.allocate(DGX, busy, kk, e, mo.GREEDY, False)["agg_bw"] == best_agg
        assert mo.allocate(DGX, busy, kk, e, mo.PRESERVE, False)["preserved_bw"] == best_pres
        assert mo.allocate(DGX, busy, kk, e, mo.PRESERVE, True)["pred_effbw_exact"] == best_eff


def test_chosen_subset_of_free_and_deterministic():
    rng = random.Random(5)
    for _ in range(20):
        busy = rng.randrange(0, 256)
        kk, e = mo.make_pattern("tree", 3)
        d1 = mo.allocate(DGX, busy, kk, e, mo.PRESERVE, True)
        d2 = mo.allocate(DGX, busy, kk, e, mo.PRESERVE, True)
        assert d1 == d2
        if d1["status"] == "ok":
            assert mo.device_mask(d1["devices"]) & busy == 0


def test_other_builtins_spec():
    s = mo.builtin("summit")
    assert mo.induced_total_bandwidth(s, range(6)) == 408  # 6x50 + 9x12
    p = mo.builtin("dgx1p")
    assert mo.induced_total_bandwidth(p, range(8)) == 464  # 16x20 + 12x12
    t = mo.builtin("torus2d16")
    assert mo.induced_total_bandwidth(t, range(16)) == 16 * 50 + 16 * 25 + (120 - 32) * 12
    c = mo.builtin("cubemesh16")
    assert mo.induced_total_bandwidth(c, range(16)) == 2 * 8 * 50 + (2 * 8 + 4) * 25 + (120 - 36) * 12
    # dgx1p ring-2 sensitive: only single NVLink1 (y) or PCIe (z) pairs; (0,1,0) wins (A5)
    d = mo.allocate(p, 0, *mo.make_pattern("ring", 2), mo.PRESERVE, True)
    assert (d["x"], d["y"], d["z"]) == (0, 1, 0)
    assert d["pred_effbw_exact"] == Fraction("21.6065")


def test_topology_text_roundtrip():
    t = mo.parse_topology(W.het32_text())
    assert t.n == 32
    assert mo.induced_total_bandwidth(t, range(32)) == 7840  # every device 2x50,2x25,2x20,25x12
    for v in range(32):
        assert sum(t.w[v]) == 490
    with pytest.raises(ValueError):
        mo.parse_topology("devices 4\nlink 1 1 pcie\n")
    with pytest.raises(ValueError):
        mo.parse_topology("devices 4\nlink 1 9 pcie\n")
    with pytest.raises(ValueError):
        mo.parse_topology("devices 4\nlink 1 2 pcie\nlink 2 1 nv2x2\n")
