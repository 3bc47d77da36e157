"""GPU parity of the deep path (esa_deep, 256-bit key, k <= 16; SURVEY §8(f)
NEXT 1) through the C-ABI, against the CPU oracles on the same seeded inputs:
decision fields and counts bit-exact, Eq. 2 double within 1e-6 relative."""
import math
import random

import pytest

import workloads as W
from oracle import coracle as co
from oracle import mapa_oracle as mo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

FIELDS = ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "raw")
SELS = [(0, False), (1, True), (1, False), (2, False)]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.init()


def same(o, g, ctx=""):
    assert o["status"] == g["status"], (ctx, o, g)
    if o["status"] != "ok":
        return
    for f in FIELDS:
        assert o[f] == g[f], (ctx, f, o[f], g[f])
    assert abs(o["pred_effbw"] - g["pred_effbw"]) <= 1e-6 * max(1.0, abs(o["pred_effbw"])), ctx


def deep(t, busy, shape, k, sel, sens, raw):
    t.set_busy(busy)
    return mp.allocate(t, mp.Pattern.make(shape, k), sel, sens, raw=raw, deep=True)


@pytest.mark.parametrize("name", ["dgx1v", "summit", "cubemesh16", "torus2d16"])
def test_deep_kernel_small_k_vs_oracle(name):
    """k <= 7 forced onto the deep kernel (MAPA_F_DEEP): every field and both
    counts equal the narrow C oracle's (itself pinned)."""
    o = mo.builtin(name)
    t = mp.Topology(name)
    rng = random.Random(4242 + len(name))
    for trial in range(40):
        shape = rng.choice(["ring", "tree", "ringtree", "full", "edgeless"])
        k = rng.randint(2 if shape == "ring" else 1, min(o.n, 7 if o.n <= 8 else 6))
        busy = rng.randrange(0, 1 << o.n)
        if o.n > 8:
            busy |= (1 << rng.randint(0, 5)) - 1
        sel, sens = rng.choice(SELS)
        raw = bool(trial & 1)
        kk, e = mo.make_pattern(shape, k)
        ob = co.allocate(o, busy, kk, e, sel, sens)
        g = deep(t, busy, shape, k, sel, sens, raw)
        same(ob, g, (name, trial, shape, k, hex(busy), sel, sens, raw))
        if ob["status"] == "ok":
            assert g["raw"] == ob["raw"] and g["distinct"] == ob["distinct"]
            assert g["leaves"] == (ob["raw"] if raw else ob["distinct"])


def test_deep_equals_narrow_kernel_n32():
    """N = 32 (het32 / rand32), k <= 6, random busy: the deep kernel's decision
    equals the narrow kernel's (parity-tested against the oracle) field by field."""
    rng = random.Random(99)
    for text in (W.het32_text(), W.rand_text(32, W.MASTER_SEED)):
        t = mp.Topology(text=text)
        for trial in range(16):
            shape = rng.choice(["ring", "tree", "ringtree", "full"])
            k = rng.randint(3, 6)
            busy = sum(1 << d for d in rng.sample(range(32), rng.randint(0, 20)))
            sel, sens = rng.choice(SELS)
            raw = bool(trial & 1)
            t.set_busy(busy)
            p = mp.Pattern.make(shape, k)
            a = mp.allocate(t, p, sel, sens, raw=raw)
            b = mp.allocate(t, p, sel, sens, raw=raw, deep=True)
            for f in FIELDS + ("distinct", "leaves", "pred_effbw"):
                assert a[f] == b[f], (trial, shape, k, hex(busy), sel, sens, raw, f, a[f], b[f])


@pytest.mark.parametrize("k", [9, 10, 11])
def test_deep_k_vs_deep_oracle(k):
    """k = 9..11 on the 16-GPU graphs with |F| in {k, k+1} (ragged): decision
    fields and raw counts equal the deep C oracle's; canonical leaves =
    raw / |Aut| (orbit theorem)."""
    rng = random.Random(1000 + k)
    for name in ("cubemesh16", "torus2d16"):
        o = mo.builtin(name)
        t = mp.Topology(name)
        for shape in ("ring", "tree", "ringtree", "full"):
            nf = k + (rng.randint(0, 1) if k < 11 else 0)
            busy = sum(1 << d for d in rng.sample(range(16), 16 - nf))
            sel, sens = rng.choice(SELS[:3])
            kk, e = mo.make_pattern(shape, k)
            ob = co.allocate_deep(o, busy, kk, e, sel, sens)
            aut = mp.Pattern.make(shape, k).info()["aut"]
            for raw in (False, True):
                g = deep(t, busy, shape, k, sel, sens, raw)
                same(ob, g, (name, shape, k, hex(busy), sel, sens, raw))
                assert g["raw"] == ob["raw"] == math.perm(nf, k)
                assert g["leaves"] == (ob["raw"] if raw else ob["raw"] // aut)


def test_deep_k12_16_counts_and_validity():
    """k = 12..16 (the paper's "9 GPUs and above" on 16-GPU graphs):
    canonical leaves = P(|F|,k)/|Aut|, the decision uses only free devices,
    the mapping is a permutation of them and the decoded scores re-verify
    (decode self-check); RAW mode returns the same decision."""
    t = mp.Topology("cubemesh16")
    for shape, k, nfree in (("ring", 12, 13), ("full", 14, 16), ("ring", 16, 16), ("tree", 15, 15),
                            ("ringtree", 13, 14), ("ringtree", 13, 13)):
        p = mp.Pattern.make(shape, k)
        aut = p.info()["aut"]
        busy = ((1 << 16) - 1) & ~((1 << nfree) - 1)
        t.set_busy(busy)
        leaves = math.perm(nfree, k) // aut
        if leaves > 3e10:
            continue
        for sel, sens in SELS[:3]:
            g = mp.allocate(t, p, sel, sens)
            assert g["status"] == "ok"
            assert g["leaves"] == leaves, (shape, k)
            assert len(g["devices"]) == k and sorted(g["mapping"]) == list(g["devices"])
            assert not set(g["devices"]) & {d for d in range(16) if (busy >> d) & 1}
    p = mp.Pattern.make("ring", 11)
    t.set_busy(0b111 << 13)  # 13 free: raw P(13,11) = 3.1e9
    for sel, sens in SELS[:3]:
        a = mp.allocate(t, p, sel, sens)
        b = mp.allocate(t, p, sel, sens, raw=True)
        for f in FIELDS + ("pred_effbw",):
            assert a[f] == b[f], (sel, sens, f)
        assert b["leaves"] == math.perm(13, 11)


def test_deep_full_clique_vs_subset_bruteforce():
    """full-k (clique): one orbit per device set, so the oracle decision is the
    best k-subset by (score, lex-smallest) — a plain subset brute force with
    itertools.combinations (SURVEY §8(c) C4 pin, applied at k = 12, N = 16)."""
    import itertools
    o = mo.builtin("torus2d16")
    t = mp.Topology("torus2d16")
    t.set_busy(0)
    k = 12
    for sel, sens in SELS[:3]:
        best = None
        for S in itertools.combinations(range(16), k):
            E = [(a, b) for a, b in itertools.combinations(S, 2)]
            x, y, z = mo.link_census(o, E)
            if sel == 0:
                s = mo.aggregated_bw(o, E)
            elif sens:
                s = mo.eq2_exact(x, y, z)
            else:
                s = mo.preserved_bw(o, range(16), S)
            if best is None or s > best[0]:
                best = (s, S, (x, y, z))
        g = mp.allocate(t, mp.Pattern.make("full", k), sel, sens)
        assert g["devices"] == best[1] and (g["x"], g["y"], g["z"]) == best[2], (sel, sens)
        assert g["mapping"] == best[1]


def test_deep_sharded_virtual_ranks_and_determinism():
    """Shards r = 0..R-1 of one deep query combine (lexicographic 256-bit max,
    sum of leaves) to the unsharded record for R = 1, 2, 3, 5; repeated runs
    give identical records; on 11 free devices the combined 3-rank record
    decodes to the deep C oracle's decision."""
    t = mp.Topology("cubemesh16")
    o = mo.builtin("cubemesh16")
    busy = 0b0000000000100001
    for shape, k, sel, sens in (("ring", 10, 0, False), ("tree", 11, 1, True), ("ringtree", 9, 1, False)):
        p = mp.Pattern.make(shape, k)
        # 11 free devices for the oracle comparison of the combined shards
        ob = 0b1000110000100001
        kk, ee = mo.make_pattern(shape, k)
        exp = co.allocate_deep(o, ob, kk, ee, sel, sens)
        recs = []
        for rank in range(3):
            rec, _q = md.run_query_wide(t, p, sel, sens, ob, rank=rank, world=3)
            torch.cuda.synchronize()
            recs.append(md.wide_records_from_tensor(rec)[0])
        same(exp, mp.decode_wide(t, p, ob, sel, sens, mp.reduce_wide_records(recs)), (shape, k, "world 3 vs oracle"))
        ref = None
        for world in (1, 2, 3, 5):
            recs = []
            for rank in range(world):
                rec, _q = md.run_query_wide(t, p, sel, sens, busy, rank=rank, world=world)
                torch.cuda.synchronize()
                recs.append(md.wide_records_from_tensor(rec)[0])
            comb = mp.reduce_wide_records(recs)
            if ref is None:
                ref = comb
            assert (comb.score, comb.set, comb.ecode_hi, comb.ecode_lo, comb.leaves) == \
                (ref.score, ref.set, ref.ecode_hi, ref.ecode_lo, ref.leaves), (shape, k, world)
        d = mp.decode_wide(t, p, busy, sel, sens, ref)
        t.set_busy(busy)
        assert mp.allocate(t, p, sel, sens)["key"] == d["key"]


def test_deep_edge_cases():
    t = mp.Topology("cubemesh16")
    # no capacity through the deep path
    t.set_busy((1 << 16) - 1 - 0xFF)
    assert mp.allocate(t, mp.Pattern.make("ring", 9), 0, False)["status"] == "no_capacity"
    # k == |F| = 16 canonical tree, and k = 16 edgeless (|Aut| = 16!: a single leaf)
    t.set_busy(0)
    g = mp.allocate(t, mp.Pattern.make("edgeless", 16), 1, False)
    assert g["devices"] == tuple(range(16)) and g["leaves"] == 1 and g["preserved_bw"] == 0
    # N = 32 with k = 9 (key wider than 63 bits there: deep path automatically)
    text = W.het32_text()
    o32, t32 = mo.parse_topology(text), mp.Topology(text=text)
    busy = ((1 << 32) - 1) & ~sum(1 << d for d in (0, 3, 7, 9, 14, 18, 21, 25, 29, 31))
    kk, e = mo.make_pattern("ring", 9)
    for sel, sens in SELS:
        ob = co.allocate_deep(o32, busy, kk, e, sel, sens)
        t32.set_busy(busy)
        same(ob, mp.allocate(t32, mp.Pattern.make("ring", 9), sel, sens), (sel, sens))


def test_deep_n64_vs_deep_oracle():
    """N = 64 (het64: 8 dgx1v islands) on the deep path
    with u64 masks and the 256-bit key: random busy masks leaving 9..11 free
    devices spread over both halves of the id space, k = 3..9, every selector,
    RAW and canonical, vs the deep C oracle."""
    text = W.het64_text()
    o = mo.parse_topology(text)
    t = mp.Topology(text=text)
    assert t.n == 64 and t.width == 64
    rng = random.Random(6464)
    for trial in range(16):
        nf = rng.randint(9, 11)
        free = rng.sample(range(64), nf)
        busy = ((1 << 64) - 1) & ~sum(1 << d for d in free)
        shape = rng.choice(["ring", "tree", "ringtree", "full"])
        k = rng.randint(3, 9 if nf <= 10 else 8)
        sel, sens = rng.choice(SELS)
        kk, e = mo.make_pattern(shape, k)
        ob = co.allocate_deep(o, busy, kk, e, sel, sens)
        for raw in (False, True):
            t.set_busy(busy)
            g = mp.allocate(t, mp.Pattern.make(shape, k), sel, sens, raw=raw)
            same(ob, g, (trial, shape, k, hex(busy), sel, sens, raw))
            assert g["raw"] == ob["raw"] == math.perm(nf, k)


def test_deep_n64_all_free_clique_and_narrow_refusal():
    """het64 all free, full-4: 635,376 device sets (one orbit each), vs the
    deep C oracle over every subset; the narrow entry point refuses N > 32."""
    text = W.het64_text()
    o = mo.parse_topology(text)
    t = mp.Topology(text=text)
    kk, e = mo.make_pattern("full", 4)
    for sel, sens in SELS[:3]:
        ob = co.allocate_deep(o, 0, kk, e, sel, sens, max_subsets=700000)
        g = mp.allocate(t, mp.Pattern.make("full", 4), sel, sens)
        same(ob, g, (sel, sens))
        assert g["leaves"] == math.comb(64, 4)
    q, rec = md.query_tensor(0), torch.zeros(4, dtype=torch.int64, device="cuda")
    with pytest.raises(mp.MapaError) as ei:
        mp.launch_query(t, mp.Pattern.make("ring", 3), 0, False, q.data_ptr(), rec.data_ptr(), busy_hint=0)
    assert ei.value.status == mp.E_UNSUPPORTED


def test_deep_prune_equals_exhaustive():
    """Deep branch and bound (MAPA_F_PRUNE: Greedy's Eq. 1 bounds, Preserve-
    sensitive's Eq. 2 rank bounds; Preserve-insensitive routes to the set
    search): the decision equals the
    exhaustive deep search's and the deep C oracle's (small cases), fewer leaves
    are scored, and raw / distinct are the closed forms."""
    rng = random.Random(2024)
    for name in ("cubemesh16", "torus2d16"):
        o = mo.builtin(name)
        t = mp.Topology(name)
        for shape, k in (("ring", 9), ("tree", 10), ("ringtree", 11), ("ring", 12), ("full", 9), ("ring", 5)):
            busy = sum(1 << d for d in rng.sample(range(16), rng.randint(0, 16 - k)))
            nf = 16 - bin(busy).count("1")
            p = mp.Pattern.make(shape, k)
            t.set_busy(busy)
            for sel, sens in ((0, False), (1, False), (1, True)):
                for raw in (False, True):
                    if raw and math.perm(nf, k) > 3e10:
                        continue
                    ex = mp.allocate(t, p, sel, sens, raw=raw, deep=True)
                    pr = mp.allocate(t, p, sel, sens, raw=raw, deep=True, prune=True)
                    for f in FIELDS + ("distinct", "pred_effbw", "key", "ecode"):
                        assert pr[f] == ex[f], (name, shape, k, hex(busy), sel, raw, f)
                    if sel == 0 or sens:
                        assert pr["leaves"] <= ex["leaves"]
                if math.perm(nf, k) <= 2e7:
                    kk, e = mo.make_pattern(shape, k)
                    same(co.allocate_deep(o, busy, kk, e, sel, sens, max_subsets=200000), pr,
                         (name, shape, k, hex(busy), sel))


def test_deep_prune_n64_and_sharded():
    """Branch and bound on het64 (u64 masks) and across virtual ranks: the
    combined pruned record decodes to the exhaustive decision."""
    text = W.het64_text()
    t = mp.Topology(text=text)
    busy = ((1 << 64) - 1) & ~sum(1 << d for d in (1, 5, 9, 12, 20, 33, 40, 41, 47, 50, 58, 63))
    p = mp.Pattern.make("ring", 10)
    t.set_busy(busy)
    ex = mp.allocate(t, p, 0, False, deep=True)
    pr = mp.allocate(t, p, 0, False, deep=True, prune=True)
    for f in FIELDS + ("key", "ecode"):
        assert pr[f] == ex[f], f
    ex_s = mp.allocate(t, p, 1, True, deep=True)
    pr_s = mp.allocate(t, p, 1, True, deep=True, prune=True)
    for f in FIELDS + ("key", "ecode", "pred_effbw", "distinct"):
        assert pr_s[f] == ex_s[f], f
    for sel, sens, want in ((0, False, ex), (1, True, ex_s)):
        recs = []
        for rank in range(3):
            q = md.query64_tensor(busy, sel, sens)
            rec = torch.zeros(8, dtype=torch.int64, device="cuda")
            mp.launch_query_wide(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), busy, rank=rank, world=3,
                                 prune=True)
            torch.cuda.synchronize()
            recs.append(md.wide_records_from_tensor(rec)[0])
        d = mp.decode_wide(t, p, busy, sel, sens, mp.reduce_wide_records(recs), prune=True)
        for f in FIELDS + ("key", "ecode", "distinct"):
            assert d[f] == want[f], (sel, f)


def test_deep_insensitive_set_search_equals_exhaustive():
    """Preserve-insensitive with MAPA_F_PRUNE on the deep path: best set by the
    full-k pattern + the pattern's cached lex-smallest labelling; every field
    equals the exhaustive deep search's and (small cases) the deep oracle's."""
    rng = random.Random(77)
    for name in ("cubemesh16", "torus2d16"):
        o = mo.builtin(name)
        t = mp.Topology(name)
        for shape, k in (("ring", 9), ("tree", 10), ("ringtree", 11), ("ring", 12), ("tree", 9)):
            busy = sum(1 << d for d in rng.sample(range(16), rng.randint(0, 16 - k)))
            nf = 16 - bin(busy).count("1")
            p = mp.Pattern.make(shape, k)
            t.set_busy(busy)
            ex = mp.allocate(t, p, 1, False, deep=True)
            for raw in (False, True, False):  # later calls: cached labelling; RAW changes nothing
                fa = mp.allocate(t, p, 1, False, deep=True, prune=True, raw=raw)
                for f in FIELDS + ("distinct", "pred_effbw", "key", "ecode"):
                    assert fa[f] == ex[f], (name, shape, k, hex(busy), f, fa[f], ex[f])
            if math.perm(nf, k) <= 2e7:
                kk, e = mo.make_pattern(shape, k)
                same(co.allocate_deep(o, busy, kk, e, 1, False, max_subsets=200000), fa, (name, shape, k, hex(busy)))


def test_deep_baseline_set_shortcut_equals_exhaustive():
    """Baseline with MAPA_F_PRUNE on the deep path: the k lowest free ids and
    the pattern's lex-smallest labelling, equal to the exhaustive deep search
    (every leaf ties there) and to the deep oracle."""
    rng = random.Random(5)
    o, t = mo.builtin("torus2d16"), mp.Topology("torus2d16")
    for shape, k in (("ring", 9), ("tree", 9), ("ringtree", 10)):
        busy = sum(1 << d for d in rng.sample(range(16), 16 - k))  # exactly k free: exhaustive stays small
        t.set_busy(busy)
        p = mp.Pattern.make(shape, k)
        ex = mp.allocate(t, p, 2, False, deep=True)
        fa = mp.allocate(t, p, 2, False, deep=True, prune=True)
        for f in FIELDS + ("distinct", "key", "ecode"):
            assert fa[f] == ex[f], (shape, k, f)
        kk, e = mo.make_pattern(shape, k)
        same(co.allocate_deep(o, busy, kk, e, 2, False), fa, (shape, k))


def test_deep_prune_forced_set_ties():
    """Exactly k free devices (the set is forced, every top-score leaf ties on
    it and the edge code decides): the pruned decision equals the exhaustive
    deep search's for Greedy and Preserve-sensitive, N = 16 and 32, RAW and
    canonical, and k = N = 16 all free."""
    rng = random.Random(31)
    cases = [("cubemesh16", None), ("torus2d16", None), ("het32", W.het32_text())]
    for name, text in cases:
        t = mp.Topology(text=text) if text else mp.Topology(name)
        n = 32 if text else 16
        for shape, k in (("ring", 10), ("tree", 11), ("ringtree", 12), ("ring", 12)):
            free = rng.sample(range(n), k)
            busy = ((1 << n) - 1) & ~sum(1 << d for d in free)
            t.set_busy(busy)
            p = mp.Pattern.make(shape, k)
            for sel, sens in ((0, False), (1, True)):
                for raw in (False, True):
                    ex = mp.allocate(t, p, sel, sens, raw=raw, deep=True)
                    pr = mp.allocate(t, p, sel, sens, raw=raw, deep=True, prune=True)
                    for f in FIELDS + ("distinct", "pred_effbw", "key", "ecode"):
                        assert pr[f] == ex[f], (name, shape, k, hex(busy), sel, raw, f)
    t = mp.Topology("torus2d16")
    p = mp.Pattern.make("ring", 16)
    ex = mp.allocate(t, p, 1, True, deep=True)
    pr = mp.allocate(t, p, 1, True, deep=True, prune=True)
    for f in FIELDS + ("distinct", "pred_effbw", "key", "ecode"):
        assert pr[f] == ex[f], ("ring16", f)
    assert pr["leaves"] < ex["leaves"]


def test_deep_k12_13_vs_oracle_golden(golden_dir):
    """k = 12 and 13 NON-clique patterns (ring / tree / ringtree) on the
    16-GPU graphs with exactly k or k+1 free devices: every decision field of
    the deep path (RAW and canonical) equals the deep C oracle's, stored in
    tests/golden/deep_k12_13.json by tests/golden/make_golden_deep.py (oracle/
    only; 12! = 4.8e8 and 13! = 6.2e9 permutations per case); canonical
    leaves = raw / |Aut| (orbit theorem)."""
    import json
    import os
    path = os.path.join(golden_dir, "deep_k12_13.json")
    if not os.path.exists(path):
        pytest.skip("deep golden not generated")
    cases = json.load(open(path))["cases"]
    assert len(cases) == 16
    tops = {n: mp.Topology(n) for n in ("cubemesh16", "torus2d16")}
    for c in cases:
        t = tops[c["topology"]]
        p = mp.Pattern.make(c["shape"], c["k"])
        exp = dict(c, devices=tuple(c["devices"]), mapping=tuple(c["mapping"]),
                   used_edges=[tuple(e) for e in c["used_edges"]])
        nf = 16 - bin(c["busy"]).count("1")
        assert exp["raw"] == math.perm(nf, c["k"])
        t.set_busy(c["busy"])
        for raw in (False, True):
            g = mp.allocate(t, p, c["selector"], bool(c["sensitive"]), raw=raw)
            same(exp, g, (c["topology"], c["shape"], c["k"], nf, c["selector"], c["sensitive"], raw))
            assert g["leaves"] == (exp["raw"] if raw else exp["raw"] // p.info()["aut"])
