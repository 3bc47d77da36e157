"""Host side of libmapa through the C-ABI (no GPU, no compute launches):
symbol exports, topology encode, pattern compile (Aut, lex-leader
constraints), Eq. 2 rank tables, key decode and record combine.  Expected
values come from the pinned oracle or from first principles, never from the
CUDA path."""
import ctypes
import itertools
import math
import os
import random
import re

import pytest

import workloads as W
from oracle import mapa_oracle as mo
from tests.keyutil import encode_key, selector_score

import paper_2110_03214_b200 as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "mapa.h")).read()
    names = set(re.findall(r"\b(mapa_\w+)\s*\(", hdr))
    assert len(names) >= 20
    lib = ctypes.CDLL(mp.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
        assert n in mp.EXPORTS, n
    assert mp.version().startswith("mapa-b200")


@pytest.mark.parametrize("name", ["dgx1v", "dgx1p", "summit", "torus2d16", "cubemesh16"])
def test_builtins_equal_oracle(name):
    t = mp.Topology(name)
    o = mo.builtin(name)
    info = t.info()
    assert info["n"] == o.n
    assert info["width"] == (8 if o.n <= 8 else 16 if o.n <= 16 else 32)
    assert info["bw"] == [[0 if u == v else o.w[u][v] for v in range(o.n)] for u in range(o.n)]


def test_text_topologies_equal_oracle():
    for text in (W.het32_text(), W.rand_text(32, W.MASTER_SEED), W.rand_text(13, 5)):
        t = mp.Topology(text=text)
        o = mo.parse_topology(text)
        assert t.info()["bw"] == [[0 if u == v else o.w[u][v] for v in range(o.n)] for u in range(o.n)]


def test_topology_parse_errors():
    with pytest.raises(mp.MapaError) as e:
        mp.Topology(text="devices 4\nlink 1 1 pcie\n")
    assert e.value.status == mp.E_PARSE and "line 2" in str(e.value)
    with pytest.raises(mp.MapaError) as e:
        mp.Topology(text="devices 4\nlink 1 9 nv2x2\n")
    assert e.value.status == mp.E_ID_RANGE
    with pytest.raises(mp.MapaError) as e:
        mp.Topology(text="devices 4\nlink 1 2 nv2x2\nlink 2 1 nv2x1\n")
    assert e.value.status == mp.E_PARSE
    with pytest.raises(mp.MapaError) as e:
        mp.Topology(text="devices 4\nsockets 1,2 2,3,4\n")
    assert e.value.status == mp.E_PARSE
    with pytest.raises(mp.MapaError) as e:
        mp.Topology(text="devices 65\n")
    assert e.value.status == mp.E_UNSUPPORTED
    with pytest.raises(mp.MapaError):
        mp.Topology("dgx2")


def test_state_management_spec_examples():
    t = mp.Topology("dgx1v")
    t.claim(0b11)                       # S:76 allocate {1,2}
    assert t.busy == 0b11
    with pytest.raises(mp.MapaError) as e:
        t.claim(0b1)                    # S:77 double allocation
    assert e.value.status == mp.E_ALREADY_BUSY and t.busy == 0b11
    t.release(0b11)                     # S:85 inverse
    assert t.busy == 0
    with pytest.raises(mp.MapaError) as e:
        t.release(0b100)                # S:86 not busy
    assert e.value.status == mp.E_NOT_BUSY
    t.claim(0b10011)                    # S:87 allocate {1,2,5}, release {2}
    t.release(0b10)
    assert t.busy == 0b10001
    with pytest.raises(mp.MapaError) as e:
        t.claim(1 << 8)
    assert e.value.status == mp.E_ID_RANGE
    t.set_busy(0xFF)                    # S:78 exhaustion
    assert t.busy == 0xFF


@pytest.mark.parametrize("shape", ["ring", "tree", "ringtree", "full", "edgeless"])
def test_patterns_equal_oracle(shape):
    for k in range(1, 9):
        if shape == "ring" and k == 1:
            with pytest.raises(mp.MapaError):
                mp.Pattern.make("ring", 1)
            continue
        p = mp.Pattern.make(shape, k).info()
        kk, e = mo.make_pattern(shape, k)
        assert p["k"] == kk and p["edges"] == e
        if k <= 7:
            assert p["aut"] == mo.automorphism_count(kk, e)


def test_pattern_errors():
    with pytest.raises(mp.MapaError) as e:
        mp.Pattern(4, [(0, 1), (2, 3)])
    assert e.value.status == mp.E_DISCONNECTED
    assert mp.Pattern(4, [(0, 1), (2, 3)], allow_disconnected=True).info()["m"] == 2
    with pytest.raises(mp.MapaError):
        mp.Pattern(3, [(0, 0)])
    with pytest.raises(mp.MapaError):
        mp.Pattern(3, [(0, 1), (1, 0)])
    with pytest.raises(mp.MapaError) as e:
        mp.Pattern(17, [])
    assert e.value.status == mp.E_UNSUPPORTED
    with pytest.raises(mp.MapaError) as e:
        mp.Pattern.make("ring", 17)
    assert e.value.status == mp.E_UNSUPPORTED


def _count_automorphisms(k, edges):
    """|Aut| by exhaustive backtracking over vertex images (every complete
    adjacency-preserving bijection is counted once; no stabiliser chain)."""
    adj = [set() for _ in range(k)]
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    img = [-1] * k

    def go(v, used):
        if v == k:
            return 1
        tot = 0
        for c in range(k):
            if c in used or len(adj[c]) != len(adj[v]):
                continue
            if all((w in adj[v]) == (img[w] in adj[c]) for w in range(v)):
                img[v] = c
                tot += go(v + 1, used | {c})
        return tot

    return go(0, frozenset())


@pytest.mark.parametrize("shape", ["ring", "tree", "ringtree", "full", "edgeless"])
def test_deep_patterns_aut_order(shape):
    """k = 9..16 (deep path): |Aut| from the library's stabiliser chain equals
    the closed forms (ring 2k, full / edgeless k!) and, for sparse shapes, an
    exhaustive automorphism count; edges equal SPEC make_pattern's."""
    for k in range(9, 17):
        p = mp.Pattern.make(shape, k).info()
        kk, e = mo.make_pattern(shape, k)
        assert p["k"] == kk and p["edges"] == e
        if shape == "ring":
            assert p["aut"] == 2 * k
        elif shape in ("full", "edgeless"):
            assert p["aut"] == math.factorial(k)
        else:
            assert p["aut"] == _count_automorphisms(k, e)


def _lex_leader_ok(f, lex_src):
    return all(f[i] < f[u] for u in range(len(f)) for i in range(len(f)) if (lex_src[u] >> i) & 1)


@pytest.mark.parametrize("shape", ["ring", "tree", "ringtree", "full", "edgeless"])
def test_lex_leader_keeps_exactly_the_lexmin_of_each_orbit(shape):
    """Canonical mode's constraint set (host-compiled) keeps exactly one
    mapping per (device set, edge set) class — the lex-min one (reading A1,
    SURVEY §8(c) orbit theorem).  Brute force over all injective maps."""
    for k in range(2 if shape == "ring" else 1, 7):
        p = mp.Pattern.make(shape, k).info()
        n = k + 1
        groups = {}
        for f in itertools.permutations(range(n), k):
            key = (tuple(sorted(f)), tuple(mo.used_edges(f, p["edges"])))
            groups.setdefault(key, []).append(f)
        kept = 0
        for key, fs in groups.items():
            ok = [f for f in fs if _lex_leader_ok(f, p["lex_src"])]
            assert ok == [min(fs)], (shape, k, key)
            kept += 1
        assert kept * p["aut"] == math.perm(n, k)


def test_rank_table_orders_like_exact_eq2():
    for m in range(0, 29):
        tab = mp.effbw_rank_table(m)
        cens = [(x, y, m - x - y) for x in range(m + 1) for y in range(m + 1 - x)]
        by_rank = sorted(cens, key=lambda c: tab[c[0] * (m + 1) + c[1]])
        by_exact = sorted(cens, key=lambda c: mo.eq2_exact(*c))
        assert by_rank == by_exact
        assert sorted(tab[c[0] * (m + 1) + c[1]] for c in cens) == list(range(len(cens)))


def test_pred_effbw_matches_oracle():
    for x, y, z in itertools.product(range(7), repeat=3):
        assert abs(mp.pred_effbw(x, y, z) - float(mo.eq2_exact(x, y, z))) < 1e-9


def _oracle_case(rng, topo_name):
    o = mo.builtin(topo_name)
    busy = rng.randrange(0, 1 << o.n)
    shape = rng.choice(["ring", "tree", "ringtree", "full"])
    k = rng.randint(2, 5)
    sel, sens = rng.choice([(0, False), (1, True), (1, False)])
    return o, busy, shape, k, sel, sens


@pytest.mark.parametrize("topo_name", ["dgx1v", "summit", "cubemesh16"])
def test_decode_recovers_oracle_decision(topo_name):
    """Key encoded (test-side, from the header definition) from the oracle's
    decision -> mapa_decode must give back the oracle's devices, mapping,
    edges, census and scores."""
    rng = random.Random(sum(map(ord, topo_name)))
    t = mp.Topology(topo_name)
    width = t.width
    done = 0
    while done < 25:
        o, busy, shape, k, sel, sens = _oracle_case(rng, topo_name)
        if topo_name == "cubemesh16":
            k = min(k, 4)
        kk, e = mo.make_pattern(shape, k)
        d = mo.allocate(o, busy, kk, e, sel, sens)
        if d["status"] != "ok":
            continue
        pat = mp.Pattern.make(shape, k)
        tab = mp.effbw_rank_table(len(e))
        key = encode_key(d, selector_score(d, sel, sens, tab, len(e)), width, k)
        rec = mp.Record(key=key, leaves=d["distinct"])
        got = mp.decode(t, pat, busy, sel, sens, rec)
        for f in ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "distinct"):
            assert got[f] == d[f], (f, got[f], d[f])
        assert got["raw"] == d["raw"]
        assert abs(got["pred_effbw"] - d["pred_effbw"]) <= 1e-6 * max(1, abs(d["pred_effbw"]))
        done += 1


def test_decode_rejects_inconsistent_key():
    t = mp.Topology("dgx1v")
    pat = mp.Pattern.make("ring", 3)
    good = encode_key(dict(devices=(0, 2, 3), used_edges=[(0, 2), (0, 3), (2, 3)]), 125, 8, 3)
    assert mp.decode(t, pat, 0, 0, False, mp.Record(key=good))["devices"] == (0, 2, 3)
    bad = encode_key(dict(devices=(0, 2, 3), used_edges=[(0, 2), (0, 3), (2, 3)]), 124, 8, 3)
    with pytest.raises(mp.MapaError) as e:
        mp.decode(t, pat, 0, 0, False, mp.Record(key=bad))
    assert e.value.status == mp.E_INTERNAL
    with pytest.raises(mp.MapaError):  # device 0 busy
        mp.decode(t, pat, 1, 0, False, mp.Record(key=good))
    assert mp.decode(t, pat, 0, 0, False, mp.Record(key=0))["status"] == "no_capacity"


def test_reduce_records_max_and_sum():
    recs = [mp.Record(key=5, leaves=10), mp.Record(key=9, leaves=1), mp.Record(key=7, leaves=100)]
    r = mp.reduce_records(recs)
    assert r.key == 9 and r.leaves == 111


def test_decode_trace_recovers_oracle_replay():
    """mapa_decode_trace on keys encoded (test side) from the oracle's replay
    of a 120-job FIFO trace on summit: every decision is decoded against the
    busy mask of its moment and equals the oracle's field by field; raw /
    distinct are the closed forms (§3.6)."""
    jobs = W.c2_jobs(7, 120)
    o = mo.builtin("summit")
    ops = W.fifo_ops(jobs, o.n)
    shapes = sorted({(j["shape"], j["k"]) for j in jobs})
    patd = {sk: mo.make_pattern(*sk) for sk in shapes}
    exp = mo.replay_trace(o, jobs, ops, patd, "preserve")
    t = mp.Topology("summit")
    pats = [mp.Pattern.make(s, k) for s, k in shapes]
    rows = [(shapes.index((j["shape"], j["k"])), 1, j["sensitive"]) for j in jobs]
    keys = []
    for j, job in enumerate(jobs):
        d, m = exp[j], len(patd[(job["shape"], job["k"])][1])
        score = selector_score(d, 1, job["sensitive"], mp.effbw_rank_table(m), m)
        keys.append(encode_key(d, score, t.width, job["k"]))
    got = mp.decode_trace(t, pats, ops, rows, keys)
    for j, d in exp.items():
        for f in ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "raw", "distinct"):
            assert got[j][f] == d[f], (j, f, got[j][f], d[f])
        assert abs(got[j]["pred_effbw"] - d["pred_effbw"]) <= 1e-6 * max(1, abs(d["pred_effbw"]))
    # a key that overlaps a running job is rejected; a zero key is no capacity
    first = [j for op, j in ops if op == 0][:2]
    bad = list(keys)
    bad[first[1]] = keys[first[0]]
    with pytest.raises(mp.MapaError) as e:
        mp.decode_trace(t, pats, ops, rows, bad)
    assert e.value.status == mp.E_INTERNAL
    zero = list(keys)
    zero[first[1]] = 0
    assert mp.decode_trace(t, pats, ops, rows, zero)[first[1]]["status"] == "no_capacity"


def test_shard_queries_lpt():
    """mapa_shard_queries (SURVEY §8(e) batches): every query owned by one rank
    in [0, world); loads = the per-rank sums of P(|F|,k) (RAW) or
    P(|F|,k)/|Aut| (canonical); LPT bound max load <= mean + largest query;
    deterministic; world 1 owns everything."""
    t = mp.Topology("cubemesh16")
    shapes = [(s, k) for s in ("ring", "tree", "full") for k in range(2, 6)]
    pats = [mp.Pattern.make(s, k) for s, k in shapes]
    qs = W.c5_queries(16, count=2000, seed=5)
    pid = {sk: i for i, sk in enumerate(shapes)}
    rows = [(q["busy"], pid[(q["shape"], q["k"])], q["selector"], q["sensitive"]) for q in qs]
    for raw in (True, False):
        work = []
        for q in qs:
            nf = 16 - bin(q["busy"]).count("1")
            w = math.perm(nf, q["k"]) if q["k"] <= nf else 0
            if not raw:
                w //= mo.automorphism_count(*mo.make_pattern(q["shape"], q["k"]))
            work.append(w)
        for world in (1, 2, 3, 8):
            own, load = mp.shard_queries(t, pats, rows, world, raw=raw)
            assert own == mp.shard_queries(t, pats, rows, world, raw=raw)[0]
            assert all(0 <= o < world for o in own)
            exp = [sum(w for w, o in zip(work, own) if o == r) for r in range(world)]
            assert [round(x) for x in load] == exp
            assert max(exp) <= sum(work) / world + max(work)
            if world == 1:
                assert set(own) == {0}
    with pytest.raises(mp.MapaError):
        mp.shard_queries(t, pats, [(0, 99, 0, 0)], 2)
