"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle, element by
element on the same seeded inputs (decision fields and counts bit-exact,
Eq. 2 double within 1e-6 relative — north_star tolerance)."""
import itertools
import json
import math
import os
import random

import pytest

import workloads as W
from oracle import coracle as co
from oracle import mapa_oracle as mo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

FIELDS = ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "raw", "distinct")
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


def gpu(topo: mp.Topology, busy, shape, k, sel, sens, raw):
    topo.set_busy(busy)
    return mp.allocate(topo, mp.Pattern.make(shape, k), sel, sens, raw=raw)


def oracle(o, busy, shape, k, sel, sens, use_c=False):
    kk, e = mo.make_pattern(shape, k)
    if use_c:
        return co.allocate(o, busy, kk, e, sel, sens)
    return mo.allocate(o, busy, kk, e, sel, sens)


def test_c1_expected_answer():
    """C1: dgx1v ring-3 all free -> {1,3,4} (1-based), (2,1,0), 125, 311,
    57.857167; raw 336 / distinct 56 in both modes."""
    t = mp.Topology("dgx1v")
    o = mo.builtin("dgx1v")
    for sel, sens in SELS:
        for raw in (False, True):
            g = gpu(t, 0, "ring", 3, sel, sens, raw)
            same(oracle(o, 0, "ring", 3, sel, sens), g, (sel, sens, raw))
            assert g["leaves"] == (336 if raw else 56)
            if sel != 2:
                assert g["devices"] == (0, 2, 3)


@pytest.mark.parametrize("name", ["dgx1v", "dgx1p", "summit", "torus2d16", "cubemesh16"])
def test_random_small_vs_oracle(name):
    o = mo.builtin(name)
    t = mp.Topology(name)
    rng = random.Random(sum(map(ord, name)) * 7)
    ntr = 60 if o.n <= 8 else 40
    for trial in range(ntr):
        shape = rng.choice(["ring", "tree", "ringtree", "full"])
        k = rng.randint(2 if shape == "ring" else 1, 6 if o.n <= 8 else 5)
        busy = rng.randrange(0, 1 << o.n)
        if o.n > 8:  # keep the python-free C oracle fast
            busy |= (1 << rng.randint(0, 3)) - 1
        sel, sens = rng.choice(SELS)
        raw = bool(trial & 1)
        g = gpu(t, busy, shape, k, sel, sens, raw)
        ob = oracle(o, busy, shape, k, sel, sens, use_c=True)
        same(ob, g, (name, trial, shape, k, hex(busy), sel, sens, raw))
        if ob["status"] == "ok":
            assert g["leaves"] == (ob["raw"] if raw else ob["distinct"])


def test_text_topologies_vs_oracle():
    rng = random.Random(1234)
    for text in (W.rand_text(8, 3), W.rand_text(13, 4), W.rand_text(21, 5), W.het32_text(),
                 W.rand_text(32, W.MASTER_SEED)):
        o = mo.parse_topology(text)
        t = mp.Topology(text=text)
        for trial in range(12):
            shape = rng.choice(["ring", "tree", "ringtree", "full"])
            k = rng.randint(2, 4 if o.n > 16 else 5)
            nb = max(0, o.n - rng.randint(k, min(o.n, 12)))
            busy = sum(1 << d for d in rng.sample(range(o.n), nb))
            sel, sens = rng.choice(SELS)
            raw = bool(trial & 1)
            same(oracle(o, busy, shape, k, sel, sens, use_c=True), gpu(t, busy, shape, k, sel, sens, raw),
                 (o.name, trial, shape, k, hex(busy), sel, sens, raw))


def test_large_k_vs_oracle():
    """k = 7, 8 (key budget holds for W <= 16), ragged free sets."""
    rng = random.Random(77)
    for name in ("dgx1v", "cubemesh16", "torus2d16"):
        o = mo.builtin(name)
        t = mp.Topology(name)
        for k in (7, 8):
            for shape in ("ring", "tree", "full"):
                nf = min(o.n, k + rng.randint(0, 1))
                busy = sum(1 << d for d in rng.sample(range(o.n), o.n - nf))
                sel, sens = rng.choice(SELS[:3])
                for raw in (False, True):
                    same(oracle(o, busy, shape, k, sel, sens, use_c=True), gpu(t, busy, shape, k, sel, sens, raw),
                         (name, k, shape, hex(busy), sel, sens, raw))


def test_edge_cases():
    o = mo.builtin("dgx1v")
    t = mp.Topology("dgx1v")
    # no capacity
    assert gpu(t, 0b11111110, "ring", 2, 0, False, False)["status"] == "no_capacity"
    assert gpu(t, 0xFF, "full", 1, 0, False, True)["status"] == "no_capacity"
    # k == |F|, k = 1, empty pattern on many devices
    for busy in (0b00001111, 0b10100101, 0):
        for shape, k in (("full", 4), ("tree", 4), ("full", 1), ("edgeless", 3)):
            for sel, sens in SELS:
                for raw in (False, True):
                    same(oracle(o, busy, shape, k, sel, sens), gpu(t, busy, shape, k, sel, sens, raw),
                         (hex(busy), shape, k, sel, sens, raw))
    # N = 32 with the top device free / busy
    text = W.het32_text()
    o32, t32 = mo.parse_topology(text), mp.Topology(text=text)
    for busy in (0x7FFFFFF0 ^ 0x00F0F000, 0xFFFFFF00 ^ 0x80000000, 0x0FFFFFFF):
        for sel, sens in SELS:
            same(oracle(o32, busy, "ring", 3, sel, sens, use_c=True), gpu(t32, busy, "ring", 3, sel, sens, True))


def test_unsupported_key_budget():
    """ring-8 on 32 devices needs 15 + 32 + 28 > 63 key bits: the narrow
    entry point refuses it; mapa_allocate routes it to the deep path."""
    t = mp.Topology(text=W.het32_text())
    p = mp.Pattern.make("ring", 8)
    q, rec = md.query_tensor(0), torch.zeros(4, dtype=torch.int64, device="cuda")
    with pytest.raises(mp.MapaError) as e:
        mp.launch_query(t, p, 0, False, q.data_ptr(), rec.data_ptr(), busy_hint=0)
    assert e.value.status == mp.E_UNSUPPORTED
    t.set_busy(((1 << 32) - 1) & ~0x3FF)  # 10 free: P(10,8)/16 canonical leaves
    d = mp.allocate(t, p, 0, False)
    assert d["status"] == "ok" and d["leaves"] == 1814400 // 16


def test_commit_and_release_roundtrip():
    t = mp.Topology("dgx1v")
    p = mp.Pattern.make("ring", 3)
    d1 = mp.allocate(t, p, 0, False, commit=True)
    assert t.busy == sum(1 << d for d in d1["devices"])
    d2 = mp.allocate(t, p, 0, False, commit=True)
    assert d2["devices"] == (4, 6, 7)  # S:354 analogue: next best triangle {5,7,8}
    t.release(sum(1 << d for d in d1["devices"]))
    assert t.busy == sum(1 << d for d in d2["devices"])


def test_sharded_virtual_ranks_equal_unsharded():
    """Sharding by work item (rank = i % world) + max/sum combine gives the
    unsharded record for every world size (S:369 determinism), and the
    combined record decodes to the C oracle's decision."""
    text = W.rand_text(32, W.MASTER_SEED)
    t = mp.Topology(text=text)
    o = mo.parse_topology(text)
    for shape, k, busy in (("full", 5, 0), ("ring", 5, 0x0000FF00), ("tree", 6, 0xF0F0F0F0)):
        pat = mp.Pattern.make(shape, k)
        kk, ee = mo.make_pattern(shape, k)
        for sel, sens in SELS[:3]:
            exp = co.allocate(o, busy, kk, ee, sel, sens)
            for raw in (True, False):
                ref, _ = md.run_query(t, pat, sel, sens, busy, raw=raw)
                torch.cuda.synchronize()
                ref = md.records_from_tensor(ref)[0]
                for world in (2, 3, 8):
                    recs = []
                    for r in range(world):
                        rt, _ = md.run_query(t, pat, sel, sens, busy, raw=raw, rank=r, world=world)
                        torch.cuda.synchronize()
                        recs.append(md.records_from_tensor(rt)[0])
                    comb = mp.reduce_records(recs)
                    assert comb.key == ref.key and comb.leaves == ref.leaves, (shape, k, world, raw)
                    # the combined shards decode to the oracle's decision
                    same(exp, mp.decode(t, pat, busy, sel, sens, comb, raw=raw), (shape, k, world, raw))
                d = mp.decode(t, pat, busy, sel, sens, ref, raw=raw)
                nf = 32 - bin(busy).count("1")
                assert d["raw"] == math.perm(nf, k)


def test_determinism_repeat():
    t = mp.Topology(text=W.het32_text())
    pat = mp.Pattern.make("tree", 5)
    keys = {mp.allocate(t, pat, 1, False, raw=True)["key"] for _ in range(5)}
    assert len(keys) == 1


def test_c4_full_size_golden(golden_dir):
    """C4 at full size in the bench launch configuration: het32 / rand32,
    full-6, all free, RAW mode (652,458,240 embeddings) vs the oracle's
    decisions (tests/golden/make_golden.py, oracle/ only)."""
    gold = json.load(open(os.path.join(golden_dir, "c4_expected.json")))
    tops = {"het32": W.het32_text(), "rand32_2110": W.rand_text(32, W.MASTER_SEED)}
    sel_of = {"greedy": (0, False), "sensitive": (1, True), "insensitive": (1, False)}
    pat = mp.Pattern.make("full", 6)
    for case in gold["cases"]:
        t = mp.Topology(text=tops[case["topology"]])
        sel, sens = sel_of[case["selector"]]
        for raw in (True, False):
            g = mp.allocate(t, pat, sel, sens, raw=raw)
            exp = dict(case)
            exp["devices"] = tuple(exp["devices"])
            exp["mapping"] = tuple(exp["mapping"])
            exp["used_edges"] = [tuple(e) for e in exp["used_edges"]]
            same(exp, g, (case["topology"], case["selector"], raw))
            assert g["leaves"] == (652458240 if raw else 906192)


# ---------------------------------------------------------------- MAPA_F_PRUNE
# Branch-and-bound mode: the same decision as the
# exhaustive search (the bound is exact and the test strict), fewer leaves
# scored; raw / distinct are then the closed forms.


@pytest.mark.parametrize("name", ["dgx1v", "cubemesh16", "torus2d16"])
def test_prune_random_vs_oracle(name):
    o = mo.builtin(name)
    t = mp.Topology(name)
    rng = random.Random(sum(map(ord, name)) * 11 + 5)
    for trial in range(36):
        shape = rng.choice(["ring", "tree", "ringtree", "full"])
        k = rng.randint(4, 6 if o.n <= 8 else 5)
        busy = rng.randrange(0, 1 << o.n) & rng.randrange(0, 1 << o.n)
        if o.n > 8:
            busy |= (1 << rng.randint(0, 3)) - 1
        sel, sens = rng.choice(SELS)
        raw = bool(trial & 1)
        t.set_busy(busy)
        g = mp.allocate(t, mp.Pattern.make(shape, k), sel, sens, raw=raw, prune=True)
        ob = oracle(o, busy, shape, k, sel, sens, use_c=True)
        same(ob, g, (name, trial, shape, k, hex(busy), sel, sens, raw))
        if ob["status"] == "ok":
            assert g["leaves"] <= (ob["raw"] if raw else ob["distinct"])


def test_prune_text_topologies_vs_oracle():
    rng = random.Random(4321)
    for text in (W.rand_text(13, 4), W.rand_text(21, 5), W.het32_text(), W.rand_text(32, W.MASTER_SEED)):
        o = mo.parse_topology(text)
        t = mp.Topology(text=text)
        for trial in range(10):
            shape = rng.choice(["ring", "tree", "ringtree", "full"])
            k = rng.randint(4, 5)
            nb = max(0, o.n - rng.randint(k, min(o.n, 12)))
            busy = sum(1 << d for d in rng.sample(range(o.n), nb))
            sel, sens = rng.choice(SELS)
            raw = bool(trial & 1)
            t.set_busy(busy)
            g = mp.allocate(t, mp.Pattern.make(shape, k), sel, sens, raw=raw, prune=True)
            same(oracle(o, busy, shape, k, sel, sens, use_c=True), g, (o.name, trial, shape, k, hex(busy), sel, sens))


def test_prune_c4_full_size_golden(golden_dir):
    """C4 full size with MAPA_F_PRUNE: the golden decisions, raw / distinct
    the closed forms, strictly fewer leaves scored than the exhaustive count."""
    gold = json.load(open(os.path.join(golden_dir, "c4_expected.json")))
    tops = {"het32": W.het32_text(), "rand32_2110": W.rand_text(32, W.MASTER_SEED)}
    sel_of = {"greedy": (0, False), "sensitive": (1, True), "insensitive": (1, False)}
    pat = mp.Pattern.make("full", 6)
    for case in gold["cases"]:
        t = mp.Topology(text=tops[case["topology"]])
        sel, sens = sel_of[case["selector"]]
        for raw in (True, False):
            g = mp.allocate(t, pat, sel, sens, raw=raw, prune=True)
            exp = dict(case)
            exp["devices"] = tuple(exp["devices"])
            exp["mapping"] = tuple(exp["mapping"])
            exp["used_edges"] = [tuple(e) for e in exp["used_edges"]]
            same(exp, g, (case["topology"], case["selector"], raw, "prune"))
            assert g["raw"] == 652458240 and g["distinct"] == 906192
            assert 0 < g["leaves"] < (652458240 if raw else 906192)


def test_prune_sharded_virtual_ranks():
    """Prune mode per shard (each rank prunes against its own best) combined
    over 3 virtual ranks = the unsharded decision."""
    t = mp.Topology(text=W.het32_text())
    pat = mp.Pattern.make("tree", 5)
    for sel, sens in SELS[:3]:
        ref = mp.allocate(t, pat, sel, sens, raw=True)
        recs = []
        for r in range(3):
            rec, _q = md.run_query(t, pat, sel, sens, 0, raw=True, rank=r, world=3, prune=True)
            recs.append(md.records_from_tensor(rec)[0])
        torch.cuda.synchronize()
        d = mp.decode(t, pat, 0, sel, sens, mp.reduce_records(recs), raw=True, prune=True)
        for f in ("devices", "mapping", "used_edges", "key"):
            assert d[f] == ref[f], (sel, sens, f)


def test_prune_rejected_for_batch():
    t = mp.Topology("dgx1v")
    with pytest.raises(mp.MapaError):
        mp._check(mp._lib.mapa_allocate_batch(t.handle, (mp._vp * 1)(mp.Pattern.make("ring", 3).handle), 1, 0,
                                               None, None, None, mp.F_PRUNE, None))


def test_batch_vs_oracle_and_counts():
    """C5-shaped batch: every query's leaf count equals the closed form, a
    sample of decisions equals the oracle."""
    for name, text in (("cubemesh16", None), ("het32", W.het32_text())):
        o = mo.builtin(name) if text is None else mo.parse_topology(text)
        t = mp.Topology(name) if text is None else mp.Topology(text=text)
        qs = W.c5_queries(o.n, count=2000, seed=99)
        shapes = [(s, k) for s in ("ring", "tree", "full") for k in range(2, 6)]
        pats = [mp.Pattern.make(s, k) for s, k in shapes]
        auts = [p.info()["aut"] for p in pats]
        pid = {sk: i for i, sk in enumerate(shapes)}
        rows = [(q["busy"], pid[(q["shape"], q["k"])], q["selector"], q["sensitive"]) for q in qs]
        for raw in (True, False):
            res = md.run_batch(t, pats, md.queries_tensor(rows), raw=raw)
            torch.cuda.synchronize()
            recs = md.records_from_tensor(res)
            for i, (q, r) in enumerate(zip(qs, recs)):
                nf = o.n - bin(q["busy"]).count("1")
                p = math.perm(nf, q["k"])
                assert r.leaves == (p if raw else p // auts[rows[i][1]]), (name, i)
                assert r.status == 0
            rng = random.Random(5)
            for i in rng.sample(range(len(qs)), 25):
                q = qs[i]
                d = mp.decode(t, pats[rows[i][1]], q["busy"], q["selector"], q["sensitive"], recs[i], raw=raw)
                same(oracle(o, q["busy"], q["shape"], q["k"], q["selector"], q["sensitive"], use_c=True), d,
                     (name, i, raw))


def test_batch_mixed_code_paths_and_bad_index():
    """Queries of every (k, selector) code path interleaved with bad pattern
    indices: the device bucketing by code path leaves every record where its
    query is (status 1 only for the bad ones, the rest equal to the oracle)."""
    o, t = mo.builtin("dgx1v"), mp.Topology("dgx1v")
    shapes = [("full", 1), ("ring", 2), ("ring", 3), ("tree", 4), ("ringtree", 5), ("full", 6), ("ring", 7)]
    pats = [mp.Pattern.make(s, k) for s, k in shapes]
    rng = random.Random(17)
    rows, exp = [], []
    for i in range(3000):
        pi = rng.randrange(len(shapes) + 1)
        busy = rng.randrange(0, 256) & rng.randrange(0, 256)
        sel, sens = rng.choice(SELS)
        rows.append((busy, pi if pi < len(shapes) else 99, sel, sens))
        exp.append(None if pi == len(shapes) else (busy, shapes[pi], sel, sens))
    recs = md.records_from_tensor(md.run_batch(t, pats, md.queries_tensor(rows), raw=True))
    for i in rng.sample(range(len(rows)), 200):
        if exp[i] is None:
            assert recs[i].status == 1 and recs[i].key == 0
            continue
        busy, (shape, k), sel, sens = exp[i]
        d = mp.decode(t, pats[rows[i][1]], busy, sel, sens, recs[i], raw=True)
        same(oracle(o, busy, shape, k, sel, sens, use_c=True), d, (i, shape, k, hex(busy), sel, sens))


def test_launch_query_inside_user_cuda_graph():
    """mapa_launch_query is capturable into the caller's CUDA graph.  With a
    fresh topology the cached pair-table image cannot be allocated during the
    capture, so the kernel builds its tables itself: the replayed record must
    equal a normal launch's (which uses the cached image)."""
    text = W.het32_text()
    ref_t = mp.Topology(text=text)
    p = mp.Pattern.make("ring", 5)
    busy = 0x00F0000F
    for sel, sens in SELS:
        rec0, _q0 = md.run_query(ref_t, p, sel, sens, busy, raw=True)
        torch.cuda.synchronize()
        ref = md.records_from_tensor(rec0)[0]
        t = mp.Topology(text=text)  # empty cache
        q = md.query_tensor(busy, 0, sel, sens)
        rec = torch.zeros(4, dtype=torch.int64, device="cuda")
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, busy_hint=busy, stream=s)
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        got = md.records_from_tensor(rec)[0]
        assert (got.key, got.leaves) == (ref.key, ref.leaves), (sel, sens)


def _trace_inputs(topo_name, seed, policy):
    jobs = W.c2_jobs(seed, 1000)
    n = mo.builtin(topo_name).n
    ops = W.fifo_ops(jobs, n)
    shapes = [(s, k) for s in ("ring", "tree", "full") for k in range(2, 6)]
    pid = {sk: i for i, sk in enumerate(shapes)}
    jrows = []
    for j in jobs:
        if policy == "preserve":
            jrows.append([0, pid[(j["shape"], j["k"])], 1, j["sensitive"]])
        else:
            jrows.append([0, pid[(j["shape"], j["k"])], 0, 0])
    return jobs, ops, shapes, jrows


@pytest.mark.parametrize("topo_name", ["dgx1p", "summit"])
@pytest.mark.parametrize("policy", ["preserve", "greedy"])
def test_c2_trace_replay_vs_oracle(topo_name, policy):
    """C2: 1000-job FIFO trace replayed entirely on the device; every
    allocation must equal the oracle's replay (§3.6 state management)."""
    jobs, ops, shapes, jrows = _trace_inputs(topo_name, 2110 + len(topo_name), policy)
    t = mp.Topology(topo_name)
    pats = [mp.Pattern.make(s, k) for s, k in shapes]
    dops = torch.tensor([[o, j] for o, j in ops], dtype=torch.int32, device="cuda").reshape(1, -1, 2)
    djobs = torch.tensor(jrows, dtype=torch.int32, device="cuda").reshape(1, -1, 4)
    for raw in (False, True):
        keys = md.run_trace(t, pats, dops, djobs, raw=raw)
        torch.cuda.synchronize()
        keys = keys.cpu().tolist()[0]
        o = mo.builtin(topo_name)
        patd = {(s, k): mo.make_pattern(s, k) for s, k in shapes}

        def alloc(topo, busy, k, pe, sel, sens):
            return co.allocate(topo, busy, k, pe, sel, sens, nthreads=1)

        exp = mo.replay_trace(o, jobs, ops, patd, policy, allocate_fn=alloc)
        # every key decoded through the C-ABI (mapa_decode_trace replays the
        # busy state) and compared field by field with the oracle's replay
        got = mp.decode_trace(t, pats, ops, [(r[1], r[2], r[3]) for r in jrows], keys, raw=raw)
        for j, d in exp.items():
            same(d, got[j], (topo_name, policy, j, raw))


def test_c3_sampled_vs_oracle():
    """C3: cubemesh16, {ring,tree,full} x k in {4,6,8}, random busy; sampled
    queries in the single-query launch configuration vs the C oracle."""
    o = mo.builtin("cubemesh16")
    t = mp.Topology("cubemesh16")
    qs = W.c3_queries(per_case=1000)
    rng = random.Random(3)
    picked = 0
    for i in rng.sample(range(len(qs)), 400):
        q = qs[i]
        nf = 16 - bin(q["busy"]).count("1")
        if q["k"] <= nf and math.perm(nf, q["k"]) > 3e6:  # keep the CPU oracle within seconds
            continue
        for raw in (True, False):
            same(oracle(o, q["busy"], q["shape"], q["k"], q["selector"], q["sensitive"], use_c=True),
                 gpu(t, q["busy"], q["shape"], q["k"], q["selector"], q["sensitive"], raw), (i, q, raw))
        picked += 1
        if picked >= 40:
            break
    assert picked >= 20


def test_run_queries_multistream_vs_oracle():
    """md.run_queries (independent launches over 8 streams): every record
    decodes to the oracle's decision, counts = closed forms."""
    o, t = mo.builtin("cubemesh16"), mp.Topology("cubemesh16")
    keys = [(s, k) for s in ("ring", "tree", "full") for k in (3, 4, 5)]
    pats = [mp.Pattern.make(s, k) for s, k in keys]
    rng = random.Random(33)
    rows = []
    for _ in range(120):
        ki = rng.randrange(len(keys))
        busy = rng.randrange(0, 1 << 16) | 0xFF
        sel, sens = rng.choice(SELS)
        rows.append((busy, ki, sel, sens))
    recs = md.records_from_tensor(md.run_queries(t, pats, rows, raw=True))
    for (busy, ki, sel, sens), r in zip(rows, recs):
        shape, k = keys[ki]
        nf = 16 - bin(busy).count("1")
        assert r.leaves == (math.perm(nf, k) if k <= nf else 0)
        d = mp.decode(t, pats[ki], busy, sel, sens, r, raw=True)
        same(oracle(o, busy, shape, k, sel, sens, use_c=True), d, (shape, k, hex(busy), sel, sens))


def _hub_text(n=32):
    """Device 1 has a double NVLink to every other device; all other pairs
    are PCIe: inc_F(hub) = 50 (n-1) while inc_F(other) = 50 + 12 (n-2), an
    Eq. 3 spread far beyond the 16-bit scan's range (lin16_fits)."""
    lines = [f"name hub{n}", f"devices {n}", "sockets " + ",".join(str(i) for i in range(1, n // 2 + 1)) + " "
             + ",".join(str(i) for i in range(n // 2 + 1, n + 1))]
    lines += [f"link 1 {b} nv2x2" for b in range(2, n + 1)]
    return "\n".join(lines) + "\n"


def test_lin16_range_fallback_and_refusal():
    """Eq. 3 on a hub topology (spread 1140 > the s16 budget): with the hub
    free the host keeps the 32-bit scan and decisions equal the oracle's; with
    the hub busy the 16-bit scan is used and decisions still equal the
    oracle's; a launch whose busy_hint claims the hub busy while the device
    query has it free is refused by the kernel (record status -> decode
    error), never mis-scored."""
    text = _hub_text()
    o, t = mo.parse_topology(text), mp.Topology(text=text)
    rng = random.Random(5)
    for trial in range(6):
        # hub free with 24 others: spread 38 nf - 76 = 874 > 972 - 50 (k-2) -> 32-bit scan;
        # hub busy (or few free): spread small -> 16-bit scan
        hub_busy = trial % 2 == 1
        free = rng.sample(range(1, 32), 24 if not hub_busy else 10) + ([] if hub_busy else [0])
        busy = ((1 << 32) - 1) & ~sum(1 << d for d in free)
        shape = rng.choice(["ring", "tree", "full"])
        k = rng.randint(4, 5)
        for raw in (True, False):
            same(oracle(o, busy, shape, k, 1, False, use_c=True), gpu(t, busy, shape, k, 1, False, raw),
                 ("hub", trial, hub_busy, shape, k, raw))
    pat = mp.Pattern.make("full", 5)
    busy_true = 0                                 # all 32 free: spread 1140
    hint = 1                                      # claims the hub busy: spread 0 -> 16-bit scan chosen
    q = md.query_tensor(busy_true)
    rec = torch.zeros(4, dtype=torch.int64, device="cuda")
    mp.launch_query(t, pat, 1, False, q.data_ptr(), rec.data_ptr(), raw=True, busy_hint=hint)
    torch.cuda.synchronize()
    r = md.records_from_tensor(rec)[0]
    assert r.status != 0
    with pytest.raises(mp.MapaError) as e:
        mp.decode(t, pat, busy_true, 1, False, r, raw=True)
    assert e.value.status == mp.E_INVALID_ARG


def test_allocate_many_equals_single_allocations_and_oracle():
    """mapa_allocate_many (one graph: one H2D copy, parallel launches, one D2H
    copy, host decode): every decision equals mapa_allocate's for the same
    query and the oracle's; narrow and deep queries and a no-capacity query in
    one call; the cached graph is reused when only the busy mask changes."""
    o, t = mo.builtin("cubemesh16"), mp.Topology("cubemesh16")
    qs = [("ring", 4, 0, False), ("tree", 5, 1, True), ("full", 4, 1, False), ("ring", 9, 0, False),
          ("tree", 13, 1, True)]
    pats = {(s, k): mp.Pattern.make(s, k) for s, k, _, _ in qs}
    for busy in (0b1010000000000001, 0b0000000100100110, 0b1111111100000000):
        t.set_busy(busy)
        for raw in (True, False):
            got = mp.allocate_many(t, [(pats[(s, k)], sel, sens) for s, k, sel, sens in qs], raw=raw)
            for (s, k, sel, sens), g in zip(qs, got):
                one = mp.allocate(t, pats[(s, k)], sel, sens, raw=raw)
                assert g["status"] == one["status"]
                if g["status"] == "ok":
                    for f in FIELDS + ("leaves", "key", "pred_effbw"):
                        assert g[f] == one[f], (s, k, hex(busy), raw, f)
                if k <= 5:
                    same(oracle(o, busy, s, k, sel, sens, use_c=True), g, (s, k, hex(busy), raw))
    assert t.busy == 0b1111111100000000  # never commits
    with pytest.raises(mp.MapaError):
        mp._check(mp._lib.mapa_allocate_many(t.handle, None, 0, None, None, 0, None, None))
