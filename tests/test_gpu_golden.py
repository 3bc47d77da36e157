"""GPU parity on the FULL C3 / C5 parity sets (SURVEY.md §8(d) "Full parity
sets"): every query of the oracle-written goldens (tests/golden/*.npz,
tests/golden/make_golden_c3c5.py, oracle/ only) through the launch
configuration the bench times, every record decoded through the C-ABI and
compared field by field -- device set, mapping, used edges, census, AggBW,
PreservedBW, raw / distinct counts bit-exact, Eq. 2 within 1e-6 relative
(north_star tolerance).

  C5  mapa_allocate_batch (one batch launch per topology), RAW and canonical
  C3  mapa_launch_queries (one full-GPU launch per query over 8 streams),
      RAW and canonical; k = 8 on up to 16 free devices (P(16,8) = 5.19e8)."""
import pytest

from tests import goldenutil as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

FIELDS = ("devices", "mapping", "used_edges", "x", "y", "z", "agg_bw", "preserved_bw", "raw", "distinct")
SHAPE_K = [(s, k) for s in ("ring", "tree", "full") for k in range(2, 6)]


def _cmp(exp, g, ctx):
    assert exp["status"] == g["status"], (ctx, exp, g)
    if exp["status"] != "ok":
        return
    for f in FIELDS:
        assert exp[f] == g[f], (ctx, f, exp[f], g[f])
    assert abs(exp["pred_effbw"] - g["pred_effbw"]) <= 1e-6 * max(1.0, abs(exp["pred_effbw"])), ctx


def _check_all(topo, pats, pid_of, rec, qs, recs, raw, part):
    bad = 0
    for i, (q, r) in enumerate(zip(qs, recs)):
        exp = G.expected(rec[i])
        pi = pid_of(q)
        if exp["status"] != "ok":
            assert r.key == 0 and r.leaves == 0, (part, i)
            continue
        assert r.leaves == (exp["raw"] if raw else exp["distinct"]), (part, i, raw)
        d = mp.decode(topo, pats[pi], q["busy"], q["selector"], q["sensitive"], r, raw=raw)
        _cmp(exp, d, (part, i, raw, q))
    return bad


@pytest.mark.parametrize("part", ["c5_cubemesh16", "c5_het32"])
def test_c5_full_set_vs_oracle_golden(part):
    if not G.have(part):
        pytest.skip(f"{part} golden not generated")
    rec, qs = G.load(part)
    topo = mp.Topology("cubemesh16") if part == "c5_cubemesh16" else mp.Topology(text=__import__("workloads").het32_text())
    pats = [mp.Pattern.make(s, k) for s, k in SHAPE_K]
    pid = {sk: i for i, sk in enumerate(SHAPE_K)}
    rows = [(q["busy"], pid[(q["shape"], q["k"])], q["selector"], q["sensitive"]) for q in qs]
    qt = md.queries_tensor(rows)
    for raw in (True, False):
        res = md.run_batch(topo, pats, qt, raw=raw)
        torch.cuda.synchronize()
        recs = md.records_from_tensor(res)
        _check_all(topo, pats, lambda q: pid[(q["shape"], q["k"])], rec, qs, recs, raw, part)


@pytest.mark.parametrize("part", ["c3_k46", "c3_k8"])
def test_c3_full_set_vs_oracle_golden(part):
    if not G.have(part):
        pytest.skip(f"{part} golden not generated")
    rec, qs = G.load(part)
    topo = mp.Topology("cubemesh16")
    keys = [(s, k) for s in ("ring", "tree", "full") for k in (4, 6, 8)]
    pats = [mp.Pattern.make(s, k) for s, k in keys]
    rows = [(q["busy"], keys.index((q["shape"], q["k"])), q["selector"], q["sensitive"]) for q in qs]
    for raw in (True, False):
        recs = md.records_from_tensor(md.run_queries(topo, pats, rows, raw=raw))
        _check_all(topo, pats, lambda q: keys.index((q["shape"], q["k"])), rec, qs, recs, raw, part)
