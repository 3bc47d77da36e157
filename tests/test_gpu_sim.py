"""GPU parity of the simulator: mapa_simulate replays
every allocation of a FIFO job stream on the device (Topo-aware / Baseline /
Greedy / Preserve, state kept in shared memory) and must produce the oracle's
job log (oracle/mapa_oracle.simulate) record by record; plus the paper's
directional result (Preserve lifts the lower tail of predicted EffBW for
bandwidth-sensitive jobs, Fig. 12c / P:966-970)."""
import pytest

import workloads as W
from oracle import coracle as co
from oracle import mapa_oracle as mo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_03214_b200 as mp  # noqa: E402

POLICIES = ("baseline", "topo", "greedy", "preserve")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.init()


def _run(name, seed, count, kmax, policy, raw=False):
    js = W.sim_jobs(seed, count, kmax)
    shapes = sorted({(j["shape"], j["k"]) for j in js})
    pid = {sk: i for i, sk in enumerate(shapes)}
    t = mp.Topology(name)
    pats = [mp.Pattern.make(s, k) for s, k in shapes]
    got = mp.simulate(t, pats, [(pid[(j["shape"], j["k"])], j["sensitive"], j["duration"]) for j in js], policy,
                      raw=raw)
    o = mo.builtin(name)
    jobs = [dict(k=j["k"], edges=mo.make_pattern(j["shape"], j["k"])[1], sensitive=j["sensitive"],
                 duration=float(j["duration"])) for j in js]

    def alloc(topo, busy, k, pe, sel, sens):
        return co.allocate(topo, busy, k, pe, sel, sens, nthreads=1)

    exp = mo.simulate(o, jobs, policy, allocate_fn=alloc)
    return js, got, exp


@pytest.mark.parametrize("name,count,kmax", [("dgx1v", 150, 5), ("summit", 80, 5), ("cubemesh16", 100, 6),
                                             ("torus2d16", 60, 5)])
@pytest.mark.parametrize("policy", POLICIES)
def test_simulate_vs_oracle(name, count, kmax, policy):
    js, got, exp = _run(name, 77 + count, count, kmax, policy, raw=(count % 2 == 0))
    for g, e in zip(got, exp):
        for f in ("devices", "x", "y", "z", "agg_bw", "preserved_bw", "start", "end", "wait"):
            assert g[f] == e[f], (name, policy, g["job"], f, g[f], e[f])
        assert abs(g["pred_effbw"] - e["pred_effbw"]) <= 1e-6 * max(1.0, abs(e["pred_effbw"]))


def test_preserve_lifts_lower_tail_300_jobs():
    """300-job dgx1v run (§4): for bandwidth-sensitive jobs the 25th
    percentile of predicted EffBW under Preserve is >= Baseline's (
    Fig. 12c direction); summaries come from mapa_quantiles."""
    out = {}
    for pol in POLICIES:
        js = W.sim_jobs(2110, 300, 5)
        shapes = sorted({(j["shape"], j["k"]) for j in js})
        pid = {sk: i for i, sk in enumerate(shapes)}
        t = mp.Topology("dgx1v")
        pats = [mp.Pattern.make(s, k) for s, k in shapes]
        log = mp.simulate(t, pats, [(pid[(j["shape"], j["k"])], j["sensitive"], j["duration"]) for j in js], pol)
        for r, j in zip(log, js):
            r["sensitive"] = j["sensitive"]
        out[pol] = mp.summarize(log, "sensitive")
    assert out["preserve"][1]["pred_effbw"][1] >= out["baseline"][1]["pred_effbw"][1]
    assert out["preserve"][1]["makespan"] == out["baseline"][1]["makespan"]  # schedule is policy independent
