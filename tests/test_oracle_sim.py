"""The simulator layer above the path (SPEC policies
S:326-344, simulator S:386-439; paper §4, §5) — CPU only.

Oracle pins: SPEC's worked examples for select_baseline / select_topo_aware,
run_simulation and summarize_log; invariants of a seeded 300-job run
(conservation, FIFO order, census sums, replay consistency).  Host C-ABI
checks (no GPU): mapa_fifo_schedule and mapa_quantiles against the oracle."""
import random

import pytest

import workloads as W
from oracle import mapa_oracle as mo

import paper_2110_03214_b200 as mp


def _jobs(shape_k_sens_dur):
    out = []
    for shape, k, sens, dur in shape_k_sens_dur:
        kk, e = mo.make_pattern(shape, k)
        out.append(dict(k=kk, edges=e, sensitive=sens, duration=dur))
    return out


def test_spec_topo_aware_examples():
    o = mo.builtin("dgx1v")
    assert mo.select_topo_aware(o, 0, 3) == (0, 1, 2)            # {1,2,3}
    assert mo.select_topo_aware(o, 0b11, 3) == (4, 5, 6)         # {1,2} busy -> {5,6,7}
    assert mo.select_topo_aware(o, 0, 5) == (0, 1, 2, 3, 4)      # global fallback
    assert mo.select_topo_aware(o, 0b01111111, 2) is None


def test_spec_baseline_examples():
    o = mo.builtin("dgx1v")
    k, e = mo.make_pattern("ring", 3)
    assert mo.allocate_policy(o, 0, k, e, "baseline", False)["devices"] == (0, 1, 2)
    busy = 0xFF & ~((1 << 2) | (1 << 4) | (1 << 5) | (1 << 7))  # free {3,5,6,8}
    k2, e2 = mo.make_pattern("ring", 2)
    assert mo.allocate_policy(o, busy, k2, e2, "baseline", False)["devices"] == (2, 4)


def test_spec_simulation_examples():
    o = mo.builtin("dgx1v")
    r = mo.simulate(o, _jobs([("ring", 4, 1, 10), ("ring", 4, 1, 10)]), "baseline")
    assert [x["devices"] for x in r] == [(0, 1, 2, 3), (4, 5, 6, 7)] and [x["start"] for x in r] == [0, 0]
    assert max(x["end"] for x in r) == 10
    for pol in ("baseline", "topo", "greedy", "preserve"):
        r = mo.simulate(o, _jobs([("ring", 5, 1, 10)] * 3), pol)
        assert [x["start"] for x in r] == [0, 10, 20]
    r = mo.simulate(o, _jobs([("ring", 2, 1, 7)]), "preserve")[0]
    assert (r["x"], r["y"], r["z"]) == (1, 0, 0) and abs(r["pred_effbw"] - 39.08) < 1e-9


def test_spec_quantile_examples():
    assert mo.quantiles7([10, 20, 30, 40]) == (10, 17.5, 25, 32.5, 40)
    assert mo.quantiles7([3.5]) == (3.5,) * 5


@pytest.mark.parametrize("policy", ["baseline", "topo", "greedy", "preserve"])
def test_simulation_invariants(policy):
    o = mo.builtin("dgx1v")
    jobs = [dict(k=j["k"], edges=mo.make_pattern(j["shape"], j["k"])[1], sensitive=j["sensitive"],
                 duration=j["duration"]) for j in W.sim_jobs(2110, 120)]
    log = mo.simulate(o, jobs, policy)
    starts = [r["start"] for r in log]
    assert starts == sorted(starts)                                       # strict FIFO
    for r, j in zip(log, jobs):
        assert r["x"] + r["y"] + r["z"] == len(j["edges"]) and len(r["devices"]) == j["k"]
        assert r["end"] == r["start"] + j["duration"] and r["wait"] == r["start"] >= 0
    times = sorted({r["start"] for r in log} | {r["end"] for r in log})
    for t in times:                                                       # conservation, no overlap
        run = [r for r in log if r["start"] <= t < r["end"]]
        used = [d for r in run for d in r["devices"]]
        assert len(used) == len(set(used)) and sum(r["k"] for r in run) <= o.n


def test_host_fifo_schedule_equals_oracle():
    """mapa_fifo_schedule (C-ABI, host) vs the oracle event loop: start / end
    times of every job, with and without arrival times."""
    rng = random.Random(5)
    o = mo.builtin("dgx1v")
    for trial in range(6):
        js = W.sim_jobs(100 + trial, 80)
        arr = [0.0] * len(js) if trial % 2 == 0 else sorted(rng.uniform(0, 3000) for _ in js)
        jobs = [dict(k=j["k"], edges=mo.make_pattern(j["shape"], j["k"])[1], sensitive=j["sensitive"],
                     duration=float(j["duration"]), arrival=a) for j, a in zip(js, arr)]
        log = mo.simulate(o, jobs, "baseline")
        ops, st, en = mp.fifo_schedule(8, [j["k"] for j in jobs], [j["duration"] for j in jobs], arr)
        assert st == [r["start"] for r in log] and en == [r["end"] for r in log]
        assert sorted(j for op, j in ops if op == 0) == list(range(len(jobs)))
    with pytest.raises(mp.MapaError):
        mp.fifo_schedule(8, [9], [1.0])


def test_host_quantiles_equal_oracle():
    rng = random.Random(9)
    for n in (1, 2, 3, 7, 300):
        v = [rng.uniform(-5, 100) for _ in range(n)]
        assert all(abs(a - b) < 1e-12 for a, b in zip(mp.quantiles(v), mo.quantiles7(v)))
    assert mp.quantiles([10, 20, 30, 40]) == (10, 17.5, 25, 32.5, 40)
    with pytest.raises(mp.MapaError):
        mp.quantiles([])


def test_spec_generate_jobs_mix():
    """SPEC generate_jobs examples: deterministic for a seed; 300
    jobs of U{1..5} GPUs -> every gpu_count class within the binomial 99 %
    bounds of 60 (60 +- 2.576 sqrt(300 * 0.2 * 0.8) = [42, 78]); 6 networks ->
    each within those of 50 ([34, 66]); Ring for k >= 2, the singleton for k = 1."""
    a, b = W.spec_jobs(2110, 300), W.spec_jobs(2110, 300)
    assert a == b
    for seed in (2110, 2111, 2112):
        js = W.spec_jobs(seed, 300)
        for k in range(1, 6):
            assert 42 <= sum(j["k"] == k for j in js) <= 78, (seed, k)
        for name, _, _ in W.NETWORKS:
            assert 34 <= sum(j["network"] == name for j in js) <= 66, (seed, name)
        assert all(j["shape"] == ("ring" if j["k"] >= 2 else "full") for j in js)
        assert all(bool(j["sensitive"]) == (j["network"] in ("alexnet", "vgg16", "resnet50", "inceptionv3"))
                   for j in js)
