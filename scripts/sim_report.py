"""Paper-style simulation report (§4 P:770-777 job mix; §5 P:936-970,
fig:16-GPU_simulation): 300-job FIFO streams of SPEC's generated mix
(workloads.spec_jobs: k U{1..5}, Ring for k >= 2, networks U(6)) on dgx1v,
torus2d16 and cubemesh16 under Baseline / Topo-aware / Greedy / Preserve,
replayed on the device by mapa_simulate; per policy the five quantiles of
predicted EffBW (Eq. 2) of the bandwidth-sensitive multi-GPU jobs (k >= 2,
reading A24) and the simulate() wall time.  Prints one JSON document."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_03214_b200 as mp  # noqa: E402
import workloads as W  # noqa: E402

out = {"jobs": 300, "seeds": [2110, 2111, 2112], "mix": "workloads.spec_jobs (SPEC generate_jobs: Ring for k >= 2)",
       "note": "quantiles pooled over the seeds' sensitive jobs with k >= 2"}
for name in ("dgx1v", "torus2d16", "cubemesh16"):
    t = mp.Topology(name)
    res = {}
    for pol in ("baseline", "topo", "greedy", "preserve"):
        vals, ms = [], []
        for seed in out["seeds"]:
            js = W.spec_jobs(seed, 300)
            shapes = sorted({(j["shape"], j["k"]) for j in js})
            pid = {sk: i for i, sk in enumerate(shapes)}
            pats = [mp.Pattern.make(s, k) for s, k in shapes]
            jl = [(pid[(j["shape"], j["k"])], j["sensitive"], j["duration"]) for j in js]
            mp.simulate(t, pats, jl, pol)  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            log = mp.simulate(t, pats, jl, pol)
            ms.append((time.perf_counter() - t0) * 1e3)
            vals += [r["pred_effbw"] for r, j in zip(log, js) if j["sensitive"] and j["k"] >= 2]
        q = mp.quantiles(vals)
        res[pol] = {"pred_effbw_sensitive": dict(zip(("min", "p25", "p50", "p75", "max"), q)),
                    "n": len(vals), "simulate_ms": min(ms)}
    out[name] = res
print(json.dumps(out, indent=1))
