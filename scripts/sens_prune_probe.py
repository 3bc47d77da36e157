"""Latency of deep Preserve-sensitive allocations with and without MAPA_F_PRUNE (Eq. 2 bound)."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_03214_b200 as mp

out = {}
for tname in ("cubemesh16", "torus2d16"):
    t = mp.Topology(tname)
    for shape, k in (("ring", 9), ("ring", 12), ("tree", 12), ("ring", 14), ("ring", 16), ("tree", 14)):
        p = mp.Pattern.make(shape, k)
        for prune in (True, False):
            if not prune and k > 12:
                continue
            mp.allocate(t, p, 1, True, prune=prune)
            t0 = time.perf_counter()
            d = mp.allocate(t, p, 1, True, prune=prune)
            ms = (time.perf_counter() - t0) * 1e3
            out[f"{tname}_{shape}{k}_{'prune' if prune else 'exh'}"] = dict(ms=ms, leaves=d["leaves"], devices=list(d["devices"]), pred=d["pred_effbw"])
            print(tname, shape, k, prune, round(ms, 3), d["leaves"], d["devices"], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/sens_prune_probe.json", "w"), indent=1)
