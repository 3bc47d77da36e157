"""Round-2 kernel paths under compute-sanitizer (memcheck / racecheck /
synccheck): lin16 single-query scans (W = 32 / 16, RAW + canonical + prune),
the static first work chunk, the small-query batch of mapa_launch_queries,
the deep lanes2 suffix (N = 64, u64 masks) and the 32-bit fallback on a hub
topology.  Small sizes (the sanitizer runs ~100x slower)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

het = mp.Topology(text=W.het32_text())
het.set_busy(((1 << 32) - 1) & ~0xFFF)  # 12 free
for shape, k in (("full", 6), ("ring", 5), ("tree", 4)):
    p = mp.Pattern.make(shape, k)
    for sel, sens in ((0, False), (1, True), (1, False)):
        for raw in (False, True):
            mp.allocate(het, p, sel, sens, raw=raw)
        mp.allocate(het, p, sel, sens, raw=True, prune=True)
cm = mp.Topology("cubemesh16")
keys = [(s, k) for s in ("ring", "tree", "full") for k in (4, 6, 8)]
pats = [mp.Pattern.make(s, k) for s, k in keys]
qs = W.c3_queries(per_case=4)
rows = [(q["busy"], keys.index((q["shape"], q["k"])), q["selector"], q["sensitive"]) for q in qs]
rows.append((0xFF00, keys.index(("ring", 8)), 0, 0))  # a big one next to the batched small ones
md.run_queries(cm, pats, rows, raw=True)
h64 = mp.Topology(text=W.het64_text())
busy = ((1 << 64) - 1) & ~((1 << 24) - 1)  # 24 free: ring-5 -> lanes2 (r = 21)
h64.set_busy(busy)
for sel, sens in ((0, False), (1, True), (1, False)):
    for raw in (False, True):
        mp.allocate(h64, mp.Pattern.make("ring", 5), sel, sens, raw=raw)
hub = "name hub16\ndevices 16\nsockets 1,2,3,4,5,6,7,8 9,10,11,12,13,14,15,16\n" + \
      "".join(f"link 1 {b} nv2x2\n" for b in range(2, 17))
th = mp.Topology(text=hub)
th.set_busy(0xF000)
mp.allocate(th, mp.Pattern.make("full", 5), 1, False, raw=True)
torch.cuda.synchronize()
print("sanitize r02 done")
