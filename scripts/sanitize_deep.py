"""Small launches of the kernels added in round 1's second half, for
compute-sanitizer (memcheck / racecheck / synccheck): the deep kernel (u32 and
u64 masks, every term-count class, every selector, RAW and canonical, L = 1..4,
exhaustive and branch and bound),
the trace kernel's Topo-aware path (mapa_simulate), and the cached-graph
mapa_allocate path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402

for topo, busy in ((mp.Topology("cubemesh16"), 0b0110000000100001), (mp.Topology(text=W.het32_text()), (1 << 32) - 1 - 0x7FF0),
                   (mp.Topology(text=W.het64_text()), ((1 << 64) - 1) & ~(0x3F << 20 | 0xF))):
    topo.set_busy(busy)
    for shape, k in (("ring", 9), ("tree", 8), ("full", 5), ("ringtree", 7), ("ring", 4), ("full", 1), ("edgeless", 3)):
        for sel, sens in ((0, False), (1, True), (1, False), (2, False)):
            for raw in (False, True):
                for prune in (False, True):  # branch and bound: Greedy / Preserve-sensitive kernels, set search
                    mp.allocate(topo, mp.Pattern.make(shape, k), sel, sens, raw=raw, deep=True, prune=prune)
# cached-graph replays of the narrow path
t = mp.Topology("dgx1v")
p = mp.Pattern.make("ring", 3)
for _ in range(3):
    mp.allocate(t, p, 0, False)
# simulator with all four policies (Topo-aware in the trace kernel)
js = W.sim_jobs(9, 40, 5)
shapes = sorted({(j["shape"], j["k"]) for j in js})
pats = [mp.Pattern.make(s, k) for s, k in shapes]
jl = [(shapes.index((j["shape"], j["k"])), j["sensitive"], j["duration"]) for j in js]
for pol in ("baseline", "topo", "greedy", "preserve"):
    mp.simulate(mp.Topology("dgx1v"), pats, jl, pol)
torch.cuda.synchronize()
print("sanitize deep probe done")
