"""Small launches of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): W = 8 / 16 / 32, LIN and SENS, raw and canonical,
batch and trace."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2110_03214_b200 as mp
from paper_2110_03214_b200 import dist as md
for topo in (mp.Topology("dgx1v"), mp.Topology("cubemesh16"), mp.Topology(text=W.rand_text(32, 7))):
    topo.set_busy(0b1011)
    for shape, k in (("ring", 3), ("tree", 5), ("full", 4), ("ringtree", 6), ("full", 1), ("ring", 2)):
        for sel, sens in ((0, False), (1, True), (1, False), (2, False)):
            for raw in (False, True):
                mp.allocate(topo, mp.Pattern.make(shape, k), sel, sens, raw=raw)
t = mp.Topology("cubemesh16")
shapes = [(s, k) for s in ("ring", "tree", "full") for k in range(2, 6)]
pats = [mp.Pattern.make(s, k) for s, k in shapes]
pid = {sk: i for i, sk in enumerate(shapes)}
qs = W.c5_queries(16, count=200, seed=3)
rows = [(q["busy"], pid[(q["shape"], q["k"])], q["selector"], q["sensitive"]) for q in qs]
md.run_batch(t, pats, md.queries_tensor(rows))
jobs = W.c2_jobs(5, 40); ops = W.fifo_ops(jobs, 8)
t8 = mp.Topology("dgx1p")
dops = torch.tensor([[o, j] for o, j in ops], dtype=torch.int32, device="cuda").reshape(1, -1, 2)
djobs = torch.tensor([[0, pid[(j["shape"], j["k"])], 1, j["sensitive"]] for j in jobs], dtype=torch.int32, device="cuda").reshape(1, -1, 4)
md.run_trace(t8, pats, dops, djobs)
torch.cuda.synchronize()
print("sanitize probe done")
