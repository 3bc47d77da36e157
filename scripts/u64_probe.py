"""Deep kernel throughput with u64 masks: het64, 40 free devices, ring-7 RAW, per selector."""
import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2110_03214_b200 as mp
from paper_2110_03214_b200 import dist as md
t = mp.Topology(text=W.het64_text())
busy = ((1 << 64) - 1) & ~((1 << 40) - 1)
p = mp.Pattern.make("ring", 7)
q = md.query64_tensor(busy)
rec = torch.zeros(8, dtype=torch.int64, device="cuda")
for sel, sens in ((0, False), (1, True), (1, False)):
    f = lambda: mp.launch_query_wide(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), busy, raw=True)
    for _ in range(2): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(3)]; b.record(); b.synchronize()
    ms = a.elapsed_time(b) / 3
    print(sel, sens, round(ms, 2), "%.3g emb/s" % (math.perm(40, 7) / ms * 1e3))
