import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2110_03214_b200 as mp
from paper_2110_03214_b200 import dist as md
t = mp.Topology(text=W.het32_text())
pat = mp.Pattern.make("full", 6)
for sel, sens in ((0, False), (1, True), (1, False)):
    for raw in (True, False):
        for _ in range(3):
            rec, q = md.run_query(t, pat, sel, sens, 0, raw=raw)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        n = 10
        for _ in range(n):
            rec, q = md.run_query(t, pat, sel, sens, 0, raw=raw)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / n
        r = md.records_from_tensor(rec)[0]
        print(f"sel={sel} sens={sens} raw={raw} ms={ms:.3f} leaves={r.leaves} rate={r.leaves/ms/1e6:.3e} leaves/s", flush=True)
