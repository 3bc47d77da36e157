"""Times the deep kernel (device events) on a few idle-graph configurations."""
import math
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402
import workloads as W  # noqa: E402

cases = [("cubemesh16", "ring", 9, False), ("cubemesh16", "ring", 12, False), ("cubemesh16", "ring", 12, True),
         ("cubemesh16", "tree", 12, False), ("cubemesh16", "ring", 14, False), ("cubemesh16", "ring", 16, False),
         ("het32", "full", 6, True), ("het32", "ring", 8, False), ("cubemesh16", "ring", 8, True)]
if len(sys.argv) > 1:
    cases = [cases[int(i)] for i in sys.argv[1].split(",")]
for topo, shape, k, raw in cases:
    t = mp.Topology(text=W.het32_text()) if topo == "het32" else mp.Topology(topo)
    n = t.n
    p = mp.Pattern.make(shape, k)
    for sel, sens in ((0, False), (1, True), (1, False)):
        rec, q = md.run_query_wide(t, p, sel, sens, 0, raw=raw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rec, q = md.run_query_wide(t, p, sel, sens, 0, raw=raw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        r = md.wide_records_from_tensor(rec)[0]
        print(f"{topo} {shape}-{k} raw={raw} sel={sel}{'s' if sens else ''}: {ms:.3f} ms leaves={r.leaves} "
              f"{r.leaves / ms * 1e3:.3e} leaves/s status={r.status}", flush=True)
