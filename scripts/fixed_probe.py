"""Fixed cost of a single-query launch: C4 (het32 full-6 RAW) rank 0 of world
W for W in argv (default 1 8 64 100000), one launch per selector; run under
ncu for per-launch durations (scripts/ncu_sass_hot.py for where the time goes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

t = mp.Topology(text=W.het32_text())
p = mp.Pattern.make("full", 6)
q = md.query_tensor(0)
rec = torch.zeros(4, dtype=torch.int64, device="cuda")
worlds = [int(a) for a in sys.argv[1:]] or [1, 8, 64, 100000]
for world in worlds:
    for sel, sens in ((0, False), (1, True), (1, False)):
        rec.zero_()
        mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, rank=0, world=world, busy_hint=0,
                        zeroed=True)
        torch.cuda.synchronize()
        print(world, sel, sens, md.records_from_tensor(rec)[0].leaves, flush=True)
