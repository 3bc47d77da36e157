"""ncu target: one C4 shard launch (rank 0 of 8) per selector, het32 full-6 RAW.
  ncu --set full -k regex:esa_single -c 3 -o gpurun_out/x python scripts/prof_shard.py"""
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
world = int(os.environ.get("PROF_WORLD", "8"))
for sel, sens in ((0, False), (1, True), (1, False)):
    mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, rank=0, world=world, busy_hint=0)
    torch.cuda.synchronize()
