"""One het64 ring-7 RAW Greedy deep launch (40 free devices, u64 masks) for ncu:
  ncu --set full --import-source on -k regex:esa_deep -c 1 -o gpurun_out/x python scripts/prof_u64.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

t = mp.Topology(text=W.het64_text())
busy = ((1 << 64) - 1) & ~((1 << 40) - 1)
p = mp.Pattern.make("ring", int(os.environ.get("PROF_K", "7")))
q = md.query64_tensor(busy)
rec = torch.zeros(8, dtype=torch.int64, device="cuda")
mp.launch_query_wide(t, p, int(os.environ.get("PROF_SEL", "0")), False, q.data_ptr(), rec.data_ptr(), busy, raw=True)
torch.cuda.synchronize()
print(md.wide_records_from_tensor(rec)[0].leaves)
